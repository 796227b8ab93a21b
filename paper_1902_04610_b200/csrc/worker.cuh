// worker.cuh — worker CTAs of the persistent kernel.
//
// Workers run as CTA pairs (a cluster of 2 on one TPC): every task is a
// 256 x N super-tile computed by one tcgen05.mma.cta_group::2 issued by the
// pair's leader (cluster rank 0).  CTA h holds rows [128h, 128h+128) of A
// and columns [h N/2, h N/2 + N/2) of B in its shared memory and receives
// its 128 accumulator rows in its own TMEM, so each SM loads half of the
// shared B operand.  Both CTAs run the same roles on the same
// task sequence; the leader claims tasks and mails the payload to its peer.
// Each worker CTA is a warp-specialized, persistent tile engine (13 warps):
//   warp 0     decoder: (leader) claims tasks from the device task ring up
//              to NDESC ahead and mails them to the peer; (both) decodes its
//              half (stage -> GEMM / epilogue kind, tensors, coordinates) and
//              translates the epilogue's page addresses, lanes in parallel.
//   warp 1     operand loader (1 thread): issues every K-chunk of the A/B
//              operands as 2-D tensor TMAs (one 8/16 KiB block each) into a
//              4-stage mbarrier ring (page-table reads two chunks ahead).
//   warp 2     leader: MMA (1 thread): tcgen05.mma.cta_group::2 kind::f16
//              (bf16 in, fp32 accumulate) into one of two TMEM accumulators
//              of 256 columns in both CTAs (double buffered: the epilogue of
//              tile i overlaps the MMA of tile i+1).  Both CTAs' operand TMAs
//              complete on the leader's stage barrier (.cta_group::2).
//   warp 3     epilogue-input loader (1 thread): streams the tile's epilogue
//              input (fp32 master weights of a dW tile, ReLU mask of a dX
//              tile) in 32 KiB chunks through two 48 KiB smem buffers (the
//              last 16 KiB stage an SGD chunk's bf16 copy for its bulk store).
//   warps 4-11 epilogue: drain TMEM (tcgen05.ld), fused epilogue, stores.
//   warp 12    completion: gpu-scope fence, stage accounting, publication of
//              the next stage / start of the slot's next iteration (run-ahead)
//              -- off the epilogue's critical path.
// No host round-trip and no context teardown between iterations or jobs: a
// "job switch" is just a task whose slot points at a different job.
//
// Per CTA a tile is M = 128 x N (N = 256 when it divides the output width,
// else 128), K in chunks of 64 bf16.  Operands are bf16 tensors stored as 128-byte-
// swizzled 64-column panels, so a K-chunk is one 16 KiB block
// per 128 rows (K-major) or one 8 KiB block per 64 columns (MN-major).
#pragma once
#include <cuda_bf16.h>
#include "salus_dev.h"
#include "ptx.cuh"
#include "datagen.cuh"
#include "runahead.cuh"

namespace salus {

#ifndef SALUS_PIPE
#define SALUS_PIPE 4
#endif
constexpr uint32_t PIPE = SALUS_PIPE;                 // operand stages in flight
constexpr uint32_t STAGE_A_BYTES = 16384;             // 128 x 64 bf16 (this CTA's rows)
constexpr uint32_t STAGE_B_BYTES = 16384;             // <= 128 x 64 bf16 (this CTA's half of N)
constexpr uint32_t STAGE_BYTES = STAGE_A_BYTES + STAGE_B_BYTES;
constexpr uint32_t ECH_BYTES = 32768;                 // epilogue-input chunk
// SGD epilogue: the bf16 weight copy of a chunk (one 16 KiB panel block) is
// staged in smem behind the chunk's fp32 master and both leave as bulk
// stores -- 2 buffers of 48 KiB instead of 3 of 32 KiB (same smem)
#ifndef SALUS_WB_BULK
#define SALUS_WB_BULK 1
#endif
#if SALUS_WB_BULK
constexpr uint32_t ECH_STRIDE = ECH_BYTES + 16384;
#ifndef SALUS_EBUF
#define SALUS_EBUF 2
#endif
#else
constexpr uint32_t ECH_STRIDE = ECH_BYTES;
#ifndef SALUS_EBUF
#define SALUS_EBUF 3
#endif
#endif
// epilogue-input chunk buffers: the first chunks of a 128 x 256 fp32 master
// tile are read from HBM while the tile's MMA runs, not during its epilogue
// (smem: 4 operand stages x 32 KiB + 2 x 48 KiB + descriptors = 227 KiB)
constexpr uint32_t EBUF = SALUS_EBUF;
#ifndef SALUS_NDESC
#define SALUS_NDESC 4
#endif
constexpr uint32_t NDESC = SALUS_NDESC;               // decoder lookahead (tiles)
#ifndef SALUS_EPI_WARPS
#define SALUS_EPI_WARPS 8
#endif
// 4 or 8 epilogue warps: warp w reads TMEM lane quarter w % 4; with 8, the
// two warps of a quarter split the columns (two warps per SM sub-partition
// hide each other's TMEM / smem / store latencies)
constexpr uint32_t EPI_WARPS = SALUS_EPI_WARPS;
constexpr uint32_t EPI_HALVES = EPI_WARPS / 4;
static_assert(EPI_WARPS == 4 || EPI_WARPS == 8, "epilogue warps: 4 or 8");
constexpr uint32_t EPI_THREADS = 32 * EPI_WARPS;
constexpr uint32_t EPI_WARP0 = 4;
constexpr uint32_t DONE_WARP = EPI_WARP0 + EPI_WARPS;          // completion warp
constexpr uint32_t WORKER_THREADS = 32 * (DONE_WARP + 1);
constexpr uint32_t ACC_COLS = 256;
constexpr uint32_t TMEM_COLS = 2 * ACC_COLS;          // all of TMEM: 2 accumulators

enum : uint32_t { T_EXIT = 0, T_INIT = 1, T_GEN = 2, T_GEMM = 3, T_COPY = 4 };
enum : uint32_t { EPI_RELU = 0, EPI_OUT = 1, EPI_LOSS = 2, EPI_DX = 3, EPI_SGD = 4 };
// translated pointers of a tile: bf16 output panels, Wb panels (SGD/INIT),
// fp32 master pages, epilogue-input panels (DX mask); split-K partial
// pages k = 0..7 (slice q, page p of an N/128-page partial: k = q N/128 + p)
// in PTR_AUX..+3 then PTR_SK2..+3
enum : uint32_t { PTR_OUT = 0, PTR_AUX = 4, PTR_W32 = 8, PTR_EPI = 10, PTR_SK2 = 14,
                  NPTR = SALUS_SPLITK_BUILD ? 18 : 14 };
__host__ __device__ __forceinline__ uint32_t sk_ptr(uint32_t k) { return k < 4 ? PTR_AUX + k : PTR_SK2 + (k - 4); }

struct OpDesc {
  const uint32_t *table;   // page table of the operand's space
  uint32_t off, R, start, mn;
};

#ifndef SALUS_L2HINT
#define SALUS_L2HINT 1
#endif
// double K-chunks for dW / dX tiles (off: no net gain, profiles/r02/ab_kd.txt;
// together with split-K a C4 PACK run can hang, DESIGN.md §6 open issue)
#ifndef SALUS_KD
#define SALUS_KD 0
#endif
#ifndef SALUS_W32_PF
#define SALUS_W32_PF 0
#endif
#ifndef SALUS_WAIT_ACQ
#define SALUS_WAIT_ACQ 0
#endif
static_assert(PIPE % 2 == 0, "double K-chunks take two operand stages");
// SGD epilogue: the fp32 master chunk is updated in its smem buffer and
// written back with one 32 KiB bulk (TMA) store per chunk
#ifndef SALUS_W32_BULK
#define SALUS_W32_BULK 1
#endif


struct TileDesc {
  // next_stage / next_ntiles: the stage this one's completion publishes (its
  // successor; eager records: the successor's successor, 0 tiles if none)
  uint32_t kind, payload, slot, stage, job, iter, ntiles, next_ntiles, first_stage, next_stage;
  uint8_t eager, wait, dep_stage, end2;   // eager record; wait for counter dep_stage (dep_want counts);
                                          // end2: relaxed record's B_2 / B_1 (end ticket)
  // dx_ctr: relaxed record, this dX tile also counts on stage_done[dx_ctr] (0 = no);
  // next_tk: next_stage needs a publication ticket; next2_stage: a relaxed
  // backward stage also arrives on the ticket of the stage three after it
  uint8_t is_last, dx_ctr, next_tk, next2_stage;
  uint32_t dep_want, next2_ntiles;
  // K9: transposed (swap-AB) tile; ech_load: the epilogue-input chunk is
  // loaded (else only reserved as the output block's staging buffer)
  uint8_t swap, ech_load, pad_k9;
  // double K-chunks (tiles with an MN-major B: dW and dX): each operand
  // block is a 128-row (16 KiB) box, one K-chunk of 128 spans two ring
  // stages (A in the first, B in the second) -- half the copies per byte
  uint8_t kd;
  // split-K: K-slices of this tile (1 = none), this slice, base tile index
  uint8_t sk, skz;
  uint16_t sku;
  uint32_t valid;          // this CTA's half exists (odd block counts leave the peer's empty)
  uint32_t peer_valid;     // the pair's second M block exists
  uint32_t peer_nca;       // (leader) A copies per K-chunk of the peer CTA
  uint64_t seq, t_claim, t_ready, t_mma, t_end;   // physical record seq, trace stamps
  uint64_t lseq;           // logical dispatch seq (wall stamps)
  // GEMM
  uint32_t N, nk, idesc, epi, layer, ncopy_a, ncopy_b, abytes, bbytes;
  uint32_t n_ech;          // epilogue-input chunks (0 = none)
  OpDesc a, b;
  uint8_t *ptr[NPTR];
  const uint32_t *xt_tab[2];   // page tables deferred translations use: lane (0), job (1)
  uint32_t xt_off[NPTR];
  uint32_t xt_mask, xt_sel;    // pending translations; bit set in xt_sel = through xt_tab[1]
  uint32_t m0, n0;
  uint32_t rows_valid, cols_valid, ld_logical;
  uint64_t key;
  float scale, lr;
  int64_t dump_off;
};

struct WorkerSmem {
  uint8_t stage[PIPE][STAGE_BYTES];   // 1024-aligned (first member)
  uint8_t epi_in[EBUF][ECH_STRIDE];   // 1024-aligned
  TileDesc desc[NDESC];
  uint64_t full[PIPE], empty[PIPE];
  uint64_t desc_full[NDESC], desc_empty[NDESC];
  uint64_t desc_ptrs[NDESC];          // the descriptor's translated pointers are in place
  uint64_t acc_full[2], acc_empty[2];
  uint64_t epi_full[EBUF], epi_empty[EBUF];
  uint64_t epi_done[NDESC];           // epilogue -> completion warp
  uint64_t mail_full[NDESC];          // peer: the leader mailed task d
  struct alignas(16) { uint32_t payload, pad; uint64_t t_claim; } mail[NDESC];
  uint32_t sink[4];                   // target of the peer's signalling st.async
  uint32_t tmem_base;
  alignas(16) uint32_t job_cache[128]; // decoder scratch: the task's DevJob (<= 512 B)
};

static_assert(sizeof(DevJob) <= 512, "DevJob must fit the decoder cache");

#ifndef SALUS_DBG_BOUNDS
#define SALUS_DBG_BOUNDS 0
#endif
// Debugging builds (SALUS_DBG_BOUNDS): a page number outside the arena --
// with SALUS_POISON's all-ones meta, a table entry the scheduler never
// wrote -- is reported through the mapped abort slot (words 4..7: site,
// offset, entry, table address low bits) and traps.
__device__ __forceinline__ uint32_t check_page(const Params &P, uint32_t page, uint32_t site, uint32_t off,
                                               const uint32_t *table) {
#if SALUS_DBG_BOUNDS
  if (page >= P.Cp) {
    if (P.host_abort) {
      volatile uint32_t *h = const_cast<volatile uint32_t *>(P.host_abort);
      h[4] = site; h[5] = off; h[6] = page; h[7] = (uint32_t)(uintptr_t)table;
      __threadfence_system();
    }
    __trap();
  }
#else
  (void)P; (void)site; (void)off; (void)table;
#endif
  return page;
}

__device__ __forceinline__ uint8_t *xlate(const Params &P, const uint32_t *table, uint32_t off) {
  const uint32_t page = check_page(P, table[off >> PAGE_SHIFT], 1, off, table);
  return P.arena + ((uint64_t)page << PAGE_SHIFT) + (off & (PAGE_BYTES - 1));
}

__device__ __forceinline__ void defer(TileDesc &td, uint32_t which, const uint32_t *table, uint32_t off) {
  if (table == td.xt_tab[1]) td.xt_sel |= 1u << which;
  td.xt_off[which] = off;
  td.xt_mask |= 1u << which;
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t *>(&h);
}

// 16-byte chunk (8 columns) `chunk` of row r inside a swizzled panel row block
__device__ __forceinline__ uint32_t swz(uint32_t r, uint32_t chunk) {
  return r * 128u + (((chunk ^ (r & 7u)) & 7u) << 4);
}

__device__ __forceinline__ uint4 shfl_xor_u4(uint4 v, int m) {
  v.x = __shfl_xor_sync(0xffffffffu, v.x, m);
  v.y = __shfl_xor_sync(0xffffffffu, v.y, m);
  v.z = __shfl_xor_sync(0xffffffffu, v.z, m);
  v.w = __shfl_xor_sync(0xffffffffu, v.w, m);
  return v;
}

// Store 32 bf16 columns (4 x 16-byte chunks, chunk index ch0..ch0+3) of the
// warp's 32 rows into a swizzled panel row block.  A 4x4 transpose of the
// chunks inside each group of 4 lanes (two shfl_xor stages) lets every store
// instruction write 8 rows x 64 contiguous bytes (the swizzle keeps a
// row-half's 4 chunks inside one 64-byte half) instead of 32 rows x 16 bytes.
// `r` = this lane's row in the tile (warp-uniform quarter base + lane).
template <bool kStream = false>
__device__ __forceinline__ void store_bf16_rows(uint8_t *panel, uint4 (&u)[4], uint32_t r, uint32_t ch0,
                                                uint64_t policy = 0) {
  const uint32_t lane = r & 31u, base = r & ~31u;
  const bool b0 = lane & 1u, b1 = lane & 2u;
#pragma unroll
  for (int p = 0; p < 4; p += 2) {                 // stage 1: pairs (xor 1)
    const uint4 recv = shfl_xor_u4(b0 ? u[p] : u[p + 1], 1);
    if (b0) u[p] = recv; else u[p + 1] = recv;
  }
#pragma unroll
  for (int p = 0; p < 2; p++) {                    // stage 2: pairs of pairs (xor 2)
    const uint4 recv = shfl_xor_u4(b1 ? u[p] : u[p + 2], 2);
    if (b1) u[p] = recv; else u[p + 2] = recv;
  }
  // lane now holds chunk c = lane & 3 of rows 4*(lane>>2) + k, k = 0..3
  const uint32_t c = ch0 + (lane & 3u), g = base + 4u * (lane >> 2);
#pragma unroll
  for (int k = 0; k < 4; k++) {
    if (kStream) ptx::st_global_v4_hint(panel + swz(g + k, c), u[k], policy);
    else *reinterpret_cast<uint4 *>(panel + swz(g + k, c)) = u[k];
  }
}

__device__ __forceinline__ void named_bar(uint32_t id, uint32_t n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// ---------------------------------------------------------------------------
// Decode (lane 0 of the decoder warp, from the smem copy of the DevJob).
// Stage numbering: 0 INIT, 1 GEN, 2..L+1 F_1..F_L, L+2.. B_L..B_1.
// Page translations are only recorded here (defer) and resolved by the
// decoder warp's lanes in parallel.
// ---------------------------------------------------------------------------
// A task is a pair task: CTA h takes block 2t + h of INIT / GEN, and M block
// 2 mp + h of a GEMM super-tile (the N block is shared).
// The slot's in-flight record as the decoder sees it (two vector loads).
struct SlotHead { uint32_t job, iter; uint64_t seq, lseq; };

__device__ __forceinline__ SlotHead load_slot_head(const Slot &sl) {
  static_assert(offsetof(Slot, job) == 0 && offsetof(Slot, iter) == 4 && offsetof(Slot, seq) == 8 &&
                offsetof(Slot, lseq) == 16, "Slot head layout");
  uint4 a;
  uint2 b;
  asm volatile("ld.relaxed.gpu.global.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w) : "l"(&sl) : "memory");
  asm volatile("ld.relaxed.gpu.global.v2.u32 {%0, %1}, [%2];"
               : "=r"(b.x), "=r"(b.y) : "l"(reinterpret_cast<const uint8_t *>(&sl) + 16) : "memory");
  SlotHead hd;
  hd.job = a.x; hd.iter = a.y;
  hd.seq = ((uint64_t)a.w << 32) | a.z;
  hd.lseq = ((uint64_t)b.y << 32) | b.x;
  return hd;
}

// A GEN tile: CTA h generates 128 x 128 block 2 tile + h of X_kx (or, with
// `targets`, of the MSE targets T_kx; A29) into the panels at byte offset
// `off` of the space `table` translates.
__device__ __forceinline__ void decode_gen(TileDesc &td, const DevJob &J, uint32_t tile, uint32_t h,
                                           const uint32_t *table, uint32_t off, uint32_t kx, bool targets = false) {
  td.kind = T_GEN;
  const uint32_t bp = J.bpad, L = J.n_layers, d = targets ? L : 0;
  const uint32_t ncb = J.dpad[d] / 128, blk = 2 * tile + h, mb = blk / ncb, cb = blk % ncb;
  if (mb >= bp / 128) { td.valid = 0; return; }
  td.m0 = mb * 128; td.n0 = cb * 128;
  td.rows_valid = J.batch; td.cols_valid = J.dims[d];
  for (uint32_t q = 0; q < 2; q++) defer(td, PTR_OUT + q, table, off + (2 * cb + q) * bp * 128u + mb * 16384u);
  td.key = targets ? gen_key(J.seed, J.job_id, GEN_T, L, kx) : gen_key(J.seed, J.job_id, GEN_X, 0, kx);
}

// split-K: the partial pages of every slice of base tile u, CTA half h
// (np = N / 128 pages per partial) -- the last slice reads them all
__device__ __forceinline__ void defer_partials(TileDesc &td, const uint32_t *lt, uint32_t ws_off, uint32_t u,
                                               uint32_t h, uint32_t S, uint32_t np) {
  for (uint32_t q = 0; q < S; q++)
    for (uint32_t p = 0; p < np; p++)
      if (sk_ptr(q * np + p) < NPTR) defer(td, sk_ptr(q * np + p), lt, ws_off + (((2 * u + h) * S + q) * np + p) * 65536u);
}

__device__ void decode_task(const Params &P, uint32_t payload, const DevJob &J, const SlotHead &sl,
                            TileDesc &td, uint32_t h) {
  td.payload = payload;
  const uint32_t slot = payload >> 26, stage = (payload >> 21) & 31u, tile = payload & ((1u << 21) - 1);
  const uint32_t k = sl.iter & ~ITER_FLAG_BITS;       // this context's iteration index
  const uint32_t kg = k + J.iter_base;                // the job's own (migration, NEXT-4)
  const uint32_t L = J.n_layers, bp = J.bpad;
  td.slot = slot; td.stage = stage; td.job = sl.job; td.iter = k; td.seq = sl.seq; td.lseq = sl.lseq;
  td.eager = 0; td.wait = 0;
  td.first_stage = stage >= STAGE_SWAP_OUT ? stage
                   : (k == 0 && !(J.dump & DUMP_INTERNAL_RESUME)) ? 0u : (J.xpre ? 2u : 1u);
  // latency mode (eager record): eager publication, narrow tiles on the
  // stages lat_narrow marks, relaxed backward barrier for relax jobs
  const bool lat = (sl.iter & ITER_EAGER_BIT) != 0 && stage < STAGE_SWAP_OUT;
  const bool narrow = lat && (sl.iter & ITER_NARROW_BIT) != 0;
  const bool relaxed = lat && J.relax && J.kind == SALUS_TRAIN && L >= 2;
  const uint32_t lastS = last_stage(J.kind, L);
  td.eager = lat;
  td.ntiles = stage_ntiles(J, stage, narrow);
  td.is_last = stage >= STAGE_SWAP_OUT || (stage == lastS && !relaxed);
  // relaxed: B_2 and B_1 may finish in either order; the second to finish ends the record
  td.end2 = relaxed && stage + 1 >= lastS;
  td.dx_ctr = 0;
  td.next_stage = stage == lastS || stage >= STAGE_SWAP_OUT ? 0 : next_stage(J, stage);
  if (td.eager && td.next_stage) {
    // the successor was published with this stage: publish the one after it
    td.next_stage = td.next_stage == lastS ? 0 : next_stage(J, td.next_stage);
  }
  td.next_ntiles = td.next_stage ? stage_ntiles(J, td.next_stage, narrow) : 0;
  // relaxed: stage u >= L+5 is published on the completions of u-2 and u-3
  td.next_tk = relaxed && td.next_stage >= L + 5;
  td.next2_stage = relaxed && stage >= L + 2 && stage + 3 <= lastS ? stage + 3 : 0;
  td.next2_ntiles = td.next2_stage ? stage_ntiles(J, td.next2_stage, narrow) : 0;
  // every stage of an eager record but its first was published while its
  // predecessor ran: wait for it before touching what it produces -- in a
  // relaxed record, a backward stage after B_L waits only for its
  // predecessor's dX tiles (counter dx_counter), which produce its G input
  td.wait = td.eager && stage != td.first_stage;
  td.dep_stage = td.wait ? (uint8_t)prev_stage(J, stage) : 0;
  td.dep_want = td.wait ? 2 * stage_ntiles(J, td.dep_stage, narrow) : 0;
  if (td.wait && relaxed && stage > L + 2) {
    const uint32_t lp = L - (td.dep_stage - (L + 2));            // the predecessor is B_lp
    const uint32_t Np = narrow && ((J.lat_narrow >> td.dep_stage) & 1u) ? 128u : ntile_for(J.dpad[lp - 1]);
    const uint32_t nWp = ((J.dpad[lp] / 128 + 1) / 2) * (J.dpad[lp - 1] / Np);
    td.dep_want = 2 * (stage_ntiles(J, td.dep_stage, narrow) - nWp);
    td.dep_stage = (uint8_t)dx_counter(L, td.dep_stage);
  }
  td.dump_off = -1;
  td.n_ech = 0;
  td.xt_mask = 0;
  td.xt_sel = 0;
  td.swap = 0; td.ech_load = 1; td.kd = 0; td.sk = 1; td.skz = 0; td.sku = 0;
  td.valid = 1;
  td.ptr[PTR_W32] = nullptr;
  const uint32_t *lt = P.lpt + (uint64_t)slot * P.lpt_stride;   // lane (ephemeral) space
  const uint32_t *jt = P.ppt + J.pt_off;                        // job (persistent) space
  td.xt_tab[0] = lt;
  td.xt_tab[1] = jt;

  if (stage >= STAGE_SWAP_OUT) {                      // A35 swap: CTA h copies page 2 tile + h
    td.kind = T_COPY;
    const uint32_t pg = 2 * tile + h;
    td.valid = pg < J.ap_pages;
    td.m0 = pg;
    if (td.valid) {
      uint8_t *dev = P.arena + ((uint64_t)jt[pg] << PAGE_SHIFT);
      uint8_t *host = P.swap + ((uint64_t)(J.pt_off + pg) << PAGE_SHIFT);
      td.ptr[PTR_OUT] = stage == STAGE_SWAP_OUT ? host : dev;      // destination
      td.ptr[PTR_OUT + 1] = stage == STAGE_SWAP_OUT ? dev : host;  // source
    }
    return;
  }
  // GEN-prefetch jobs: the INIT stage (X_k) and the F_1 stage (X_{k+1}) end
  // with the GEN tiles of stage 1's shape, into the per-job X buffers
  if (J.xpre && (stage == 0 || stage == 2)) {
    const uint32_t ngx = J.stage_tiles[1], base = stage_ntiles(J, stage, narrow) - ngx - J.t_gen_tiles;
    const uint32_t kx = stage == 0 ? kg : kg + 1;
    if (tile >= base + ngx) { decode_gen(td, J, tile - base - ngx, h, jt, J.t_off[kx & 1], kx, true); return; }
    if (tile >= base) { decode_gen(td, J, tile - base, h, jt, J.x_off[kx & 1], kx); return; }
  }
  if (stage == 0) {                                   // INIT weights (128 x 128 blocks)
    td.kind = T_INIT;
    uint32_t t = 2 * tile + h, l = 1;
    for (; l <= L; l++) {
      const uint32_t nb = (J.dpad[l] / 128) * (J.dpad[l - 1] / 128);
      if (t < nb) break;
      t -= nb;
    }
    if (l > L) { td.valid = 0; return; }
    const uint32_t nib = J.dpad[l - 1] / 128, jb = t / nib, ib = t % nib;
    td.layer = l; td.m0 = jb * 128; td.n0 = ib * 128;
    td.rows_valid = J.dims[l]; td.cols_valid = J.dims[l - 1];
    // inference jobs keep only the bf16 copy (2 B/param): no fp32 master
    if (J.kind == SALUS_TRAIN)
      defer(td, PTR_W32, jt, J.w32_off[l - 1] + (jb * (J.dpad[l - 1] / 4) + 32 * ib) * 2048u);
    for (uint32_t q = 0; q < 2; q++)
      defer(td, PTR_AUX + q, jt, J.wb_off[l - 1][0] + (2 * ib + q) * J.dpad[l] * 128u + jb * 16384u);
    td.key = gen_key(J.seed, J.job_id, GEN_W, l, 0);
    td.scale = gen_wscale(J.dims[l - 1]);
    return;
  }
  if (stage == 1) {                                   // GEN input batch X (128 x 128 blocks)
    const uint32_t ngx = J.stage_tiles[1] - J.t_in_g;
    if (tile >= ngx) decode_gen(td, J, tile - ngx, h, lt, J.g_off[0], kg, true);   // T_k into G (t_in_g)
    else decode_gen(td, J, tile, h, lt, J.act_off[0], kg);
    return;
  }
  // where X_k is read from: the lane (GEN stage) or the job's prefetch buffer
  const uint32_t *xt = J.xpre ? jt : lt;
  const uint32_t xo = J.xpre ? J.x_off[kg & 1] : J.act_off[0];
  td.kind = T_GEMM;
  // K9 tiles (inference requests of b <= 128) except in narrow records,
  // whose non-transposed N = 128 tiles give a skinny stage twice the tasks
  const bool swap = !narrow && ((J.swap_mask >> stage) & 1u);
  if (stage <= L + 1 && swap) {                       // K9 forward F_l^T = W_l^T A_{l-1}^T
    const uint32_t l = stage - 1, mb = 2 * tile + h;
    td.swap = 1;
    td.valid = mb < J.dpad[l] / 128;
    td.peer_valid = (mb | 1u) < J.dpad[l] / 128;
    td.layer = l; td.N = bp; td.nk = J.dpad[l - 1] / 64;
    // A: 128 rows (output features) of W_l^T, K-major; B: this CTA's 64 batch rows, K-major
    td.a = OpDesc{jt, J.wb_off[l - 1][kg & 1], J.dpad[l], mb * 128, 0};
    td.b = l == 1 ? OpDesc{xt, xo, bp, h * 64, 0} : OpDesc{lt, J.act_off[l - 1], bp, h * 64, 0};
    td.m0 = mb * 128; td.n0 = 0;
    td.rows_valid = J.dims[l]; td.cols_valid = J.batch; td.ld_logical = J.dims[l];
    uint32_t out_off;
    td.ech_load = 0;
    if (l < L) { td.epi = EPI_RELU; out_off = J.act_off[l]; }
    else if (J.kind == SALUS_TRAIN) {
      td.epi = EPI_LOSS; out_off = J.g_off[0];
      td.key = gen_key(J.seed, J.job_id, GEN_T, L, kg);
      if (J.t_gen_tiles && td.valid) {                 // prefetched T_k: the block's 2 target panels
        for (uint32_t q = 0; q < 2; q++) defer(td, PTR_EPI + q, jt, J.t_off[kg & 1] + (2 * mb + q) * bp * 128u);
        td.ech_load = 1;
      }
    } else { td.epi = EPI_OUT; out_off = J.act_off[L]; }
    if (td.valid) {
      if (l == L && (J.dump & SALUS_DUMP_OUTPUTS))
        td.dump_off = (int64_t)(J.dump_out_off + (uint64_t)k * J.batch * J.dims[L]);
      for (uint32_t q = 0; q < 2; q++) defer(td, PTR_OUT + q, lt, out_off + (2 * mb + q) * bp * 128u);
      td.n_ech = 1;                                    // the output block's staging chunk
    }
  } else if (stage <= L + 1) {                        // forward F_l
    const uint32_t l = stage - 1;
    const uint32_t S = (SALUS_SPLITK_BUILD && narrow) ? J.splitk[stage] : 1u;
    const uint32_t N = S > 1 ? (((J.sk_wide >> stage) & 1u) ? 256u : 128u)
                             : (narrow && ((J.lat_narrow >> stage) & 1u)) ? 128u : ntile_for(J.dpad[l]);
    const uint32_t ntn = J.dpad[l] / N, z = tile % S, u = tile / S;
    const uint32_t mb = 2 * (u / ntn) + h, nb = u % ntn;
    td.valid = mb < bp / 128;
    td.peer_valid = (mb | 1u) < bp / 128;
    td.layer = l; td.N = N; td.nk = J.dpad[l - 1] / 64 / S;
    // K-slice z: chunks [z nk, (z+1) nk) of both K-major operands
    const uint32_t kc0 = z * td.nk;
    td.a = l == 1 ? OpDesc{xt, xo + kc0 * bp * 128u, bp, mb * 128, 0}
                  : OpDesc{lt, J.act_off[l - 1] + kc0 * bp * 128u, bp, mb * 128, 0};
    td.b = OpDesc{jt, J.wb_off[l - 1][kg & 1] + kc0 * J.dpad[l] * 128u, J.dpad[l], nb * N + h * (N / 2), 0};
    if (S > 1) {
      td.sk = (uint8_t)S; td.skz = (uint8_t)z; td.sku = (uint16_t)u;
      if (td.valid) defer_partials(td, lt, J.ws_off, u, h, S, N / 128);
    }
    td.m0 = mb * 128; td.n0 = nb * N;
    td.rows_valid = J.batch; td.cols_valid = J.dims[l]; td.ld_logical = J.dims[l];
    uint32_t out_off;
    if (l < L) { td.epi = EPI_RELU; out_off = J.act_off[l]; }
    else if (J.kind == SALUS_TRAIN) {
      td.epi = EPI_LOSS; out_off = J.g_off[0];
      td.key = gen_key(J.seed, J.job_id, GEN_T, L, kg);
      if (J.t_gen_tiles && td.valid) {               // prefetched T_k: 2 target panels per input chunk
        for (uint32_t q = 0; q < N / 64; q++)
          defer(td, PTR_EPI + q, jt, J.t_off[kg & 1] + (nb * N / 64 + q) * bp * 128u + mb * 16384u);
        td.n_ech = N / 128;
      } else if (J.t_in_g && td.valid) {             // T_k from this record's GEN stage, in G_L's place
        for (uint32_t q = 0; q < N / 64; q++)
          defer(td, PTR_EPI + q, lt, J.g_off[0] + (nb * N / 64 + q) * bp * 128u + mb * 16384u);
        td.n_ech = N / 128;
      }
    } else { td.epi = EPI_OUT; out_off = J.act_off[L]; }
    if (td.valid) {
      if (l == L && (J.dump & SALUS_DUMP_OUTPUTS))
        td.dump_off = (int64_t)(J.dump_out_off + (uint64_t)k * J.batch * J.dims[L]);
      for (uint32_t q = 0; q < N / 64; q++)
        defer(td, PTR_OUT + q, lt, out_off + (td.n0 / 64 + q) * bp * 128u + mb * 16384u);
    }
  } else {                                            // backward B_l
    const uint32_t tile_in = tile;
    const uint32_t l = L - (stage - (L + 2));
    const uint32_t Nw = narrow && ((J.lat_narrow >> stage) & 1u) ? 128u : ntile_for(J.dpad[l - 1]);
    const uint32_t S = (SALUS_SPLITK_BUILD && narrow) ? J.splitk[stage] : 1u;   // K-slices of the dX part
    const uint32_t nW = ((J.dpad[l] / 128 + 1) / 2) * (J.dpad[l - 1] / Nw);     // dW pair tasks
    // G_l lives in buffer (L - l) mod 2, or mod 3 in a relaxed record
    const uint32_t g3[3] = {J.g_off[0], J.g_off[1], J.g_off3};
    const uint32_t gin = relaxed ? g3[(L - l) % 3] : J.g_off[(L - l) & 1];
    const uint32_t gout = relaxed ? g3[(L - l + 1) % 3] : J.g_off[(L - l + 1) & 1];
    td.layer = l;
    // the long-K dX tiles take the stage's first task indices, so they are
    // claimed first (longest first within the stage)
    const uint32_t nX = td.ntiles - nW;
    if (relaxed && tile_in < nX) td.dx_ctr = dx_counter(L, stage);
    const uint32_t tile = tile_in < nX ? nW + tile_in : tile_in - nX;
    if (tile < nW) {                                  // dW_l^T = G_l^T A_{l-1}; SGD
      const uint32_t N = Nw, ntn = J.dpad[l - 1] / N;
      td.N = N;
      const uint32_t mb = 2 * (tile / ntn) + h, nb = tile % ntn;
      td.valid = mb < J.dpad[l] / 128;
      td.peer_valid = (mb | 1u) < J.dpad[l] / 128;
      td.epi = EPI_SGD; td.nk = bp / 64;
      td.a = OpDesc{lt, gin, bp, mb * 128, 1};
      td.b = l == 1 ? OpDesc{xt, xo, bp, nb * N + h * (N / 2), 1}
                    : OpDesc{lt, J.act_off[l - 1], bp, nb * N + h * (N / 2), 1};
      td.m0 = mb * 128; td.n0 = nb * N;
      td.rows_valid = J.dims[l]; td.cols_valid = J.dims[l - 1]; td.ld_logical = J.dims[l];
      td.lr = J.lr;
      // the 128 x N fp32 master tile is N/128 contiguous 64 KiB pages
      // (j-blocked layout), streamed to the epilogue in 64-column chunks
      const uint32_t w32 = J.w32_off[l - 1] + (mb * (J.dpad[l - 1] / 4) + nb * N / 4) * 2048u;
      if (td.valid) {
        for (uint32_t q = 0; q < N / 128; q++) defer(td, PTR_W32 + q, jt, w32 + q * 65536u);
        td.n_ech = N / 64;
        for (uint32_t q = 0; q < N / 64; q++)
          defer(td, PTR_AUX + q, jt, J.wb_off[l - 1][(kg + 1) & 1] + (td.n0 / 64 + q) * J.dpad[l] * 128u + mb * 16384u);
      }
      const bool wsteps = (J.dump & SALUS_DUMP_WEIGHT_STEPS) != 0;
      if (td.valid && (wsteps || ((J.dump & SALUS_DUMP_WEIGHTS) && k + 1 == J.n_iters))) {
        uint64_t base = J.dump_w_off + (wsteps ? (uint64_t)k * J.w_count : 0);
        for (uint32_t q = 1; q < l; q++) base += (uint64_t)J.dims[q - 1] * J.dims[q];
        td.dump_off = (int64_t)base;
      }
    } else {                                          // G_{l-1} = (G_l W_l^T) * [A_{l-1} > 0]
      const uint32_t N = S > 1 ? (((J.sk_wide >> stage) & 1u) ? 256u : 128u) : Nw, ntn = J.dpad[l - 1] / N;
      td.N = N;
      const uint32_t ux = tile - nW, z = ux % S, u = ux / S, mb = 2 * (u / ntn) + h, nb = u % ntn;
      td.valid = mb < bp / 128;
      td.peer_valid = (mb | 1u) < bp / 128;
      td.epi = EPI_DX; td.nk = J.dpad[l] / 64 / S;
      // K-slice z: A (G, K-major) chunks [z nk, +nk), B (W, MN-major) rows of the panels
      const uint32_t kc0 = z * td.nk;
      td.a = OpDesc{lt, gin + kc0 * bp * 128u, bp, mb * 128, 0};
      td.b = OpDesc{jt, J.wb_off[l - 1][kg & 1] + kc0 * 8192u, J.dpad[l], nb * N + h * (N / 2), 1};
      if (S > 1) {
        td.sk = (uint8_t)S; td.skz = (uint8_t)z; td.sku = (uint16_t)u;
        if (td.valid) defer_partials(td, lt, J.ws_off, u, h, S, N / 128);
      }
      td.m0 = mb * 128; td.n0 = nb * N;
      td.rows_valid = J.batch; td.cols_valid = J.dims[l - 1];
      if (td.valid) {
        for (uint32_t q = 0; q < N / 64; q++) {
          defer(td, PTR_OUT + q, lt, gout + (td.n0 / 64 + q) * bp * 128u + mb * 16384u);
          defer(td, PTR_EPI + q, lt, J.act_off[l - 1] + (td.n0 / 64 + q) * bp * 128u + mb * 16384u);
        }
        td.n_ech = N / 128;                           // 2 mask panels (32 KiB) per chunk
      }
    }
  }
  // this CTA's A is M = 128 rows (none if its half is empty); its B is N/2
  // rows (K-major, 64 or 128 rows per copy) or N/128 panels (MN-major)
  const uint32_t nh = td.N / 2;
  td.ncopy_a = td.valid ? (td.a.mn ? 2 : 1) : 0;
  td.peer_nca = td.peer_valid ? (td.a.mn ? 2 : 1) : 0;
  td.abytes = td.a.mn ? 8192u : 16384u;
  td.ncopy_b = td.b.mn ? nh / 64 : (nh + 127) / 128;
  td.bbytes = td.b.mn ? 8192u : (nh >= 128 ? 16384u : nh * 128u);
  td.idesc = ptx::idesc_bf16(256, td.N, td.a.mn, td.b.mn);
  td.kd = SALUS_KD && td.b.mn && !td.swap;
}

// global byte offset (inside the operand's space) of copy q of K-chunk kc
__device__ __forceinline__ uint32_t copy_off(const OpDesc &o, uint32_t kc, uint32_t q) {
  return o.mn ? o.off + (o.start / 64 + q) * o.R * 128u + kc * 8192u
              : o.off + kc * o.R * 128u + (o.start + 128 * q) * 128u;
}

// ---------------------------------------------------------------------------
// Epilogue over accumulator column blocks [cc0, cc1) (32 columns each):
// thread r of an epilogue warp owns accumulator row r (TMEM lane r, warp % 4
// = lane quarter).  `buf` is the smem epilogue-input chunk holding the W32
// columns [32*ccb, +64) (SGD) or the mask columns [32*ccb, +128) (DX).
// ---------------------------------------------------------------------------
struct EpiView {   // register copy of the descriptor fields the epilogue uses
  uint32_t m0, n0, rows_valid, cols_valid, ld_logical, epi;
  float lr;
  uint64_t key;
  int64_t dump_off;
};

__device__ void epilogue_cols(const Params &P, const TileDesc &tds, const EpiView &td, uint32_t tacc,
                              uint32_t r, uint32_t ccb, uint32_t cc0, uint32_t cc1, uint8_t *buf) {
  const uint32_t qw = r >> 5;
  const uint32_t row = td.m0 + r;
  const bool row_ok = row < td.rows_valid;
  float *dump = td.dump_off >= 0 ? P.dump + td.dump_off : nullptr;
#pragma unroll 1
  for (uint32_t cc = cc0; cc < cc1; cc++) {
    uint32_t raw[32];
    ptx::tmem_ld32(tacc + ((qw * 32u) << 16) + cc * 32u, raw);
    ptx::tmem_ld_wait();
    float v[32];
#pragma unroll
    for (int x = 0; x < 32; x++) v[x] = __uint_as_float(raw[x]);
    const uint32_t col0 = td.n0 + cc * 32;
    const uint32_t pan = cc >> 1, ch0 = (cc & 1) * 4;
    if (td.epi == EPI_SGD) {
      // rows are j (d_l), columns i (d_{l-1}): W32[j][i] -= lr * dW^T[j][i]
#if SALUS_L2HINT
      const uint64_t pol_stream = ptx::policy_evict_first();   // masters + Wb: streamed
#endif
#pragma unroll
      for (int g = 0; g < 8; g++) {
        const uint32_t grp = cc * 8 + g;                    // float4 column group in the tile
        const float4 *wp = reinterpret_cast<const float4 *>(buf + ((cc - ccb) * 8 + g) * 2048u + r * 16u);
        float4 w = *wp;
        w.x = fmaf(-td.lr, v[4 * g + 0], w.x);
        w.y = fmaf(-td.lr, v[4 * g + 1], w.y);
        w.z = fmaf(-td.lr, v[4 * g + 2], w.z);
        w.w = fmaf(-td.lr, v[4 * g + 3], w.w);
#if SALUS_W32_BULK
        // updated in place: the chunk goes back to HBM as one bulk store
        // (epilogue_warps) instead of 128 KiB of register stores per tile
        *const_cast<float4 *>(wp) = w;
        (void)grp;
#elif SALUS_L2HINT
        ptx::st_global_v4_hint(tds.ptr[PTR_W32 + (grp >> 5)] + (grp & 31u) * 2048u + r * 16u,
                               make_uint4(__float_as_uint(w.x), __float_as_uint(w.y), __float_as_uint(w.z),
                                          __float_as_uint(w.w)),
                               pol_stream);
#else
        *reinterpret_cast<float4 *>(tds.ptr[PTR_W32 + (grp >> 5)] + (grp & 31u) * 2048u + r * 16u) = w;
#endif
        v[4 * g + 0] = w.x; v[4 * g + 1] = w.y; v[4 * g + 2] = w.z; v[4 * g + 3] = w.w;
      }
      {
        uint4 u[4];
#pragma unroll
        for (int q = 0; q < 4; q++) {
          u[q].x = pack_bf16x2(v[8 * q + 0], v[8 * q + 1]);
          u[q].y = pack_bf16x2(v[8 * q + 2], v[8 * q + 3]);
          u[q].z = pack_bf16x2(v[8 * q + 4], v[8 * q + 5]);
          u[q].w = pack_bf16x2(v[8 * q + 6], v[8 * q + 7]);
        }
#if SALUS_WB_BULK
        // into the chunk's staging panel (the global panel's exact image)
        {
          uint8_t *stg = buf + ECH_BYTES;
#pragma unroll
          for (int q = 0; q < 4; q++) *reinterpret_cast<uint4 *>(stg + swz(r, ch0 + q)) = u[q];
          (void)pan;
        }
#elif SALUS_L2HINT
        store_bf16_rows<true>(tds.ptr[PTR_AUX + pan], u, r, ch0, pol_stream);
#else
        store_bf16_rows(tds.ptr[PTR_AUX + pan], u, r, ch0);
#endif
      }
      if (dump && row_ok) {                     // W[i][j], logical d_{l-1} x d_l
        for (int x = 0; x < 32; x++)
          if (col0 + x < td.cols_valid) dump[(uint64_t)(col0 + x) * td.ld_logical + row] = v[x];
      }
      continue;
    }
    if (td.epi == EPI_DX) {
      const uint8_t *mp = buf + ((cc - ccb) >> 1) * 16384u;
#pragma unroll
      for (int q = 0; q < 4; q++) {
        const uint4 m = *reinterpret_cast<const uint4 *>(mp + swz(r, ch0 + q));
        const uint32_t w[4] = {m.x, m.y, m.z, m.w};
#pragma unroll
        for (int hh = 0; hh < 4; hh++) {
          const uint32_t lo = w[hh] & 0xFFFFu, hi = w[hh] >> 16;
          if (!((lo & 0x8000u) == 0 && (lo & 0x7FFFu) != 0)) v[8 * q + 2 * hh] = 0.f;
          if (!((hi & 0x8000u) == 0 && (hi & 0x7FFFu) != 0)) v[8 * q + 2 * hh + 1] = 0.f;
        }
      }
    } else {
      if (dump && row_ok) {
        for (int x = 0; x < 32; x++)
          if (col0 + x < td.cols_valid) dump[(uint64_t)row * td.ld_logical + col0 + x] = v[x];
      }
      if (td.epi == EPI_RELU) {
#pragma unroll
        for (int x = 0; x < 32; x++) v[x] = row_ok ? fmaxf(v[x], 0.f) : 0.f;
      } else if (td.epi == EPI_OUT) {
#pragma unroll
        for (int x = 0; x < 32; x++) v[x] = row_ok ? v[x] : 0.f;
      } else if (buf) {  // EPI_LOSS with T prefetched (bf16 panels, exact: A29 values are bf16)
        const float inv_b = 1.0f / (float)td.rows_valid;
        const int ncol = row_ok ? (int)td.cols_valid - (int)col0 : 0;
        const uint8_t *tp = buf + ((cc - ccb) >> 1) * 16384u;
#pragma unroll
        for (int q = 0; q < 4; q++) {
          const uint4 m = *reinterpret_cast<const uint4 *>(tp + swz(r, ch0 + q));
          const uint32_t w[4] = {m.x, m.y, m.z, m.w};
#pragma unroll
          for (int hh = 0; hh < 4; hh++) {
            const int x0 = 8 * q + 2 * hh;
            const float t0 = __uint_as_float(w[hh] << 16), t1 = __uint_as_float(w[hh] & 0xFFFF0000u);
            v[x0] = x0 < ncol ? (v[x0] - t0) * inv_b : 0.f;
            v[x0 + 1] = x0 + 1 < ncol ? (v[x0 + 1] - t1) * inv_b : 0.f;
          }
        }
      } else {  // EPI_LOSS: G_L = (A_L - T) / B  (MSE)
        // branch-free so the 32 independent hash chains interleave (ILP)
        const float inv_b = 1.0f / (float)td.rows_valid;
        const uint64_t key = td.key, base = (uint64_t)row * td.ld_logical + col0;
        const int ncol = row_ok ? (int)td.cols_valid - (int)col0 : 0;
        if ((base & 1) == 0) {          // one hash per element pair (A29)
#pragma unroll
          for (int p = 0; p < 16; p++) {
            const uint64_t hv = splitmix64(key ^ ((base >> 1) + p));
            const float t0 = gen_from_bits((uint32_t)(hv >> 40), 1.0f);
            const float t1 = gen_from_bits((uint32_t)(hv >> 16) & 0xFFFFFFu, 1.0f);
            v[2 * p] = 2 * p < ncol ? (v[2 * p] - t0) * inv_b : 0.f;
            v[2 * p + 1] = 2 * p + 1 < ncol ? (v[2 * p + 1] - t1) * inv_b : 0.f;
          }
        } else {
#pragma unroll
          for (int x = 0; x < 32; x++) {
            const float gl = (v[x] - gen_value(key, base + x, 1.0f)) * inv_b;
            v[x] = x < ncol ? gl : 0.f;
          }
        }
      }
    }
    uint4 u[4];
#pragma unroll
    for (int q = 0; q < 4; q++) {
      u[q].x = pack_bf16x2(v[8 * q + 0], v[8 * q + 1]);
      u[q].y = pack_bf16x2(v[8 * q + 2], v[8 * q + 3]);
      u[q].z = pack_bf16x2(v[8 * q + 4], v[8 * q + 5]);
      u[q].w = pack_bf16x2(v[8 * q + 6], v[8 * q + 7]);
    }
    store_bf16_rows(tds.ptr[PTR_OUT + pan], u, r, ch0);
  }
}

// K9 transposed tile: TMEM lane r = output feature m0 + r, column c = batch
// row c (N = the 128-row padded batch).  The output block (2 panels of the
// batch-row-major tensor: 128 rows x 64 features each, 16 KiB) is staged in
// the tile's epilogue-input chunk (an input chunk -- a mask or prefetched
// loss targets -- would be read and overwritten in place element by element)
// and copied out by all epilogue threads with 16-byte stores.  `hh` = this
// warp's column half.
__device__ __forceinline__ uint32_t swap_off(uint32_t r, uint32_t b) {
  return (r >> 6) * 16384u + swz(b, (r & 63u) >> 3) + (r & 7u) * 2u;
}

__device__ void epilogue_swap(const Params &P, WorkerSmem &W, const TileDesc &td, uint32_t tacc, uint32_t r,
                              uint32_t hh, uint32_t et, uint32_t lane, uint32_t &e, uint32_t &e_phase) {
  const uint32_t taddr = tacc + (((r >> 5) * 32u) << 16);
  const uint32_t ncc = td.N / 32, sub = ncc / EPI_HALVES, cc0 = hh * sub;
  ptx::mbar_wait_abortable(&W.epi_full[e], e_phase, &P.ctrl->abort);
  uint8_t *buf = W.epi_in[e];
  const uint32_t f = td.m0 + r;
  const bool fok = f < td.rows_valid;
  const uint32_t batch = td.cols_valid;
  const float inv_b = 1.0f / (float)batch;
  float *dump = td.dump_off >= 0 ? P.dump + td.dump_off : nullptr;
  for (uint32_t cc = cc0; cc < cc0 + sub; cc++) {
    uint32_t raw[32];
    ptx::tmem_ld32(taddr + cc * 32u, raw);
    ptx::tmem_ld_wait();
#pragma unroll 4
    for (int x = 0; x < 32; x++) {
      const float v = __uint_as_float(raw[x]);
      const uint32_t b = cc * 32 + x;
      const bool ok = fok && b < batch;
      uint16_t *slot16 = reinterpret_cast<uint16_t *>(buf + swap_off(r, b));
      float y;
      if (td.epi == EPI_DX) {
        const uint32_t m = *slot16;
        y = ((m & 0x8000u) == 0 && (m & 0x7FFFu) != 0) ? v : 0.f;
      } else {
        if (dump && ok) dump[(uint64_t)b * td.ld_logical + f] = v;
        if (td.epi == EPI_RELU) y = ok ? fmaxf(v, 0.f) : 0.f;
        else if (td.epi == EPI_OUT) y = ok ? v : 0.f;
        else {                                          // EPI_LOSS: G_L = (A_L - T) / B
          const float t = td.ech_load ? __uint_as_float((uint32_t)*slot16 << 16)
                                      : gen_value(td.key, (uint64_t)b * td.ld_logical + f, 1.0f);
          y = ok ? (v - t) * inv_b : 0.f;
        }
      }
      __nv_bfloat16 hb = __float2bfloat16_rn(y);
      *slot16 = *reinterpret_cast<uint16_t *>(&hb);
    }
  }
  named_bar(1, EPI_THREADS);                            // the block is staged
#pragma unroll
  for (uint32_t k = 0; k < 2 * 16384u / (16u * EPI_THREADS); k++) {
    const uint32_t o = (k * EPI_THREADS + et) * 16u;
    const uint4 val = *reinterpret_cast<const uint4 *>(buf + o);
    uint8_t *dst = o < 16384u ? td.ptr[PTR_OUT] + o : td.ptr[PTR_OUT + 1] + (o - 16384u);
    *reinterpret_cast<uint4 *>(dst) = val;
  }
  __syncwarp();
  if (lane == 0) ptx::mbar_arrive(&W.epi_empty[e]);
  if (++e == EBUF) { e = 0; e_phase ^= 1; }
}

// INIT: W_l block (rows j = m0 + r of W^T storage, 128 columns i)
__device__ void init_tile(const TileDesc &td, uint32_t r, uint32_t h) {
  // descriptor fields in registers: global stores below may alias smem for
  // the compiler, which would otherwise reload them after every store
  const uint32_t j = td.m0 + r, n0 = td.n0, rows = td.rows_valid, cols = td.cols_valid;
  const uint64_t key = td.key;
  const float scale = td.scale;
  uint8_t *const w32 = td.ptr[PTR_W32];
  uint8_t *const aux0 = td.ptr[PTR_AUX], *const aux1 = td.ptr[PTR_AUX + 1];
  const int ncol = j < rows ? (int)cols - (int)n0 : 0;
#pragma unroll 2
  for (uint32_t cg = h * (128 / EPI_HALVES); cg < (h + 1) * (128 / EPI_HALVES); cg += 8) {
    float v[8];
#pragma unroll
    for (int x = 0; x < 8; x++) {
      const uint32_t i = n0 + cg + x;
      const float g = gen_value(key, (uint64_t)i * rows + j, scale);
      v[x] = (int)(cg + x) < ncol ? g : 0.f;
    }
    // W32 j-blocked layout: ((j/128)*(dp_in/4) + i/4)*2048 + (j%128)*16 + (i%4)*4
    if (w32) {
      *reinterpret_cast<float4 *>(w32 + (cg / 4) * 2048u + r * 16u) = make_float4(v[0], v[1], v[2], v[3]);
      *reinterpret_cast<float4 *>(w32 + (cg / 4 + 1) * 2048u + r * 16u) = make_float4(v[4], v[5], v[6], v[7]);
    }
    uint4 u;
    u.x = pack_bf16x2(v[0], v[1]); u.y = pack_bf16x2(v[2], v[3]);
    u.z = pack_bf16x2(v[4], v[5]); u.w = pack_bf16x2(v[6], v[7]);
    *reinterpret_cast<uint4 *>((cg < 64 ? aux0 : aux1) + swz(r, (cg % 64) / 8)) = u;
  }
}

// GEN: X block (rows m = m0 + r, 128 columns)
__device__ void gen_tile(const TileDesc &td, uint32_t r, uint32_t h) {
  const uint32_t m = td.m0 + r, n0 = td.n0, cols = td.cols_valid;
  const uint64_t key = td.key, base = (uint64_t)m * cols + n0;
  uint8_t *const out0 = td.ptr[PTR_OUT], *const out1 = td.ptr[PTR_OUT + 1];
  const int ncol = m < td.rows_valid ? (int)cols - (int)n0 : 0;
#pragma unroll 2
  for (uint32_t cg = h * (128 / EPI_HALVES); cg < (h + 1) * (128 / EPI_HALVES); cg += 8) {
    float v[8];
    gen_run(key, base + cg, 1.0f, v);
#pragma unroll
    for (int x = 0; x < 8; x++) v[x] = (int)(cg + x) < ncol ? v[x] : 0.f;
    uint4 u;
    u.x = pack_bf16x2(v[0], v[1]); u.y = pack_bf16x2(v[2], v[3]);
    u.z = pack_bf16x2(v[4], v[5]); u.w = pack_bf16x2(v[6], v[7]);
    *reinterpret_cast<uint4 *>((cg < 64 ? out0 : out1) + swz(r, (cg % 64) / 8)) = u;
  }
}

// A35 swap copy: one 64 KiB page between the arena and the pinned host swap
// area (PCIe), 16 x 16 B per epilogue thread, all loads in flight before the
// stores.  The system-scope fence makes the host-side bytes visible to the
// SM that later copies them back (another slot's record).
__device__ void copy_page(const TileDesc &td, uint32_t et) {
  const uint4 *src = reinterpret_cast<const uint4 *>(td.ptr[PTR_OUT + 1]);
  uint4 *dst = reinterpret_cast<uint4 *>(td.ptr[PTR_OUT]);
  constexpr uint32_t PER = PAGE_BYTES / 16 / EPI_THREADS;
  uint4 v[PER];
#pragma unroll
  for (uint32_t k = 0; k < PER; k++) v[k] = __ldcv(src + k * EPI_THREADS + et);
#pragma unroll
  for (uint32_t k = 0; k < PER; k++) __stcg(dst + k * EPI_THREADS + et, v[k]);
  __threadfence_system();
}

// ---------------------------------------------------------------------------
// Roles
// ---------------------------------------------------------------------------
// Barrier scopes: waits on barriers the peer CTA (or the pair's MMA commit)
// arrives on use CTA-scope try_wait like CUTLASS's cluster barriers -- the
// data they guard is shared memory / TMEM written by the async proxy, and a
// cluster-scope acquire would invalidate the SM's L1 on every wait.  Only the
// mailbox (a generic st.shared::cluster from the leader) is acquired at
// cluster scope.
// Every consumer of descriptor slot d, in both CTAs, releases it on the
// leader's desc_empty[d]: the leader's four consumers arrive (its MMA thread
// also arms 16 transaction bytes), the peer's four each complete 4 bytes with
// an st.async -- the async-proxy path, observed far sooner than a
// thread-issued remote mbarrier.arrive.  The leader mails task d only when
// the slot is free in both CTAs.
__device__ __forceinline__ void release_desc(WorkerSmem &W, uint32_t d, uint32_t h, bool arm = false) {
  if (h == 0) {
    if (arm) ptx::mbar_arrive_expect_tx(&W.desc_empty[d], 16);
    else ptx::mbar_arrive(&W.desc_empty[d]);
  } else {
    ptx::st_async_b32(ptx::mapa(&W.sink[0], 0), 0u, ptx::mapa(&W.desc_empty[d], 0));
  }
}

__device__ void decoder_warp(const Params &P, WorkerSmem &W, uint32_t lane, uint32_t h) {
  uint32_t d = 0, d_phase = 0;
  uint32_t cached_job = NONE32;               // dense index of the DevJob in W.job_cache
  for (;;) {
    TileDesc &td = W.desc[d];
    uint32_t payload = TASK_EXIT;
    uint64_t t_claim = 0;
    if (h == 0) {                             // leader: claim, mail to the peer
      ptx::mbar_wait_abortable(&W.desc_empty[d], d_phase ^ 1, &P.ctrl->abort);
      if (lane == 0) {
        const unsigned long long pos = atomicAdd(&P.ctrl->q_tail, 1ull);
        uint32_t spins = 0;
        // spin relaxed (an acquire load invalidates the SM's L1 every time),
        // then one acquire load of the published entry
        for (;;) {
          const unsigned long long v = ptx::ld_relaxed_u64(&P.ring[pos & P.ring_mask]);
          if ((uint32_t)(v >> 32) == (uint32_t)(pos + 1)) {
            payload = (uint32_t)ptx::ld_acquire_u64(&P.ring[pos & P.ring_mask]);
            break;
          }
          if ((++spins & 255) == 0 && *(volatile uint32_t *)&P.ctrl->abort) break;
        }
        t_claim = ptx::globaltimer();
        ptx::st_async_v4(ptx::mapa(&W.mail[d], 1), payload, 0u, (uint32_t)t_claim, (uint32_t)(t_claim >> 32),
                         ptx::mapa(&W.mail_full[d], 1));
      }
      payload = __shfl_sync(0xffffffffu, payload, 0);
    } else {                                  // peer: take the leader's mail
      if (lane == 0) ptx::mbar_arrive_expect_tx(&W.mail_full[d], 16);   // armed for this use
      ptx::mbar_wait_abortable(&W.mail_full[d], d_phase, &P.ctrl->abort);
      payload = W.mail[d].payload;
      t_claim = W.mail[d].t_claim;
    }
    __syncwarp();   // lane 0's acquire orders the other lanes' reads below
    if (payload == TASK_EXIT) {
      if (lane == 0) {
        td.kind = T_EXIT;
        td.payload = TASK_EXIT;
        ptx::mbar_arrive(&W.desc_full[d]);
      }
      if (lane < NPTR) ptx::mbar_arrive(&W.desc_ptrs[d]);
      break;
    }
    SlotHead head;
    if (lane == 0) head = load_slot_head(P.slots[payload >> 26]);
    const uint32_t j = __shfl_sync(0xffffffffu, head.job, 0);
    if (j != cached_job) {            // descriptors are static while a job has tasks in flight
      const uint32_t *src = reinterpret_cast<const uint32_t *>(P.jobs + j);
      for (uint32_t x = lane; x < sizeof(DevJob) / 4; x += 32) W.job_cache[x] = src[x];
      cached_job = j;
    }
    __syncwarp();
    if (lane == 0) {
      decode_task(P, payload, *reinterpret_cast<const DevJob *>(W.job_cache), head, td, h);
      td.t_claim = t_claim;
    }
    __syncwarp();
    // the operand loader and the MMA need no translated pointers: hand them
    // the descriptor first, translate the epilogue's pointers meanwhile
    if (lane == 0) {
      if (h == 0 && td.stage == td.first_stage)
        atomicMin((unsigned long long *)&P.slots[td.slot].start_ns, (unsigned long long)ptx::globaltimer());
      ptx::fence_proxy_async_global();
      ptx::mbar_arrive(&W.desc_full[d]);
    }
    // every pointer-writing lane releases its own write (desc_ptrs counts
    // NPTR arrivals) rather than lane 0 on the others' behalf
    if (lane < NPTR && ((td.xt_mask >> lane) & 1u)) {
      td.ptr[lane] = xlate(P, td.xt_tab[(td.xt_sel >> lane) & 1u], td.xt_off[lane]);
#if SALUS_W32_PF
      // SGD tiles: start pulling the fp32 master pages into L2 now, up to
      // NDESC tiles before the epilogue-input loader streams them -- in
      // eager (latency-mode) records only (SALUS_W32_PF=1; 2 = every
      // record, measured -3.5% on C2a): a claimed eager tile usually waits
      // for its predecessor stage, and with few lanes L2 has the room
      if (lane >= PTR_W32 && lane < PTR_W32 + 2 && td.kind == T_GEMM && td.epi == EPI_SGD &&
          (SALUS_W32_PF == 2 || td.eager))
        ptx::bulk_prefetch_l2(td.ptr[lane], PAGE_BYTES);
#endif
    }
    if (lane < NPTR) ptx::mbar_arrive(&W.desc_ptrs[d]);
    __syncwarp();
    if (++d == NDESC) { d = 0; d_phase ^= 1; }
  }
}

// Page numbers of one K-chunk's copies (A: <= 2, B: <= 2)
struct ChunkPages { uint32_t a0, a1, b0, b1; };

__device__ __forceinline__ ChunkPages chunk_pages(const OpDesc &a, const OpDesc &b, uint32_t nca, uint32_t ncb,
                                                  uint32_t kc) {
  ChunkPages p = {0, 0, 0, 0};
  if (nca > 0) p.a0 = a.table[copy_off(a, kc, 0) >> PAGE_SHIFT];
  if (nca > 1) p.a1 = a.table[copy_off(a, kc, 1) >> PAGE_SHIFT];
  if (ncb > 0) p.b0 = b.table[copy_off(b, kc, 0) >> PAGE_SHIFT];
  if (ncb > 1) p.b1 = b.table[copy_off(b, kc, 1) >> PAGE_SHIFT];
  return p;
}

// row coordinate of byte `off` of a page in the arena's 128-byte-row tensor map
__device__ __forceinline__ int32_t tma_row(uint32_t page, uint32_t off) {
  return (int32_t)((page << (PAGE_SHIFT - 7)) + ((off & (PAGE_BYTES - 1)) >> 7));
}

// Eager records (REC_FLAG_EAGER): block until the slot's stage `stage` has
// completed (`want` = its pair tasks x 2 CTA halves), then make the
// producers' generic-proxy stores visible to this CTA's async-proxy (TMA)
// reads.  Spins relaxed (an acquire load per spin would invalidate L1),
// then one acquire load, like the decoder's ring poll.
__device__ __forceinline__ void wait_stage(const Params &P, uint32_t slot, uint32_t stage, uint32_t want) {
  const uint32_t *c = &P.slots[slot].stage_done[stage];
  uint32_t spins = 0;
  for (;;) {
    uint32_t v;
#if SALUS_WAIT_ACQ   // every poll an acquire: no re-load round trip once the count is seen
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(c) : "memory");
    if (v >= want) { ptx::fence_proxy_async_global(); return; }
#else
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(c) : "memory");
    if (v >= want) break;
#endif
    if ((++spins & 4095u) == 0 && *(volatile uint32_t *)&P.ctrl->abort) {
#if SALUS_DBG_NOTRAP
      return;
#else
      __trap();
#endif
    }
  }
  (void)ld_acquire_u32(c);
  ptx::fence_proxy_async_global();
}

// Double K-chunk kc2 (K rows [128 kc2, +128)): byte offset of copy q.  An
// MN-major operand's copy q is panel q's 128-row block (16 KiB, inside one
// page: panels are multiples of 16 KiB); a K-major A's copy q is the
// 128-row block of the 64-wide K-chunk 2 kc2 + q.
__device__ __forceinline__ uint32_t kd_off(const OpDesc &o, uint32_t kc2, uint32_t q) {
  return o.mn ? o.off + (o.start / 64 + q) * o.R * 128u + kc2 * 16384u
              : o.off + (2 * kc2 + q) * o.R * 128u + o.start * 128u;
}

__device__ __forceinline__ ChunkPages kd_pages(const OpDesc &a, const OpDesc &b, uint32_t nca, uint32_t ncb,
                                               uint32_t kc2) {
  ChunkPages p = {0, 0, 0, 0};
  if (nca > 0) { p.a0 = a.table[kd_off(a, kc2, 0) >> PAGE_SHIFT]; p.a1 = a.table[kd_off(a, kc2, 1) >> PAGE_SHIFT]; }
  if (ncb > 0) p.b0 = b.table[kd_off(b, kc2, 0) >> PAGE_SHIFT];
  if (ncb > 1) p.b1 = b.table[kd_off(b, kc2, 1) >> PAGE_SHIFT];
  return p;
}

__device__ __forceinline__ void check_chunk(const Params &P, const ChunkPages &p, uint32_t nca, uint32_t ncb,
                                            uint32_t site, uint32_t kc) {
#if SALUS_DBG_BOUNDS
  if (nca > 0) check_page(P, p.a0, site, kc, nullptr);
  if (nca > 1) check_page(P, p.a1, site + 1, kc, nullptr);
  if (ncb > 0) check_page(P, p.b0, site + 2, kc, nullptr);
  if (ncb > 1) check_page(P, p.b1, site + 3, kc, nullptr);
#else
  (void)P; (void)p; (void)nca; (void)ncb; (void)site; (void)kc;
#endif
}

// Operand loads of a double-K tile: double chunk kc2 takes two ring stages,
// A (two 16 KiB blocks) in the first and B (one 16 KiB block per 64 columns
// of this CTA's half of N) in the second, each armed on its own leader
// barrier.  Eager tiles issue the first PIPE/2 chunks' B (weights / earlier
// activations) before waiting for the predecessor stage, whose output A is.
__device__ void load_kd(const Params &P, WorkerSmem &W, const TileDesc &td, uint32_t h, uint32_t &s,
                        uint32_t &s_phase, uint64_t pol_a, uint64_t pol_b) {
  const OpDesc a = td.a, b = td.b;
  const uint32_t nk2 = td.nk / 2, nca = td.valid ? 2u : 0u, ncb = td.N / 128;
  const uint32_t tx_a = (nca + (td.peer_valid ? 2u : 0u)) * 16384u, tx_b = 2 * ncb * 16384u;
  const void *tm = &P.tmap16;
  const bool dep_init = td.wait && td.dep_stage == 0;
  if (dep_init) wait_stage(P, td.slot, 0, td.dep_want);
  const uint32_t pre = (td.wait && !dep_init) ? min(nk2, PIPE / 2) : 0;
  if (pre) {
    uint32_t s2 = s, ph2 = s_phase;
    ChunkPages pg[PIPE / 2];
    for (uint32_t kc = 0; kc < pre; kc++) {
      pg[kc] = kd_pages(a, b, nca, ncb, kc);
      check_chunk(P, pg[kc], nca, ncb, 10, kc);
      const uint32_t sa = s2;
      if (++s2 == PIPE) { s2 = 0; ph2 ^= 1; }
      const uint32_t sb = s2, phb = ph2;
      if (++s2 == PIPE) { s2 = 0; ph2 ^= 1; }
      ptx::mbar_wait_abortable(&W.empty[sb], phb ^ 1, &P.ctrl->abort);
      if (h == 0) ptx::mbar_arrive_expect_tx(&W.full[sb], tx_b);
      const uint32_t bar = ptx::mapa(&W.full[sb], 0);
      ptx::tma_load_2d_pair(W.stage[sb], tm, 0, tma_row(pg[kc].b0, kd_off(b, kc, 0)), bar, pol_b);
      if (ncb > 1) ptx::tma_load_2d_pair(W.stage[sb] + 16384u, tm, 0, tma_row(pg[kc].b1, kd_off(b, kc, 1)), bar, pol_b);
      (void)sa;
    }
    wait_stage(P, td.slot, td.dep_stage, td.dep_want);
    for (uint32_t kc = 0; kc < pre; kc++) {
      const uint32_t sa = s, pha = s_phase;
      if (++s == PIPE) { s = 0; s_phase ^= 1; }
      if (++s == PIPE) { s = 0; s_phase ^= 1; }
      ptx::mbar_wait_abortable(&W.empty[sa], pha ^ 1, &P.ctrl->abort);
      if (h == 0) ptx::mbar_arrive_expect_tx(&W.full[sa], tx_a);
      if (nca) {
        const uint32_t bar = ptx::mapa(&W.full[sa], 0);
        ptx::tma_load_2d_pair(W.stage[sa], tm, 0, tma_row(pg[kc].a0, kd_off(a, kc, 0)), bar, pol_a);
        ptx::tma_load_2d_pair(W.stage[sa] + 16384u, tm, 0, tma_row(pg[kc].a1, kd_off(a, kc, 1)), bar, pol_a);
      }
    }
  }
  ChunkPages p0 = pre < nk2 ? kd_pages(a, b, nca, ncb, pre) : ChunkPages{0, 0, 0, 0};
  for (uint32_t kc = pre; kc < nk2; kc++) {
    const ChunkPages cur = p0;
    check_chunk(P, cur, nca, ncb, 20, kc);
    if (kc + 1 < nk2) p0 = kd_pages(a, b, nca, ncb, kc + 1);
    const uint32_t sa = s, pha = s_phase;
    if (++s == PIPE) { s = 0; s_phase ^= 1; }
    const uint32_t sb = s, phb = s_phase;
    if (++s == PIPE) { s = 0; s_phase ^= 1; }
    ptx::mbar_wait_abortable(&W.empty[sa], pha ^ 1, &P.ctrl->abort);
    ptx::mbar_wait_abortable(&W.empty[sb], phb ^ 1, &P.ctrl->abort);
    if (h == 0) { ptx::mbar_arrive_expect_tx(&W.full[sa], tx_a); ptx::mbar_arrive_expect_tx(&W.full[sb], tx_b); }
    const uint32_t bar_a = ptx::mapa(&W.full[sa], 0), bar_b = ptx::mapa(&W.full[sb], 0);
    if (nca) {
      ptx::tma_load_2d_pair(W.stage[sa], tm, 0, tma_row(cur.a0, kd_off(a, kc, 0)), bar_a, pol_a);
      ptx::tma_load_2d_pair(W.stage[sa] + 16384u, tm, 0, tma_row(cur.a1, kd_off(a, kc, 1)), bar_a, pol_a);
    }
    ptx::tma_load_2d_pair(W.stage[sb], tm, 0, tma_row(cur.b0, kd_off(b, kc, 0)), bar_b, pol_b);
    if (ncb > 1) ptx::tma_load_2d_pair(W.stage[sb] + 16384u, tm, 0, tma_row(cur.b1, kd_off(b, kc, 1)), bar_b, pol_b);
  }
}

// Operand loader (1 thread).  The page-table reads of chunk kc + 2 are issued
// before the copies of chunk kc, so their latency (an L2 round trip: the
// completion warp's gpu-scope fences keep invalidating L1) is off the
// per-chunk critical path.
__device__ void operand_loader(const Params &P, WorkerSmem &W, uint32_t h) {
  uint32_t d = 0, d_phase = 0, s = 0, s_phase = 0;
  const uint64_t first = ptx::policy_evict_first(), last = ptx::policy_evict_last();
  const uint64_t normal = ptx::policy_evict_normal();
  for (;;) {
    ptx::mbar_wait_abortable(&W.desc_full[d], d_phase, &P.ctrl->abort);
    const TileDesc &td = W.desc[d];
    if (td.kind == T_EXIT) break;
    if (td.kind == T_GEMM) {
      const OpDesc a = td.a, b = td.b;
      const uint32_t nk = td.nk, nca = td.ncopy_a, ncb = td.ncopy_b, ab = td.abytes, bb = td.bbytes;
      // bytes of one K-chunk in both CTAs: B halves are symmetric, A exists
      // in the peer iff its M block does
      const uint32_t tx_pair = (nca + td.peer_nca) * ab + 2 * ncb * bb;
      const uint32_t *jt = P.ppt + P.jobs[td.job].pt_off;
      // weights (the job's persistent space) stream; a lane's activations stay
#if SALUS_L2HINT
      const uint64_t pol_a = a.table == jt ? first : last, pol_b = b.table == jt ? first : last;
#else
      const uint64_t pol_a = normal, pol_b = normal;
#endif
      if (td.kd) {
        load_kd(P, W, td, h, s, s_phase, pol_a, pol_b);
        release_desc(W, d, h);
        if (++d == NDESC) { d = 0; d_phase ^= 1; }
        continue;
      }
      const void *ta = ab == 16384u ? (const void *)&P.tmap16 : (const void *)&P.tmap8;
      const void *tb = bb == 16384u ? (const void *)&P.tmap16 : (const void *)&P.tmap8;
      // eager (td.wait): operand A is what the previous stage produces.  The
      // first `pre` chunks' stages are armed and their B (weights /
      // activations of earlier stages) issued before the wait; their A after.
      // Exception: when the predecessor is INIT (iteration 0 of a
      // GEN-prefetch job, whose F_1 directly follows INIT), B is the weights
      // INIT is still writing -- wait before any load.
      const bool dep_init = td.wait && td.dep_stage == 0;
      if (dep_init) wait_stage(P, td.slot, 0, td.dep_want);
      // the operand the predecessor produces: A, except in a K9 transposed
      // tile, whose A is the weights and B the activations / gradients
      const bool dep_b = td.swap;
      const uint32_t pre = (td.wait && !dep_init && (dep_b ? ncb : nca) > 0) ? min(nk, PIPE) : 0;
      if (pre) {
        uint32_t s2 = s, ph2 = s_phase;
        ChunkPages pg[PIPE];
        for (uint32_t kc = 0; kc < pre; kc++) {
          pg[kc] = chunk_pages(a, b, nca, ncb, kc);
          check_chunk(P, pg[kc], nca, ncb, 40, kc);
          ptx::mbar_wait_abortable(&W.empty[s2], ph2 ^ 1, &P.ctrl->abort);
          const uint32_t bar = ptx::mapa(&W.full[s2], 0);
          if (h == 0) ptx::mbar_arrive_expect_tx(&W.full[s2], tx_pair);
          uint8_t *sa = W.stage[s2], *sb = W.stage[s2] + STAGE_A_BYTES;
          if (dep_b) {
            if (nca > 0) ptx::tma_load_2d_pair(sa, ta, 0, tma_row(pg[kc].a0, copy_off(a, kc, 0)), bar, pol_a);
            if (nca > 1) ptx::tma_load_2d_pair(sa + ab, ta, 0, tma_row(pg[kc].a1, copy_off(a, kc, 1)), bar, pol_a);
          } else {
            if (ncb > 0) ptx::tma_load_2d_pair(sb, tb, 0, tma_row(pg[kc].b0, copy_off(b, kc, 0)), bar, pol_b);
            if (ncb > 1) ptx::tma_load_2d_pair(sb + bb, tb, 0, tma_row(pg[kc].b1, copy_off(b, kc, 1)), bar, pol_b);
          }
          if (++s2 == PIPE) { s2 = 0; ph2 ^= 1; }
        }
        wait_stage(P, td.slot, td.dep_stage, td.dep_want);
        for (uint32_t kc = 0; kc < pre; kc++) {
          const uint32_t bar = ptx::mapa(&W.full[s], 0);
          uint8_t *sa = W.stage[s], *sb = W.stage[s] + STAGE_A_BYTES;
          if (dep_b) {
            if (ncb > 0) ptx::tma_load_2d_pair(sb, tb, 0, tma_row(pg[kc].b0, copy_off(b, kc, 0)), bar, pol_b);
            if (ncb > 1) ptx::tma_load_2d_pair(sb + bb, tb, 0, tma_row(pg[kc].b1, copy_off(b, kc, 1)), bar, pol_b);
          } else {
            ptx::tma_load_2d_pair(sa, ta, 0, tma_row(pg[kc].a0, copy_off(a, kc, 0)), bar, pol_a);
            if (nca > 1) ptx::tma_load_2d_pair(sa + ab, ta, 0, tma_row(pg[kc].a1, copy_off(a, kc, 1)), bar, pol_a);
          }
          if (++s == PIPE) { s = 0; s_phase ^= 1; }
        }
      }
      ChunkPages p0 = pre < nk ? chunk_pages(a, b, nca, ncb, pre) : ChunkPages{0, 0, 0, 0};
      ChunkPages p1 = pre + 1 < nk ? chunk_pages(a, b, nca, ncb, pre + 1) : p0;
      for (uint32_t kc = pre; kc < nk; kc++) {
        const ChunkPages cur = p0;
        check_chunk(P, cur, nca, ncb, 30, kc);
        p0 = p1;
        if (kc + 2 < nk) p1 = chunk_pages(a, b, nca, ncb, kc + 2);
        // stage s is free once the pair's MMA has consumed it (multicast commit)
        ptx::mbar_wait_abortable(&W.empty[s], s_phase ^ 1, &P.ctrl->abort);
        // both CTAs' copies complete on the LEADER's full[s]: the leader alone
        // arms it with the pair's bytes (one arrival); the peer's TMAs only
        // add their bytes through the async proxy -- no thread-issued remote
        // arrive on the per-chunk path (those take ~1 us to be observed)
        const uint32_t bar = ptx::mapa(&W.full[s], 0);
        if (h == 0) ptx::mbar_arrive_expect_tx(&W.full[s], tx_pair);
        uint8_t *sa = W.stage[s], *sb = W.stage[s] + STAGE_A_BYTES;
        if (nca > 0) ptx::tma_load_2d_pair(sa, ta, 0, tma_row(cur.a0, copy_off(a, kc, 0)), bar, pol_a);
        if (nca > 1) ptx::tma_load_2d_pair(sa + ab, ta, 0, tma_row(cur.a1, copy_off(a, kc, 1)), bar, pol_a);
        if (ncb > 0) ptx::tma_load_2d_pair(sb, tb, 0, tma_row(cur.b0, copy_off(b, kc, 0)), bar, pol_b);
        if (ncb > 1) ptx::tma_load_2d_pair(sb + bb, tb, 0, tma_row(cur.b1, copy_off(b, kc, 1)), bar, pol_b);
#if SALUS_DBG_CHUNKS   // trace fields re-purposed: loader issue of chunk 0 / last chunk
        if (kc == 0) const_cast<TileDesc &>(td).t_ready = ptx::globaltimer();
        if (kc + 1 == nk) const_cast<TileDesc &>(td).t_mma = ptx::globaltimer();
#endif
#if SALUS_DBG_CHUNKS2  // per-chunk stamps of one F tile (job 0, iter 10, stage 2, task 0) -> trace tail
        if (td.job == 0 && td.iter == 10 && td.stage == 2 && (td.payload & 0x1FFFFF) == 0 && kc < 32) {
          uint64_t *dbg = reinterpret_cast<uint64_t *>(P.trace + P.trace_cap) - 256;
          dbg[ptx::cluster_ctarank() * 64 + kc] = ptx::globaltimer();
        }
#endif
        if (++s == PIPE) { s = 0; s_phase ^= 1; }
      }
    }
    release_desc(W, d, h);
    if (++d == NDESC) { d = 0; d_phase ^= 1; }
  }
}

// Streams a tile's epilogue input in 32 KiB chunks: SGD chunk c = W32 columns
// [64c, 64c+64) (half of a 64 KiB page); DX chunk c = mask panels 2c, 2c+1.
__device__ void epi_loader(const Params &P, WorkerSmem &W, uint32_t h) {
  uint32_t d = 0, d_phase = 0, e = 0, e_phase = 0;
#if SALUS_L2HINT
  const uint64_t pol_w = ptx::policy_evict_first(), pol_a = ptx::policy_evict_last();
#else
  const uint64_t pol_w = ptx::policy_evict_normal(), pol_a = pol_w;
#endif
  for (;;) {
    ptx::mbar_wait_abortable(&W.desc_full[d], d_phase, &P.ctrl->abort);
    const TileDesc &td = W.desc[d];
    if (td.kind == T_EXIT) break;
    ptx::mbar_wait_abortable(&W.desc_ptrs[d], d_phase, &P.ctrl->abort);
    if (td.kind == T_GEMM) {
      const uint32_t n = td.n_ech;
      const bool sgd = td.epi == EPI_SGD;
      // eager: every epilogue input was produced before the predecessor
      // stage began (earlier stages or iterations), except the prefetched
      // targets T_0 of a 1-layer GEN-prefetch job, which its INIT stage --
      // the loss stage's own predecessor -- generates
      // (and a 1-layer job's T from the GEN stage right before its F_1 = F_L)
      if (td.wait && td.epi == EPI_LOSS && n && (td.iter == 0 || td.dep_stage == 1))
        wait_stage(P, td.slot, td.dep_stage, td.dep_want);
      for (uint32_t c = 0; c < n; c++) {
        ptx::mbar_wait_abortable(&W.epi_empty[e], e_phase ^ 1, &P.ctrl->abort);
        if (!td.ech_load) {                   // K9 staging chunk: reserved, nothing to load
          ptx::mbar_arrive(&W.epi_full[e]);
          if (++e == EBUF) { e = 0; e_phase ^= 1; }
          continue;
        }
        ptx::mbar_arrive_expect_tx(&W.epi_full[e], ECH_BYTES);
        if (sgd) {
          ptx::bulk_g2s_hint(W.epi_in[e], td.ptr[PTR_W32 + (c >> 1)] + (c & 1) * 32768u, ECH_BYTES, &W.epi_full[e],
                             pol_w);
        } else {
          ptx::bulk_g2s_hint(W.epi_in[e], td.ptr[PTR_EPI + 2 * c], 16384u, &W.epi_full[e], pol_a);
          ptx::bulk_g2s_hint(W.epi_in[e] + 16384u, td.ptr[PTR_EPI + 2 * c + 1], 16384u, &W.epi_full[e], pol_a);
        }
        if (++e == EBUF) { e = 0; e_phase ^= 1; }
      }
    }
    release_desc(W, d, h);
    if (++d == NDESC) { d = 0; d_phase ^= 1; }
  }
}

// Leader: one tcgen05.mma.cta_group::2 per K16 step over both CTAs' smem;
// commits arrive on the stage / accumulator barriers of both CTAs.
__device__ void mma_thread(const Params &P, WorkerSmem &W, uint32_t tmem) {
  uint32_t d = 0, d_phase = 0, s = 0, s_phase = 0, b = 0, b_phase = 0;
  for (;;) {
    ptx::mbar_wait_abortable(&W.desc_full[d], d_phase, &P.ctrl->abort);
    const TileDesc &td = W.desc[d];
    if (td.kind == T_EXIT) break;
    if (td.kind == T_GEMM) {
      // both CTAs' epilogues have drained accumulator b
      ptx::mbar_wait_abortable(&W.acc_empty[b], b_phase ^ 1, &P.ctrl->abort);
      ptx::tc_fence_after();
      const uint32_t tacc = tmem + b * ACC_COLS, idesc = td.idesc, nk = td.nk;
      if (td.kd) {
        // double chunks: A's two 16 KiB blocks in stage sa (MN-major: the
        // 128-row panels, LBO 16 KiB; K-major: K-chunks 2kc, 2kc+1), B's
        // 128-row panels in stage sb
        const bool amn = td.a.mn;
        for (uint32_t kc = 0; kc < nk / 2; kc++) {
          const uint32_t sa_i = s;
          ptx::mbar_wait_abortable(&W.full[s], s_phase, &P.ctrl->abort);
          if (++s == PIPE) { s = 0; s_phase ^= 1; }
          const uint32_t sb_i = s;
          ptx::mbar_wait_abortable(&W.full[s], s_phase, &P.ctrl->abort);
          if (++s == PIPE) { s = 0; s_phase ^= 1; }
          ptx::tc_fence_after();
          const uint32_t sa = ptx::smem_u32(W.stage[sa_i]), sb = ptx::smem_u32(W.stage[sb_i]);
#pragma unroll
          for (uint32_t ks = 0; ks < 8; ks++) {
            const uint64_t ad = amn ? ptx::smem_desc_sw128(sa + ks * 2048u, 16384u, 1024)
                                    : ptx::smem_desc_sw128(sa + (ks >> 2) * 16384u + (ks & 3u) * 32u, 16u, 1024);
            const uint64_t bd = ptx::smem_desc_sw128(sb + ks * 2048u, 16384u, 1024);
            ptx::mma_bf16(tacc, ad, bd, idesc, (kc | ks) != 0);
          }
          ptx::mma_commit_pair(&W.empty[sa_i]);
          ptx::mma_commit_pair(&W.empty[sb_i]);
        }
        ptx::mma_commit_pair(&W.acc_full[b]);
        if (++b == 2) { b = 0; b_phase ^= 1; }
        release_desc(W, d, 0, true);
        if (++d == NDESC) { d = 0; d_phase ^= 1; }
        continue;
      }
      const uint32_t a_lbo = td.a.mn ? 8192u : 16u, b_lbo = td.b.mn ? 8192u : 16u;
      const uint32_t a_step = td.a.mn ? 2048u : 32u, b_step = td.b.mn ? 2048u : 32u;
      for (uint32_t kc = 0; kc < nk; kc++) {
        // the chunk has landed in both CTAs (both loaders' copies complete here)
        ptx::mbar_wait_abortable(&W.full[s], s_phase, &P.ctrl->abort);
#if SALUS_DBG_CHUNKS2
        if (td.job == 0 && td.iter == 10 && td.stage == 2 && (td.payload & 0x1FFFFF) == 0 && kc < 32) {
          uint64_t *dbg = reinterpret_cast<uint64_t *>(P.trace + P.trace_cap) - 256;
          dbg[160 + kc] = ptx::globaltimer();                      // chunk landed (both CTAs)
        }
#endif
#if SALUS_DBG_CHUNKS   // MMA thread: last chunk landed in both CTAs
        if (kc + 1 == nk) const_cast<TileDesc &>(td).t_end = ptx::globaltimer();
#endif
        ptx::tc_fence_after();
        const uint32_t sa = ptx::smem_u32(W.stage[s]), sb = sa + STAGE_A_BYTES;
#pragma unroll
        for (uint32_t ks = 0; ks < 4; ks++) {
          const uint64_t ad = ptx::smem_desc_sw128(sa + ks * a_step, a_lbo, 1024);
          const uint64_t bd = ptx::smem_desc_sw128(sb + ks * b_step, b_lbo, 1024);
          ptx::mma_bf16(tacc, ad, bd, idesc, (kc | ks) != 0);
        }
        ptx::mma_commit_pair(&W.empty[s]);
#if SALUS_DBG_CHUNKS2
        if (td.job == 0 && td.iter == 10 && td.stage == 2 && (td.payload & 0x1FFFFF) == 0 && kc < 32) {
          uint64_t *dbg = reinterpret_cast<uint64_t *>(P.trace + P.trace_cap) - 256;
          dbg[192 + kc] = ptx::globaltimer();                      // MMAs issued
        }
#endif
        if (++s == PIPE) { s = 0; s_phase ^= 1; }
      }
      ptx::mma_commit_pair(&W.acc_full[b]);
      if (++b == 2) { b = 0; b_phase ^= 1; }
    }
    release_desc(W, d, 0, true);
    if (++d == NDESC) { d = 0; d_phase ^= 1; }
  }
}

// Peer: no MMA to issue (the leader's covers both CTAs); it only releases
// its descriptors like the leader's MMA thread does.
__device__ void peer_mma_role(const Params &P, WorkerSmem &W) {
  uint32_t d = 0, d_phase = 0;
  for (;;) {
    ptx::mbar_wait_abortable(&W.desc_full[d], d_phase, &P.ctrl->abort);
    if (W.desc[d].kind == T_EXIT) break;
    release_desc(W, d, 1);
    if (++d == NDESC) { d = 0; d_phase ^= 1; }
  }
}

// Split-K (DevJob.splitk): every K-slice of a tile writes its fp32 partial
// (this CTA's 128 rows x N columns, 64 KiB per 128 columns, layout sk_off)
// to its workspace pages, then counts itself on the
// slot's counter for (base tile, CTA half, epilogue warp).  The slice that
// arrives last at a warp's counter sums that warp's region of the S
// partials in slice order -- its own straight from TMEM -- and
// stores the sum back into its accumulator, so the ordinary epilogue
// (ReLU / loss / mask, bf16 stores) runs once per tile on the full sum,
// independent of which slice finished last.  Returns whether this warp runs
// that epilogue on its region.
// Partial layout (private to the slices of one tile): column block cc of
// TMEM lane quarter w is 4 KiB at cc x 16 KiB + w x 4 KiB, holding float4 g
// (columns 4g..4g+3) of lane t at g x 512 B + t x 16 B -- every warp store
// and load of a float4 column group covers 512 contiguous bytes.
__device__ __forceinline__ uint32_t sk_off(uint32_t cc, uint32_t r) {
  return cc * 16384u + (r >> 5) * 4096u + (r & 31u) * 16u;
}

__device__ bool splitk_reduce(const Params &P, WorkerSmem &W, const TileDesc &td, uint32_t tacc, uint32_t r,
                              uint32_t hh, uint32_t et) {
  const uint32_t S = td.sk, z = td.skz, np = td.N / 128;   // partial pages (N = 128 or 256)
  const uint32_t taddr = tacc + (((r >> 5) * 32u) << 16);
  const uint32_t sub = (td.N / 32) / EPI_HALVES, cc0 = hh * sub;
  for (uint32_t cc = cc0; cc < cc0 + sub; cc++) {
    uint32_t raw[32];
    ptx::tmem_ld32(taddr + cc * 32u, raw);
    ptx::tmem_ld_wait();
    float4 *dst = reinterpret_cast<float4 *>(td.ptr[sk_ptr(z * np + (cc >> 2))] + sk_off(cc & 3u, r));
#pragma unroll
    for (int q = 0; q < 8; q++)
      __stcg(dst + 32 * q, make_float4(__uint_as_float(raw[4 * q]), __uint_as_float(raw[4 * q + 1]),
                                  __uint_as_float(raw[4 * q + 2]), __uint_as_float(raw[4 * q + 3])));
  }
  // per warp (each owns 32 rows x its column half of the tile): one acq_rel
  // atomic on the warp's own counter -- its release is cumulative over the
  // warp's partial stores (ordered before it by __syncwarp), its acquire
  // orders the other slices' partials of the same region before the reads
  __syncwarp();
  uint32_t last = 0;
  if ((r & 31u) == 0) {
    uint32_t *cnt = &P.slots[td.slot].sk_cnt[(2 * td.sku + ptx::cluster_ctarank()) * EPI_WARPS + (et >> 5)];
    last = ptx::atom_add_acqrel_u32(cnt, 1u) + 1 == S;
    // the next split stage of this slot starts from 0 (it runs after this
    // stage's completion, which the completion warp releases after this tile)
    if (last) asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(cnt), "r"(0u) : "memory");
  }
  last = __shfl_sync(0xffffffffu, last, 0);
#if SALUS_DBG_SK   // trace field re-purposed: partials written and counted
  if (et == 0) const_cast<TileDesc &>(td).t_claim = ptx::globaltimer();
#endif
  if (!last) return false;
  // all other slices' loads of a 16-column half in flight at once (one L2
  // round trip per half instead of one per slice), then the sum in slice order
  for (uint32_t c16 = 2 * cc0; c16 < 2 * (cc0 + sub); c16++) {
    uint32_t raw[16];
    ptx::tmem_ld16(taddr + c16 * 16u, raw);
    float4 pv[SK_MAX - 1][4];                 // remote slice i = q < z ? q : q - 1
#pragma unroll
    for (uint32_t i = 0; i < SK_MAX - 1; i++) {
      if (i + 1 < S) {
        const uint32_t q = i < z ? i : i + 1;
        const uint32_t cc = c16 >> 1;
        const float4 *src = reinterpret_cast<const float4 *>(td.ptr[sk_ptr(q * np + (cc >> 2))] + sk_off(cc & 3u, r)) +
                            32 * 4 * (c16 & 1u);
#pragma unroll
        for (int g = 0; g < 4; g++) pv[i][g] = __ldcg(src + 32 * g);
      }
    }
    ptx::tmem_ld_wait();
#pragma unroll
    for (int g = 0; g < 4; g++) {
      float a[4];
#pragma unroll
      for (uint32_t q = 0; q < SK_MAX; q++) {
        if (q >= S) break;
        // static indices only (q is unrolled): remote slice q sits at q - 1 above z, else at q
        const float4 lo = pv[q < SK_MAX - 1 ? q : SK_MAX - 2][g], hi = pv[q > 0 ? q - 1 : 0][g];
        const float4 f = q < z ? lo : hi;
        float v[4] = {f.x, f.y, f.z, f.w};
        if (q == z) {
#pragma unroll
          for (int x = 0; x < 4; x++) v[x] = __uint_as_float(raw[4 * g + x]);
        }
#pragma unroll
        for (int x = 0; x < 4; x++) a[x] = q == 0 ? v[x] : a[x] + v[x];
      }
#pragma unroll
      for (int x = 0; x < 4; x++) raw[4 * g + x] = __float_as_uint(a[x]);
    }
    ptx::tmem_st16(taddr + c16 * 16u, raw);
  }
  ptx::tmem_st_wait();
  return true;
}

__device__ void epilogue_warps(const Params &P, WorkerSmem &W, uint32_t tmem, uint32_t tid,
                               unsigned long long &my_tasks) {
  const uint32_t warp = tid >> 5, lane = tid & 31;
  const uint32_t r = ((warp & 3u) << 5) | lane;   // TMEM lane quarter = warp % 4
  const uint32_t h = (warp - EPI_WARP0) >> 2;     // column half (8 epilogue warps)
  const uint32_t et = tid - 32 * EPI_WARP0;       // 0..EPI_THREADS-1
  uint32_t d = 0, d_phase = 0, b = 0, b_phase = 0, e = 0, e_phase = 0;
#if SALUS_W32_BULK
  const uint64_t pol_w32 = ptx::policy_evict_first();   // fp32 masters stream
#endif
  for (;;) {
    ptx::mbar_wait_abortable(&W.desc_full[d], d_phase, &P.ctrl->abort);
    const TileDesc &td = W.desc[d];
    if (td.kind == T_EXIT) break;
    ptx::mbar_wait_abortable(&W.desc_ptrs[d], d_phase, &P.ctrl->abort);
    if (td.valid) my_tasks++;
    const uint64_t t_ready = ptx::globaltimer();
    uint64_t t_mma = t_ready;
    if (td.kind == T_GEMM) {
      const EpiView ev = {td.m0, td.n0, td.rows_valid, td.cols_valid, td.ld_logical, td.epi, td.lr, td.key,
                          td.dump_off};
      const uint32_t ncc = td.N / 32, n = td.n_ech;
      ptx::mbar_wait_abortable(&W.acc_full[b], b_phase, &P.ctrl->abort);
      ptx::tc_fence_after();
      t_mma = ptx::globaltimer();
      const uint32_t tacc = tmem + b * ACC_COLS;
      // split-K: only the tile's last K-slice (holding the summed partials) runs the epilogue
#if SALUS_SPLITK_BUILD
      const bool epi = !td.valid || td.sk < 2 || splitk_reduce(P, W, td, tacc, r, h, et);
#else
      constexpr bool epi = true;
#endif
      if (!td.valid) {
        // the peer half of a super-tile past the last M block: nothing to store
      } else if (td.swap) {
        epilogue_swap(P, W, td, tacc, r, h, et, lane, e, e_phase);
      } else if (n == 0) {
        const uint32_t sub = ncc / EPI_HALVES;
        if (epi) epilogue_cols(P, td, ev, tacc, r, 0, h * sub, (h + 1) * sub, nullptr);
      } else {
        const uint32_t per = ncc / n;                 // column blocks per input chunk
        const uint32_t sub = per / EPI_HALVES;
        for (uint32_t c = 0; c < n; c++) {
          ptx::mbar_wait_abortable(&W.epi_full[e], e_phase, &P.ctrl->abort);
          if (epi)
            epilogue_cols(P, td, ev, tacc, r, c * per, c * per + h * sub, c * per + (h + 1) * sub, W.epi_in[e]);
#if SALUS_W32_BULK
          if (td.epi == EPI_SGD) {
            // the updated master chunk (contiguous in HBM: half a 64 KiB page)
            // leaves smem in one bulk store; the buffer is handed back only
            // once the TMA unit has read it
            ptx::fence_proxy_async_smem();
            named_bar(2, EPI_THREADS);
            if (et == 0) {
              ptx::bulk_s2g_hint(td.ptr[PTR_W32 + (c >> 1)] + (c & 1) * 32768u, W.epi_in[e], ECH_BYTES, pol_w32);
#if SALUS_WB_BULK
              // chunk c = columns [64c, 64c + 64) = the bf16 copy's panel c (this M block's 16 KiB)
              ptx::bulk_s2g_hint(td.ptr[PTR_AUX + c], W.epi_in[e] + ECH_BYTES, 16384u, pol_w32);
#endif
              ptx::bulk_commit();
              ptx::bulk_wait_read0();
            }
          }
#endif
          __syncwarp();                               // each warp releases the chunk on its own
          if (lane == 0) ptx::mbar_arrive(&W.epi_empty[e]);
          if (++e == EBUF) { e = 0; e_phase ^= 1; }
        }
#if SALUS_W32_BULK
        // the tile completes only once its master writes are performed
        if (td.epi == EPI_SGD && et == 0) { ptx::bulk_wait0(); ptx::fence_proxy_async_global(); }
#endif
      }
      ptx::tc_fence_before();
      named_bar(1, EPI_THREADS);
      if (et == 0) {                                // the leader's MMA may reuse it (both CTAs drained)
        if (ptx::cluster_ctarank() == 0) ptx::mbar_arrive_expect_tx(&W.acc_empty[b], 4);
        else ptx::st_async_b32(ptx::mapa(&W.sink[1], 0), 0u, ptx::mapa(&W.acc_empty[b], 0));
      }
      if (++b == 2) { b = 0; b_phase ^= 1; }
    } else if (!td.valid) {
    } else if (td.kind == T_COPY) {
      copy_page(td, et);
    } else {
      if (td.wait) {   // eager: a GEN tile of a non-first stage completes only after its predecessor
        if (et == 0) wait_stage(P, td.slot, td.dep_stage, td.dep_want);
        named_bar(1, EPI_THREADS);
      }
      if (td.kind == T_INIT) init_tile(td, r, h);
      else gen_tile(td, r, h);
    }
    // hand the tile to the completion warp: all epilogue stores are issued
    // before the CTA barrier; the completion thread's gpu-scope fence after
    // the mbarrier handoff is cumulative over them (the grid-sync pattern)
    ptx::fence_proxy_async_global();
    named_bar(1, EPI_THREADS);
    if (et == 0) {
#if !SALUS_DBG_CHUNKS
      W.desc[d].t_ready = t_ready; W.desc[d].t_mma = t_mma; W.desc[d].t_end = ptx::globaltimer();
#else
      (void)t_ready; (void)t_mma;
#endif
      ptx::mbar_arrive(&W.epi_done[d]);
    }
    if (++d == NDESC) { d = 0; d_phase ^= 1; }
  }
}

// Completion warp: per tile, in order — fence, stage counter, and publication
// of the next stage's tiles or (last stage) the slot's next iteration.  Each
// CTA of the pair counts its half: a stage of n pair tasks is complete at 2n.
__device__ void completion_warp(const Params &P, WorkerSmem &W, uint32_t lane, uint32_t h) {
  uint32_t d = 0, d_phase = 0;
  for (;;) {
    ptx::mbar_wait_abortable(&W.desc_full[d], d_phase, &P.ctrl->abort);
    const TileDesc &td = W.desc[d];
    if (td.kind == T_EXIT) break;
    ptx::mbar_wait_abortable(&W.epi_done[d], d_phase, &P.ctrl->abort);
    uint32_t pub = 0, ps = 0, pst = 0, pn = 0, pst2 = NONE32, pn2 = 0;
    unsigned long long pb = 0;
    if (lane == 0) {
      // The epilogue's stores happen-before this thread's acq_rel stage-counter
      // atomic (CTA-scope mbarrier handoff after a named barrier); its release
      // at gpu scope is cumulative over them, so no separate fence is needed.
      if ((P.flags & SALUS_FLAG_TRACE) && td.valid) {
        const unsigned long long i = atomicAdd(&P.ctrl->n_trace, 1ull);
        if (i < P.trace_cap) {
          uint32_t smid;
          asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
          salus_trace_rec t;
          t.task = td.payload; t.smid = smid; t.job = td.job; t.iter = td.iter;
          t.t_claim = td.t_claim; t.t_ready = td.t_ready; t.t_mma = td.t_mma; t.t_end = td.t_end;
          P.trace[i] = t;
        }
      }
      Slot &sl = P.slots[td.slot];
      // relaxed record: a dX tile first releases its G output to the next
      // backward stage (the counter that stage waits on)
      if (td.dx_ctr) ptx::atom_add_acqrel_u32(&sl.stage_done[td.dx_ctr], 1u);
      const uint32_t old = ptx::atom_add_acqrel_u32(&sl.stage_done[td.stage], 1u);
      if (old + 1 == 2 * td.ntiles) {
        // relaxed: B_2 and B_1 each take an end ticket; the second one ends the record
        const bool end = td.is_last || (td.end2 && ptx::atom_add_acqrel_u32(&sl.end_ticket, 1u) == 1u);
        if (end) {                             // the record is physically complete
          const uint64_t end = ptx::globaltimer(), start = sl.start_ns;
          sl.end_ns = end;
          const DevJob &J = P.jobs[td.job];
          if (td.kind == T_COPY) {             // A35 swap record
            __threadfence_system();
            atomicAdd(td.stage == STAGE_SWAP_OUT ? &P.ctrl->n_swap_out : &P.ctrl->n_swap_in, 1ull);
            atomicAdd(&P.ctrl->swap_bytes, (unsigned long long)J.ap_pages << PAGE_SHIFT);
            atomicAdd(&P.ctrl->swap_ns, (unsigned long long)(end - start));
          } else {
            if ((P.flags & SALUS_FLAG_LOG) && td.lseq < P.log_cap) {
              salus_wall_rec w;
              w.seq = td.lseq; w.lane = sl.lane_id; w.job = J.job_id; w.start_ns = start; w.end_ns = end;
              w.append_ns = sl.append_ns;
              P.wall[td.lseq] = w;
            }
            if (td.iter == 0) P.stats[td.job].wall_start_ns = start;
            if (td.iter + 1 == J.n_iters) P.stats[td.job].wall_end_ns = end;
          }
          ptx::st_release_u64(&sl.done_seq, td.seq + 1);
          // run-ahead: start the slot's next queued iteration right here
          DispRec rec;
          if (take_next(sl, &rec)) {
            pub = 1; ps = td.slot; pst = rec.first; pn = rec.n1; pst2 = rec.second; pn2 = rec.n2;
            // reserve the ring positions first: the atomic's round trip
            // overlaps begin_iteration's fence
            pb = atomicAdd(&P.ctrl->q_head, (unsigned long long)(pn + pn2));
            begin_iteration(sl, rec);
          }
        } else {
          // the stage two after this one (eager), and in a relaxed record
          // the one three after it, once their publication tickets are full
          const bool p1 = td.next_ntiles &&
                          (!td.next_tk || ptx::atom_add_acqrel_u32(&sl.pub_ticket[td.next_stage], 1u) == 1u);
          const bool p2 = td.next2_stage && ptx::atom_add_acqrel_u32(&sl.pub_ticket[td.next2_stage], 1u) == 1u;
          if (p1 || p2) {
            pub = 1; ps = td.slot;
            pst = p1 ? td.next_stage : td.next2_stage;
            pn = p1 ? td.next_ntiles : td.next2_ntiles;
            if (p1 && p2) { pst2 = td.next2_stage; pn2 = td.next2_ntiles; }
            pb = atomicAdd(&P.ctrl->q_head, (unsigned long long)(pn + pn2));
          }
        }
      }
    }
    pub = __shfl_sync(0xffffffffu, pub, 0);
    if (pub) {                                 // publish the next tiles (32 lanes)
      ps = __shfl_sync(0xffffffffu, ps, 0);
      pst = __shfl_sync(0xffffffffu, pst, 0);
      pn = __shfl_sync(0xffffffffu, pn, 0);
      pst2 = __shfl_sync(0xffffffffu, pst2, 0);
      pn2 = __shfl_sync(0xffffffffu, pn2, 0);
      pb = __shfl_sync(0xffffffffu, pb, 0);
      // the first stage's tiles, then (eager) the second's at higher positions
      publish_tiles(P.ring, P.ring_mask, lane, pb, ps, pst, pn, pst2, pn2);
    }
    __syncwarp();
    if (lane == 0) release_desc(W, d, h);
    if (++d == NDESC) { d = 0; d_phase ^= 1; }
  }
}

__device__ void run_worker(const Params &P, uint8_t *smem_raw) {
  // the dynamic smem window starts 1 KiB-aligned (no static smem); the
  // SWIZZLE_128B operand stages rely on it, and there is no room for slack
  if (ptx::smem_u32(smem_raw) & 1023u) __trap();
  WorkerSmem &W = *reinterpret_cast<WorkerSmem *>(smem_raw);
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t h = ptx::cluster_ctarank();

  if (tid == 0) {
    // full[s]: the leader's, armed by the leader's loader for both CTAs' bytes
    for (uint32_t s = 0; s < PIPE; s++) { ptx::mbar_init(&W.full[s], 1); ptx::mbar_init(&W.empty[s], 1); }
    // (leader) a descriptor is released by its 4 consumers in each CTA:
    // operand loader, epilogue-input loader, MMA thread (peer: its stand-in),
    // completion warp (after the epilogue is done)
    for (uint32_t d = 0; d < NDESC; d++) {
      ptx::mbar_init(&W.desc_full[d], 1);
      ptx::mbar_init(&W.desc_ptrs[d], NPTR);
      ptx::mbar_init(&W.desc_empty[d], 4);
      ptx::mbar_init(&W.epi_done[d], 1);
      ptx::mbar_init(&W.mail_full[d], 1);
    }
    for (uint32_t b = 0; b < 2; b++) { ptx::mbar_init(&W.acc_full[b], 1); ptx::mbar_init(&W.acc_empty[b], 1); }
    for (uint32_t e = 0; e < EBUF; e++) { ptx::mbar_init(&W.epi_full[e], 1); ptx::mbar_init(&W.epi_empty[e], EPI_WARPS); }
    ptx::fence_mbar_init();
  }
  if (warp == 2) { ptx::tmem_alloc(&W.tmem_base, TMEM_COLS); ptx::tmem_relinquish(); }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync();           // the peer's barriers exist before any remote arrive
  ptx::tc_fence_after();
  const uint32_t tmem = W.tmem_base;
  unsigned long long my_tasks = 0;

  if (warp == 0) {
    decoder_warp(P, W, lane, h);
  } else if (warp < EPI_WARP0) {
    if (lane == 0) {
      if (warp == 1) operand_loader(P, W, h);
      else if (warp == 2) { if (h == 0) mma_thread(P, W, tmem); else peer_mma_role(P, W); }
      else epi_loader(P, W, h);
    }
    __syncwarp();
  } else if (warp < DONE_WARP) {
    epilogue_warps(P, W, tmem, tid, my_tasks);
  } else {
    completion_warp(P, W, lane, h);
  }
  __syncthreads();
  if (tid == 32 * EPI_WARP0) atomicAdd(&P.ctrl->n_tasks, my_tasks);
  ptx::tc_fence_before();
  ptx::cluster_sync();           // no remote smem / TMEM traffic after this point
  ptx::tc_fence_after();
  if (warp == 2) ptx::tmem_dealloc(tmem, TMEM_COLS);
}

}  // namespace salus
