// worker.cuh — worker CTAs of the persistent kernel.  Each worker loops:
// claim a tile task from the device task ring, execute it, and, if it was the
// last tile of its stage, publish the next stage of that iteration (or mark
// the iteration complete for the scheduler).  No host round-trip and no
// context teardown between iterations or jobs: TMEM and barriers are set up
// once per kernel, and a "job switch" is just a task with a different slot.
//
// GEMM tiles (the only tensor-core work, north star): M = 128 rows, N = 128
// or 256, K in chunks of 64 bf16.  Operands are bf16 tensors stored in HBM as
// 128-byte-swizzled column panels, so every K-chunk
// of an operand is one or a few contiguous 8/16 KiB blocks moved by the bulk
// async copy engine (cp.async.bulk, TMA unit) into a 4-stage mbarrier ring;
// one thread issues tcgen05.mma (kind::f16, fp32 accumulate in TMEM); four
// epilogue warps drain TMEM with tcgen05.ld and apply the fused epilogue.
#pragma once
#include <cuda_bf16.h>
#include "salus_dev.h"
#include "ptx.cuh"
#include "datagen.cuh"

namespace salus {

constexpr uint32_t PIPE = 4;
constexpr uint32_t STAGE_A_BYTES = 16384;             // 128 x 64 bf16
constexpr uint32_t STAGE_B_BYTES = 32768;             // 256 x 64 bf16
constexpr uint32_t STAGE_BYTES = STAGE_A_BYTES + STAGE_B_BYTES;
constexpr uint32_t MAX_COPIES = 1024;
constexpr uint32_t WORKER_THREADS = 192;              // w0 producer, w1 MMA, w2-5 epilogue
constexpr uint32_t TMEM_COLS = 256;

enum : uint32_t { T_EXIT = 0, T_INIT = 1, T_GEN = 2, T_GEMM = 3 };
enum : uint32_t { EPI_RELU = 0, EPI_OUT = 1, EPI_LOSS = 2, EPI_DX = 3, EPI_SGD = 4 };

struct OpDesc {
  const uint32_t *table;   // page table of the operand's space
  uint32_t off, R, start, mn;
};

struct TileDesc {
  uint32_t kind, payload, slot, stage, job, iter, ntiles, next_ntiles, is_last;
  uint64_t seq;
  // GEMM
  uint32_t N, nk, idesc, epi, layer, a_mn, b_mn, ncopy_a, ncopy_b, bytes_chunk;
  OpDesc a, b;
  // epilogue / elementwise addressing (row block base pointers, translated)
  uint8_t *out[4];         // output panels (bf16)
  uint8_t *aux[4];         // EPI_DX: mask panels; SGD/INIT: Wb panels
  uint8_t *w32[2];         // SGD/INIT: W32 pages
  uint32_t m0, n0;         // tile origin in logical (row, col) of the output
  uint32_t rows_valid, cols_valid, ld_logical;   // batch / d for masking & indexing
  uint64_t key;            // datagen key (T for LOSS, W for INIT, X for GEN)
  float scale, lr;
  int64_t dump_off;        // float offset, -1 = no dump
};

struct WorkerSmem {
  uint8_t stage[PIPE][STAGE_BYTES];   // 1024-aligned (first member)
  uint64_t src[MAX_COPIES];           // translated global addresses of copies
  uint64_t full[PIPE], empty[PIPE], accum;
  uint32_t tmem_base;
  uint32_t pub_flag;
  unsigned long long pub_base;
  uint64_t tr_claim, tr_ready, tr_mma;   // SALUS_FLAG_TRACE stamps
  TileDesc td;
};

__device__ __forceinline__ uint8_t *xlate(const Params &P, const uint32_t *table, uint32_t off) {
  const uint32_t page = table[off >> PAGE_SHIFT];
  return P.arena + ((uint64_t)page << PAGE_SHIFT) + (off & (PAGE_BYTES - 1));
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t *>(&h);
}

// 8 consecutive columns (one 16-byte chunk) of row r in a swizzled panel block
__device__ __forceinline__ uint4 *panel_chunk(uint8_t *panel_rowblock, uint32_t r, uint32_t chunk) {
  return reinterpret_cast<uint4 *>(panel_rowblock + r * 128u + (((chunk ^ (r & 7u)) & 7u) << 4));
}

// ---------------------------------------------------------------------------
// Decode a task into a TileDesc (thread 0).  Stage numbering: 0 INIT,
// 1 GEN, 2..L+1 F_1..F_L, L+2.. B_L..B_1 (salus_dev.h).
// ---------------------------------------------------------------------------
__device__ void decode_task(const Params &P, uint32_t payload, TileDesc &td) {
  td.payload = payload;
  if (payload == TASK_EXIT) { td.kind = T_EXIT; return; }
  const uint32_t slot = payload >> 26, stage = (payload >> 21) & 31u, tile = payload & ((1u << 21) - 1);
  const Slot &sl = P.slots[slot];
  const uint32_t j = sl.job, k = sl.iter;
  const DevJob &J = P.jobs[j];
  const uint32_t L = J.n_layers, bp = J.bpad;
  td.slot = slot; td.stage = stage; td.job = j; td.iter = k; td.seq = sl.seq;
  td.ntiles = J.stage_tiles[stage];
  const uint32_t ls = last_stage(J.kind, L);
  td.is_last = stage == ls;
  td.next_ntiles = td.is_last ? 0 : J.stage_tiles[stage + 1];
  td.dump_off = -1;
  const uint32_t *lt = P.lpt + (uint64_t)slot * P.lpt_stride;   // lane (ephemeral) space
  const uint32_t *jt = P.ppt + J.pt_off;                        // job (persistent) space

  if (stage == 0) {                                   // INIT weights
    td.kind = T_INIT;
    uint32_t t = tile, l = 1;
    for (; l <= L; l++) {
      const uint32_t nb = (J.dpad[l] / 128) * (J.dpad[l - 1] / 128);
      if (t < nb) break;
      t -= nb;
    }
    const uint32_t nib = J.dpad[l - 1] / 128, jb = t / nib, ib = t % nib;
    td.layer = l; td.m0 = jb * 128; td.n0 = ib * 128;
    td.rows_valid = J.dims[l]; td.cols_valid = J.dims[l - 1];
    // inference jobs keep only the bf16 copy (2 B/param): no fp32 master
    td.w32[0] = J.kind == SALUS_TRAIN
                    ? xlate(P, jt, J.w32_off[l - 1] + (jb * (J.dpad[l - 1] / 4) + 32 * ib) * 2048u)
                    : nullptr;
    for (uint32_t q = 0; q < 2; q++)
      td.aux[q] = xlate(P, jt, J.wb_off[l - 1][0] + (2 * ib + q) * J.dpad[l] * 128u + jb * 16384u);
    td.key = gen_key(J.seed, J.job_id, GEN_W, l, 0);
    td.scale = gen_wscale(J.dims[l - 1]);
    return;
  }
  if (stage == 1) {                                   // GEN input batch X
    td.kind = T_GEN;
    const uint32_t ncb = J.dpad[0] / 128, mb = tile / ncb, cb = tile % ncb;
    td.m0 = mb * 128; td.n0 = cb * 128;
    td.rows_valid = J.batch; td.cols_valid = J.dims[0];
    for (uint32_t q = 0; q < 2; q++)
      td.out[q] = xlate(P, lt, J.act_off[0] + (2 * cb + q) * bp * 128u + mb * 16384u);
    td.key = gen_key(J.seed, J.job_id, GEN_X, 0, k);
    return;
  }
  td.kind = T_GEMM;
  if (stage <= L + 1) {                               // forward F_l
    const uint32_t l = stage - 1, NT = ntile_for(J.dpad[l]), ntn = J.dpad[l] / NT;
    const uint32_t mb = tile / ntn, nb = tile % ntn;
    td.layer = l; td.N = NT; td.nk = J.dpad[l - 1] / 64;
    td.a = OpDesc{lt, J.act_off[l - 1], bp, mb * 128, 0};
    td.b = OpDesc{jt, J.wb_off[l - 1][k & 1], J.dpad[l], nb * NT, 0};
    td.m0 = mb * 128; td.n0 = nb * NT;
    td.rows_valid = J.batch; td.cols_valid = J.dims[l]; td.ld_logical = J.dims[l];
    uint32_t out_off;
    if (l < L) { td.epi = EPI_RELU; out_off = J.act_off[l]; }
    else if (J.kind == SALUS_TRAIN) {
      td.epi = EPI_LOSS; out_off = J.g_off[0];
      td.key = gen_key(J.seed, J.job_id, GEN_T, L, k);
    } else { td.epi = EPI_OUT; out_off = J.act_off[L]; }
    if (l == L && (J.dump & SALUS_DUMP_OUTPUTS))
      td.dump_off = (int64_t)(J.dump_out_off + (uint64_t)k * J.batch * J.dims[L]);
    for (uint32_t q = 0; q < NT / 64; q++)
      td.out[q] = xlate(P, lt, out_off + (td.n0 / 64 + q) * bp * 128u + mb * 16384u);
  } else {                                            // backward B_l
    const uint32_t l = L - (stage - (L + 2)), NT = ntile_for(J.dpad[l - 1]);
    const uint32_t ntn = J.dpad[l - 1] / NT, nW = (J.dpad[l] / 128) * ntn;
    const uint32_t gin = J.g_off[(L - l) & 1], gout = J.g_off[(L - l + 1) & 1];
    td.layer = l; td.N = NT;
    if (tile < nW) {                                  // dW_l^T = G_l^T A_{l-1}; SGD
      const uint32_t mb = tile / ntn, nb = tile % ntn;
      td.epi = EPI_SGD; td.nk = bp / 64;
      td.a = OpDesc{lt, gin, bp, mb * 128, 1};
      td.b = OpDesc{lt, J.act_off[l - 1], bp, nb * NT, 1};
      td.m0 = mb * 128; td.n0 = nb * NT;
      td.rows_valid = J.dims[l]; td.cols_valid = J.dims[l - 1]; td.ld_logical = J.dims[l];
      td.lr = J.lr;
      const uint32_t w32 = J.w32_off[l - 1] + (mb * (J.dpad[l - 1] / 4) + nb * NT / 4) * 2048u;
      for (uint32_t q = 0; q < NT / 128; q++) td.w32[q] = xlate(P, jt, w32 + q * 65536u);
      for (uint32_t q = 0; q < NT / 64; q++)
        td.aux[q] = xlate(P, jt, J.wb_off[l - 1][(k + 1) & 1] + (td.n0 / 64 + q) * J.dpad[l] * 128u + mb * 16384u);
      if ((J.dump & SALUS_DUMP_WEIGHTS) && k + 1 == J.n_iters) {
        uint64_t base = J.dump_w_off;
        for (uint32_t q = 1; q < l; q++) base += (uint64_t)J.dims[q - 1] * J.dims[q];
        td.dump_off = (int64_t)base;
      }
    } else {                                          // G_{l-1} = (G_l W_l^T) * [A_{l-1} > 0]
      const uint32_t u = tile - nW, mb = u / ntn, nb = u % ntn;
      td.epi = EPI_DX; td.nk = J.dpad[l] / 64;
      td.a = OpDesc{lt, gin, bp, mb * 128, 0};
      td.b = OpDesc{jt, J.wb_off[l - 1][k & 1], J.dpad[l], nb * NT, 1};
      td.m0 = mb * 128; td.n0 = nb * NT;
      td.rows_valid = J.batch; td.cols_valid = J.dims[l - 1];
      for (uint32_t q = 0; q < NT / 64; q++) {
        td.out[q] = xlate(P, lt, gout + (td.n0 / 64 + q) * bp * 128u + mb * 16384u);
        td.aux[q] = xlate(P, lt, J.act_off[l - 1] + (td.n0 / 64 + q) * bp * 128u + mb * 16384u);
      }
    }
  }
  td.a_mn = td.a.mn; td.b_mn = td.b.mn;
  td.ncopy_a = td.a.mn ? 2 : 1;
  td.ncopy_b = td.b.mn ? td.N / 64 : td.N / 128;
  td.bytes_chunk = STAGE_A_BYTES + td.N * 128u;
  td.idesc = ptx::idesc_bf16(128, td.N, td.a.mn, td.b.mn);
}

// global byte offset (inside the operand's space) of copy q of K-chunk kc
__device__ __forceinline__ uint32_t copy_off(const OpDesc &o, uint32_t kc, uint32_t q) {
  return o.mn ? o.off + (o.start / 64 + q) * o.R * 128u + kc * 8192u
              : o.off + kc * o.R * 128u + (o.start + 128 * q) * 128u;
}

// ---------------------------------------------------------------------------
// Epilogues: thread r of the 4 epilogue warps owns accumulator row r
// (TMEM lane r); columns are drained 32 at a time.
// ---------------------------------------------------------------------------
__device__ void epilogue(const Params &P, const TileDesc &td, uint32_t tmem, uint32_t r) {
  const uint32_t qw = r >> 5;
  const uint32_t row = td.m0 + r;
  const bool row_ok = row < td.rows_valid;
  float *dump = td.dump_off >= 0 ? P.dump + td.dump_off : nullptr;
  for (uint32_t cc = 0; cc < td.N / 32; cc++) {
    uint32_t raw[32];
    ptx::tmem_ld32(tmem + ((qw * 32u) << 16) + cc * 32u, raw);
    ptx::tmem_ld_wait();
    float v[32];
#pragma unroll
    for (int x = 0; x < 32; x++) v[x] = __uint_as_float(raw[x]);
    const uint32_t col0 = td.n0 + cc * 32;
    uint8_t *ob = td.out[cc >> 1];
    const uint32_t ch0 = (cc & 1) * 4;
    if (td.epi == EPI_SGD) {
      // rows are j (d_l), columns i (d_{l-1}): W32[j][i] -= lr * dW^T[j][i]
      uint8_t *wp = td.w32[cc >> 2];
#pragma unroll
      for (int g = 0; g < 8; g++) {
        float4 *a = reinterpret_cast<float4 *>(wp + (((cc * 8 + g) & 31u) * 2048u) + r * 16u);
        float4 w = *a;
        w.x = fmaf(-td.lr, v[4 * g + 0], w.x);
        w.y = fmaf(-td.lr, v[4 * g + 1], w.y);
        w.z = fmaf(-td.lr, v[4 * g + 2], w.z);
        w.w = fmaf(-td.lr, v[4 * g + 3], w.w);
        *a = w;
        v[4 * g + 0] = w.x; v[4 * g + 1] = w.y; v[4 * g + 2] = w.z; v[4 * g + 3] = w.w;
      }
      uint8_t *wb = td.aux[cc >> 1];
#pragma unroll
      for (int q = 0; q < 4; q++) {
        uint4 u;
        u.x = pack_bf16x2(v[8 * q + 0], v[8 * q + 1]);
        u.y = pack_bf16x2(v[8 * q + 2], v[8 * q + 3]);
        u.z = pack_bf16x2(v[8 * q + 4], v[8 * q + 5]);
        u.w = pack_bf16x2(v[8 * q + 6], v[8 * q + 7]);
        *panel_chunk(wb, r, ch0 + q) = u;
      }
      if (dump && row_ok) {                     // W[i][j], logical d_{l-1} x d_l
        for (int x = 0; x < 32; x++)
          if (col0 + x < td.cols_valid) dump[(uint64_t)(col0 + x) * td.ld_logical + row] = v[x];
      }
      continue;
    }
    if (td.epi == EPI_DX) {
      uint8_t *mb = td.aux[cc >> 1];
#pragma unroll
      for (int q = 0; q < 4; q++) {
        const uint4 m = *panel_chunk(mb, r, ch0 + q);
        const uint32_t w[4] = {m.x, m.y, m.z, m.w};
#pragma unroll
        for (int h = 0; h < 4; h++) {
          const uint32_t lo = w[h] & 0xFFFFu, hi = w[h] >> 16;
          if (!((lo & 0x8000u) == 0 && (lo & 0x7FFFu) != 0)) v[8 * q + 2 * h] = 0.f;
          if (!((hi & 0x8000u) == 0 && (hi & 0x7FFFu) != 0)) v[8 * q + 2 * h + 1] = 0.f;
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
      } else {  // EPI_LOSS: G_L = (A_L - T) / B  (MSE)
        const float fb = (float)td.rows_valid;
#pragma unroll 4
        for (int x = 0; x < 32; x++) {
          const uint32_t col = col0 + x;
          if (row_ok && col < td.cols_valid) {
            const float tv = gen_value(td.key, (uint64_t)row * td.ld_logical + col, 1.0f);
            v[x] = __fdiv_rn(v[x] - tv, fb);
          } else {
            v[x] = 0.f;
          }
        }
      }
    }
#pragma unroll
    for (int q = 0; q < 4; q++) {
      uint4 u;
      u.x = pack_bf16x2(v[8 * q + 0], v[8 * q + 1]);
      u.y = pack_bf16x2(v[8 * q + 2], v[8 * q + 3]);
      u.z = pack_bf16x2(v[8 * q + 4], v[8 * q + 5]);
      u.w = pack_bf16x2(v[8 * q + 6], v[8 * q + 7]);
      *panel_chunk(ob, r, ch0 + q) = u;
    }
  }
}

// INIT: W_l block (rows j = m0 + r of W^T storage, 128 columns i)
__device__ void init_tile(const TileDesc &td, uint32_t r) {
  const uint32_t j = td.m0 + r;
  for (uint32_t cg = 0; cg < 128; cg += 8) {
    float v[8];
#pragma unroll
    for (int x = 0; x < 8; x++) {
      const uint32_t i = td.n0 + cg + x;
      v[x] = (j < td.rows_valid && i < td.cols_valid)
                 ? gen_value(td.key, (uint64_t)i * td.rows_valid + j, td.scale) : 0.f;
    }
    // W32 j-blocked layout: ((j/128)*(dp_in/4) + i/4)*2048 + (j%128)*16 + (i%4)*4
    if (td.w32[0]) {
      *reinterpret_cast<float4 *>(td.w32[0] + ((cg / 4) * 2048u) + r * 16u) = make_float4(v[0], v[1], v[2], v[3]);
      *reinterpret_cast<float4 *>(td.w32[0] + ((cg / 4 + 1) * 2048u) + r * 16u) = make_float4(v[4], v[5], v[6], v[7]);
    }
    uint4 u;
    u.x = pack_bf16x2(v[0], v[1]); u.y = pack_bf16x2(v[2], v[3]);
    u.z = pack_bf16x2(v[4], v[5]); u.w = pack_bf16x2(v[6], v[7]);
    *panel_chunk(td.aux[cg / 64], r, (cg % 64) / 8) = u;
  }
}

// GEN: X block (rows m = m0 + r, 128 columns)
__device__ void gen_tile(const TileDesc &td, uint32_t r) {
  const uint32_t m = td.m0 + r;
  for (uint32_t cg = 0; cg < 128; cg += 8) {
    float v[8];
#pragma unroll
    for (int x = 0; x < 8; x++) {
      const uint32_t c = td.n0 + cg + x;
      v[x] = (m < td.rows_valid && c < td.cols_valid)
                 ? gen_value(td.key, (uint64_t)m * td.cols_valid + c, 1.0f) : 0.f;
    }
    uint4 u;
    u.x = pack_bf16x2(v[0], v[1]); u.y = pack_bf16x2(v[2], v[3]);
    u.z = pack_bf16x2(v[4], v[5]); u.w = pack_bf16x2(v[6], v[7]);
    *panel_chunk(td.out[cg / 64], r, (cg % 64) / 8) = u;
  }
}

__device__ void run_worker(const Params &P, uint8_t *smem_raw) {
  const uint32_t base = ptx::smem_u32(smem_raw);
  WorkerSmem &W = *reinterpret_cast<WorkerSmem *>(smem_raw + (((base + 1023u) & ~1023u) - base));
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  if (tid == 0) {
    for (uint32_t s = 0; s < PIPE; s++) { ptx::mbar_init(&W.full[s], 1); ptx::mbar_init(&W.empty[s], 1); }
    ptx::mbar_init(&W.accum, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 2) { ptx::tmem_alloc(&W.tmem_base, TMEM_COLS); ptx::tmem_relinquish(); }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = W.tmem_base;

  uint32_t p_stage = 0, p_phase = 0;     // producer ring position (warp 0 lane 0)
  uint32_t m_stage = 0, m_phase = 0;     // MMA ring position (warp 1 lane 0)
  uint32_t acc_phase = 0;
  unsigned long long my_tasks = 0;

  for (;;) {
    __syncthreads();
    if (tid == 0) {
      const unsigned long long pos = atomicAdd(&P.ctrl->q_tail, 1ull);
      uint32_t payload = TASK_EXIT;
      uint32_t spins = 0;
      for (;;) {
        const unsigned long long v = ptx::ld_acquire_u64(&P.ring[pos & P.ring_mask]);
        if ((uint32_t)(v >> 32) == (uint32_t)(pos + 1)) { payload = (uint32_t)v; break; }
        if ((++spins & 255) == 0 && *(volatile uint32_t *)&P.ctrl->abort) break;
      }
      W.tr_claim = ptx::globaltimer();
      decode_task(P, payload, W.td);
      if (W.td.kind != T_EXIT) {
        const uint32_t first = W.td.iter == 0 ? 0u : 1u;
        if (W.td.stage == first) atomicMin((unsigned long long *)&P.slots[W.td.slot].start_ns,
                                           (unsigned long long)ptx::globaltimer());
      }
    }
    __syncthreads();
    const TileDesc &td = W.td;
    if (td.kind == T_EXIT) break;
    my_tasks++;

    if (td.kind == T_GEMM) {
      const uint32_t nc = td.ncopy_a + td.ncopy_b, total = td.nk * nc;
      if (warp == 0) {
        for (uint32_t x = lane; x < total; x += 32) {
          const uint32_t kc = x / nc, q = x % nc;
          const OpDesc &o = q < td.ncopy_a ? td.a : td.b;
          const uint32_t qq = q < td.ncopy_a ? q : q - td.ncopy_a;
          W.src[x] = reinterpret_cast<uint64_t>(xlate(P, o.table, copy_off(o, kc, qq)));
        }
      }
      __syncthreads();
      if (tid == 0) W.tr_ready = ptx::globaltimer();
      if (warp == 0 && lane == 0) {
        ptx::fence_proxy_async_global();
        const uint32_t abytes = td.a_mn ? 8192u : 16384u, bbytes = td.b_mn ? 8192u : 16384u;
        for (uint32_t kc = 0; kc < td.nk; kc++) {
          ptx::mbar_wait_abortable(&W.empty[p_stage], p_phase ^ 1, &P.ctrl->abort);
          ptx::mbar_arrive_expect_tx(&W.full[p_stage], td.bytes_chunk);
          uint8_t *sa = W.stage[p_stage], *sb = W.stage[p_stage] + STAGE_A_BYTES;
          for (uint32_t q = 0; q < td.ncopy_a; q++)
            ptx::bulk_g2s(sa + q * abytes, reinterpret_cast<void *>(W.src[kc * nc + q]), abytes, &W.full[p_stage]);
          for (uint32_t q = 0; q < td.ncopy_b; q++)
            ptx::bulk_g2s(sb + q * bbytes, reinterpret_cast<void *>(W.src[kc * nc + td.ncopy_a + q]), bbytes,
                          &W.full[p_stage]);
          if (++p_stage == PIPE) { p_stage = 0; p_phase ^= 1; }
        }
      } else if (warp == 1 && lane == 0) {
        const uint32_t a_lbo = td.a_mn ? 8192u : 16u, b_lbo = td.b_mn ? 8192u : 16u;
        const uint32_t a_step = td.a_mn ? 2048u : 32u, b_step = td.b_mn ? 2048u : 32u;
        for (uint32_t kc = 0; kc < td.nk; kc++) {
          ptx::mbar_wait_abortable(&W.full[m_stage], m_phase, &P.ctrl->abort);
          ptx::tc_fence_after();
          const uint32_t sa = ptx::smem_u32(W.stage[m_stage]), sb = sa + STAGE_A_BYTES;
#pragma unroll
          for (uint32_t ks = 0; ks < 4; ks++) {
            const uint64_t ad = ptx::smem_desc_sw128(sa + ks * a_step, a_lbo, 1024);
            const uint64_t bd = ptx::smem_desc_sw128(sb + ks * b_step, b_lbo, 1024);
            ptx::mma_bf16(tmem, ad, bd, td.idesc, (kc | ks) != 0);
          }
          ptx::mma_commit(&W.empty[m_stage]);
          if (++m_stage == PIPE) { m_stage = 0; m_phase ^= 1; }
        }
        ptx::mma_commit(&W.accum);
      } else if (warp >= 2) {
        ptx::mbar_wait_abortable(&W.accum, acc_phase, &P.ctrl->abort);
        ptx::tc_fence_after();
        if (tid == 64) W.tr_mma = ptx::globaltimer();
        // a warp may only touch TMEM lanes [32*(warp%4), +32): warps 2,3,4,5
        // own accumulator rows 64-95, 96-127, 0-31, 32-63
        epilogue(P, td, tmem, ((warp & 3u) << 5) | lane);
      }
      acc_phase ^= 1;
    } else if (warp >= 2) {
      if (tid == 64) { W.tr_ready = W.tr_claim; W.tr_mma = ptx::globaltimer(); }
      if (td.kind == T_INIT) init_tile(td, ((warp & 3u) << 5) | lane);
      else gen_tile(td, ((warp & 3u) << 5) | lane);
    }
    if (warp >= 2) {
      __threadfence();
      ptx::fence_proxy_async_global();
      ptx::tc_fence_before();
    }
    __syncthreads();
    if (tid == 0) {
      if (P.flags & SALUS_FLAG_TRACE) {
        const unsigned long long i = atomicAdd(&P.ctrl->n_trace, 1ull);
        if (i < P.trace_cap) {
          uint32_t smid;
          asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
          salus_trace_rec t;
          t.task = td.payload; t.smid = smid; t.job = td.job; t.iter = td.iter;
          t.t_claim = W.tr_claim; t.t_ready = W.tr_ready; t.t_mma = W.tr_mma; t.t_end = ptx::globaltimer();
          P.trace[i] = t;
        }
      }
      Slot &sl = P.slots[td.slot];
      const uint32_t old = ptx::atom_add_acqrel_u32(&sl.stage_done[td.stage], 1u);
      W.pub_flag = 0;
      if (old + 1 == td.ntiles) {
        if (td.is_last) {
          sl.end_ns = ptx::globaltimer();
          ptx::st_release_u64(&sl.done_seq, td.seq + 1);
        } else {
          W.pub_flag = 1;
          W.pub_base = atomicAdd(&P.ctrl->q_head, (unsigned long long)td.next_ntiles);
        }
      }
    }
    __syncthreads();
    if (W.pub_flag) {                          // publish the next stage's tiles
      const unsigned long long b0 = W.pub_base;
      for (uint32_t x = tid; x < td.next_ntiles; x += WORKER_THREADS) {
        const unsigned long long pos = b0 + x;
        ptx::st_release_u64(&P.ring[pos & P.ring_mask],
                            ((pos + 1) << 32) | task_pack(td.slot, td.stage + 1, x));
      }
    }
  }
  if (tid == 0) atomicAdd(&P.ctrl->n_tasks, my_tasks);
  __syncthreads();
  if (warp == 2) ptx::tmem_dealloc(tmem, TMEM_COLS);
}

}  // namespace salus
