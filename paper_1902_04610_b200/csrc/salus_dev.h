// salus_dev.h — internal structures shared by the host library and the
// persistent kernel (never by oracle/).  Layouts are described in DESIGN.md
// ("Data layout in HBM", "Meta buffer").
#pragma once
#include <stdint.h>
#include <cuda.h>
#include "../../include/salus.h"

namespace salus {

constexpr int MAX_LANES = 64;          // lane table (A9)
constexpr int MAX_JOBS = 2048;         // scheduler SMEM tables
constexpr int MAX_LAYERS = 8;
constexpr int MAX_STAGES = 2 + 2 * MAX_LAYERS;   // INIT, GEN, F_1..F_L, B_L..B_1
constexpr uint32_t PAGE_SHIFT = 16;    // 64 KiB pages (A18)
constexpr uint32_t PAGE_BYTES = 1u << PAGE_SHIFT;
constexpr uint32_t NONE32 = 0xFFFFFFFFu;
constexpr uint32_t TASK_EXIT = 0xFFFFFFFFu;

// Job states (oracle: NOT_ARRIVED, QUEUED, ADMITTED, DONE)
// + SWAPPED (A35, SALUS_FLAG_EVICT): admitted once, persistent pages on the host, in Q
enum : uint8_t { ST_NOT_ARRIVED = 0, ST_QUEUED = 1, ST_ADMITTED = 2, ST_DONE = 3, ST_SWAPPED = 4 };

// Static per-job descriptor, uploaded by salus_prepare.  The dense index of
// a job is its rank in (arrival_tick, job_id) order, so every "(arrival, id)"
// tie-break of the readings (A11-A15) is a comparison of dense indices.
struct alignas(128) DevJob {   // whole cache lines: a live job's descriptor never
                               // shares one with a descriptor already read
  uint32_t job_id, kind, n_layers, batch;
  int64_t arrival, iter_ticks;
  uint32_t n_iters, p_pages, e_pages;     // declared sizes in pages (schedule)
  uint32_t ap_pages, ae_pages;            // actual backing pages (device layout)
  uint32_t bpad;                          // batch padded to 128
  uint32_t dims[MAX_LAYERS + 1];          // logical widths
  uint32_t dpad[MAX_LAYERS + 1];          // padded to 128
  float lr;
  uint32_t dump;
  uint64_t seed;
  uint32_t req_off;                       // index into request tick array
  uint32_t pt_off;                        // index into the persistent page-table pool
  uint64_t dump_out_off;                  // float offset of outputs in the dump area
  uint64_t dump_w_off;                    // float offset of final weights
  // byte offsets inside the job's persistent space: per layer W32, Wb[0], Wb[1]
  uint32_t w32_off[MAX_LAYERS], wb_off[MAX_LAYERS][2];
  // byte offsets inside the lane's ephemeral space: act[0]=X, act[l]=A_l; g[2]
  uint32_t act_off[MAX_LAYERS + 1], g_off[2];
  uint32_t n_stages;                      // stages of a non-first iteration path
  uint32_t stage_tiles[MAX_STAGES];       // tiles per stage
  uint32_t iter_base;                     // migration (NEXT-4): global index of local iteration 0
};

// DevJob.dump bit set by the host: the job resumes from a state image
// (its first iteration copies the image in instead of initialising weights)
constexpr uint32_t DUMP_INTERNAL_RESUME = 1u << 31;

// Run-ahead execution (A30 mode 2): the scheduler appends dispatch records to
// a per-slot ring; the thread that completes an iteration starts the slot's
// next record itself, so a lane never waits for the scheduler.
#ifndef SALUS_RQ
#define SALUS_RQ 4096
#endif
// records queued per slot (run-ahead depth): deep enough that the scheduler,
// which emits dispatches in logical order, is never held back by one lane's
// full ring while another lane runs dry (C3: 1k+ requests per lane)
constexpr uint32_t RQ = SALUS_RQ;

// Record kinds: an iteration, or (A35) a swap of the job's persistent pages
enum : uint32_t { REC_ITER = 0, REC_SWAP_OUT = 1, REC_SWAP_IN = 2 };

struct DispRec {
  uint32_t job, iter;                  // dense job index, iteration index
  uint64_t seq;                        // physical record seq (done_seq, page fences)
  uint32_t lane_id, kind;              // logical lane id (for the wall log), REC_*
  uint64_t append_ns;                  // globaltimer of the scheduler's append
  uint64_t lseq;                       // logical dispatch seq (log, wall stamps)
};

// One physical lane slot.  256-B aligned.
struct alignas(256) Slot {
  // the in-flight iteration (written by whoever started it)
  uint32_t job;             // dense job index of the in-flight iteration
  uint32_t iter;            // iteration index k
  uint64_t seq;             // physical record seq
  uint64_t lseq;            // logical dispatch seq (REC_ITER)
  uint32_t rkind;           // REC_*
  uint64_t start_ns;        // min globaltimer over first-stage tiles (atomicMin)
  uint64_t end_ns;          // globaltimer when the last stage completed
  uint64_t done_seq;        // seq + 1 of the last physically completed iteration (monotonic)
  uint32_t lane_id;
  uint64_t append_ns;       // when the in-flight iteration's record was appended
  uint32_t stage_done[32];         // per stage number (5 bits; 30, 31 = swap copies)
  // dispatch ring: qstate = records appended << 32 | running (1 while an
  // iteration is in flight or being started), one word so that append and
  // release race through single atomics
  unsigned long long qstate;
  uint32_t q_head;          // records started (only the holder of `running`)
  DispRec recs[RQ];
};

// Control block at the start of meta.
struct alignas(256) Ctrl {
  unsigned long long q_head;     // task ring: next position to publish
  unsigned long long q_tail;     // next position to claim
  unsigned long long n_tasks;
  uint32_t abort;                // set on device error or host abort
  int32_t status;                // SALUS_OK or SALUS_E_*
  uint32_t err_info[4];
  uint64_t n_dispatch, n_ticks, n_log, sched_wait_ns, sched_fence_ns, sched_ring_ns;
  uint64_t wall_first_ns, wall_last_ns;
  uint32_t log_overflow, n_workers;
  unsigned long long n_trace;
  unsigned long long n_swap_out, n_swap_in, swap_bytes, swap_ns;   // A35 swap records
};

struct Params {
  // The arena viewed as a 2-D tensor of 128-byte rows (uint8, no swizzle:
  // the data are already stored in the smem image).  Box = 128 or 64 rows,
  // i.e. one 16 KiB / 8 KiB operand block per TMA.  Tensor copies are the
  // only bulk copies that can complete on the PEER CTA's mbarrier
  // (.cta_group::2), which lets both CTAs of a pair fill the leader's stage
  // barrier directly.
  CUtensorMap tmap16, tmap8;
  uint8_t *arena;
  Ctrl *ctrl;
  const DevJob *jobs;
  const int64_t *req_ticks;
  const uint16_t *infer_list;      // dense indices of INFER jobs, ascending
  uint32_t *ppt;                   // persistent page tables (pool)
  uint32_t *lpt;                   // lane page tables: MAX_LANES x lpt_stride
  uint32_t lpt_stride;
  uint32_t *free_stack;            // Cp entries
  uint8_t *fence_slot;             // per page: slot of its last user (A30 mode 2 fences)
  uint64_t *fence_seq;             // per page: last user's final seq + 1 (0 = none)
  unsigned long long *pend_fence;  // [target slot][source slot]: seq + 1 to wait for
  Slot *slots;                     // MAX_LANES
  unsigned long long *ring;        // task ring (seq << 32 | payload)
  uint32_t ring_mask;
  salus_log_rec *log;
  salus_wall_rec *wall;
  uint64_t log_cap;
  salus_job_stat *stats;           // dense order
  salus_trace_rec *trace;
  uint64_t trace_cap;
  float *dump;
  const volatile uint32_t *host_abort;   // mapped pinned host flag
  uint32_t n_jobs, n_infer, Cp, policy, max_lanes, flags, n_workers;
  uint32_t n_req;                  // request ticks in req_ticks
  uint32_t max_jobs;               // descriptor capacity (online submission)
  uint32_t *live;                  // mapped {n_published, closed} (SALUS_FLAG_ONLINE), else null
  int64_t switch_ticks;
  uint64_t timeout_ns;
  // SALUS_FLAG_EVICT (A35): pinned host swap area (job j's region at
  // pt_off * PAGE_BYTES, ap_pages pages), per-job fence of its last swap-out
  // record (slot << 56 | seq + 1), victims of the current admission pass
  uint8_t *swap;
  unsigned long long *swap_fence;
  uint16_t *evl;
};

// A35 swap records run as one stage of copy tasks (two 64 KiB pages per pair task)
constexpr uint32_t STAGE_SWAP_OUT = 30, STAGE_SWAP_IN = 31;
__host__ __device__ inline uint32_t stage_ntiles(const DevJob &J, uint32_t stage) {
  return stage >= STAGE_SWAP_OUT ? (J.ap_pages + 1) / 2 : J.stage_tiles[stage];
}

// task payload: slot (6 bits) | stage (5 bits) | tile (21 bits)
__host__ __device__ inline uint32_t task_pack(uint32_t slot, uint32_t stage, uint32_t tile) {
  return (slot << 26) | (stage << 21) | tile;
}

// Stage numbering: 0 INIT (first iteration only), 1 GEN, 2..L+1 F_1..F_L,
// L+2..2L+1 B_L..B_1 (TRAIN only).
__host__ __device__ inline uint32_t last_stage(uint32_t kind, uint32_t L) {
  return kind == SALUS_TRAIN ? 2 * L + 1 : L + 1;
}

// GEMM N tile for an output width (padded to 128): 256 when it divides, else
// 128.  Wide tiles halve operand re-reads; the epilogue streams its input
// (fp32 master weights / ReLU mask) through three 32 KiB smem chunk buffers.
__host__ __device__ inline uint32_t ntile_for(uint32_t dpad) { return (dpad % 256 == 0) ? 256 : 128; }

}  // namespace salus
