// scheduler.cuh — the device-resident Salus scheduler: one warp of CTA 0 of
// the persistent kernel runs Algorithm 1 (GPU Lane Assignment, PAPER.md
// P:415-477) under the safety condition, the FIFO/SRTF/PACK/FAIR
// policies (§4) and the event loop "reacting when jobs arrive or
// finish, or at iteration boundaries", with the readings of
// DESIGN.md.
//
// Control flow is warp-uniform: every thread of the warp holds the same
// scalar state; scans over lanes / jobs / the pending queue are spread over
// the 32 threads (ballot / shuffle reductions); shared-memory writes of
// scalar state are done by thread 0 followed by __syncwarp().
//
// Run-ahead execution (A30 mode 2): decisions use logical ticks only, so the
// scheduler never waits for an iteration to finish; it appends each dispatch
// to its lane slot's ring (runahead.cuh) and moves on.  It blocks only for
// ring backpressure and for page-reuse fences (see pop_pages).
#pragma once
#include "salus_dev.h"
#include "ptx.cuh"
#include "runahead.cuh"

namespace salus {

constexpr int64_t IDLE_T = INT64_MAX;
constexpr uint16_t NONE16 = 0xFFFF;
constexpr uint32_t KEY_BITS = 11;          // dense job index < 2048 in key low bits

constexpr uint32_t REQ_STAGE = 9216;

struct SchedShared {
  // lane table, index order == lane id order
  uint32_t lane_id[MAX_LANES], lane_L[MAX_LANES], lane_slot[MAX_LANES], lane_back[MAX_LANES];
  int64_t lane_busy[MAX_LANES];
  uint64_t lane_seq[MAX_LANES];             // logical seq of the in-flight dispatch (log, stats)
  uint64_t lane_pseq[MAX_LANES];            // its physical record seq (page fences)
  uint32_t hL[MAX_LANES];                   // A35: lane sizes of a hypothetical eviction state
  uint16_t lane_cur[MAX_LANES], lane_last[MAX_LANES];
  // per job (dense index = (arrival, id) rank)
  int64_t svc[MAX_JOBS];
  int64_t c[MAX_JOBS];
  int64_t nrt[MAX_JOBS];                    // next request tick (INFER)
  uint32_t done[MAX_JOBS], pending[MAX_JOBS], next_req[MAX_JOBS];
  uint32_t n[MAX_JOBS], p[MAX_JOBS], e[MAX_JOBS], ap[MAX_JOBS], ae[MAX_JOBS];
  uint32_t id[MAX_JOBS];
  uint16_t Q[MAX_JOBS];
  uint16_t adm[MAX_JOBS];                   // admitted, unfinished
  uint8_t st[MAX_JOBS], jslot[MAX_JOBS], kind[MAX_JOBS];
  uint8_t xpre[MAX_JOBS];                   // DevJob.xpre (GEN prefetch), tagged on its records
  // run-ahead: records appended per physical slot, last appended seq + 1
  uint32_t sq_tail[MAX_LANES];
  uint64_t last_app[MAX_LANES];
  // last appended seq + 1 of a record that may translate through the slot's
  // page-table entries at or beyond the lane's current backing (set when the
  // backing shrinks or the lane closes): growing into those entries waits
  // for it, nothing else does
  uint64_t tail_seq[MAX_LANES];
  // static per-job data the per-tick loops read, cached from global memory
  uint16_t infer[MAX_JOBS];                 // dense indices of INFER jobs, ascending
  uint32_t req_off[MAX_JOBS];
  // phase_dispatch: per-slot minimum dispatch key over runnable residents
  unsigned long long slot_key[MAX_LANES];
  uint32_t q_head_seen[MAX_LANES];          // last q_head read per slot (backpressure)
  // request ticks staged in smem when they fit (C3: 8400): every request
  // arrival otherwise costs a dependent global load on the scheduler's path
  int64_t req_stage[REQ_STAGE];
};

__device__ __forceinline__ int64_t warp_min_i64(int64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    int64_t w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w < v ? w : v;
  }
  return v;
}
__device__ __forceinline__ uint64_t warp_min_u64(uint64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    uint64_t w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w < v ? w : v;
  }
  return v;
}
__device__ __forceinline__ uint64_t warp_max_u64(uint64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    uint64_t w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w > v ? w : v;
  }
  return v;
}
__device__ __forceinline__ uint32_t warp_max_u32(uint32_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    uint32_t w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w > v ? w : v;
  }
  return v;
}

struct Sched {
  const Params &P;
  SchedShared &S;
  uint32_t tid;
  // warp-uniform scalar state
  int64_t t = 0;
  uint64_t seq = 0, n_log = 0, n_ticks = 0, wait_ns = 0;
  // physical record seq: every record appended to a slot ring (iterations and
  // A35 swap records) takes the next one; done_seq, page fences and drains
  // count in it.  Equal to `seq` (logical dispatches) without eviction.
  uint64_t pseq = 0;
  uint64_t wait_fence_ns = 0, wait_ring_ns = 0;     // parts of wait_ns: page fences, full dispatch ring
  uint64_t append_ns = 0;                          // SALUS_DBG_SCHED builds
  const int64_t *rq = nullptr;                     // request ticks (smem stage or global)
  uint32_t nl = 0, qn = 0, an = 0, next_lane = 0, sumP = 0, sumL = 0, arr_ptr = 0, n_done = 0;
  uint32_t n_jobs = 0;                       // known jobs: submitted before the run + live ones seen
  bool live_done = true;                     // no more live jobs can come
  uint32_t free_top = 0, max_lanes = 0, err = 0;
  uint64_t slot_free = ~0ull;
  int64_t next_arrival = IDLE_T;
  bool dirty = false;
  bool physical = true;                      // false in SALUS_FLAG_NULL_WORK
  bool evict_mode = false;                   // SALUS_FLAG_EVICT (A35)
  uint64_t pend_mask = 0;                    // target slots with page-reuse fences
  uint32_t lreq_seen = 0;                    // live requests taken from the host ring

  __device__ Sched(const Params &p_, SchedShared &s_)
      : P(p_), S(s_), tid(threadIdx.x & 31), physical(!(p_.flags & SALUS_FLAG_NULL_WORK)),
        evict_mode((p_.flags & SALUS_FLAG_EVICT) != 0), rq(p_.req_ticks) {}

  __device__ void fail(int32_t code, uint32_t info) {
    if (tid == 0 && err == 0) {
      atomicCAS(reinterpret_cast<int *>(&P.ctrl->status), 0, code);
      P.ctrl->err_info[0] = info;
      if (P.host_abort) {   // the workers trap on the abort: leave the reason in the mapped slot
        volatile uint32_t *h = const_cast<volatile uint32_t *>(P.host_abort);
        h[1] = (uint32_t)code; h[2] = info; h[3] = (uint32_t)t;
        __threadfence_system();
      }
      atomicExch(&P.ctrl->abort, 1u);
    }
    err = 1;
    __syncwarp();
  }

  __device__ void emit(uint32_t kind, uint32_t lane, uint32_t job, uint32_t a, uint64_t b) {
    if ((P.flags & SALUS_FLAG_LOG) && tid == 0 && n_log < P.log_cap) {
      salus_log_rec r;
      r.tick = t; r.kind = kind; r.lane = lane; r.job = job; r.a = a; r.b = b;
      P.log[n_log] = r;
    }
    n_log++;
  }

  // ------------------------------------------------------------ page pool
  // A18: the arena is a pool of 64 KiB pages; a lane / persistent region is a
  // page list, so "auto defragmentation" never moves data.
  //
  // Run-ahead (A30 mode 2) makes page reuse the one physical hazard: a page
  // freed at logical tick t may still be in use by its previous owner's
  // queued iterations.  Every freed page therefore carries a fence (slot,
  // seq+1 of that owner's final iteration); popping it for a different
  // target slot records the fence, and the target's next record is appended
  // only after the fence iteration has physically completed.
  __device__ void pop_pages(uint32_t *dst, uint32_t k, uint32_t target, uint32_t lane_id) {
    if (k > free_top) { fail(SALUS_E_CAPACITY, 1); return; }
    bool any = false;
    for (uint32_t i = tid; i < k; i += 32) {
      const uint32_t pg = P.free_stack[free_top - k + i];
      dst[i] = pg;
      if (physical) {
        const uint64_t fs = P.fence_seq[pg];
        const uint32_t src = fs ? P.fence_slot[pg] : target;   // fence_slot is only set with a fence
        if (fs && src != target) {
          atomicMax(&P.pend_fence[target * MAX_LANES + src], (unsigned long long)fs);
          any = true;
          if (P.handoff_cap) {                  // I4 evidence: records of `target` from pseq on use it
            const unsigned long long n = atomicAdd(&P.ctrl->n_handoff, 1ull);
            if (n < P.handoff_cap) {
              salus_handoff_rec h;
              h.page = pg; h.to = target; h.from = src; h.to_lane = lane_id; h.from_seq = fs - 1; h.to_seq = pseq;
              P.handoff[n] = h;
            }
          }
        }
        P.fence_seq[pg] = 0;
      }
    }
    if (__any_sync(0xffffffffu, any)) pend_mask |= 1ull << target;
    free_top -= k;
    __syncwarp();
  }
  __device__ void push_pages(const uint32_t *src, uint32_t k, uint32_t fslot, uint64_t fseq) {
    for (uint32_t i = tid; i < k; i += 32) {
      const uint32_t pg = src[i];
      P.free_stack[free_top + i] = pg;
      if (physical) { P.fence_slot[pg] = (uint8_t)fslot; P.fence_seq[pg] = fseq + 1; }
    }
    free_top += k;
    __syncwarp();
  }
  __device__ uint32_t *lane_table(uint32_t slot) { return P.lpt + (uint64_t)slot * P.lpt_stride; }
  __device__ uint32_t *job_table(uint32_t j) { return P.ppt + P.jobs[j].pt_off; }

  // ------------------------------------------------------------ FindLane
  // Algorithm 1 FindLane with A1 (branch 2 keeps the safety
  // condition), A2 (best match = smallest L >= E, lowest id), A3 (branch 3
  // only for L_r < E, ascending (L_r, id)), A9 (max_lanes).
  // Returns 0 = none, 1 = new, 2 = reuse, 3 = resize; *li = lane index.
  // Over a lane table Ls[0..n_all) of which n_open exist (NONE32 = a lane
  // closed in a hypothetical eviction state, A35; it matches no branch).
  __device__ int find_lane_g(uint32_t p, uint32_t e, const uint32_t *Ls, uint32_t n_all, uint32_t n_open,
                             int64_t S_, uint32_t *li) const {
    const int64_t Cp = P.Cp;
    if (n_open < max_lanes && S_ + p + e <= Cp) return 1;
    if (S_ + p <= Cp) {
      uint32_t bestL = NONE32, bi = NONE32;
      for (uint32_t i = 0; i < n_all; i++) {
        uint32_t L = Ls[i];
        if (L >= e && L < bestL) { bestL = L; bi = i; }
      }
      if (bi != NONE32) { *li = bi; return 2; }
    }
    const int64_t thr = S_ + p + e - Cp;   // S - L + p + e <= C  <=>  L >= thr
    uint32_t bestL = NONE32, bi = NONE32;
    for (uint32_t i = 0; i < n_all; i++) {
      uint32_t L = Ls[i];
      if (L < e && (int64_t)L >= thr && L < bestL) { bestL = L; bi = i; }
    }
    if (bi != NONE32) { *li = bi; return 3; }
    return 0;
  }
  __device__ int find_lane(uint32_t p, uint32_t e, uint32_t *li) const {
    return find_lane_g(p, e, S.lane_L, nl, nl, (int64_t)sumP + (int64_t)sumL, li);
  }

  // ------------------------------------------------------------ helpers
  __device__ bool runnable(uint32_t j) const { return S.kind[j] == SALUS_TRAIN || S.pending[j] > 0; }

  // SRTF priority (A10/A11/A35): ((n - done) * c, dense index); smaller first
  __device__ uint64_t srtf_key(uint32_t j) const {
    return ((uint64_t)((int64_t)(S.n[j] - S.done[j]) * S.c[j]) << KEY_BITS) | j;
  }
  // a job with requests or iterations still to come (arrived, not finished)
  __device__ static bool live_state(uint8_t st) { return st == ST_QUEUED || st == ST_ADMITTED || st == ST_SWAPPED; }

  // min svc over admitted jobs in `slot` (excluding `skip`, optionally only
  // runnable ones); IDLE_T if none
  __device__ int64_t min_svc_in(uint32_t slot, uint32_t skip, bool only_runnable) const {
    int64_t m = IDLE_T;
    for (uint32_t a = tid; a < an; a += 32) {
      uint32_t j = S.adm[a];
      if (S.jslot[j] == slot && j != skip && (!only_runnable || runnable(j))) m = min(m, S.svc[j]);
    }
    return warp_min_i64(m);
  }

  __device__ bool host_abort() const { return P.host_abort && ptx::ld_volatile_u32(P.host_abort) != 0; }

  // Spin until `slot` has physically completed the iteration with seq + 1 ==
  // want (done_seq is monotonic per slot).
  __device__ void wait_slot(uint32_t slot, uint64_t want) {
    uint64_t t0 = ptx::globaltimer();
    uint32_t ok = 0, spins = 0;
    while (true) {
      if (tid == 0) ok = ptx::ld_acquire_u64(&P.slots[slot].done_seq) >= want;
      ok = __shfl_sync(0xffffffffu, ok, 0);
      if (ok) break;
      if ((++spins & 1023) == 0) {
        uint32_t bad = 0;
        if (tid == 0) bad = host_abort() || (ptx::globaltimer() - t0 > P.timeout_ns) ||
                            *(volatile uint32_t *)&P.ctrl->abort;
        bad = __shfl_sync(0xffffffffu, bad, 0);
        if (bad) { fail(host_abort() ? SALUS_E_TIMEOUT : SALUS_E_STUCK, 2); return; }
      }
    }
    wait_ns += ptx::globaltimer() - t0;
  }

  // ------------------------------------------------------------ phases
  __device__ void init_job(uint32_t j, const DevJob &J) {
    S.svc[j] = 0; S.c[j] = J.iter_ticks; S.done[j] = 0; S.pending[j] = 0; S.next_req[j] = 0;
    S.n[j] = J.n_iters; S.p[j] = J.p_pages; S.e[j] = J.e_pages; S.ap[j] = J.ap_pages; S.ae[j] = J.ae_pages;
    S.id[j] = J.job_id; S.st[j] = ST_NOT_ARRIVED; S.jslot[j] = 0xFF; S.kind[j] = (uint8_t)J.kind;
    // bit 0: GEN prefetch; bits 1-4: latency-mode lane limit of the job --
    // eager records only while nl x (its mean stage tasks) <= 2 x workers,
    // i.e. while the open lanes' stages cannot fill the GPU anyway (C2b's
    // 8 wide jobs would otherwise hold pairs waiting on each other's
    // stages), or while it runs alone (nl = 1: nothing else to wait for)
    S.xpre[j] = (uint8_t)(J.xpre | (min(15u, 2u * P.n_workers / max(1u, (uint32_t)J.lat_cost)) << 1));
    S.nrt[j] = J.kind == SALUS_INFER ? rq[J.req_off] : IDLE_T;
    S.req_off[j] = J.req_off;
    salus_job_stat &st = P.stats[j];
    st.job_id = J.job_id; st.first_lane = NONE32; st.admit_tick = -1; st.first_start_tick = -1;
    st.completion_tick = -1; st.completion_seq = ~0ull; st.wall_start_ns = 0; st.wall_end_ns = 0;
    st.wall_arrive_ns = 0;
  }

  // Online submission (SALUS_FLAG_ONLINE): once every
  // job known so far has arrived, take the jobs the host has published since
  // (descriptors already in P.jobs, in publication order = dense order) and
  // give them arrival tick t + 1 -- strictly after every processed tick, so
  // replaying the logged arrival ticks through the oracle gives this log.
  __device__ void poll_live() {
    if (live_done || arr_ptr < n_jobs) return;
    uint32_t np = 0, cl = 0;
    if (tid == 0) {
      // one 8-byte read of {n_published, closed}: a snapshot in one PCIe round
      // trip (the host closes only after its last publication)
      const unsigned long long v = *reinterpret_cast<const volatile unsigned long long *>(P.live);
      np = (uint32_t)v;
      cl = (uint32_t)(v >> 32);
    }
    cl = __shfl_sync(0xffffffffu, cl, 0);
    np = __shfl_sync(0xffffffffu, np, 0);
    if (np > P.max_jobs) { fail(SALUS_E_CAPACITY, 7); return; }
    if (np > n_jobs) {
      __threadfence_system();                 // their descriptors were uploaded before publication
      for (uint32_t j = n_jobs + tid; j < np; j += 32) {
        DevJob *Jw = const_cast<DevJob *>(P.jobs) + j;
        *(volatile int64_t *)&Jw->arrival = t + 1;
        DevJob J;
        const volatile uint32_t *src = reinterpret_cast<const volatile uint32_t *>(Jw);
        uint32_t *dst = reinterpret_cast<uint32_t *>(&J);
        for (uint32_t x = 0; x < sizeof(DevJob) / 4; x++) dst[x] = src[x];
        init_job(j, J);
      }
      __syncwarp();
      n_jobs = np;
      next_arrival = t + 1;
    }
    if (cl && np == n_jobs) live_done = true;
  }

  // Live requests (salus_submit_requests): take the requests the host has
  // published since the last poll, in publication order, and give each the
  // arrival tick t + 1 (never before its job's arrival) -- strictly after
  // every processed tick, like A34 -- plus the globaltimer it was seen at.
  // Returns true if any arrived.
  __device__ bool poll_requests() {
    if (!P.n_lreq || lreq_seen >= P.n_lreq) return false;
    uint32_t np = 0, last = 0;
    if (tid == 0) {
      // {count, job of the last entry} in one 8-byte acquire read at system
      // scope: the entries the host wrote before are read after it, and a
      // batch of one needs no second PCIe round trip
      unsigned long long v;
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(P.lreq) : "memory");
      np = (uint32_t)v;
      last = (uint32_t)(v >> 32);
    }
    np = __shfl_sync(0xffffffffu, np, 0);
    if (np == lreq_seen) return false;
    if (np > P.n_lreq) { fail(SALUS_E_CAPACITY, 9); return false; }
    if (tid == 0) {
      const uint64_t now = ptx::globaltimer();
      for (uint32_t k = lreq_seen; k < np; k++) {
        const uint32_t j = k + 1 == np ? last : ptx::ld_volatile_u32(P.lreq + 2 + k);
        // requests of j seen so far: every earlier one got a tick <= t and was
        // counted into next_req by phase_arrivals already, unless the job has
        // not arrived or this batch holds more than one (then the global count)
        const uint32_t c = (np == lreq_seen + 1 && S.st[j] != ST_NOT_ARRIVED) ? S.next_req[j] : P.lreq_cnt[j];
        P.lreq_cnt[j] = c + 1;
        // an arrived job takes t + 1; one still to arrive, its arrival tick
        const int64_t tk = S.st[j] != ST_NOT_ARRIVED ? t + 1
                         : (t + 1 > P.jobs[j].arrival ? t + 1 : P.jobs[j].arrival);
        P.req_ticks[S.req_off[j] + c] = tk;
        if (rq != P.req_ticks) S.req_stage[S.req_off[j] + c] = tk;   // the staged copy the tick loop reads
        P.req_seen[S.req_off[j] + c] = now;
        if (S.next_req[j] == c && S.nrt[j] == IDLE_T) S.nrt[j] = tk;   // the job was waiting for it
      }
    }
    __syncwarp();
    lreq_seen = np;
    return true;
  }

  // Nothing scheduled and the host may still submit jobs or requests: wait.
  __device__ bool wait_live() {
    const uint64_t t0 = ptx::globaltimer();
    // every mapped-memory read is a PCIe round trip (~1 us): requests are
    // polled every spin, live jobs and the abort flags every 16th
    for (uint32_t spin = 0; !err; spin++) {
      if (poll_requests()) break;
      if (live_done && lreq_seen >= P.n_lreq) break;   // nothing more can come
      if ((spin & 15) == 0) {
        if (!live_done) {
          poll_live();
          if (arr_ptr < n_jobs || live_done) break;
        }
        uint32_t bad = 0;
        if (tid == 0) bad = host_abort() || *(volatile uint32_t *)&P.ctrl->abort;
        if (__shfl_sync(0xffffffffu, bad, 0)) { fail(SALUS_E_TIMEOUT, 8); return false; }
      }
    }
    wait_ns += ptx::globaltimer() - t0;
    return !err;
  }

  __device__ void init() {
    const uint32_t N = P.n_jobs;
    if (P.n_req <= REQ_STAGE) {                       // live requests write both copies
      for (uint32_t i = tid; i < P.n_req; i += 32) S.req_stage[i] = P.req_ticks[i];
      __syncwarp();
      rq = S.req_stage;
    }
    for (uint32_t j = tid; j < N; j += 32) init_job(j, P.jobs[j]);
    n_jobs = N;
    live_done = P.live == nullptr;
    for (uint32_t i = tid; i < P.Cp; i += 32) P.free_stack[i] = P.Cp - 1 - i;
    for (uint32_t i = tid; i < MAX_LANES; i += 32) {
      S.sq_tail[i] = 0; S.last_app[i] = 0; S.tail_seq[i] = 0; S.q_head_seen[i] = 0;
    }
    for (uint32_t k = tid; k < P.n_infer; k += 32) S.infer[k] = P.infer_list[k];
    free_top = P.Cp;
    max_lanes = P.max_lanes;
    next_arrival = N ? P.jobs[0].arrival : IDLE_T;
    __syncwarp();
  }

  __device__ int64_t next_event() {
    int64_t m = IDLE_T;
    for (uint32_t i = tid; i < nl; i += 32) m = min(m, S.lane_busy[i]);
    for (uint32_t k = tid; k < P.n_infer; k += 32) {
      uint32_t j = S.infer[k];
      if (live_state(S.st[j])) m = min(m, S.nrt[j]);
    }
    m = warp_min_i64(m);
    return min(m, next_arrival);
  }

  __device__ void remove_lane(uint32_t i) {     // keep id order
    __syncwarp();                                // every lane's reads of the table are done
    for (uint32_t k = i; k + 1 < nl; k++) {
      if (tid == 0) {
        S.lane_id[k] = S.lane_id[k + 1]; S.lane_L[k] = S.lane_L[k + 1]; S.lane_slot[k] = S.lane_slot[k + 1];
        S.lane_back[k] = S.lane_back[k + 1]; S.lane_busy[k] = S.lane_busy[k + 1];
        S.lane_seq[k] = S.lane_seq[k + 1]; S.lane_pseq[k] = S.lane_pseq[k + 1];
        S.lane_cur[k] = S.lane_cur[k + 1]; S.lane_last[k] = S.lane_last[k + 1];
      }
    }
    nl--;
    __syncwarp();
  }

  __device__ void remove_adm(uint32_t j) {
    uint32_t pos = NONE32;
    for (uint32_t a = tid; a < an; a += 32)
      if (S.adm[a] == j) pos = a;
    pos = warp_max_u32(pos == NONE32 ? 0 : pos + 1) - 1;
    if (tid == 0) S.adm[pos] = S.adm[an - 1];
    an--;
    __syncwarp();
  }

  // P1: iteration completions and JobFinish (A4)
  // Lanes whose iteration ends at t are found 32 at a time with a ballot and
  // processed in lane-id order; a deleted lane shifts the later entries down
  // by one, so original index o sits at o - (lanes deleted before it).
  __device__ void phase_completions() {
    const uint32_t nl0 = nl;
    uint32_t removed = 0;
    for (uint32_t b = 0; b < nl0 && !err; b += 32) {
      const uint32_t o = b + tid;
      uint32_t m = __ballot_sync(0xffffffffu, o < nl0 && S.lane_busy[o - removed] == t);
      while (m) {
        const uint32_t i = b + (uint32_t)(__ffs(m) - 1) - removed;
        m &= m - 1;
        if (complete_lane(i)) removed++;
        if (err) return;
      }
    }
  }

  // the in-flight iteration of lane index i ended at t; JobFinish if it was
  // the job's last.  Returns true if the lane was deleted.
  __device__ bool complete_lane(uint32_t i) {
    {
      const uint32_t slot = S.lane_slot[i];
      const uint32_t j = S.lane_cur[i];
      __syncwarp();                              // the lanes' earlier reads of lane_busy are done
      if (tid == 0) { S.done[j] += 1; S.svc[j] += S.c[j]; S.lane_busy[i] = IDLE_T; }
      __syncwarp();
      if (S.done[j] == S.n[j]) {
        if (tid == 0) {
          S.st[j] = ST_DONE;
          P.stats[j].completion_tick = t;
        }
        n_done++; dirty = true; sumP -= S.p[j];
        __syncwarp();
        remove_adm(j);
        // completion_seq = seq of the final iteration = the lane's in-flight one
        emit(SALUS_REC_JOB_FINISH, S.lane_id[i], S.id[j], S.n[j], S.lane_seq[i]);
        uint64_t fseq = S.lane_pseq[i];
        if (physical && S.ap[j] > 0 && (P.jobs[j].dump & SALUS_DUMP_STATE)) {
          // migration (NEXT-4): copy the final persistent state to the job's
          // swap region behind its last iteration; its pages wait for the copy
          append(slot, S.lane_id[i], j, REC_SWAP_OUT);
          if (err) return false;
          fseq = S.last_app[slot] - 1;
        }
        push_pages(job_table(j), S.ap[j], slot, fseq);
        return lane_left(i, j, fseq);
      }
    }
    return false;
  }

  // Job j has left lane index i (JobFinish; eviction, A35): delete
  // the lane if ref(lane) == 0, else L = max E of its residents (A4) and the
  // backing shrinks to their max actual E.  Freed pages are fenced on the
  // slot's physical record `fseq` (~0 = none).  Returns true if deleted.
  __device__ bool lane_left(uint32_t i, uint32_t j, uint64_t fseq) {
    const uint32_t slot = S.lane_slot[i];
    uint32_t cnt = 0, maxe = 0, maxae = 0;
    for (uint32_t a = tid; a < an; a += 32) {
      uint32_t r = S.adm[a];
      if (S.jslot[r] == slot) { cnt++; maxe = max(maxe, S.e[r]); maxae = max(maxae, S.ae[r]); }
    }
    cnt = __reduce_add_sync(0xffffffffu, cnt);
    maxe = warp_max_u32(maxe);
    maxae = warp_max_u32(maxae);
    if (cnt == 0) {                           // ref(lane) == 0: delete lane
      emit(SALUS_REC_LANE_CLOSE, S.lane_id[i], S.id[j], 0, 0);
      push_pages(lane_table(slot), S.lane_back[i], slot, fseq);
      sumL -= S.lane_L[i];
      if (tid == 0) S.tail_seq[slot] = S.last_app[slot];
      slot_free |= (1ull << slot);
      remove_lane(i);
      return true;
    }
    if (maxe < S.lane_L[i]) {                 // A4: L_j = max E_i of residents
      emit(SALUS_REC_LANE_SHRINK, S.lane_id[i], S.id[j], maxe, S.lane_L[i]);
      sumL -= S.lane_L[i] - maxe;
      __syncwarp();
      if (tid == 0) S.lane_L[i] = maxe;
    }
    if (maxae < S.lane_back[i]) {
      push_pages(lane_table(slot) + maxae, S.lane_back[i] - maxae, slot, fseq);
      if (tid == 0) { S.lane_back[i] = maxae; S.tail_seq[slot] = S.last_app[slot]; }
    }
    __syncwarp();
    return false;
  }

  __device__ void q_insert(uint32_t j) {
    uint32_t pos = qn;
    if (P.policy == SALUS_SRTF) {            // A10: key ((n - done)*c, arrival, id) (A35: done > 0 when swapped)
      const uint64_t kj = srtf_key(j);
      uint32_t cnt = 0;
      for (uint32_t q = tid; q < qn; q += 32)
        if (srtf_key(S.Q[q]) < kj) cnt++;
      pos = __reduce_add_sync(0xffffffffu, cnt);
      // shift [pos, qn) right by one, high chunks first
      for (int64_t b = (int64_t)((qn - 1) & ~31u); qn > 0 && b >= (int64_t)(pos & ~31u); b -= 32) {
        uint32_t k = (uint32_t)b + tid;
        uint16_t v = (k < qn && k >= pos) ? S.Q[k] : 0;
        __syncwarp();
        if (k < qn && k >= pos) S.Q[k + 1] = v;
        __syncwarp();
      }
    }
    if (tid == 0) S.Q[pos] = (uint16_t)j;
    qn++;
    __syncwarp();
  }

  __device__ void q_remove(uint32_t pos) {
    for (uint32_t b = pos & ~31u; b < qn; b += 32) {
      uint32_t k = b + tid;
      uint16_t v = (k >= pos && k + 1 < qn) ? S.Q[k + 1] : 0;
      __syncwarp();
      if (k >= pos && k + 1 < qn) S.Q[k] = v;
      __syncwarp();
    }
    qn--;
    __syncwarp();
  }

  // P2: JobArrive and inference request arrivals (A27, A28)
  __device__ void phase_arrivals() {
    while (arr_ptr < n_jobs && next_arrival == t) {
      const uint32_t j = arr_ptr;
      if (tid == 0) { S.st[j] = ST_QUEUED; P.stats[j].wall_arrive_ns = ptx::globaltimer(); }
      __syncwarp();
      q_insert(j);
      emit(SALUS_REC_JOB_QUEUED, NONE32, S.id[j], 0, 0);
      dirty = true;
      arr_ptr++;
      next_arrival = arr_ptr < n_jobs ? P.jobs[arr_ptr].arrival : IDLE_T;
    }
    for (uint32_t k0 = 0; k0 < P.n_infer; k0 += 32) {
      const uint32_t k = k0 + tid;
      uint32_t j = 0, cnt = 0;
      if (k < P.n_infer) {
        j = S.infer[k];
        if (live_state(S.st[j]) && S.nrt[j] == t) {
          const uint32_t off = S.req_off[j];
          uint32_t nr = S.next_req[j];
          int64_t nt = t;                  // == rq[off + nr] (that is why we are here)
          while (nt == t) {
            nr++; cnt++;
            nt = nr < S.n[j] ? rq[off + nr] : IDLE_T;
          }
          S.next_req[j] = nr;
          S.nrt[j] = nt;
        }
      }
      uint32_t mask = __ballot_sync(0xffffffffu, cnt > 0);
      __syncwarp();
      while (mask) {                          // sequential in (arrival, id) order
        const int b = __ffs(mask) - 1;
        mask &= mask - 1;
        const uint32_t jj = __shfl_sync(0xffffffffu, j, b);
        const uint32_t cc = __shfl_sync(0xffffffffu, cnt, b);
        const bool was_idle = S.pending[jj] == 0;
        __syncwarp();
        if (tid == 0) S.pending[jj] += cc;
        __syncwarp();
        if (P.policy == SALUS_FAIR && S.st[jj] == ST_ADMITTED && was_idle) {
          // A28: an idle inference job re-enters at the min service of its
          // lane's runnable co-residents
          const uint32_t slot = S.jslot[jj];
          bool running = false;
          for (uint32_t i = 0; i < nl; i++)
            if (S.lane_slot[i] == slot) running = S.lane_busy[i] != IDLE_T && S.lane_cur[i] == jj;
          if (!running) {
            const int64_t co = min_svc_in(slot, jj, true);
            if (co != IDLE_T && tid == 0 && co > S.svc[jj]) S.svc[jj] = co;
            __syncwarp();
          }
        }
      }
    }
  }

  __device__ void admit(uint32_t j, int branch, uint32_t li) {
    const bool restored = S.st[j] == ST_SWAPPED;         // A35: re-admission of a victim
    uint32_t slot;
    if (branch == 1) {                                   // new lane
      // any free slot will do (slots are physical, never logged): prefer
      // one whose past records have all completed, so no drain is needed
      uint32_t idle = 0;
      for (uint32_t q = tid; q < MAX_LANES; q += 32)
        if (((slot_free >> q) & 1ull) &&
            (!physical || ptx::ld_acquire_u64(&P.slots[q].done_seq) >= S.tail_seq[q])) idle |= 1u << (q >> 5);
      // lanes hold bit q>>5 of slots q = tid, tid + 32: find the lowest idle slot
      const uint32_t m0 = __ballot_sync(0xffffffffu, idle & 1u), m1 = __ballot_sync(0xffffffffu, (idle >> 1) & 1u);
      slot = m0 ? (uint32_t)__ffs(m0) - 1 : m1 ? 32u + (uint32_t)__ffs(m1) - 1 : (uint32_t)__ffsll((long long)slot_free) - 1;
      slot_free &= ~(1ull << slot);
      li = nl;
      if (tid == 0) {
        S.lane_id[li] = next_lane; S.lane_L[li] = S.e[j]; S.lane_slot[li] = slot; S.lane_back[li] = 0;
        S.lane_busy[li] = IDLE_T; S.lane_cur[li] = NONE16; S.lane_last[li] = NONE16; S.lane_seq[li] = 0;
        S.lane_pseq[li] = 0;
      }
      next_lane++; nl++; sumL += S.e[j];
      __syncwarp();
      emit(SALUS_REC_LANE_OPEN, S.lane_id[li], S.id[j], S.e[j], 0);
    } else if (branch == 2) {                            // existing lane
      slot = S.lane_slot[li];
      emit(SALUS_REC_LANE_REUSE, S.lane_id[li], S.id[j], S.lane_L[li], 0);
    } else {                                             // replace
      slot = S.lane_slot[li];
      const uint32_t old = S.lane_L[li];
      sumL += S.e[j] - old;
      __syncwarp();
      if (tid == 0) S.lane_L[li] = S.e[j];
      __syncwarp();
      emit(SALUS_REC_LANE_RESIZE, S.lane_id[li], S.id[j], S.e[j], old);
    }
    // physical backing: the lane grows to the max actual E of its residents,
    // the job's persistent tensors get their own pages (Observation 2)
    if (S.ae[j] > S.lane_back[li]) {
      // the slot's page-table entries past the backing are about to be
      // rewritten: records that may still translate through them (queued
      // before the last shrink / close, run-ahead) must have completed.
      // Records of current residents only use entries below the backing.
      if (physical && S.tail_seq[slot]) wait_slot(slot, S.tail_seq[slot]);
      pop_pages(lane_table(slot) + S.lane_back[li], S.ae[j] - S.lane_back[li], slot, S.lane_id[li]);
      if (tid == 0) S.lane_back[li] = S.ae[j];
    }
    if (restored && physical && S.ap[j] > 0) {
      // its page-table entries are read by its swap-out record: rewrite them
      // only once that record has completed
      const uint64_t f = P.swap_fence[j];
      wait_slot((uint32_t)(f >> 56), f & ((1ull << 56) - 1));
    }
    pop_pages(job_table(j), S.ap[j], slot, S.lane_id[li]);
    if (P.policy == SALUS_FAIR) {                        // A12: virtual-time start
      const int64_t m = min_svc_in(slot, NONE32, false);
      if (tid == 0) S.svc[j] = (m == IDLE_T) ? 0 : m;
    }
    if (tid == 0) {
      S.adm[an] = (uint16_t)j; S.jslot[j] = (uint8_t)slot; S.st[j] = ST_ADMITTED;
      if (!restored) { P.stats[j].admit_tick = t; P.stats[j].first_lane = S.lane_id[li]; }
    }
    an++; sumP += S.p[j];
    __syncwarp();
    emit(restored ? SALUS_REC_JOB_RESTORE : SALUS_REC_JOB_ADMIT, S.lane_id[li], S.id[j], S.p[j], S.e[j]);
    // the copy back precedes the job's next iteration in the slot's ring; a
    // migrated job (NEXT-4) is copied in before its first iteration
    if (physical && S.ap[j] > 0 && (restored || (P.jobs[j].dump & DUMP_INTERNAL_RESUME) && S.done[j] == 0))
      append(slot, S.lane_id[li], j, REC_SWAP_IN);
  }

  // ------------------------------------------------------------ eviction (A35)
  // SALUS_FLAG_EVICT, SRTF: "the higher priority job is admitted as long as
  // its own safety condition is met ... regardless of other already-running
  // jobs".  Victims are admitted jobs with a larger SRTF key that are
  // not mid-iteration, largest key first, until FindLane succeeds on the
  // hypothetical state; all or nothing.

  __device__ uint32_t lane_index_of_slot(uint32_t slot) const {
    uint32_t i = 0;
    while (i < nl && S.lane_slot[i] != slot) i++;
    return i;
  }

  // swap out job v (its decision is final): leave the lane, free its pages
  // behind a swap-out record in its slot's ring
  __device__ void evict(uint32_t v) {
    const uint32_t slot = S.jslot[v];
    const uint32_t i = lane_index_of_slot(slot);
    if (tid == 0) S.st[v] = ST_SWAPPED;
    sumP -= S.p[v];
    __syncwarp();
    remove_adm(v);
    emit(SALUS_REC_JOB_EVICT, S.lane_id[i], S.id[v], S.p[v], S.done[v]);
    if (physical && S.ap[v] > 0) {
      append(slot, S.lane_id[i], v, REC_SWAP_OUT);
      if (err) return;
      if (tid == 0) P.swap_fence[v] = ((unsigned long long)slot << 56) | S.last_app[slot];
      __syncwarp();
    }
    // the last record of the slot (the swap-out; ~0 = none ever) fences the pages
    const uint64_t fseq = S.last_app[slot] - 1;
    push_pages(job_table(v), S.ap[v], slot, fseq);
    lane_left(i, v, fseq);
  }

  __device__ bool executing(uint32_t v) const {
    const uint32_t i = lane_index_of_slot(S.jslot[v]);
    return i < nl && S.lane_busy[i] != IDLE_T && S.lane_cur[i] == v;
  }

  // Returns FindLane's branch for j after the evictions (0: nobody evicted).
  // Victims are appended to P.evl[*nev..] (they join Q after the pass).
  __device__ int evict_for(uint32_t j, uint32_t *li, uint32_t *nev) {
    const uint64_t kj = srtf_key(j);
    int64_t hP = sumP;
    uint32_t nch = 0;
    bool fits = false;
    for (;;) {
      uint64_t best = 0;
      for (uint32_t a = tid; a < an; a += 32) {
        const uint32_t v = S.adm[a];
        if (S.st[v] != ST_ADMITTED) continue;          // chosen already in this attempt
        const uint64_t kv = srtf_key(v);
        if (kv > kj && kv > best && !executing(v)) best = kv;
      }
      best = warp_max_u64(best);
      if (best == 0) break;                             // no candidate left
      const uint32_t v = (uint32_t)(best & ((1u << KEY_BITS) - 1));
      if (tid == 0) { S.st[v] = ST_SWAPPED; P.evl[*nev + nch] = (uint16_t)v; }
      nch++;
      hP -= S.p[v];
      __syncwarp();
      int64_t hS = hP;
      uint32_t nopen = 0;
      for (uint32_t i = 0; i < nl; i++) {               // L = max e of the remaining residents
        uint32_t cnt = 0, mx = 0;
        for (uint32_t a = tid; a < an; a += 32) {
          const uint32_t r = S.adm[a];
          if (S.st[r] == ST_ADMITTED && S.jslot[r] == S.lane_slot[i]) { cnt++; mx = max(mx, S.e[r]); }
        }
        cnt = __reduce_add_sync(0xffffffffu, cnt);
        mx = warp_max_u32(mx);
        if (tid == 0) S.hL[i] = cnt ? mx : NONE32;
        if (cnt) { hS += mx; nopen++; }
      }
      __syncwarp();
      uint32_t hli;
      if (find_lane_g(S.p[j], S.e[j], S.hL, nl, nopen, hS, &hli)) { fits = true; break; }
    }
    __syncwarp();
    if (!fits) {                                        // nothing is evicted
      for (uint32_t k = tid; k < nch; k += 32) S.st[P.evl[*nev + k]] = ST_ADMITTED;
      __syncwarp();
      return 0;
    }
    for (uint32_t k = 0; k < nch && !err; k++) evict(P.evl[*nev + k]);
    *nev += nch;
    return find_lane(S.p[j], S.e[j], li);
  }

  // P3 with eviction: one in-order pass over Q (sorted by SRTF key); a job
  // FindLane rejects may evict; victims join Q after the pass (so none is
  // re-admitted in the pass that evicted it).
  __device__ void phase_admission_evict() {
    uint32_t pos = 0, nev = 0;
    while (pos < qn && !err) {
      const uint32_t j = S.Q[pos];
      uint32_t li = 0;
      int br = find_lane(S.p[j], S.e[j], &li);
      if (br == 0) br = evict_for(j, &li, &nev);
      if (br == 0) { pos++; continue; }
      q_remove(pos);
      admit(j, br, li);
    }
    for (uint32_t k = 0; k < nev; k++) q_insert(P.evl[k]);
  }

  // P3: ProcessRequests — one in-order pass over Q (A5, A7, A8, A14)
  __device__ void phase_admission() {
    uint32_t pos = 0;
    while (pos < qn && !err) {
      uint32_t first = NONE32;
      if (P.policy == SALUS_FIFO) {                      // A14: exclusive, strict HOL
        if (an > 0) break;
        uint32_t li;
        if (find_lane(S.p[S.Q[0]], S.e[S.Q[0]], &li) == 0) break;
        first = 0;
      } else {
        for (uint32_t b = pos; b < qn && first == NONE32; b += 32) {
          const uint32_t k = b + tid;
          uint32_t li;
          const bool ok = k < qn && find_lane(S.p[S.Q[k]], S.e[S.Q[k]], &li) != 0;
          const uint32_t m = __ballot_sync(0xffffffffu, ok);
          if (m) first = b + __ffs(m) - 1;
        }
        if (first == NONE32) break;
      }
      const uint32_t j = S.Q[first];
      uint32_t li = 0;
      const int br = find_lane(S.p[j], S.e[j], &li);
      __syncwarp();
      q_remove(first);
      admit(j, br, li);
      pos = first;
    }
  }

  // Page-reuse fences of `slot` (pop_pages): wait until every source slot has
  // physically completed the recorded iteration, then clear them.
  __device__ void wait_fences(uint32_t slot) {
    if (!((pend_mask >> slot) & 1ull)) return;
    for (uint32_t q = 0; q < MAX_LANES; q++) {
      unsigned long long *pf = &P.pend_fence[slot * MAX_LANES + q];
      const uint64_t want = *(volatile unsigned long long *)pf;
      if (want) {
        const uint64_t w0 = wait_ns;
        wait_slot(q, want);
        wait_fence_ns += wait_ns - w0;
        if (err) return;
        if (tid == 0) *pf = 0;
      }
    }
    __syncwarp();
    pend_mask &= ~(1ull << slot);
  }

  // Append the dispatch to the slot's ring (A30 mode 2); if the slot is idle,
  // take the `running` token and start it here, else the worker finishing
  // the slot's current iteration will.
  __device__ void append(uint32_t slot, uint32_t lane_id, uint32_t j, uint32_t kind = REC_ITER) {
#if SALUS_DBG_SCHED
    const uint64_t ta_ = ptx::globaltimer();
    append_body(slot, lane_id, j, kind);
    append_ns += ptx::globaltimer() - ta_;
  }
  __device__ void append_body(uint32_t slot, uint32_t lane_id, uint32_t j, uint32_t kind) {
#endif
    wait_fences(slot);
    if (err) return;
    Slot &sl = P.slots[slot];
    const uint32_t tl = S.sq_tail[slot];
    {                                                      // backpressure: RQ in flight
      uint64_t t0 = 0;
      uint32_t full = 1, spins = 0;
      while (true) {
        // the cached head usually proves there is room without a load
        if (tid == 0) {
          full = ((tl - S.q_head_seen[slot]) & 0x7FFFFFFFu) >= RQ;
          if (full) {
            S.q_head_seen[slot] = qs_head(ld_acquire_u64q(&sl.qstate));
            full = ((tl - S.q_head_seen[slot]) & 0x7FFFFFFFu) >= RQ;
          }
        }
        full = __shfl_sync(0xffffffffu, full, 0);
        if (!full) break;
        if (t0 == 0) t0 = ptx::globaltimer();
        if ((++spins & 1023) == 0) {
          uint32_t bad = 0;
          if (tid == 0) bad = host_abort() || (ptx::globaltimer() - t0 > P.timeout_ns) ||
                              *(volatile uint32_t *)&P.ctrl->abort;
          if (__shfl_sync(0xffffffffu, bad, 0)) { fail(host_abort() ? SALUS_E_TIMEOUT : SALUS_E_STUCK, 6); return; }
        }
      }
      if (t0) { wait_ns += ptx::globaltimer() - t0; wait_ring_ns += ptx::globaltimer() - t0; }
    }
    uint32_t won = 0;
    DispRec rec;                                           // (thread 0) the record as appended
    __syncwarp();                                          // every lane has read sq_tail
    if (tid == 0) {
      volatile DispRec *vr = &sl.recs[tl % RQ];
      const bool eager = kind == REC_ITER && nl <= P.eager_lanes && (nl == 1 || nl <= (uint32_t)(S.xpre[j] >> 1));
      rec.job = j; rec.iter = S.done[j]; rec.seq = pseq; rec.lseq = seq; rec.lane_id = lane_id;
      rec.kind = kind | ((kind == REC_ITER && (S.xpre[j] & 1u)) ? REC_FLAG_XPRE : 0u) |
                 (eager ? REC_FLAG_EAGER : 0u) | ((eager && nl <= P.narrow_lanes) ? REC_FLAG_NARROW : 0u);
      rec.append_ns = ptx::globaltimer();
      // what starting the record publishes (the record carries it, so the
      // thread that starts it -- here or a completion warp -- reads no
      // descriptor)
      const DevJob &JJ = P.jobs[rec.job];
      const bool narrow = (rec.kind & REC_FLAG_NARROW) != 0;
      rec.first = first_stage_of(rec, P.jobs);
      rec.second = eager_second(JJ, rec.kind, rec.first);
      rec.n1 = stage_ntiles(JJ, rec.first, narrow);
      rec.n2 = rec.second != NONE32 ? stage_ntiles(JJ, rec.second, narrow) : 0;
      vr->job = rec.job; vr->iter = rec.iter; vr->seq = rec.seq; vr->lseq = rec.lseq;
      vr->lane_id = rec.lane_id; vr->kind = rec.kind; vr->append_ns = rec.append_ns;
      vr->first = rec.first; vr->second = rec.second; vr->n1 = rec.n1; vr->n2 = rec.n2;
    }
    uint32_t first = 0, second = NONE32, n1 = 0, n2 = 0;
    if (tid == 0) {
      first = rec.first; second = rec.second; n1 = rec.n1; n2 = rec.n2;
      // publish (release) and learn whether the slot was idle in one atomic;
      // only the scheduler ever sets `running`, so taking it needs no CAS
      won = (atom_add_release_u64(&sl.qstate, QS_TAIL_ONE) & 1ull) == 0;
      S.sq_tail[slot] = tl + 1;
      S.last_app[slot] = pseq + 1;
    }
    pseq++;
    __syncwarp();
    won = __shfl_sync(0xffffffffu, won, 0);
    if (!won) return;
    unsigned long long base = 0;
    if (tid == 0) {
      // running was clear, so the ring was empty (a holder consumes every
      // record before releasing): the record just appended at index tl is
      // the only one -- take it from registers (set running, head + 1)
      // instead of take_next's round trips through the ring
      atomicAdd(&sl.qstate, 1ull + QS_HEAD_ONE);
      base = atomicAdd(&P.ctrl->q_head, (unsigned long long)(n1 + n2));   // overlaps the fence below
      begin_iteration(sl, rec);
    }
    first = __shfl_sync(0xffffffffu, first, 0);
    second = __shfl_sync(0xffffffffu, second, 0);
    n1 = __shfl_sync(0xffffffffu, n1, 0);
    n2 = __shfl_sync(0xffffffffu, n2, 0);
    base = __shfl_sync(0xffffffffu, base, 0);
    // eager: the second stage's tiles go behind the first's (higher ring
    // positions), so every tile's dependency sits at a lower position
    publish_tiles(P.ring, P.ring_mask, tid, base, slot, first, n1, second, n2);
  }

  // End of the schedule: wait for every slot to drain its ring.
  __device__ void drain() {
    for (uint32_t s = 0; s < MAX_LANES && !err; s++)
      if (S.last_app[s]) wait_slot(s, S.last_app[s]);
  }

  // P4: every idle lane dispatches its next iteration
  __device__ void phase_dispatch() {

    // one pass over the residents: the minimum key of each slot (a lane owns
    // one slot and a job one lane, so dispatching on one lane never changes
    // another lane's minimum)
    bool idle = false;
    for (uint32_t i = tid; i < nl; i += 32) idle |= S.lane_busy[i] == IDLE_T;
    if (!__any_sync(0xffffffffu, idle)) return;
    for (uint32_t i = tid; i < nl; i += 32) S.slot_key[S.lane_slot[i]] = ~0ull;
    __syncwarp();
    for (uint32_t a = tid; a < an; a += 32) {
      const uint32_t j = S.adm[a];
      if (!runnable(j)) continue;
      uint64_t key;
      if (P.policy == SALUS_SRTF)          // A11: remaining = (n - done) * c
        key = ((uint64_t)((int64_t)(S.n[j] - S.done[j]) * S.c[j]) << KEY_BITS) | j;
      else if (P.policy == SALUS_FAIR)     // least service
        key = ((uint64_t)S.svc[j] << KEY_BITS) | j;
      else                                 // FIFO / PACK (A13): earliest arrival
        key = j;
      atomicMin(&S.slot_key[S.jslot[j]], (unsigned long long)key);
    }
    __syncwarp();
    // idle lanes with a runnable resident, 32 at a time, in lane-id order
    for (uint32_t b = 0; b < nl && !err; b += 32) {
      const uint32_t k = b + tid;
      uint32_t m = __ballot_sync(0xffffffffu, k < nl && S.lane_busy[k] == IDLE_T && S.slot_key[S.lane_slot[k]] != ~0ull);
      while (m && !err) {
        const uint32_t i = b + (uint32_t)(__ffs(m) - 1);
        m &= m - 1;
        dispatch_lane(i);
      }
    }
  }

  __device__ void dispatch_lane(uint32_t i) {
    {
      const uint32_t slot = S.lane_slot[i];
      const uint64_t best = S.slot_key[slot];
      const uint32_t j = (uint32_t)(best & ((1u << KEY_BITS) - 1));
      const uint16_t last = S.lane_last[i];
      const int64_t pen = (last != NONE16 && last != j) ? P.switch_ticks : 0;   // A16
      if (tid == 0) {
        S.lane_busy[i] = t + pen + S.c[j];
        S.lane_cur[i] = (uint16_t)j; S.lane_last[i] = (uint16_t)j; S.lane_seq[i] = seq; S.lane_pseq[i] = pseq;
        if (S.kind[j] == SALUS_INFER) S.pending[j] -= 1;
        salus_job_stat &st = P.stats[j];
        if (S.done[j] == 0) st.first_start_tick = t;   // a job's iterations never overlap
        st.completion_seq = seq;
      }
      __syncwarp();
      emit(SALUS_REC_DISPATCH, S.lane_id[i], S.id[j], S.done[j], seq);
      if (physical) append(slot, S.lane_id[i], j);
      seq++;
    }
  }

  __device__ void check_safety() {
    if ((uint64_t)sumP + sumL > P.Cp) fail(SALUS_E_STATE, 3);   // I1
  }

  __device__ void run() {
    init();
    const uint64_t wall0 = ptx::globaltimer();
#if SALUS_DBG_SCHED   // per-phase time (ns) -> the tail of the trace buffer
    uint64_t ph[6] = {0, 0, 0, 0, 0, 0};
#define SALUS_PH(i, stmt) { const uint64_t t0_ = ptx::globaltimer(); stmt; ph[i] += ptx::globaltimer() - t0_; }
#else
#define SALUS_PH(i, stmt) stmt;
#endif
    bool woke = false;                       // wait_live just polled the host
    while (!err) {
      if (!woke) {
        if (!live_done && (n_ticks & 15) == 0) poll_live();
        if ((n_ticks & 7) == 0) poll_requests();
      }
      woke = false;
      if (n_done == n_jobs && live_done) break;
      int64_t tn;
      SALUS_PH(0, tn = next_event())
      if (tn == IDLE_T) {
        if (!live_done || lreq_seen < P.n_lreq) { if (!wait_live()) break; woke = true; continue; }
        fail(SALUS_E_STUCK, 4);
        break;
      }
      t = tn;
      n_ticks++;
      dirty = false;
      SALUS_PH(1, phase_completions())
      if (err) break;
      SALUS_PH(2, phase_arrivals())
      // A35: with eviction an iteration end can make its job evictable, so
      // the pass runs at every tick with a queued job
      if (qn > 0 && evict_mode) SALUS_PH(3, phase_admission_evict())
      else if (qn > 0 && dirty) SALUS_PH(3, phase_admission())
      if (P.flags & SALUS_FLAG_CHECK) check_safety();
      SALUS_PH(4, phase_dispatch())
      if ((n_ticks & 255) == 0) {
        uint32_t bad = 0;
        if (tid == 0) bad = host_abort();
        if (__shfl_sync(0xffffffffu, bad, 0)) fail(SALUS_E_TIMEOUT, 5);
      }
    }
#if SALUS_DBG_SCHED
    if (tid == 0 && P.trace_cap) {
      uint64_t *dbg = reinterpret_cast<uint64_t *>(P.trace + P.trace_cap) - 8;
      for (int i = 0; i < 6; i++) dbg[i] = ph[i];
      dbg[6] = append_ns;
    }
#endif
#undef SALUS_PH
    if (physical && !err) drain();
    // release the workers
    {
      unsigned long long base = 0;
      if (tid == 0) base = atomicAdd(&P.ctrl->q_head, (unsigned long long)P.n_workers);
      base = __shfl_sync(0xffffffffu, base, 0);
      for (uint32_t k = tid; k < P.n_workers; k += 32) {
        unsigned long long pos = base + k;
        ptx::st_release_u64(&P.ring[pos & P.ring_mask], ((pos + 1) << 32) | TASK_EXIT);
      }
    }
    if (tid == 0) {
      P.ctrl->n_dispatch = seq; P.ctrl->n_ticks = n_ticks; P.ctrl->n_log = n_log;
      P.ctrl->sched_wait_ns = wait_ns; P.ctrl->wall_first_ns = wall0;
      P.ctrl->sched_fence_ns = wait_fence_ns; P.ctrl->sched_ring_ns = wait_ring_ns;
      P.ctrl->wall_last_ns = ptx::globaltimer();
      P.ctrl->log_overflow = ((P.flags & SALUS_FLAG_LOG) && n_log > P.log_cap) ? 1u : 0u;
    }
  }
};

}  // namespace salus
