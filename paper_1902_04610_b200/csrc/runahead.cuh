// runahead.cuh — per-slot dispatch rings for run-ahead execution (SURVEY
// §8(c)-A30 mode 2).
//
// The schedule is decided purely in logical ticks by the scheduler warp,
// which appends each DISPATCH to its lane slot's ring of RQ records.  A slot
// executes its records strictly in order ("iteration execution is serialised
// within a lane"): whoever holds the slot's `running` token —
// the scheduler after an append to an idle slot, or the worker thread that
// completes an iteration's last tile — takes the next record and starts it.
// The handoff goes through one 64-bit word per slot, qstate = tail << 32 |
// head << 1 | running: the appender's atomic add (release) publishes a record and tells
// it whether the slot was idle; the holder releases `running` only with a
// CAS that expects the tail it has consumed up to, so an append racing with
// the last completion is never lost and no store/fence/load Dekker pair (two
// full fences per handoff) is needed.
#pragma once
#include "salus_dev.h"
#include "ptx.cuh"

namespace salus {

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(uint32_t *p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ unsigned long long ld_acquire_u64q(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long atom_add_release_u64(unsigned long long *p, unsigned long long v) {
  unsigned long long old;
  asm volatile("atom.add.release.gpu.global.u64 %0, [%1], %2;" : "=l"(old) : "l"(p), "l"(v) : "memory");
  return old;
}

// qstate = tail << 32 | head << 1 | running: records appended (tail, 32
// bits), records started (head, 31 bits), running bit.  One acquire load
// gives the holder both counters; it bumps head with one release add.
constexpr unsigned long long QS_HEAD_ONE = 2ull, QS_TAIL_ONE = 1ull << 32;
__host__ __device__ __forceinline__ uint32_t qs_head(unsigned long long st) { return (uint32_t)(st >> 1) & 0x7FFFFFFFu; }
__host__ __device__ __forceinline__ uint32_t qs_tail(unsigned long long st) { return (uint32_t)(st >> 32) & 0x7FFFFFFFu; }

__device__ __forceinline__ void red_add_release_u64(unsigned long long *p, unsigned long long v) {
  asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Caller holds `running`.  Takes the next record (true) or releases the token
// (false): the CAS succeeds only if no record was appended since the load.
// The head bump is a release so the record's slot in the ring (reused RQ
// records later) is only handed back after it was read.
__device__ __forceinline__ bool take_next(Slot &sl, DispRec *rec) {
  for (;;) {
    const unsigned long long st = ld_acquire_u64q(&sl.qstate);
    const uint32_t h = qs_head(st);
    if (qs_tail(st) != h) {
      const volatile DispRec *vr = &sl.recs[h % RQ];
      rec->job = vr->job; rec->iter = vr->iter; rec->seq = vr->seq; rec->lane_id = vr->lane_id; rec->kind = vr->kind;
      rec->append_ns = vr->append_ns; rec->lseq = vr->lseq;
      rec->first = vr->first; rec->second = vr->second; rec->n1 = vr->n1; rec->n2 = vr->n2;
      red_add_release_u64(&sl.qstate, QS_HEAD_ONE);
      return true;
    }
    if (atomicCAS(&sl.qstate, st, st & ~1ull) == st) return false;   // released
  }
}

// The first stage of record `rec` (INIT before a job's first iteration, else
// GEN, or F_1 for a GEN-prefetch job; the copy stage of a swap record).
__device__ __forceinline__ uint32_t first_stage_of(const DispRec &rec, const DevJob *jobs) {
  const uint32_t kind = rec.kind & REC_KIND_MASK;
  if (kind == REC_SWAP_OUT) return STAGE_SWAP_OUT;
  if (kind == REC_SWAP_IN) return STAGE_SWAP_IN;
  // a job's first iteration initialises its weights -- unless it resumes a
  // migrated state (NEXT-4), whose swap-in record already put them in place;
  // a GEN-prefetch job's X is already there (stage 1 skipped)
  if (rec.iter == 0 && !(jobs[rec.job].dump & DUMP_INTERNAL_RESUME)) return 0u;
  return (rec.kind & REC_FLAG_XPRE) ? 2u : 1u;
}

// Publish `n1` tiles of stage st1 of `slot` (then `n2` of st2) at ring
// positions base..: by lane 0 alone behind one fence.acq_rel for a handful
// of tiles (release pattern: the fence orders everything lane 0 wrote or
// acquired before it -- begin_iteration's slot fields, a stage counter --
// ahead of every entry), by all lanes with release stores for more (lane 0
// fences its own writes first).  Warp-collective.
constexpr uint32_t PUBLISH_BY_ONE = 16;
__device__ __forceinline__ void publish_tiles(unsigned long long *ring, uint32_t ring_mask, uint32_t lane,
                                              unsigned long long base, uint32_t slot, uint32_t st1, uint32_t n1,
                                              uint32_t st2, uint32_t n2) {
  const uint32_t n = n1 + n2;
  if (n <= PUBLISH_BY_ONE) {
    if (lane == 0) {
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
      for (uint32_t x = 0; x < n; x++) {
        const unsigned long long pos = base + x;
        const uint32_t task = x < n1 ? task_pack(slot, st1, x) : task_pack(slot, st2, x - n1);
        asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(&ring[pos & ring_mask]),
                     "l"(((pos + 1) << 32) | task) : "memory");
      }
    }
  } else {
    if (lane == 0) __threadfence();
    __syncwarp();
    for (uint32_t x = lane; x < n; x += 32) {
      const unsigned long long pos = base + x;
      const uint32_t task = x < n1 ? task_pack(slot, st1, x) : task_pack(slot, st2, x - n1);
      ptx::st_release_u64(&ring[pos & ring_mask], ((pos + 1) << 32) | task);
    }
  }
  __syncwarp();
}

// Single thread: make `rec` the slot's in-flight record.  The caller
// publishes the first stage's tiles after this returns with publish_tiles,
// whose fence orders these writes first; it may reserve their ring
// positions before calling, so that atomic's round trip overlaps the fence.
__device__ __forceinline__ void begin_iteration(Slot &sl, const DispRec &rec) {
  sl.job = rec.job;
  sl.iter = rec.iter | ((rec.kind & REC_FLAG_EAGER) ? ITER_EAGER_BIT : 0u) |
            ((rec.kind & REC_FLAG_NARROW) ? ITER_NARROW_BIT : 0u);
  sl.seq = rec.seq;
  sl.lseq = rec.lseq;
  sl.rkind = rec.kind;
  sl.lane_id = rec.lane_id;
  sl.append_ns = rec.append_ns;
  sl.start_ns = ~0ull;
  sl.end_ns = 0;
  for (uint32_t k = 0; k < N_STAGE_COUNTERS; k++) sl.stage_done[k] = 0;
  sl.end_ticket = 0;
  for (uint32_t k = 0; k < MAX_STAGES; k++) sl.pub_ticket[k] = 0;
  if ((rec.kind & REC_KIND_MASK) != REC_ITER) { sl.stage_done[STAGE_SWAP_OUT] = 0; sl.stage_done[STAGE_SWAP_IN] = 0; }
}

}  // namespace salus
