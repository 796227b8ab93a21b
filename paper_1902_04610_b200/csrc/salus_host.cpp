// salus_host.cpp — host side of the C ABI (include/salus.h): validation,
// page rounding (A18), device-layout footprints, meta-buffer layout, job
// table upload, cooperative launch of the persistent kernel, watchdog, and
// readback.  No per-iteration host work: one launch per salus_run.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <chrono>
#include <cmath>
#include <cstring>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "salus_dev.h"

namespace salus {
int launch_persistent(const Params &P, uint32_t grid, cudaStream_t stream);
int max_coresident_grid(int device, int *grid);
}  // namespace salus

using namespace salus;

#ifndef SALUS_DEFAULT_EAGER_LANES
#define SALUS_DEFAULT_EAGER_LANES 8
#endif

namespace {

inline uint64_t pad128(uint64_t x) { return (x + 127) / 128 * 128; }
inline uint64_t align_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

struct Footprint {
  uint64_t p, e;
};

Footprint footprint(const salus_job &j) {
  const uint32_t L = j.n_layers;
  uint64_t dp[MAX_LAYERS + 1], mx = 0;
  for (uint32_t l = 0; l <= L; l++) { dp[l] = pad128(j.dims[l]); mx = std::max(mx, dp[l]); }
  const uint64_t bp = pad128(j.batch);
  uint64_t w = 0;
  for (uint32_t l = 1; l <= L; l++) w += dp[l - 1] * dp[l];
  Footprint f;
  if (j.kind == SALUS_TRAIN) {
    uint64_t inner = 0;
    for (uint32_t l = 1; l < L; l++) inner += dp[l];
    f.p = 8 * w;
    f.e = 2 * bp * (dp[0] + inner) + 2 * (2 * bp * mx);
  } else {
    uint64_t s = 0;
    for (uint32_t l = 0; l <= L; l++) s += dp[l];
    f.p = 2 * w;
    f.e = 2 * bp * s;
  }
  return f;
}

struct HostJob {
  salus_job j;
  bool live_req = false;              // INFER job whose requests arrive live (salus_submit_requests)
  std::vector<int64_t> req;
  std::vector<uint8_t> resume;        // migration: the persistent image to resume from
  Footprint fp;
  uint32_t submit_idx;
};

}  // namespace

struct salus_ctx {
  salus_config cfg{};
  int state = 0;                       // 0 open, 1 prepared
  std::vector<HostJob> jobs;
  std::unordered_map<uint32_t, uint32_t> id_to_submit;
  std::string err;
  uint32_t Cp = 0;
  uint64_t dump_floats = 0;
  // prepared state
  uint8_t *meta = nullptr;
  uint64_t meta_bytes = 0;
  Params P{};
  std::vector<DevJob> djobs;           // dense order
  std::vector<uint32_t> dense_to_submit;
  std::unordered_map<uint32_t, uint32_t> id_to_dense;
  uint32_t grid = 0;
  uint64_t ring_cap = 0, log_cap = 0;
  uint64_t off_ctrl = 0, off_jobs = 0, off_req = 0, off_inf = 0, off_ppt = 0, off_lpt = 0, off_free = 0,
           off_slots = 0, off_ring = 0, off_fslot = 0, off_fseq = 0, off_pend = 0, off_log = 0, off_wall = 0, off_stats = 0, off_dump = 0, off_trace = 0,
           off_swfence = 0, off_evl = 0, off_reqseen = 0, off_lreqcnt = 0, off_handoff = 0, total = 0;
  uint64_t handoff_cap = 0, n_handoff = 0;
  // caller-owned pinned host swap area: SALUS_FLAG_EVICT (A35) and migration
  // (SALUS_DUMP_STATE / resume_state, NEXT-4); job j's region at pt_off pages
  uint8_t *swap_dev = nullptr, *swap_host = nullptr;
  uint64_t swap_set_bytes = 0;
  uint64_t trace_cap = 0, n_trace = 0, h2d_bytes = 0;
  uint32_t lpt_stride = 0;
  uint32_t *host_abort = nullptr;
  uint32_t *host_abort_dev = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  salus_run_stats last{};
  bool ran = false;
  // online submission (SALUS_FLAG_ONLINE)
  bool running = false, ended = false;
  std::mutex live_mu;
  uint32_t *live = nullptr, *live_dev = nullptr;   // mapped pinned {n_published, closed}
  // live requests: mapped pinned {n_published, pad, dense job index[lreq_cap]}
  uint32_t *lreq = nullptr, *lreq_dev = nullptr;
  uint32_t lreq_cap = 0, lreq_pub = 0;
  std::vector<uint32_t> lreq_left;                 // per dense job: live requests still to come
  cudaStream_t side = nullptr;                     // private stream for descriptor uploads
  uint64_t ppt_used = 0, ppt_cap = 0, ring_tiles = 0, dump_cur = 0, dump_cap = 0;
  uint32_t max_id = 0, n_pre = 0;
  bool t_out = false;
  // the kernel ignored the abort flag past the grace period: buffers it may
  // still touch (mapped flags, caller arena/meta/swap) must never be freed
  bool poisoned = false;
  uint32_t n_cap = 0;                              // stats records reserved (max_jobs when online)
  uint64_t run_h2d = 0;                            // per-run H2D bytes (stats reset image)
  std::vector<salus_job_stat> stats_img;           // host source of that copy (outlives it)
  std::chrono::steady_clock::time_point t0;
};

namespace {

int fail(salus_ctx *c, int code, const std::string &msg) {
  if (c) c->err = msg;
  return code;
}
int cuda_fail(salus_ctx *c, cudaError_t e, const char *where) {
  return fail(c, SALUS_E_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

uint32_t default_max_lanes(uint32_t policy) {
  switch (policy) {
    case SALUS_PACK: return 64;
    default: return 1;   // FIFO, SRTF, FAIR (A9)
  }
}

// Latency-mode knobs (DevJob.lat_narrow / relax): SALUS_NARROW_BELOW (pair
// tasks at N = 256 below which a stage takes N = 128 in latency mode; 0 =
// never) and SALUS_RELAX ("0" disables the relaxed backward barrier).
uint32_t narrow_below() {
  const char *e = getenv("SALUS_NARROW_BELOW");   // read per call: tests change it between contexts
  return e ? (uint32_t)atoi(e) : 32u;
}
// K9 transposed tiles are opt-in (SALUS_SWAP=1): measured on C3 they cost
// 20 us per request in latency mode and gained 0.6% in throughput mode
// (profiles/r02/ab_c3.txt)
bool swap_enabled() {
  const char *e = getenv("SALUS_SWAP");
  return e && e[0] == '1';
}
// Split-K in narrow records (DevJob.splitk) is opt-in (the SALUS_SPLITK_BUILD
// library, libsalus_splitk.so, with SALUS_SPLITK=1): it
// gains 1-3% on C4 / C5 and 15% on a lone 4096-wide job, but long runs in
// the full bench process hung in 3 of 3 attempts while every
// isolated run and test passed; until that is understood it stays off
bool splitk_enabled() {
  const char *e = getenv("SALUS_SPLITK");
  return SALUS_SPLITK_BUILD && e && e[0] == '1';
}
// Targets generated in the GEN stage (DevJob.t_in_g): SALUS_TG=0 disables
bool tg_enabled() {
  const char *e = getenv("SALUS_TG");
  return !(e && e[0] == '0');
}
bool relax_enabled() {
  const char *e = getenv("SALUS_RELAX");
  return !(e && e[0] == '0');
}

// Persistent backing pages of a job: its footprint, plus two X buffers for
// the GEN prefetch when the declared P leaves room for them (and the
// SALUS_XPRE environment variable is not "0"); never more than declared.
uint32_t backing_pages(const salus_job &j, const Footprint &fp, bool null_work, uint32_t *xpre,
                       uint64_t *xbytes) {
  const uint64_t G = PAGE_BYTES;
  const uint64_t p_pages = (j.persistent_bytes + G - 1) / G;
  const uint64_t xb = 2ull * pad128(j.batch) * pad128(j.dims[0]);
  const uint64_t tb = j.kind == SALUS_TRAIN ? 2ull * pad128(j.batch) * pad128(j.dims[j.n_layers]) : 0;
  const char *xe = getenv("SALUS_XPRE");
  const bool enabled = !(xe && xe[0] == '0');
  *xpre = 0;
  *xbytes = xb;
  // DevJob byte offsets inside a job's persistent space are 32-bit: the
  // prefetch buffers go past the footprint, so they need it to stay < 4 GiB
  if (!null_work && enabled && p_pages * G >= fp.p + 2 * xb + 2 * tb && fp.p + 2 * xb + 2 * tb <= 0xFFFFFFFFull) {
    *xpre = 1;
    return (uint32_t)((fp.p + 2 * xb + 2 * tb + G - 1) / G);
  }
  return (uint32_t)std::min<uint64_t>((fp.p + G - 1) / G, p_pages);
}

int validate_job(const salus_job *j, bool null_work, std::string *why, bool live_req_ok = false) {
  if (j->kind > SALUS_INFER) { *why = "kind"; return SALUS_E_INVAL; }
  if (j->n_layers < 1 || j->n_layers > MAX_LAYERS) { *why = "n_layers must be 1..8"; return SALUS_E_INVAL; }
  for (uint32_t l = 0; l <= j->n_layers; l++)
    if (j->dims[l] < 1 || j->dims[l] > 8192) { *why = "dims must be 1..8192"; return SALUS_E_INVAL; }
  if (j->batch < 1 || j->batch > 8192) { *why = "batch must be 1..8192"; return SALUS_E_INVAL; }
  if (j->n_iters < 1 || j->iter_ticks < 1) { *why = "n_iters and iter_ticks must be >= 1"; return SALUS_E_INVAL; }
  if (j->arrival_tick < 0 || j->arrival_tick > (int64_t)1 << 60) { *why = "arrival_tick"; return SALUS_E_INVAL; }
  if ((long double)j->n_iters * (long double)j->iter_ticks >= (long double)(1ull << 52)) {
    *why = "n_iters * iter_ticks must be < 2^52";
    return SALUS_E_INVAL;
  }
  if (j->kind == SALUS_INFER) {
    if (!j->request_ticks && !live_req_ok) {
      *why = "INFER job needs request_ticks (NULL = live requests, online contexts only)";
      return SALUS_E_INVAL;
    }
    int64_t prev = j->arrival_tick;
    for (uint32_t k = 0; j->request_ticks && k < j->n_iters; k++) {
      if (j->request_ticks[k] < prev) { *why = "request_ticks must be sorted and >= arrival"; return SALUS_E_INVAL; }
      prev = j->request_ticks[k];
    }
  }
  if (!std::isfinite(j->lr)) { *why = "lr"; return SALUS_E_INVAL; }
  Footprint f = footprint(*j);
  if (!null_work && (j->persistent_bytes < f.p || j->ephemeral_bytes < f.e)) {
    *why = "declared persistent/ephemeral bytes below the device footprint (salus_job_footprint)";
    return SALUS_E_INVAL;
  }
  if (j->resume_state) {                 // migration: an image of this very layout
    uint32_t xpre;
    uint64_t xb;
    const uint64_t img = (uint64_t)backing_pages(*j, f, null_work, &xpre, &xb) * PAGE_BYTES;
    if (j->resume_bytes != img || null_work) {
      *why = "resume_bytes must equal the job's persistent backing (salus_read_state), real work only";
      return SALUS_E_INVAL;
    }
    if ((uint64_t)j->resume_iter + j->n_iters > 0xFFFFu) { *why = "resume_iter + n_iters must be < 65536"; return SALUS_E_INVAL; }
  } else if (j->resume_iter) {
    *why = "resume_iter without resume_state";
    return SALUS_E_INVAL;
  }
  return SALUS_OK;
}

}  // namespace

extern "C" {

int salus_job_footprint(const salus_job *job, uint64_t *persistent_bytes, uint64_t *ephemeral_bytes) {
  if (!job || job->n_layers < 1 || job->n_layers > MAX_LAYERS) return SALUS_E_INVAL;
  Footprint f = footprint(*job);
  if (persistent_bytes) *persistent_bytes = f.p;
  if (ephemeral_bytes) *ephemeral_bytes = f.e;
  return SALUS_OK;
}

int salus_open(const salus_config *cfg, salus_ctx **out) {
  if (!cfg || !out) return SALUS_E_INVAL;
  *out = nullptr;
  salus_config c = *cfg;
  if (c.page_bytes == 0) c.page_bytes = PAGE_BYTES;
  if (c.page_bytes != PAGE_BYTES) return SALUS_E_INVAL;
  if (c.policy > SALUS_FAIR) return SALUS_E_INVAL;
  if (c.max_lanes == 0) c.max_lanes = default_max_lanes(c.policy);
  if (c.max_lanes > MAX_LANES) return SALUS_E_INVAL;
  if (c.max_jobs == 0 || c.max_jobs > MAX_JOBS) return SALUS_E_INVAL;
  const uint64_t Cp = c.capacity_bytes / c.page_bytes;
  if (Cp == 0 || Cp > 0xFFFFFFF0ull) return SALUS_E_INVAL;
  if (!c.arena || (reinterpret_cast<uintptr_t>(c.arena) & 255) || c.arena_bytes < Cp * c.page_bytes)
    return SALUS_E_INVAL;
  if (c.timeout_ms == 0) c.timeout_ms = 600000;
  // A35: eviction is the SRTF admission rule of P:530, for offline traces
  if ((c.flags & SALUS_FLAG_EVICT) && (c.policy != SALUS_SRTF || (c.flags & SALUS_FLAG_ONLINE)))
    return SALUS_E_INVAL;
  salus_ctx *ctx = new salus_ctx();
  ctx->cfg = c;
  ctx->Cp = (uint32_t)Cp;
  *out = ctx;
  return SALUS_OK;
}

int salus_submit_job(salus_ctx *ctx, const salus_job *job) {
  if (!ctx || !job) return SALUS_E_INVAL;
  if (ctx->state != 0) return fail(ctx, SALUS_E_STATE, "submit after prepare");
  if (ctx->id_to_submit.count(job->job_id)) return fail(ctx, SALUS_E_DUPLICATE, "duplicate job id");
  std::string why;
  int rc = validate_job(job, (ctx->cfg.flags & SALUS_FLAG_NULL_WORK) != 0, &why,
                        (ctx->cfg.flags & SALUS_FLAG_ONLINE) != 0);
  if (rc) return fail(ctx, rc, "job " + std::to_string(job->job_id) + ": " + why);
  const uint64_t G = ctx->cfg.page_bytes;
  const uint64_t p = (job->persistent_bytes + G - 1) / G, e = (job->ephemeral_bytes + G - 1) / G;
  if (p + e > ctx->Cp) return fail(ctx, SALUS_E_UNSCHEDULABLE, "p + e > C pages (A22)");
  if (ctx->jobs.size() >= ctx->cfg.max_jobs) return fail(ctx, SALUS_E_CAPACITY, "max_jobs reached");
  uint64_t df = 0;
  if (job->dump & SALUS_DUMP_OUTPUTS) df += (uint64_t)job->n_iters * job->batch * job->dims[job->n_layers];
  if (job->dump & (SALUS_DUMP_WEIGHTS | SALUS_DUMP_WEIGHT_STEPS)) {
    uint64_t wc = 0;
    for (uint32_t l = 1; l <= job->n_layers; l++) wc += (uint64_t)job->dims[l - 1] * job->dims[l];
    df += (job->dump & SALUS_DUMP_WEIGHT_STEPS) ? wc * job->n_iters : wc;
  }
  if ((job->dump & SALUS_DUMP_WEIGHT_STEPS) && job->kind != SALUS_TRAIN)
    return fail(ctx, SALUS_E_INVAL, "SALUS_DUMP_WEIGHT_STEPS is for TRAIN jobs");
  if (ctx->cfg.dump_bytes && (ctx->dump_floats + df) * 4 > ctx->cfg.dump_bytes)
    return fail(ctx, SALUS_E_CAPACITY, "dump_bytes exceeded");
  HostJob h;
  h.j = *job;
  if (job->kind == SALUS_INFER && job->request_ticks) h.req.assign(job->request_ticks, job->request_ticks + job->n_iters);
  if (job->kind == SALUS_INFER && !job->request_ticks) {   // live requests: ticks assigned on arrival
    h.live_req = true;
    h.req.assign(job->n_iters, INT64_MAX);
  }
  h.j.request_ticks = nullptr;
  if (job->resume_state) {
    const uint8_t *r = static_cast<const uint8_t *>(job->resume_state);
    h.resume.assign(r, r + job->resume_bytes);
  }
  h.j.resume_state = nullptr;
  h.fp = footprint(*job);
  h.submit_idx = (uint32_t)ctx->jobs.size();
  ctx->dump_floats += df;
  ctx->id_to_submit[job->job_id] = h.submit_idx;
  ctx->jobs.push_back(std::move(h));
  return SALUS_OK;
}

// Mapped pinned 64-byte flags (the per-context abort flag), carved from
// process-wide 64 KiB pages: cudaHostAlloc of a fresh pinned buffer can take
// tens of ms, which a context per run (bench.py's e2e) would pay every time.
namespace {
std::mutex g_flag_mu;
std::vector<std::pair<uint32_t *, uint32_t *>> g_flag_free;   // (host, device)
}
static cudaError_t flag_alloc(uint32_t **host, uint32_t **dev) {
  std::lock_guard<std::mutex> g(g_flag_mu);
  if (g_flag_free.empty()) {
    uint8_t *base = nullptr, *dbase = nullptr;
    cudaError_t e = cudaHostAlloc(reinterpret_cast<void **>(&base), 65536, cudaHostAllocMapped | cudaHostAllocPortable);
    if (e != cudaSuccess) return e;
    if ((e = cudaHostGetDevicePointer(reinterpret_cast<void **>(&dbase), base, 0)) != cudaSuccess) return e;
    for (uint32_t o = 65536 - 64;; o -= 64) {
      g_flag_free.emplace_back(reinterpret_cast<uint32_t *>(base + o), reinterpret_cast<uint32_t *>(dbase + o));
      if (o == 0) break;
    }
  }
  *host = g_flag_free.back().first;
  *dev = g_flag_free.back().second;
  g_flag_free.pop_back();
  return cudaSuccess;
}
static void flag_free(uint32_t *host, uint32_t *dev) {
  std::lock_guard<std::mutex> g(g_flag_mu);
  g_flag_free.emplace_back(host, dev);
}

static void fill_devjob(salus_ctx *c, const HostJob &h, DevJob &D, uint64_t &req_total, uint64_t &ppt_total,
                        uint64_t &dump_cur) {
    const salus_job &j = h.j;
    const uint64_t G = c->cfg.page_bytes;
    D.job_id = j.job_id; D.kind = j.kind; D.n_layers = j.n_layers; D.batch = j.batch;
    D.arrival = j.arrival_tick; D.iter_ticks = (int64_t)j.iter_ticks; D.n_iters = j.n_iters;
    D.p_pages = (uint32_t)((j.persistent_bytes + G - 1) / G);
    D.e_pages = (uint32_t)((j.ephemeral_bytes + G - 1) / G);
    // backing pages: the device footprint (<= declared, so the pool of Cp pages
    // can never run dry under the safety condition); in NULL_WORK mode the
    // allocator still runs, bounded by the declared sizes
    uint64_t xbytes = 0;
    D.ap_pages = backing_pages(j, h.fp, (c->cfg.flags & SALUS_FLAG_NULL_WORK) != 0, &D.xpre, &xbytes);
    D.x_off[0] = D.xpre ? (uint32_t)h.fp.p : 0;
    D.x_off[1] = D.xpre ? (uint32_t)(h.fp.p + xbytes) : 0;
    const uint64_t tbytes = 2ull * pad128(j.batch) * pad128(j.dims[j.n_layers]);
    const bool tpre = D.xpre && j.kind == SALUS_TRAIN;
    D.t_off[0] = tpre ? (uint32_t)(h.fp.p + 2 * xbytes) : 0;
    D.t_off[1] = tpre ? (uint32_t)(h.fp.p + 2 * xbytes + tbytes) : 0;
    D.ae_pages = (uint32_t)std::min<uint64_t>((h.fp.e + G - 1) / G, D.e_pages);
    D.bpad = (uint32_t)pad128(j.batch);
    const uint32_t L = j.n_layers;
    for (uint32_t l = 0; l <= MAX_LAYERS; l++) {
      D.dims[l] = l <= L ? j.dims[l] : 0;
      D.dpad[l] = l <= L ? (uint32_t)pad128(j.dims[l]) : 0;
    }
    D.lr = j.lr; D.dump = j.dump | (h.resume.empty() ? 0u : DUMP_INTERNAL_RESUME); D.seed = j.seed;
    D.iter_base = j.resume_iter;
    D.req_off = (uint32_t)req_total;
    if (j.kind == SALUS_INFER) req_total += j.n_iters;
    D.pt_off = (uint32_t)ppt_total;
    ppt_total += D.ap_pages;
    // persistent tensors
    uint64_t off = 0;
    for (uint32_t l = 1; l <= L; l++) {
      const uint64_t w = (uint64_t)D.dpad[l - 1] * D.dpad[l];
      if (j.kind == SALUS_TRAIN) {
        D.w32_off[l - 1] = (uint32_t)off; off += 4 * w;
        D.wb_off[l - 1][0] = (uint32_t)off; off += 2 * w;
        D.wb_off[l - 1][1] = (uint32_t)off; off += 2 * w;
      } else {
        D.w32_off[l - 1] = 0;
        D.wb_off[l - 1][0] = D.wb_off[l - 1][1] = (uint32_t)off; off += 2 * w;
      }
    }
    // ephemeral tensors
    off = 0;
    const uint64_t bp = D.bpad;
    const uint32_t nact = j.kind == SALUS_TRAIN ? L : L + 1;   // act[0..nact-1]
    uint32_t mx = 0;
    for (uint32_t l = 0; l <= L; l++) mx = std::max(mx, D.dpad[l]);
    for (uint32_t l = 0; l < nact; l++) { D.act_off[l] = (uint32_t)off; off += 2 * bp * D.dpad[l]; }
    if (j.kind == SALUS_TRAIN) {
      D.g_off[0] = (uint32_t)off; off += 2 * bp * mx;
      D.g_off[1] = (uint32_t)off; off += 2 * bp * mx;
    }
    // latency mode's relaxed backward barrier: a third G buffer from the
    // declared E's slack (jobs that declare exactly their footprint keep the
    // full stage barrier)
    D.relax = 0; D.g_off3 = 0;
    if (j.kind == SALUS_TRAIN && L >= 2 && !(c->cfg.flags & SALUS_FLAG_NULL_WORK) && relax_enabled() &&
        (uint64_t)D.e_pages * G >= off + 2 * bp * mx) {
      D.relax = 1;
      D.g_off3 = (uint32_t)off;
      D.ae_pages = (uint32_t)((off + 2 * bp * mx + G - 1) / G);
    }
    // stage tasks: pair tasks (a CTA pair computes 2 blocks / a 256-row super-tile)
    auto pairs = [](uint32_t n) { return (n + 1) / 2; };
    uint32_t ti = 0;
    for (uint32_t l = 1; l <= L; l++) ti += (D.dpad[l] / 128) * (D.dpad[l - 1] / 128);
    D.stage_tiles[0] = pairs(ti);
    D.stage_tiles[1] = pairs((D.bpad / 128) * (D.dpad[0] / 128));
    D.t_gen_tiles = (D.xpre && j.kind == SALUS_TRAIN) ? pairs((D.bpad / 128) * (D.dpad[L] / 128)) : 0;
    D.t_in_g = (!D.xpre && j.kind == SALUS_TRAIN && !(c->cfg.flags & SALUS_FLAG_NULL_WORK) && tg_enabled())
                   ? pairs((D.bpad / 128) * (D.dpad[L] / 128)) : 0;
    D.stage_tiles[1] += D.t_in_g;
    D.n_stages = last_stage(j.kind, L) + 1;
    // K9 (opt-in, swap_enabled): an inference job with a 128-row batch
    // (b <= 128; C3's requests of b = 1..16) takes transposed
    // (swap-AB) F_l tiles except in narrow records: pairs of 128-feature
    // output blocks.  (Measured on C4's training jobs, transposed F / dX
    // tiles were 1% slower -- half the tasks of the N = 128 tiles,
    // profiles/r02/ab_k9.txt -- so training jobs never take them.)
    const bool skinny = D.bpad == 128 && j.kind == SALUS_INFER && swap_enabled();
    D.swap_mask = 0;
    D.lat_narrow = 0;
    // GEN-prefetch tiles ride on INIT (stage 0) and F_1 (stage 2)
    const uint32_t gen_extra = D.xpre ? D.stage_tiles[1] + D.t_gen_tiles : 0;
    if (D.xpre) D.stage_tiles[0] += gen_extra;
    for (uint32_t s = 0; s < 2; s++) D.stage_tiles_lat[s] = (uint16_t)std::min<uint32_t>(D.stage_tiles[s], 0xFFFF);
    for (uint32_t s = 2; s < D.n_stages; s++) {
      const bool fwd = s <= L + 1;
      if (!fwd && j.kind != SALUS_TRAIN) break;
      const uint32_t l = fwd ? s - 1 : L - (s - (L + 2));
      const uint32_t dn = fwd ? D.dpad[l] : D.dpad[l - 1];      // N of the stage's (non-swap) GEMMs
      const uint32_t extra = (s == 2) ? gen_extra : 0;
      const bool has_x = fwd || l > 1;                          // F tiles / dX tiles (B_1 has none)
      // tasks of the F / dX part and of the dW part at N tile nt (non-swap)
      auto x_tiles = [&](uint32_t nt) { return has_x ? pairs(D.bpad / 128) * (dn / nt) : 0u; };
      auto w_tiles = [&](uint32_t nt) { return fwd ? 0u : pairs(D.dpad[l] / 128) * (dn / nt); };
      const uint32_t nt0 = ntile_for(dn);
      uint32_t xw = x_tiles(nt0), ww = w_tiles(nt0);
      if (skinny && has_x) { D.swap_mask |= 1u << s; xw = pairs(dn / 128); }
      D.stage_tiles[s] = xw + ww + extra;
      // narrow latency mode (no K9 tiles): N = 128 on the stages with few tasks
      uint32_t xl = x_tiles(nt0), wl = ww;
      if (nt0 == 256 && xl + ww < narrow_below()) {
        D.lat_narrow |= 1u << s;
        wl = w_tiles(128);
        xl = x_tiles(128);
      }
      D.stage_tiles_lat[s] = (uint16_t)std::min<uint32_t>(xl + wl + extra, 0xFFFF);
    }
    // split-K (narrow records): a stage whose F / dX part has few pair tasks
    // and a long K (>= 2048: below, a slice's partial write and reduction,
    // ~4 us, cost what the shorter K saves) runs S K-slices of it.  Among
    // N in {128, 256} and S in {2, 4} with npair(N) x S <= SK_PAIRS (one wave
    // of CTA pairs), slices of >= 8 chunks and whole double chunks, take the
    // least bytes per CTA per task: (K / S) x (16 KiB of A + N/2 rows of B)
    // per 64-chunk, plus the S partials (128 x N fp32 each) the last slice
    // writes and reads (measured: N = 256 x 4 slices lost to N = 128 x 2 on
    // a 4096-wide layer of batch 64).  The workspace comes from the declared E's
    // slack like the relaxed barrier's third G buffer.
    for (uint32_t s = 0; s < MAX_STAGES; s++) D.splitk[s] = 1;
    D.ws_off = 0;
    D.sk_wide = 0;
    if (splitk_enabled() && !(c->cfg.flags & SALUS_FLAG_NULL_WORK)) {
      constexpr uint32_t SK_PAIRS = 74;
      uint8_t sk[MAX_STAGES];
      uint32_t np[MAX_STAGES], wide = 0;
      uint64_t need = 0;
      for (uint32_t s = 0; s < MAX_STAGES; s++) { sk[s] = 1; np[s] = 0; }
      for (uint32_t s = 2; s < D.n_stages; s++) {
        const bool fwd = s <= L + 1;
        if (!fwd && j.kind != SALUS_TRAIN) break;
        const uint32_t l = fwd ? s - 1 : L - (s - (L + 2));
        if (!fwd && l == 1) continue;                           // B_1 has no dX part
        const uint32_t dn = fwd ? D.dpad[l] : D.dpad[l - 1];
        const uint32_t nk = (fwd ? D.dpad[l - 1] : D.dpad[l]) / 64;
        if (nk < 32) continue;
        uint64_t best = ~0ull;
        for (uint32_t nt = 128; nt <= 256; nt *= 2) {
          if (dn % nt) continue;
          const uint32_t npair = pairs(D.bpad / 128) * (dn / nt);
          for (uint32_t cand = 2; cand <= SK_MAX; cand *= 2) {
            if (npair * cand > SK_PAIRS || nk % (2 * cand) || nk / cand < 8 || 16 * npair > SK_COUNTERS) continue;
            // operand bytes of one slice + the last slice's partial traffic
            const uint64_t cost = (uint64_t)(nk / cand) * (16384 + nt * 64) + (uint64_t)cand * nt * 512;
            if (cost < best) {
              best = cost;
              sk[s] = (uint8_t)cand;
              np[s] = npair;
              wide = nt == 256 ? (wide | 1u << s) : (wide & ~(1u << s));
            }
          }
        }
        if (sk[s] > 1)
          need = std::max<uint64_t>(need, (uint64_t)np[s] * 2 * sk[s] * (((wide >> s) & 1u) ? 2 : 1) * 65536);
      }
      const uint64_t end = D.relax ? (uint64_t)D.g_off3 + 2 * bp * mx : off;
      const uint64_t ws = align_up(end, 65536);
      if (need && (uint64_t)D.e_pages * G >= ws + need && ws + need < (1ull << 32)) {
        D.ws_off = (uint32_t)ws;
        D.sk_wide = wide;
        D.ae_pages = std::max<uint32_t>(D.ae_pages, (uint32_t)((ws + need + G - 1) / G));
        for (uint32_t s = 2; s < D.n_stages; s++) {
          if (sk[s] < 2) continue;
          const bool fwd = s <= L + 1;
          const uint32_t l = fwd ? s - 1 : L - (s - (L + 2));
          const uint32_t dn = fwd ? D.dpad[l] : D.dpad[l - 1];
          const uint32_t nt0 = ntile_for(dn);
          const uint32_t nx_old = pairs(D.bpad / 128) * (dn / (((D.lat_narrow >> s) & 1u) ? 128u : nt0));
          D.splitk[s] = sk[s];
          D.stage_tiles_lat[s] = (uint16_t)std::min<uint32_t>(D.stage_tiles_lat[s] - nx_old + np[s] * sk[s], 0xFFFF);
        }
      }
    }
    {
      uint64_t tot = 0;
      for (uint32_t s = 2; s < D.n_stages; s++) tot += D.stage_tiles[s];
      D.lat_cost = (uint16_t)std::min<uint64_t>(0xFFFF, tot / std::max<uint32_t>(1, D.n_stages - 2));
    }
    D.dump_out_off = dump_cur;
    if (j.dump & SALUS_DUMP_OUTPUTS) dump_cur += (uint64_t)j.n_iters * j.batch * j.dims[L];
    D.dump_w_off = dump_cur;
    D.w_count = 0;
    for (uint32_t l = 1; l <= L; l++) D.w_count += (uint64_t)j.dims[l - 1] * j.dims[l];
    if (j.dump & SALUS_DUMP_WEIGHT_STEPS) dump_cur += D.w_count * j.n_iters;
    else if (j.dump & SALUS_DUMP_WEIGHTS) dump_cur += D.w_count;
}

static void compute_layout(salus_ctx *c) {
  const uint32_t n = (uint32_t)c->jobs.size();
  // dense order = (arrival, id) rank
  std::vector<uint32_t> order(n);
  for (uint32_t i = 0; i < n; i++) order[i] = i;
  std::sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) {
    const salus_job &x = c->jobs[a].j, &y = c->jobs[b].j;
    return x.arrival_tick != y.arrival_tick ? x.arrival_tick < y.arrival_tick : x.job_id < y.job_id;
  });
  c->dense_to_submit = order;
  c->djobs.assign(n, DevJob{});
  c->id_to_dense.clear();
  const uint64_t G = c->cfg.page_bytes;
  uint64_t req_total = 0, ppt_total = 0, dump_cur = 0, max_ae = 1, max_tiles = 1, dispatches = 0;
  for (uint32_t d = 0; d < n; d++) {
    const HostJob &h = c->jobs[order[d]];
    const salus_job &j = h.j;
    DevJob &D = c->djobs[d];
    c->id_to_dense[j.job_id] = d;
    fill_devjob(c, h, D, req_total, ppt_total, dump_cur);
    for (uint32_t s = 0; s < D.n_stages; s++)
      max_tiles = std::max<uint64_t>(max_tiles, std::max<uint32_t>(D.stage_tiles[s], D.stage_tiles_lat[s]));
    if (c->cfg.flags & SALUS_FLAG_EVICT) max_tiles = std::max<uint64_t>(max_tiles, (D.ap_pages + 1) / 2);
    max_ae = std::max<uint64_t>(max_ae, D.ae_pages);
    dispatches += j.n_iters;
  }
  const bool online = (c->cfg.flags & SALUS_FLAG_ONLINE) != 0;
  c->ppt_used = ppt_total;
  c->ppt_cap = ppt_total;
  c->dump_cur = dump_cur;
  c->n_pre = n;
  uint32_t n_cap = n;
  c->n_cap = n;
  if (online) {
    // room for live jobs: descriptors and stats up to max_jobs, page-table
    // entries for 4 x C of persistent memory over the run, lanes up to C,
    // stages of up to 4096 pair tasks (checked at salus_submit_live)
    c->ppt_cap += 4ull * c->Cp;
    max_ae = std::max<uint64_t>(max_ae, c->Cp);
    max_tiles = std::max<uint64_t>(max_tiles, 4096);
    n_cap = c->cfg.max_jobs;
    c->n_cap = n_cap;
  }
  c->ring_tiles = max_tiles;
  c->lpt_stride = (uint32_t)max_ae;
  uint64_t rc = 1024;
  const uint64_t need = 2 * (MAX_LANES * max_tiles + 4096);
  while (rc < need) rc <<= 1;
  c->ring_cap = rc;
  c->log_cap = 0;
  if (c->cfg.flags & SALUS_FLAG_LOG)
    c->log_cap = c->cfg.log_capacity ? c->cfg.log_capacity
                                     : dispatches + 6ull * n + 16 + (online ? (1ull << 20) : 0) +
                                       // A35: an eviction logs <= 4 records and happens at most
                                       // once per iteration boundary of its victim
                                       ((c->cfg.flags & SALUS_FLAG_EVICT) ? 4 * dispatches : 0);
  uint64_t o = 0;
  auto take = [&](uint64_t bytes) { uint64_t r = o; o = align_up(o + bytes, 256); return r; };
  c->off_ctrl = take(sizeof(Ctrl));
  c->off_jobs = take(sizeof(DevJob) * std::max<uint64_t>(n_cap, 1));
  c->off_req = take(8 * std::max<uint64_t>(req_total, 1));
  c->off_inf = take(2 * std::max<uint64_t>(n, 1));
  c->off_ppt = take(4 * std::max<uint64_t>(c->ppt_cap, 1));
  c->off_lpt = take(4ull * MAX_LANES * c->lpt_stride);
  c->off_free = take(4ull * c->Cp);
  c->off_fslot = take(1ull * c->Cp);
  c->off_fseq = take(8ull * c->Cp);
  c->off_pend = take(8ull * MAX_LANES * MAX_LANES);
  c->off_slots = take(sizeof(Slot) * MAX_LANES);
  c->off_ring = take(8 * c->ring_cap);
  c->off_log = take(sizeof(salus_log_rec) * std::max<uint64_t>(c->log_cap, 1));
  c->off_wall = take(sizeof(salus_wall_rec) * std::max<uint64_t>(c->log_cap, 1));
  c->off_stats = take(sizeof(salus_job_stat) * std::max<uint64_t>(n_cap, 1));
  // online: cfg.dump_bytes reserves room for live jobs' dumps as well
  c->dump_cap = online ? std::max<uint64_t>(dump_cur, c->cfg.dump_bytes / 4) : dump_cur;
  c->off_dump = take(4 * std::max<uint64_t>(c->dump_cap, 1));
  c->trace_cap = (c->cfg.flags & SALUS_FLAG_TRACE) ? (c->cfg.trace_capacity ? c->cfg.trace_capacity : (1ull << 20)) : 0;
  c->off_trace = take(sizeof(salus_trace_rec) * std::max<uint64_t>(c->trace_cap, 1));
  c->off_swfence = take(8 * std::max<uint64_t>(n_cap, 1));
  c->off_evl = take(2 * std::max<uint64_t>(n_cap, 1));
  c->off_reqseen = take(8 * std::max<uint64_t>(req_total, 1));   // live requests: globaltimer when seen
  c->off_lreqcnt = take(4 * std::max<uint64_t>(n_cap, 1));        // live requests received per job
  c->handoff_cap = (c->cfg.flags & SALUS_FLAG_CHECK) ? (1ull << 20) : 0;
  c->off_handoff = take(sizeof(salus_handoff_rec) * std::max<uint64_t>(c->handoff_cap, 1));
  c->total = o;
}

int salus_meta_bytes(const salus_ctx *ctx, uint64_t *bytes) {
  if (!ctx || !bytes) return SALUS_E_INVAL;
  // the layout is frozen at prepare (live jobs only consume reserved space):
  // recomputing it afterwards would move the offsets Params already holds
  if (ctx->state == 0) compute_layout(const_cast<salus_ctx *>(ctx));
  *bytes = ctx->total;
  return SALUS_OK;
}

static bool needs_swap(const salus_ctx *ctx) {
  if (ctx->cfg.flags & SALUS_FLAG_EVICT) return true;
  for (const HostJob &h : ctx->jobs)
    if ((h.j.dump & SALUS_DUMP_STATE) || !h.resume.empty()) return true;
  return false;
}

int salus_swap_bytes(const salus_ctx *ctx, uint64_t *bytes) {
  if (!ctx || !bytes) return SALUS_E_INVAL;
  if (ctx->state == 0) compute_layout(const_cast<salus_ctx *>(ctx));
  // job j's region: its persistent backing pages, at pt_off pages (dense order)
  *bytes = needs_swap(ctx) ? ctx->ppt_used * ctx->cfg.page_bytes : 0;
  return SALUS_OK;
}

int salus_set_swap(salus_ctx *ctx, void *host, uint64_t bytes) {
  if (!ctx) return SALUS_E_INVAL;
  if (ctx->state != 0) return fail(ctx, SALUS_E_STATE, "salus_set_swap after salus_prepare");
  if (!needs_swap(ctx)) return fail(ctx, SALUS_E_STATE, "no swap area needed (no EVICT flag, DUMP_STATE or resume)");
  if (!host || (reinterpret_cast<uintptr_t>(host) & 255)) return fail(ctx, SALUS_E_INVAL, "swap must be 256-B aligned");
  uint64_t need = 0;
  salus_swap_bytes(ctx, &need);
  if (bytes < need) return fail(ctx, SALUS_E_CAPACITY, "swap area too small");
  cudaError_t e = cudaSetDevice(ctx->cfg.device);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaSetDevice");
  void *dev = nullptr;
  if ((e = cudaHostGetDevicePointer(&dev, host, 0)) != cudaSuccess) {
    cudaGetLastError();
    return fail(ctx, SALUS_E_INVAL, "swap area is not page-locked host memory the device can access");
  }
  ctx->swap_dev = static_cast<uint8_t *>(dev);
  ctx->swap_host = static_cast<uint8_t *>(host);
  ctx->swap_set_bytes = bytes;
  return SALUS_OK;
}

int salus_prepare(salus_ctx *ctx, void *meta, uint64_t meta_bytes) {
  if (!ctx) return SALUS_E_INVAL;
  if (ctx->state != 0) return fail(ctx, SALUS_E_STATE, "already prepared");
  const bool online = (ctx->cfg.flags & SALUS_FLAG_ONLINE) != 0;
  if (ctx->jobs.empty() && !online) return fail(ctx, SALUS_E_STATE, "no jobs submitted");
  compute_layout(ctx);
  if (!meta || (reinterpret_cast<uintptr_t>(meta) & 255)) return fail(ctx, SALUS_E_INVAL, "meta must be 256-B aligned");
  if (meta_bytes < ctx->total) return fail(ctx, SALUS_E_CAPACITY, "meta buffer too small");
  if (needs_swap(ctx) && ctx->ppt_used &&
      (!ctx->swap_dev || ctx->swap_set_bytes < ctx->ppt_used * ctx->cfg.page_bytes))
    return fail(ctx, SALUS_E_STATE, "SALUS_FLAG_EVICT / DUMP_STATE / resume need salus_set_swap (>= salus_swap_bytes) first");
  cudaError_t e = cudaSetDevice(ctx->cfg.device);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaSetDevice");
  int grid = 0;
  int rc = max_coresident_grid(ctx->cfg.device, &grid);
  if (rc) return cuda_fail(ctx, (cudaError_t)rc, "occupancy");
  if (grid < 4) return fail(ctx, SALUS_E_CUDA, "persistent kernel does not fit two CTA pairs");
  // n_workers counts worker CTA pairs; pair 0 is the scheduler's cluster
  if (ctx->cfg.n_workers && 2 * ((int)ctx->cfg.n_workers + 1) < grid) grid = 2 * ((int)ctx->cfg.n_workers + 1);
  ctx->grid = (uint32_t)grid;
  ctx->meta = static_cast<uint8_t *>(meta);
  ctx->meta_bytes = meta_bytes;
  const uint32_t n = (uint32_t)ctx->jobs.size();
  cudaStream_t st = static_cast<cudaStream_t>(ctx->cfg.stream);
  std::vector<int64_t> req;
  std::vector<uint16_t> inf;
  for (uint32_t d = 0; d < n; d++) {
    const HostJob &h = ctx->jobs[ctx->dense_to_submit[d]];
    if (h.j.kind == SALUS_INFER) {
      req.insert(req.end(), h.req.begin(), h.req.end());
      inf.push_back((uint16_t)d);
    }
  }
  uint8_t *m = ctx->meta;
  if ((e = cudaMemcpyAsync(m + ctx->off_jobs, ctx->djobs.data(), sizeof(DevJob) * n, cudaMemcpyHostToDevice, st)))
    return cuda_fail(ctx, e, "upload jobs");
  if (!req.empty() &&
      (e = cudaMemcpyAsync(m + ctx->off_req, req.data(), 8 * req.size(), cudaMemcpyHostToDevice, st)))
    return cuda_fail(ctx, e, "upload requests");
  if (!inf.empty() &&
      (e = cudaMemcpyAsync(m + ctx->off_inf, inf.data(), 2 * inf.size(), cudaMemcpyHostToDevice, st)))
    return cuda_fail(ctx, e, "upload infer list");
  if ((e = cudaStreamSynchronize(st))) return cuda_fail(ctx, e, "sync");
  ctx->h2d_bytes = sizeof(DevJob) * n + 8 * req.size() + 2 * inf.size();
  if ((e = flag_alloc(&ctx->host_abort, &ctx->host_abort_dev))) return cuda_fail(ctx, e, "abort flag");
  for (int k = 0; k < 8; k++) reinterpret_cast<volatile uint32_t *>(ctx->host_abort)[k] = 0;
  if ((e = cudaEventCreate(&ctx->ev0)) || (e = cudaEventCreate(&ctx->ev1))) return cuda_fail(ctx, e, "events");

  Params &P = ctx->P;
  P.arena = static_cast<uint8_t *>(ctx->cfg.arena);
  {   // the arena as rows of 128 B for the operand TMA (see salus_dev.h)
    PFN_cuTensorMapEncodeTiled enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    if ((e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void **>(&enc), cudaEnableDefault,
                                     &q)) || !enc || q != cudaDriverEntryPointSuccess)
      return fail(ctx, SALUS_E_CUDA, "cuTensorMapEncodeTiled unavailable");
    const cuuint64_t rows = (cuuint64_t)ctx->Cp * ctx->cfg.page_bytes / 128;
    cuuint64_t gdim[2] = {128, rows};
    cuuint64_t gstride[1] = {128};
    cuuint32_t estride[2] = {1, 1};
    cuuint32_t box16[2] = {128, 128}, box8[2] = {128, 64};
    if (enc(&P.tmap16, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, ctx->cfg.arena, gdim, gstride, box16, estride,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS ||
        enc(&P.tmap8, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, ctx->cfg.arena, gdim, gstride, box8, estride,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return fail(ctx, SALUS_E_CUDA, "tensor map encoding failed");
  }
  P.ctrl = reinterpret_cast<Ctrl *>(m + ctx->off_ctrl);
  P.jobs = reinterpret_cast<const DevJob *>(m + ctx->off_jobs);
  P.req_ticks = reinterpret_cast<int64_t *>(m + ctx->off_req);
  P.req_seen = reinterpret_cast<uint64_t *>(m + ctx->off_reqseen);
  P.lreq_cnt = reinterpret_cast<uint32_t *>(m + ctx->off_lreqcnt);
  P.infer_list = reinterpret_cast<const uint16_t *>(m + ctx->off_inf);
  P.ppt = reinterpret_cast<uint32_t *>(m + ctx->off_ppt);
  P.lpt = reinterpret_cast<uint32_t *>(m + ctx->off_lpt);
  P.lpt_stride = ctx->lpt_stride;
  P.free_stack = reinterpret_cast<uint32_t *>(m + ctx->off_free);
  P.fence_slot = m + ctx->off_fslot;
  P.fence_seq = reinterpret_cast<uint64_t *>(m + ctx->off_fseq);
  P.pend_fence = reinterpret_cast<unsigned long long *>(m + ctx->off_pend);
  P.slots = reinterpret_cast<Slot *>(m + ctx->off_slots);
  P.ring = reinterpret_cast<unsigned long long *>(m + ctx->off_ring);
  P.ring_mask = (uint32_t)(ctx->ring_cap - 1);
  P.log = reinterpret_cast<salus_log_rec *>(m + ctx->off_log);
  P.wall = reinterpret_cast<salus_wall_rec *>(m + ctx->off_wall);
  P.log_cap = ctx->log_cap;
  P.stats = reinterpret_cast<salus_job_stat *>(m + ctx->off_stats);
  P.trace = reinterpret_cast<salus_trace_rec *>(m + ctx->off_trace);
  P.handoff = reinterpret_cast<salus_handoff_rec *>(m + ctx->off_handoff);
  P.handoff_cap = ctx->handoff_cap;
  P.trace_cap = ctx->trace_cap;
  P.dump = reinterpret_cast<float *>(m + ctx->off_dump);
  P.host_abort = ctx->host_abort_dev;
  P.swap = ctx->swap_dev;
  P.swap_fence = reinterpret_cast<unsigned long long *>(m + ctx->off_swfence);
  P.evl = reinterpret_cast<uint16_t *>(m + ctx->off_evl);
  P.n_jobs = n;
  P.n_infer = (uint32_t)inf.size();
  P.n_req = (uint32_t)req.size();
  P.Cp = ctx->Cp;
  P.policy = ctx->cfg.policy;
  P.max_lanes = ctx->cfg.max_lanes;
  P.flags = ctx->cfg.flags;
  P.n_workers = ctx->grid / 2 - 1;
  P.switch_ticks = (int64_t)ctx->cfg.switch_ticks;
  {   // eager stage publication (latency mode) while few lanes are open; the
      // SALUS_EAGER_LANES environment variable overrides (0 = never)
    const char *ev = getenv("SALUS_EAGER_LANES");
    P.eager_lanes = ev ? (uint32_t)atoi(ev) : SALUS_DEFAULT_EAGER_LANES;
    const char *nv = getenv("SALUS_NARROW_LANES");
    P.narrow_lanes = nv ? (uint32_t)atoi(nv) : 2u;
  }
  P.timeout_ns = (uint64_t)ctx->cfg.timeout_ms * 1000000ull;
  P.live = nullptr;
  P.max_jobs = ctx->cfg.max_jobs;
  if (online) {
    if ((e = cudaHostAlloc(reinterpret_cast<void **>(&ctx->live), 64, cudaHostAllocMapped)))
      return cuda_fail(ctx, e, "cudaHostAlloc live");
    if ((e = cudaHostGetDevicePointer(reinterpret_cast<void **>(&ctx->live_dev), ctx->live, 0)))
      return cuda_fail(ctx, e, "cudaHostGetDevicePointer live");
    if ((e = cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking))) return cuda_fail(ctx, e, "side stream");
    P.live = ctx->live_dev;
    for (const HostJob &h : ctx->jobs) ctx->max_id = std::max(ctx->max_id, h.j.job_id);
    ctx->lreq_cap = 0;
    ctx->lreq_left.assign(ctx->djobs.size(), 0);
    for (uint32_t d = 0; d < (uint32_t)ctx->djobs.size(); d++) {
      const HostJob &h = ctx->jobs[ctx->dense_to_submit[d]];
      if (h.live_req) ctx->lreq_cap += h.j.n_iters;
    }
    if (ctx->lreq_cap) {
      if ((e = cudaHostAlloc(reinterpret_cast<void **>(&ctx->lreq), 4ull * (ctx->lreq_cap + 2), cudaHostAllocMapped)))
        return cuda_fail(ctx, e, "cudaHostAlloc requests");
      if ((e = cudaHostGetDevicePointer(reinterpret_cast<void **>(&ctx->lreq_dev), ctx->lreq, 0)))
        return cuda_fail(ctx, e, "cudaHostGetDevicePointer requests");
      P.lreq = ctx->lreq_dev;
      P.n_lreq = ctx->lreq_cap;
    }
  }
  ctx->state = 1;
  return SALUS_OK;
}

int salus_run_async(salus_ctx *ctx) {
  if (!ctx) return SALUS_E_INVAL;
  if (ctx->state != 1) return fail(ctx, SALUS_E_STATE, "salus_prepare first");
  if (ctx->running) return fail(ctx, SALUS_E_STATE, "already running");
  if (ctx->poisoned) return fail(ctx, SALUS_E_STATE, "context poisoned by a kernel that ignored the abort");
  if ((ctx->cfg.flags & SALUS_FLAG_ONLINE) && ctx->ran) return fail(ctx, SALUS_E_STATE, "an online context runs once");
  cudaError_t e = cudaSetDevice(ctx->cfg.device);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaSetDevice");
  cudaStream_t st = static_cast<cudaStream_t>(ctx->cfg.stream);
  uint8_t *m = ctx->meta;
  if ((e = cudaMemsetAsync(m + ctx->off_ctrl, 0, sizeof(Ctrl), st)) ||
      (e = cudaMemsetAsync(m + ctx->off_lreqcnt, 0, 4 * std::max<uint64_t>(ctx->n_cap, 1), st)) ||
      (e = cudaMemsetAsync(m + ctx->off_slots, 0, sizeof(Slot) * MAX_LANES, st)) ||
      (e = cudaMemsetAsync(m + ctx->off_ring, 0, 8 * ctx->ring_cap, st)) ||
      (e = cudaMemsetAsync(m + ctx->off_fseq, 0, 8ull * ctx->Cp, st)) ||
      (e = cudaMemsetAsync(m + ctx->off_pend, 0, 8ull * MAX_LANES * MAX_LANES, st)))
    return cuda_fail(ctx, e, "reset");
  // per-job records start as "nothing yet" (job id, -1 ticks, 0 stamps) before
  // ev0, so a salus_poll_stats ordered after ev0 never sees a previous run's
  // records or uninitialised memory; the device's init_job rewrites the same
  {
    std::vector<salus_job_stat> img(std::max<uint32_t>(ctx->n_cap, 1));
    for (auto &r : img) {
      r.job_id = NONE32; r.first_lane = NONE32; r.admit_tick = -1; r.first_start_tick = -1;
      r.completion_tick = -1; r.completion_seq = ~0ull; r.wall_start_ns = 0; r.wall_end_ns = 0; r.wall_arrive_ns = 0;
    }
    for (uint32_t d = 0; d < (uint32_t)ctx->djobs.size() && d < img.size(); d++) img[d].job_id = ctx->djobs[d].job_id;
    ctx->stats_img.swap(img);
    if ((e = cudaMemcpyAsync(m + ctx->off_stats, ctx->stats_img.data(), sizeof(salus_job_stat) * ctx->stats_img.size(),
                             cudaMemcpyHostToDevice, st)))
      return cuda_fail(ctx, e, "reset stats");
    ctx->run_h2d = sizeof(salus_job_stat) * ctx->stats_img.size();
  }
  for (int k = 0; k < 8; k++) reinterpret_cast<volatile uint32_t *>(ctx->host_abort)[k] = 0;
  // migration: every run starts from the resume images (a DUMP_STATE job's
  // region is overwritten with its final state by the previous run)
  for (uint32_t d = 0; d < (uint32_t)ctx->djobs.size() && d < ctx->n_pre; d++) {
    const HostJob &h = ctx->jobs[ctx->dense_to_submit[d]];
    if (!h.resume.empty())
      std::memcpy(ctx->swap_host + (uint64_t)ctx->djobs[d].pt_off * ctx->cfg.page_bytes, h.resume.data(),
                  h.resume.size());
  }
  if ((e = cudaEventRecord(ctx->ev0, st))) return cuda_fail(ctx, e, "event");
  if (ctx->live) {
    std::lock_guard<std::mutex> g(ctx->live_mu);
    reinterpret_cast<volatile uint32_t *>(ctx->live)[0] = (uint32_t)ctx->jobs.size();   // published so far
    reinterpret_cast<volatile uint32_t *>(ctx->live)[1] = 0;                           // submissions open
    ctx->ended = false;
    if (ctx->lreq) {
      *reinterpret_cast<volatile uint64_t *>(ctx->lreq) = 0;
      ctx->lreq_pub = 0;
      for (uint32_t d = 0; d < (uint32_t)ctx->djobs.size(); d++) {
        const HostJob &h = ctx->jobs[ctx->dense_to_submit[d]];
        ctx->lreq_left[d] = h.live_req ? h.j.n_iters : 0;
      }
    }
  }
  int rc = launch_persistent(ctx->P, ctx->grid, st);
  if (rc) return cuda_fail(ctx, (cudaError_t)rc, "cooperative launch");
  if ((e = cudaEventRecord(ctx->ev1, st))) return cuda_fail(ctx, e, "event");
  ctx->running = true;
  ctx->t_out = false;
  ctx->t0 = std::chrono::steady_clock::now();
  return SALUS_OK;
}

int salus_wait(salus_ctx *ctx, salus_job_stat *stats, uint64_t max_stats, uint64_t *n_stats);

int salus_run(salus_ctx *ctx, salus_job_stat *stats, uint64_t max_stats, uint64_t *n_stats) {
  int rc = salus_run_async(ctx);
  if (rc) return rc;
  if (ctx->live) salus_end_submissions(ctx);
  return salus_wait(ctx, stats, max_stats, n_stats);
}

int salus_end_submissions(salus_ctx *ctx) {
  if (!ctx) return SALUS_E_INVAL;
  if (!ctx->live) return fail(ctx, SALUS_E_STATE, "not an online context");
  std::lock_guard<std::mutex> g(ctx->live_mu);
  std::atomic_thread_fence(std::memory_order_seq_cst);
  reinterpret_cast<volatile uint32_t *>(ctx->live)[1] = 1;
  ctx->ended = true;
  return SALUS_OK;
}

int salus_submit_requests(salus_ctx *ctx, const uint32_t *job_ids, uint32_t n) {
  if (!ctx || (!job_ids && n)) return SALUS_E_INVAL;
  if (!ctx->live) return fail(ctx, SALUS_E_STATE, "not an online context (SALUS_FLAG_ONLINE)");
  std::lock_guard<std::mutex> g(ctx->live_mu);
  if (!ctx->running || ctx->ended) return fail(ctx, SALUS_E_STATE, "no live run accepting submissions");
  if (!ctx->lreq) return fail(ctx, SALUS_E_INVAL, "no live-request jobs (INFER with request_ticks = NULL)");
  // check the whole batch before publishing any of it
  std::unordered_map<uint32_t, uint32_t> take;
  for (uint32_t i = 0; i < n; i++) {
    auto it = ctx->id_to_dense.find(job_ids[i]);
    if (it == ctx->id_to_dense.end() || it->second >= ctx->lreq_left.size() ||
        !ctx->jobs[ctx->dense_to_submit[it->second]].live_req)
      return fail(ctx, SALUS_E_INVAL, "job " + std::to_string(job_ids[i]) + " takes no live requests");
    if (++take[it->second] > ctx->lreq_left[it->second])
      return fail(ctx, SALUS_E_CAPACITY, "job " + std::to_string(job_ids[i]) + ": more requests than n_iters");
  }
  if (n == 0) return SALUS_OK;
  volatile uint32_t *ring = reinterpret_cast<volatile uint32_t *>(ctx->lreq);
  uint32_t d = 0;
  for (uint32_t i = 0; i < n; i++) {
    d = ctx->id_to_dense[job_ids[i]];
    ring[2 + ctx->lreq_pub + i] = d;
    ctx->lreq_left[d]--;
  }
  ctx->lreq_pub += n;
  std::atomic_thread_fence(std::memory_order_seq_cst);
  // publish {count, last entry} in one 8-byte store (the device reads both at once)
  *reinterpret_cast<volatile uint64_t *>(ctx->lreq) = ((uint64_t)d << 32) | ctx->lreq_pub;
  return SALUS_OK;
}

int salus_read_requests(salus_ctx *ctx, uint32_t job_id, int64_t *ticks, uint64_t *seen_ns, uint64_t cap,
                        uint64_t *n) {
  if (!ctx || !n) return SALUS_E_INVAL;
  if (!ctx->ran || ctx->running) return fail(ctx, SALUS_E_STATE, "no finished run");
  auto it = ctx->id_to_dense.find(job_id);
  if (it == ctx->id_to_dense.end()) return fail(ctx, SALUS_E_INVAL, "unknown job");
  const DevJob &D = ctx->djobs[it->second];
  *n = D.kind == SALUS_INFER ? D.n_iters : 0;
  if (!*n || (!ticks && !seen_ns)) return SALUS_OK;
  if (cap < *n) return fail(ctx, SALUS_E_CAPACITY, "buffer too small");
  cudaError_t e = cudaSetDevice(ctx->cfg.device);
  if (e == cudaSuccess && ticks)
    e = cudaMemcpy(ticks, ctx->meta + ctx->off_req + 8ull * D.req_off, 8 * *n, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && seen_ns) {
    if (ctx->jobs[ctx->dense_to_submit[it->second]].live_req)
      e = cudaMemcpy(seen_ns, ctx->meta + ctx->off_reqseen + 8ull * D.req_off, 8 * *n, cudaMemcpyDeviceToHost);
    else
      std::memset(seen_ns, 0, 8 * *n);
  }
  if (e != cudaSuccess) return cuda_fail(ctx, e, "read requests");
  return SALUS_OK;
}

int salus_submit_live(salus_ctx *ctx, const salus_job *job) {
  if (!ctx || !job) return SALUS_E_INVAL;
  if (!ctx->live) return fail(ctx, SALUS_E_STATE, "not an online context (SALUS_FLAG_ONLINE)");
  std::lock_guard<std::mutex> g(ctx->live_mu);
  if (!ctx->running || ctx->ended) return fail(ctx, SALUS_E_STATE, "no live run accepting submissions");
  if (ctx->id_to_submit.count(job->job_id)) return fail(ctx, SALUS_E_DUPLICATE, "duplicate job id");
  if (job->kind != SALUS_TRAIN) return fail(ctx, SALUS_E_INVAL, "live submission takes TRAIN jobs");
  if (job->resume_state || (job->dump & SALUS_DUMP_STATE))
    return fail(ctx, SALUS_E_INVAL, "migration state (resume / DUMP_STATE) is for jobs submitted before the run");
  if (!ctx->jobs.empty() && job->job_id <= ctx->max_id)
    return fail(ctx, SALUS_E_INVAL, "live job ids must increase");
  std::string why;
  int rc = validate_job(job, (ctx->cfg.flags & SALUS_FLAG_NULL_WORK) != 0, &why);
  if (rc) return fail(ctx, rc, "job " + std::to_string(job->job_id) + ": " + why);
  const uint64_t G = ctx->cfg.page_bytes;
  const uint64_t p = (job->persistent_bytes + G - 1) / G, e = (job->ephemeral_bytes + G - 1) / G;
  if (p + e > ctx->Cp) return fail(ctx, SALUS_E_UNSCHEDULABLE, "p + e > C pages (A22)");
  if (ctx->jobs.size() >= ctx->cfg.max_jobs) return fail(ctx, SALUS_E_CAPACITY, "max_jobs reached");
  HostJob h;
  h.j = *job;
  h.j.request_ticks = nullptr;
  h.j.arrival_tick = INT64_MAX;        // stamped by the device scheduler
  h.fp = footprint(*job);
  h.submit_idx = (uint32_t)ctx->jobs.size();
  DevJob D{};
  uint64_t req_dummy = 0, ppt = ctx->ppt_used, dump = ctx->dump_cur;
  fill_devjob(ctx, h, D, req_dummy, ppt, dump);
  if (ppt > ctx->ppt_cap) return fail(ctx, SALUS_E_CAPACITY, "live page-table space exhausted");
  if (dump > ctx->dump_cap) return fail(ctx, SALUS_E_CAPACITY, "dump_bytes exceeded");
  for (uint32_t s = 0; s < D.n_stages; s++)
    if (std::max<uint32_t>(D.stage_tiles[s], D.stage_tiles_lat[s]) > ctx->ring_tiles)
      return fail(ctx, SALUS_E_CAPACITY, "stage exceeds the task ring");
  const uint32_t d = (uint32_t)ctx->jobs.size();   // dense index = publication order
  cudaError_t ce = cudaSetDevice(ctx->cfg.device);
  if (ce == cudaSuccess)
    ce = cudaMemcpyAsync(ctx->meta + ctx->off_jobs + sizeof(DevJob) * d, &D, sizeof(DevJob), cudaMemcpyHostToDevice,
                         ctx->side);
  if (ce == cudaSuccess) ce = cudaStreamSynchronize(ctx->side);
  if (ce != cudaSuccess) return cuda_fail(ctx, ce, "upload live job");
  ctx->ppt_used = ppt;
  ctx->dump_cur = dump;
  ctx->max_id = job->job_id;
  ctx->id_to_submit[job->job_id] = h.submit_idx;
  ctx->id_to_dense[job->job_id] = d;
  ctx->dense_to_submit.push_back(h.submit_idx);
  ctx->djobs.push_back(D);
  ctx->jobs.push_back(std::move(h));
  ctx->h2d_bytes += sizeof(DevJob);
  std::atomic_thread_fence(std::memory_order_seq_cst);
  reinterpret_cast<volatile uint32_t *>(ctx->live)[0] = d + 1;   // publish
  return SALUS_OK;
}

int salus_wait(salus_ctx *ctx, salus_job_stat *stats, uint64_t max_stats, uint64_t *n_stats) {
  if (!ctx) return SALUS_E_INVAL;
  if (!ctx->running) return fail(ctx, SALUS_E_STATE, "salus_run_async first");
  cudaError_t e = cudaSetDevice(ctx->cfg.device);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaSetDevice");
  uint8_t *m = ctx->meta;
  // host watchdog: poll, then ask the kernel to abort (mapped pinned flag)
  const auto t0 = ctx->t0;
  bool timed_out = false;
  for (;;) {
    e = cudaEventQuery(ctx->ev1);
    if (e == cudaSuccess) break;
    if (e != cudaErrorNotReady) {
      ctx->running = false;
      // a scheduler failure aborts the workers, which trap: its code is in the mapped slot
      const volatile uint32_t *h = ctx->host_abort;
      std::string where = h[1] ? "kernel (scheduler failure " + std::to_string((int32_t)h[1]) + ", info " +
                                     std::to_string(h[2]) + ", tick " + std::to_string(h[3]) + ")"
                               : std::string("kernel");
      if (h[4])   // SALUS_DBG_BOUNDS builds: a page number outside the arena
        where += " (bad page: site " + std::to_string(h[4]) + ", offset/chunk " + std::to_string(h[5]) +
                 ", entry " + std::to_string(h[6]) + ")";
      return cuda_fail(ctx, e, where.c_str());
    }
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (!timed_out && ms > ctx->cfg.timeout_ms) {
      *reinterpret_cast<volatile uint32_t *>(ctx->host_abort) = 1;
      timed_out = true;
    }
    if (timed_out && ms > ctx->cfg.timeout_ms + 20000.0) {
      // the kernel may still read/write the mapped flags and the caller's
      // buffers: never free them (salus_close leaks them); reset the device
      ctx->running = false;
      ctx->poisoned = true;
      return fail(ctx, SALUS_E_TIMEOUT, "kernel did not exit after abort (context poisoned: reset the device)");
    }
    std::this_thread::sleep_for(std::chrono::microseconds(20));
  }
  ctx->running = false;
  Ctrl ctrl;
  if ((e = cudaMemcpy(&ctrl, m + ctx->off_ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost)))
    return cuda_fail(ctx, e, "readback");
  float ms = 0;
  cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
  salus_run_stats &rs = ctx->last;
  rs.n_dispatch = ctrl.n_dispatch; rs.n_ticks = ctrl.n_ticks; rs.n_log = std::min<uint64_t>(ctrl.n_log, ctx->log_cap);
  rs.n_tasks = ctrl.n_tasks; rs.kernel_ns = (uint64_t)((double)ms * 1e6);
  rs.wall_first_ns = ctrl.wall_first_ns; rs.wall_last_ns = ctrl.wall_last_ns;
  rs.sched_wait_ns = ctrl.sched_wait_ns; rs.sched_fence_ns = ctrl.sched_fence_ns; rs.sched_ring_ns = ctrl.sched_ring_ns; rs.status = ctrl.status; rs.n_workers = ctx->grid / 2 - 1;
  rs.n_swap_out = ctrl.n_swap_out; rs.n_swap_in = ctrl.n_swap_in; rs.swap_bytes = ctrl.swap_bytes; rs.swap_ns = ctrl.swap_ns;
  ctx->n_trace = std::min<uint64_t>(ctrl.n_trace, ctx->trace_cap);
  ctx->n_handoff = std::min<uint64_t>(ctrl.n_handoff, ctx->handoff_cap);
  rs.h2d_bytes = ctx->h2d_bytes + ctx->run_h2d;
  rs.d2h_bytes = sizeof(Ctrl) + (stats ? sizeof(salus_job_stat) * ctx->jobs.size() : 0);
  ctx->ran = true;
  const uint32_t n = (uint32_t)ctx->jobs.size();
  if (stats) {
    std::vector<salus_job_stat> dense(n);
    if ((e = cudaMemcpy(dense.data(), m + ctx->off_stats, sizeof(salus_job_stat) * n, cudaMemcpyDeviceToHost)))
      return cuda_fail(ctx, e, "readback stats");
    const uint64_t k = std::min<uint64_t>(max_stats, n);
    for (uint32_t d = 0; d < n; d++) {
      const uint32_t s = ctx->dense_to_submit[d];
      if (s < k) stats[s] = dense[d];
    }
    if (n_stats) *n_stats = k;
  } else if (n_stats) {
    *n_stats = 0;
  }
  if (timed_out) return fail(ctx, SALUS_E_TIMEOUT, "run exceeded timeout_ms");
  if (ctrl.status) return fail(ctx, ctrl.status, "device error, info " + std::to_string(ctrl.err_info[0]));
  if (ctrl.log_overflow) return fail(ctx, SALUS_E_CAPACITY, "log capacity exceeded");
  return SALUS_OK;
}

int salus_poll_stats(salus_ctx *ctx, salus_job_stat *stats, uint64_t max_stats, uint64_t *n_stats,
                     uint64_t *n_done) {
  if (!ctx) return SALUS_E_INVAL;
  if (!ctx->running) return fail(ctx, SALUS_E_STATE, "no run in flight (salus_run_async first)");
  cudaError_t e = cudaSetDevice(ctx->cfg.device);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaSetDevice");
  if (!ctx->side && (e = cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking)))
    return cuda_fail(ctx, e, "side stream");
  uint32_t n;
  std::vector<uint32_t> d2s;
  {
    std::lock_guard<std::mutex> g(ctx->live_mu);     // live submissions grow the table
    n = (uint32_t)ctx->jobs.size();
    d2s = ctx->dense_to_submit;
  }
  std::vector<salus_job_stat> dense(n);
  // never overtake run_async's reset of the records (recorded before ev0)
  if ((e = cudaStreamWaitEvent(ctx->side, ctx->ev0, 0))) return cuda_fail(ctx, e, "poll order");
  if (n && ((e = cudaMemcpyAsync(dense.data(), ctx->meta + ctx->off_stats, sizeof(salus_job_stat) * n,
                                 cudaMemcpyDeviceToHost, ctx->side)) ||
            (e = cudaStreamSynchronize(ctx->side))))
    return cuda_fail(ctx, e, "poll stats");
  uint64_t done = 0;
  for (uint32_t d = 0; d < n; d++) done += dense[d].wall_end_ns != 0;
  if (n_done) *n_done = done;
  const uint64_t k = stats ? std::min<uint64_t>(max_stats, n) : 0;
  for (uint32_t d = 0; d < n && stats; d++) {
    const uint32_t s = d < d2s.size() ? d2s[d] : d;
    if (s < k) stats[s] = dense[d];
  }
  if (n_stats) *n_stats = k;
  return SALUS_OK;
}

int salus_read_state(salus_ctx *ctx, uint32_t job_id, void *buf, uint64_t cap_bytes, uint64_t *n) {
  if (!ctx || !n) return SALUS_E_INVAL;
  if (!ctx->ran) return fail(ctx, SALUS_E_STATE, "no run yet");
  auto it = ctx->id_to_dense.find(job_id);
  if (it == ctx->id_to_dense.end()) return fail(ctx, SALUS_E_INVAL, "unknown job");
  const DevJob &D = ctx->djobs[it->second];
  if (!(D.dump & SALUS_DUMP_STATE)) return fail(ctx, SALUS_E_INVAL, "job was not submitted with SALUS_DUMP_STATE");
  const uint64_t bytes = (uint64_t)D.ap_pages * ctx->cfg.page_bytes;
  *n = bytes;
  if (!buf) return SALUS_OK;
  if (cap_bytes < bytes) return fail(ctx, SALUS_E_CAPACITY, "buffer too small");
  std::memcpy(buf, ctx->swap_host + (uint64_t)D.pt_off * ctx->cfg.page_bytes, bytes);
  return SALUS_OK;
}

int salus_read_run_stats(const salus_ctx *ctx, salus_run_stats *out) {
  if (!ctx || !out) return SALUS_E_INVAL;
  if (!ctx->ran) return SALUS_E_STATE;
  *out = ctx->last;
  return SALUS_OK;
}

int salus_read_log(salus_ctx *ctx, void *buf, uint64_t cap_bytes, uint64_t *n_bytes) {
  if (!ctx || !n_bytes) return SALUS_E_INVAL;
  if (!ctx->ran || !(ctx->cfg.flags & SALUS_FLAG_LOG)) return fail(ctx, SALUS_E_STATE, "no log");
  const uint64_t bytes = ctx->last.n_log * sizeof(salus_log_rec);
  *n_bytes = bytes;
  if (!buf) return SALUS_OK;
  if (cap_bytes < bytes) return fail(ctx, SALUS_E_CAPACITY, "log buffer too small");
  cudaError_t e = cudaMemcpy(buf, ctx->meta + ctx->off_log, bytes, cudaMemcpyDeviceToHost);
  return e ? cuda_fail(ctx, e, "read log") : SALUS_OK;
}

int salus_read_trace(salus_ctx *ctx, salus_trace_rec *buf, uint64_t cap_recs, uint64_t *n_recs) {
  if (!ctx || !n_recs) return SALUS_E_INVAL;
  if (!ctx->ran || !(ctx->cfg.flags & SALUS_FLAG_TRACE)) return fail(ctx, SALUS_E_STATE, "no trace");
  *n_recs = ctx->n_trace;
  if (!buf) return SALUS_OK;
  if (cap_recs < ctx->n_trace) return fail(ctx, SALUS_E_CAPACITY, "trace buffer too small");
  cudaError_t e = cudaMemcpy(buf, ctx->meta + ctx->off_trace, ctx->n_trace * sizeof(salus_trace_rec),
                             cudaMemcpyDeviceToHost);
  return e ? cuda_fail(ctx, e, "read trace") : SALUS_OK;
}

int salus_debug_layout(const salus_ctx *ctx, uint64_t *out, uint32_t n) {
  if (!ctx || !out || n < 9) return SALUS_E_INVAL;
  if (ctx->state == 0) return SALUS_E_STATE;
  out[0] = ctx->off_ctrl; out[1] = ctx->off_slots; out[2] = sizeof(Slot); out[3] = ctx->off_trace;
  out[4] = ctx->trace_cap; out[5] = offsetof(Slot, stage_done); out[6] = offsetof(Slot, qstate);
  out[7] = offsetof(Slot, done_seq); out[8] = offsetof(Ctrl, n_trace);
  return SALUS_OK;
}

int salus_debug_read(salus_ctx *ctx, uint64_t off, uint64_t bytes, void *host) {
  if (!ctx || !host) return SALUS_E_INVAL;
  if (ctx->state == 0) return SALUS_E_STATE;
  if (off > ctx->meta_bytes || bytes > ctx->meta_bytes - off) return SALUS_E_INVAL;
  cudaError_t e = cudaSetDevice(ctx->cfg.device);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaSetDevice");
  if (!ctx->side && (e = cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking)))
    return cuda_fail(ctx, e, "side stream");
  if ((e = cudaMemcpyAsync(host, ctx->meta + off, bytes, cudaMemcpyDeviceToHost, ctx->side)) ||
      (e = cudaStreamSynchronize(ctx->side)))
    return cuda_fail(ctx, e, "debug read");
  return SALUS_OK;
}

int salus_read_handoffs(salus_ctx *ctx, salus_handoff_rec *buf, uint64_t cap_recs, uint64_t *n_recs) {
  if (!ctx || !n_recs) return SALUS_E_INVAL;
  if (!ctx->ran || !(ctx->cfg.flags & SALUS_FLAG_CHECK)) return fail(ctx, SALUS_E_STATE, "no hand-off record (SALUS_FLAG_CHECK)");
  *n_recs = ctx->n_handoff;
  if (!buf) return SALUS_OK;
  if (cap_recs < ctx->n_handoff) return fail(ctx, SALUS_E_CAPACITY, "buffer too small");
  cudaError_t e = cudaMemcpy(buf, ctx->meta + ctx->off_handoff, ctx->n_handoff * sizeof(salus_handoff_rec),
                             cudaMemcpyDeviceToHost);
  return e ? cuda_fail(ctx, e, "read hand-offs") : SALUS_OK;
}

int salus_read_wall(salus_ctx *ctx, salus_wall_rec *buf, uint64_t cap_recs, uint64_t *n_recs) {
  if (!ctx || !n_recs) return SALUS_E_INVAL;
  if (!ctx->ran || !(ctx->cfg.flags & SALUS_FLAG_LOG)) return fail(ctx, SALUS_E_STATE, "no wall log");
  const uint64_t n = std::min<uint64_t>(ctx->last.n_dispatch, ctx->log_cap);
  *n_recs = n;
  if (!buf) return SALUS_OK;
  if (cap_recs < n) return fail(ctx, SALUS_E_CAPACITY, "wall buffer too small");
  cudaError_t e = cudaMemcpy(buf, ctx->meta + ctx->off_wall, n * sizeof(salus_wall_rec), cudaMemcpyDeviceToHost);
  return e ? cuda_fail(ctx, e, "read wall") : SALUS_OK;
}

int salus_read_layers(salus_ctx *ctx, uint32_t job_id, uint32_t iter, float *buf, uint64_t cap_floats,
                      uint64_t *n) {
  if (!ctx || !n) return SALUS_E_INVAL;
  if (!ctx->ran) return fail(ctx, SALUS_E_STATE, "not run");
  auto it = ctx->id_to_dense.find(job_id);
  if (it == ctx->id_to_dense.end()) return fail(ctx, SALUS_E_INVAL, "unknown job");
  const DevJob &D = ctx->djobs[it->second];
  uint64_t off, cnt;
  const bool steps = (D.dump & SALUS_DUMP_WEIGHT_STEPS) != 0;
  if (iter == 0xFFFFFFFFu) {
    if (!(D.dump & (SALUS_DUMP_WEIGHTS | SALUS_DUMP_WEIGHT_STEPS)))
      return fail(ctx, SALUS_E_INVAL, "job did not dump weights");
    cnt = D.w_count;
    off = D.dump_w_off + (steps ? (uint64_t)(D.n_iters - 1) * cnt : 0);
  } else if (iter & 0x80000000u) {
    const uint32_t k = iter & 0x7FFFFFFFu;
    if (!steps || k >= D.n_iters) return fail(ctx, SALUS_E_INVAL, "no such weight step (SALUS_DUMP_WEIGHT_STEPS)");
    cnt = D.w_count;
    off = D.dump_w_off + (uint64_t)k * cnt;
  } else {
    if (!(D.dump & SALUS_DUMP_OUTPUTS) || iter >= D.n_iters) return fail(ctx, SALUS_E_INVAL, "no such output");
    cnt = (uint64_t)D.batch * D.dims[D.n_layers];
    off = D.dump_out_off + (uint64_t)iter * cnt;
  }
  *n = cnt;
  if (!buf) return SALUS_OK;
  if (cap_floats < cnt) return fail(ctx, SALUS_E_CAPACITY, "buffer too small");
  cudaError_t e = cudaMemcpy(buf, ctx->meta + ctx->off_dump + 4 * off, 4 * cnt, cudaMemcpyDeviceToHost);
  return e ? cuda_fail(ctx, e, "read layers") : SALUS_OK;
}

const char *salus_last_error(const salus_ctx *ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int salus_close(salus_ctx *ctx) {
  if (!ctx) return SALUS_OK;
  if (ctx->poisoned) return SALUS_E_TIMEOUT;   // leak: a hung kernel may still use the mapped buffers
  if (ctx->running) {                      // never free under a live kernel
    if (ctx->live && !ctx->ended) salus_end_submissions(ctx);
    salus_wait(ctx, nullptr, 0, nullptr);
  }
  if (ctx->host_abort) flag_free(ctx->host_abort, ctx->host_abort_dev);
  if (ctx->live) cudaFreeHost(ctx->live);
  if (ctx->lreq) cudaFreeHost(ctx->lreq);
  if (ctx->side) cudaStreamDestroy(ctx->side);
  if (ctx->ev0) cudaEventDestroy(ctx->ev0);
  if (ctx->ev1) cudaEventDestroy(ctx->ev1);
  delete ctx;
  return SALUS_OK;
}

}  // extern "C"
