/*
 * salus.h — C ABI of the B200-native Salus execution service (libsalus.so).
 *
 * What it implements (PAPER.md = LaTeX source of arXiv 1902.04610):
 *   - a singleton execution service that consolidates all GPU access
 *     (§3.1) — here one persistent sm_100a kernel per GPU;
 *   - sessions created per job — salus_submit_job();
 *   - lane requests queued by the memory manager, Algorithm 1 "GPU Lane
 *     Assignment" (§3.3.2) under the safety condition
 *     sum P_i + sum L_j <= C, L_j = max_{i in j} E_i;
 *   - iteration-granularity scheduling per lane (§3.2.2
 *     P:353-354) with FIFO / SRTF / PACK / FAIR (§4);
 *   - persistent memory kept resident so a switch is only the next
 *     iteration record (Observations 1-2).
 *
 * Ambiguities of the paper are resolved by the readings A1..A30 of
 * SURVEY.md §8(c), restated in DESIGN.md; the ones visible at this
 * boundary are cited below.
 *
 * Conventions
 *   - Every call returns int: SALUS_OK (0) or a negative SALUS_E_* code.
 *     No call aborts the process.  salus_last_error() gives a message.
 *   - Pointers documented "device" are CUDA device pointers owned by the
 *     caller (in this repo: torch tensors); "host" pointers are ordinary
 *     host memory.  The library never cudaMalloc()s device memory and never
 *     frees caller buffers.  It owns only the host-side context and a few
 *     bytes of pinned host memory for the abort flag.
 *   - A context has a single owner; calls on one context must not overlap.
 *     Separate contexts on separate devices may run concurrently.
 *   - Sizes are bytes unless the name says pages.  Logical time is int64
 *     ticks (1 tick = 1 ns nominal, A17).
 */
#ifndef SALUS_H_
#define SALUS_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SALUS_ABI_VERSION 1

/* Scheduling policies (§4; FIFO baseline P:504, 612-613). */
enum { SALUS_FIFO = 0, SALUS_SRTF = 1, SALUS_PACK = 2, SALUS_FAIR = 3 };

/* Job kinds: a training job runs forward+backward+SGD per iteration; an
 * inference job runs one forward pass per request (§2.1, §5.3). */
enum { SALUS_TRAIN = 0, SALUS_INFER = 1 };

enum {
  SALUS_OK = 0,
  SALUS_E_INVAL = -1,          /* bad argument / descriptor                     */
  SALUS_E_DUPLICATE = -2,      /* job id already submitted               */
  SALUS_E_UNSCHEDULABLE = -3,  /* p + e > C pages: can never run alone (A22)    */
  SALUS_E_STATE = -4,          /* call not valid in the context's state          */
  SALUS_E_CAPACITY = -5,       /* a caller buffer / table is too small          */
  SALUS_E_CUDA = -6,           /* CUDA runtime error (message has the string)   */
  SALUS_E_STUCK = -7,          /* no event left with jobs unfinished (device)   */
  SALUS_E_TIMEOUT = -8         /* salus_run exceeded cfg.timeout_ms; kernel was
                                  told to abort and has exited                   */
};

/* salus_config.flags */
enum {
  SALUS_FLAG_LOG = 1,        /* record the canonical schedule log + wall stamps  */
  SALUS_FLAG_NULL_WORK = 2,  /* schedule only: no iteration work is executed     */
  SALUS_FLAG_CHECK = 4,      /* device asserts the safety invariants every tick  */
  SALUS_FLAG_TRACE = 8,      /* record one salus_trace_rec per executed tile     */
  SALUS_FLAG_ONLINE = 16,    /* online submission: the run
                                also admits jobs submitted with salus_submit_live
                                while it is live, until salus_end_submissions    */
  SALUS_FLAG_EVICT = 32      /* SRTF admission with persistent eviction (SURVEY
                                §8(f) NEXT-3, reading A35; "the
                                higher priority job is admitted as long as its own
                                safety condition is met ... regardless of other
                                already-running jobs"): when FindLane fails for a
                                queued job, idle admitted jobs of strictly lower
                                SRTF priority are swapped out (lowest first, all or
                                nothing) -- their persistent pages copied by the
                                kernel to the caller's pinned host buffer
                                (salus_set_swap) and freed -- and restored (copied
                                back into fresh pages) when re-admitted.  SRTF only,
                                not with SALUS_FLAG_ONLINE (else E_INVAL at open). */
};

/* salus_job.dump */
enum {
  SALUS_DUMP_OUTPUTS = 1,    /* keep fp32 A_L of every iteration / request       */
  SALUS_DUMP_WEIGHTS = 2,    /* keep fp32 master weights after the last iteration */
  SALUS_DUMP_WEIGHT_STEPS = 8, /* keep fp32 master weights after EVERY iteration
                                (parity checks of each step from the kernel's own
                                state; n_iters x the weight count floats)        */
  SALUS_DUMP_STATE = 4       /* migration: when the job
                                finishes, the kernel copies its persistent device
                                state (the opaque image salus_read_state returns)
                                to its region of the swap area; another context,
                                e.g. on another GPU, resumes it from that image
                                (salus_job.resume_state)                          */
};

/* ---------------------------------------------------------------------
 * Canonical schedule log: fixed-width little-endian 32-byte records.
 * The byte-compare of this log against the CPU oracle is the schedule
 * parity test (north star: "schedules must match the oracle bit-exactly").
 * Order within a tick follows the phases of A15: completions/finishes,
 * arrivals, admission, dispatch.
 * ------------------------------------------------------------------- */
typedef struct {
  int64_t  tick;
  uint32_t kind;   /* SALUS_REC_*                                   */
  uint32_t lane;   /* lane id (monotonic, never reused, I5); NONE = 0xFFFFFFFF */
  uint32_t job;    /* job id                                        */
  uint32_t a;
  uint64_t b;
} salus_log_rec;

enum {
  SALUS_REC_DISPATCH = 1,    /* a = iteration index, b = global dispatch seq     */
  SALUS_REC_LANE_OPEN = 2,   /* FindLane branch 1; a = L pages        */
  SALUS_REC_LANE_REUSE = 3,  /* branch 2 (A1/A2); a = L pages          */
  SALUS_REC_LANE_RESIZE = 4, /* branch 3 (A3); a = new L, b = old L    */
  SALUS_REC_LANE_SHRINK = 5, /* JobFinish, residents remain (A4); a = new, b = old */
  SALUS_REC_LANE_CLOSE = 6,  /* JobFinish, ref(lane) == 0             */
  SALUS_REC_JOB_QUEUED = 7,  /* JobArrive: Q <- Q u {(P,E)}           */
  SALUS_REC_JOB_ADMIT = 8,   /* ProcessRequests assigns a lane; a = p, b = e pages */
  SALUS_REC_JOB_FINISH = 9,  /* last iteration ended; a = n, b = completion_seq    */
  SALUS_REC_JOB_EVICT = 10,  /* SALUS_FLAG_EVICT: swapped out of its lane (A35);
                                lane = the lane it left, a = p pages,
                                b = iterations done so far                       */
  SALUS_REC_JOB_RESTORE = 11 /* SALUS_FLAG_EVICT: a swapped-out job re-admitted;
                                a = p, b = e pages (its first admission is
                                JOB_ADMIT)                                       */
};

/* Physical timing of one dispatched iteration (not part of the compared log):
 * globaltimer ns of its first tile start and last tile end, and of the
 * scheduler's append of its dispatch record to the lane's ring. */
typedef struct {
  uint64_t seq;
  uint32_t lane, job;
  uint64_t start_ns, end_ns;
  uint64_t append_ns;
} salus_wall_rec;

/* ---------------------------------------------------------------------
 * Configuration
 * ------------------------------------------------------------------- */
typedef struct {
  int32_t  device;           /* CUDA ordinal the arena/meta live on              */
  uint32_t policy;           /* SALUS_FIFO..SALUS_FAIR                           */
  void    *arena;            /* device, caller-owned, >= 256-byte aligned. The
                                HBM arena all persistent regions and lanes are
                                carved from (two-region layout P:365-369, paged
                                per A18).                                        */
  uint64_t arena_bytes;      /* >= floor(capacity_bytes/page_bytes)*page_bytes   */
  void    *stream;           /* cudaStream_t the kernel is launched on (NULL =
                                legacy default stream)                           */
  uint64_t capacity_bytes;   /* C of the safety condition            */
  uint32_t page_bytes;       /* 0 -> 65536. P_i, E_i and C are rounded to pages
                                before every check: p = ceil(P/G), e = ceil(E/G),
                                Cp = floor(C/G) (A18). Must be 65536 in v1.      */
  uint32_t max_lanes;        /* 0 -> policy default (FIFO 1, SRTF 1, PACK 64,
                                FAIR 1; A9); at most 64                           */
  uint32_t max_jobs;         /* submit capacity; <= 2048                          */
  uint32_t flags;            /* SALUS_FLAG_*                                      */
  uint64_t switch_ticks;     /* logical switch penalty per job change in a lane
                                (A16); 0 in parity tests                          */
  uint64_t log_capacity;     /* records reserved for the log and for wall stamps */
  uint64_t dump_bytes;       /* bytes reserved for SALUS_DUMP_* data             */
  uint32_t n_workers;        /* worker CTA pairs; 0 -> (#SMs / 2 - 1)              */
  uint32_t timeout_ms;       /* salus_run watchdog; 0 -> 600000                   */
  uint64_t trace_capacity;   /* SALUS_FLAG_TRACE records; 0 -> 1<<20              */
} salus_config;

typedef struct salus_ctx salus_ctx;

/* Create a context.  Copies *cfg.  Errors: E_INVAL (bad policy, page size,
 * capacity > arena, max_jobs out of range), E_CUDA. */
int salus_open(const salus_config *cfg, salus_ctx **out);

/* ---------------------------------------------------------------------
 * Jobs ("sessions").  A job is a dense MLP with n_layers
 * layers of widths dims[0..n_layers] (the "small-model forward/backward
 * dense layers" of the north star), batch rows per iteration.
 * ------------------------------------------------------------------- */
typedef struct {
  uint32_t job_id;           /* unique per context                               */
  uint32_t kind;             /* SALUS_TRAIN | SALUS_INFER                        */
  int64_t  arrival_tick;     /* JobArrive time                            */
  uint64_t persistent_bytes; /* declared P_i: model + framework-internal (P:292-306,
                                484); must be >= the job's device footprint       */
  uint64_t ephemeral_bytes;  /* declared E_i: per-iteration scratch   */
  uint32_t n_iters;          /* TRAIN: iterations; INFER: number of requests      */
  uint32_t n_layers;         /* 1..8                                              */
  uint64_t iter_ticks;       /* known per-iteration duration; the job's duration is
                                n_iters*iter_ticks ("we assume the job
                                execution time is known")                        */
  uint32_t dims[9];          /* d_0..d_L, each 1..8192                            */
  uint32_t batch;            /* 1..8192                                           */
  float    lr;               /* SGD learning rate (TRAIN)                          */
  uint32_t dump;             /* SALUS_DUMP_* bits                                  */
  uint64_t seed;             /* data generator seed (A29)                          */
  const int64_t *request_ticks; /* host; INFER: n_iters non-decreasing ticks
                                   >= arrival_tick; copied at submit.  NULL in an
                                   online context (SALUS_FLAG_ONLINE, submitted
                                   before the run): the job's n_iters requests
                                   arrive live via salus_submit_requests      */
  /* Migration (NEXT-4): resume a job another context ran for resume_iter
   * iterations.  resume_state (host, copied at submit) is the image that
   * context's salus_read_state returned for a job of identical kind, dims and
   * batch (resume_bytes must equal it); it replaces the weight
   * initialisation, and this context's iteration k is the job's iteration
   * resume_iter + k (data generation, A29).  NULL = a fresh job.  Needs a
   * swap area (salus_set_swap). */
  const void *resume_state;
  uint64_t resume_bytes;
  uint32_t resume_iter;
  uint32_t _reserved;
} salus_job;

/* Footprint of a job in the device layout, so a
 * caller can declare P_i/E_i >= it.  Host-only; no context needed. */
int salus_job_footprint(const salus_job *job, uint64_t *persistent_bytes,
                        uint64_t *ephemeral_bytes);

/* Copy a job into the context.  Only before salus_prepare (else E_STATE).
 * Errors: E_INVAL (shape/ticks/declared size below footprint), E_DUPLICATE,
 * E_UNSCHEDULABLE (p + e > Cp, A22), E_CAPACITY (max_jobs / dump_bytes). */
int salus_submit_job(salus_ctx *ctx, const salus_job *job);

/* Device scratch ("meta") the context needs for the submitted jobs: job
 * tables, page tables, free-page stack, lane slots, task ring, log, stats,
 * dump area.  Valid after the last submit. */
int salus_meta_bytes(const salus_ctx *ctx, uint64_t *bytes);

/* Bytes of pinned host memory the swap area needs -- one fixed region per
 * job, the size of its persistent device backing (salus_job_footprint) --
 * when the context uses one: SALUS_FLAG_EVICT, or
 * a job with SALUS_DUMP_STATE or resume_state (migration, NEXT-4); else 0.
 * Valid after the last submit. */
int salus_swap_bytes(const salus_ctx *ctx, uint64_t *bytes);

/* Bind the caller-owned swap area: page-locked host memory (cudaHostAlloc /
 * torch pin_memory; with unified addressing the kernel reads and writes it
 * directly), >= salus_swap_bytes, 256-byte aligned, outliving the context.
 * Before salus_prepare.  Errors: E_STATE (after prepare, or no swap area needed),
 * E_INVAL (alignment / not device-accessible), E_CAPACITY (too small).
 * salus_prepare fails with E_STATE if EVICT needs a swap area and none was set. */
int salus_set_swap(salus_ctx *ctx, void *host, uint64_t bytes);

/* Migration (NEXT-4): after a run, copy the persistent state image of a job
 * submitted with SALUS_DUMP_STATE (as it stood when its last iteration
 * ended) into buf (host); *n = bytes (the job's persistent backing; pass
 * buf = NULL to query).  Errors: E_STATE (no run yet), E_INVAL (unknown job,
 * no SALUS_DUMP_STATE), E_CAPACITY (cap_bytes too small). */
int salus_read_state(salus_ctx *ctx, uint32_t job_id, void *buf, uint64_t cap_bytes, uint64_t *n);

/* Bind the caller-owned device buffer `meta` (>= salus_meta_bytes, 256-byte
 * aligned) and upload the job tables on cfg.stream (host->device copies).
 * After this no more jobs can be submitted. Errors: E_STATE, E_CAPACITY, E_CUDA. */
int salus_prepare(salus_ctx *ctx, void *meta, uint64_t meta_bytes);

/* Run the whole trace once: launch the persistent kernel on cfg.stream and
 * wait for it (device-resident scheduler: no host round-trip per iteration).
 * Every call is an independent, deterministic replay of the submitted jobs
 * from an empty GPU.  `stats` (host, may be NULL) receives one record per
 * job in submission order, *n_stats the count.  Errors: E_STATE (not
 * prepared), E_CAPACITY (log/ring overflow), E_STUCK, E_TIMEOUT, E_CUDA. */
typedef struct {
  uint32_t job_id;
  uint32_t first_lane;        /* lane the job was admitted to (one for life, I6) */
  int64_t  admit_tick;
  int64_t  first_start_tick;
  int64_t  completion_tick;   /* JCT = completion_tick - arrival_tick            */
  uint64_t completion_seq;    /* dispatch seq of its final iteration (A25)       */
  uint64_t wall_start_ns;     /* globaltimer at its first tile start              */
  uint64_t wall_end_ns;       /* globaltimer at its last tile end                 */
  uint64_t wall_arrive_ns;    /* globaltimer when the scheduler processed its
                                 arrival (for a live job: ~when it was seen)      */
} salus_job_stat;

int salus_run(salus_ctx *ctx, salus_job_stat *stats, uint64_t max_stats, uint64_t *n_stats);

/* ---------------------------------------------------------------------
 * Online submission (SALUS_FLAG_ONLINE, the paper's
 * "a session is created when a job is submitted").
 *
 * salus_run = salus_run_async + salus_wait.  Between the two, on the thread
 * that owns ctx or any other, salus_submit_live hands the running kernel a
 * new TRAIN job: the host writes its device descriptor into a reserved slot
 * (cudaMemcpy on a private stream) and publishes it through mapped pinned
 * memory; the device scheduler notices it at a tick t once every job known
 * before has arrived, and gives it arrival tick t + 1 (logged as
 * JOB_QUEUED), so replaying the logged arrival ticks through the oracle
 * reproduces the whole log.  Live job ids must exceed every earlier id;
 * their dumps come out of cfg.dump_bytes; the descriptor is copied.  Errors: E_STATE (not running /
 * not online / submissions ended), E_INVAL, E_DUPLICATE, E_UNSCHEDULABLE,
 * E_CAPACITY (max_jobs or the reserved page-table / ring space).
 * salus_end_submissions lets the kernel exit once every job is done.
 * salus_wait has salus_run's outputs and errors.
 * ------------------------------------------------------------------- */
int salus_run_async(salus_ctx *ctx);
int salus_submit_live(salus_ctx *ctx, const salus_job *job);
int salus_end_submissions(salus_ctx *ctx);
int salus_wait(salus_ctx *ctx, salus_job_stat *stats, uint64_t max_stats, uint64_t *n_stats);

/* Live inference requests (online contexts; wall-clock arrival of the
 * paper's low-rate inference requests, A27: one request = one
 * iteration).  An INFER job submitted before the run with request_ticks =
 * NULL receives its n_iters requests while the kernel runs:
 * salus_submit_requests appends n job ids (host array, copied) to a mapped
 * pinned request ring and publishes them with one 8-byte store (count and
 * last entry, so a batch of one costs the device a single PCIe read); the device
 * scheduler polls the ring (every tick while idle, every 8 ticks while
 * busy), gives every request it finds at tick t the arrival tick t + 1 (as
 * A34 does for live jobs) and stamps the globaltimer it saw it at.  The
 * log is then that of an offline trace with those request ticks, which is
 * the parity check.  Thread-safe.  Errors: E_STATE (nothing running,
 * submissions ended), E_INVAL (unknown job, not a live-request job),
 * E_CAPACITY (more requests than the job's n_iters).  The run ends once
 * every job -- a live-request job after its n_iters-th request -- is done
 * and salus_end_submissions was called.
 *
 * salus_read_requests: after salus_wait, the job's request ticks (arrival
 * tick of request k; live: as assigned) and, for live requests, the
 * globaltimer at which the scheduler saw request k (0 for offline
 * requests).  Either buffer may be NULL; *n = requests (n_iters). */
int salus_submit_requests(salus_ctx *ctx, const uint32_t *job_ids, uint32_t n);
int salus_read_requests(salus_ctx *ctx, uint32_t job_id, int64_t *ticks, uint64_t *seen_ns, uint64_t cap,
                        uint64_t *n);

/* Streaming statistics: while a salus_run_async is in
 * flight, copy the per-job records as they stand (host `stats`, submit
 * order, like salus_run) over a private non-blocking stream, concurrently
 * with the running kernel.  *n_done (may be NULL) = jobs whose last
 * iteration has physically completed (wall_end_ns != 0); their records are
 * final.  Records of unfinished jobs are partial (-1 / 0 where not yet set);
 * salus_run_async resets every record to that state on cfg.stream before the
 * kernel starts, and the poll's copy is ordered after that reset, so a poll
 * never returns a previous run's records.
 * Errors: E_STATE (nothing running), E_CUDA. */
int salus_poll_stats(salus_ctx *ctx, salus_job_stat *stats, uint64_t max_stats, uint64_t *n_stats,
                     uint64_t *n_done);

/* Whole-run counters of the last salus_run. */
typedef struct {
  uint64_t n_dispatch;        /* iterations executed                              */
  uint64_t n_ticks;           /* scheduler ticks processed                        */
  uint64_t n_log;             /* log records written                              */
  uint64_t n_tasks;           /* 128-row tiles executed by workers (per CTA half) */
  uint64_t kernel_ns;         /* CUDA-event time of the persistent kernel         */
  uint64_t wall_first_ns, wall_last_ns;   /* globaltimer at kernel start / end   */
  uint64_t sched_wait_ns;     /* scheduler time spent waiting for iterations      */
  int32_t  status;            /* SALUS_OK or the device error code               */
  uint32_t n_workers;         /* worker CTA pairs                                 */
  uint64_t h2d_bytes;         /* host->device bytes of salus_prepare (job tables)
                                 plus this run's reset image of the per-job records */
  uint64_t d2h_bytes;         /* device->host bytes read back by salus_run        */
  uint64_t sched_fence_ns;    /* part of sched_wait_ns: page-reuse fences (A30)    */
  uint64_t sched_ring_ns;     /* part of sched_wait_ns: a lane's dispatch ring full */
  uint64_t n_swap_out, n_swap_in;   /* SALUS_FLAG_EVICT: swap records executed     */
  uint64_t swap_bytes;        /* bytes copied by them (device <-> pinned host)     */
  uint64_t swap_ns;           /* sum of their durations (first tile start -> last
                                 tile end, globaltimer)                           */
} salus_run_stats;

int salus_read_run_stats(const salus_ctx *ctx, salus_run_stats *out);

/* Copy the canonical log of the last run (SALUS_FLAG_LOG) into buf (host).
 * *n_bytes = bytes written.  E_CAPACITY if cap_bytes is too small. */
int salus_read_log(salus_ctx *ctx, void *buf, uint64_t cap_bytes, uint64_t *n_bytes);

/* Copy the wall stamps (salus_wall_rec, in dispatch-seq order). */
int salus_read_wall(salus_ctx *ctx, salus_wall_rec *buf, uint64_t cap_recs, uint64_t *n_recs);

/* Dumped fp32 data of a job submitted with `dump`:
 *   iter <  n_iters   : A_L of that iteration/request, batch x d_L row-major
 *   iter == 0xFFFFFFFF: final weights W_1..W_L concatenated, each
 *                       d_{l-1} x d_l row-major (Z = A W orientation)
 *                       (SALUS_DUMP_WEIGHTS or SALUS_DUMP_WEIGHT_STEPS)
 *   iter == 0x80000000 | k (k < n_iters, SALUS_DUMP_WEIGHT_STEPS): the
 *                       weights after iteration k, same layout
 * *n = floats written.  E_INVAL if the job did not dump that item. */
int salus_read_layers(salus_ctx *ctx, uint32_t job_id, uint32_t iter, float *buf,
                      uint64_t cap_floats, uint64_t *n);

/* Per-tile device trace of the last run (SALUS_FLAG_TRACE): which SM ran
 * which tile of which iteration, with globaltimer stamps.  Records are in
 * completion order; *n_recs = records written (<= trace_capacity). */
typedef struct {
  uint32_t task;              /* slot << 26 | stage << 21 | tile                  */
  uint32_t smid;
  uint32_t job;               /* dense job index                                  */
  uint32_t iter;
  uint64_t t_claim;           /* task claimed (after the ring wait)               */
  uint64_t t_ready;           /* decoded + operand pages translated               */
  uint64_t t_mma;             /* accumulator ready (GEMM) / = t_ready otherwise    */
  uint64_t t_end;             /* epilogue stores done                             */
} salus_trace_rec;

int salus_read_trace(salus_ctx *ctx, salus_trace_rec *buf, uint64_t cap_recs, uint64_t *n_recs);

/* Page hand-offs of the last run (SALUS_FLAG_CHECK; "pages
 * of a closed / shrunk lane or a finished job are re-handed out only after
 * the previous owner's last iteration completed").  One record per page the
 * free-page pool handed to lane slot `to` (logical lane `to_lane`) while it
 * was still fenced on another slot's record: the page's last user was slot
 * `from`, record `from_seq` (physical record seq); every record lane
 * `to_lane` runs from physical seq `to_seq` on may use the page.  With the run's wall stamps
 * (salus_read_wall; physical seq = logical seq without SALUS_FLAG_EVICT) a
 * test checks that each such record starts after `from_seq` ended.  Up to
 * 1 << 20 records; *n_recs = records written. */
typedef struct {
  uint32_t page, to, from;    /* page; target and source lane slots               */
  uint32_t to_lane;           /* logical lane id of the target (wall records' lane) */
  uint64_t from_seq, to_seq;
} salus_handoff_rec;

int salus_read_handoffs(salus_ctx *ctx, salus_handoff_rec *buf, uint64_t cap_recs, uint64_t *n_recs);

const char *salus_last_error(const salus_ctx *ctx);

/* Release the host context (NULL-safe).  Never frees caller buffers.
 * Returns SALUS_E_TIMEOUT without freeing anything if a salus_wait found the
 * kernel still running 20 s after the abort request (the context is
 * "poisoned": the kernel may still touch the mapped flags and the caller's
 * arena/meta/swap, so the caller must keep those alive too and reset the
 * device). */
int salus_close(salus_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif /* SALUS_H_ */
