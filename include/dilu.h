/*
 * dilu.h -- C-ABI of libdilu.so, the B200 (sm_100a) implementation of the batched
 * Dilu introspective-elasticity provisioning loop (arXiv 2503.05130).
 *
 * One handle simulates n_scenarios independent synthetic clusters ("scenarios")
 * slot by slot.  Each slot does:
 *   - at second boundaries: window push, departures, lazy horizontal scaling
 *     (s3.4.2), function arrivals, and one FIFO placement pass
 *     of Algorithm 1 (s3.3) with Principle 1-3;
 *   - every slot: arrivals and dispatch, token-based vertical scaling -- request
 *     floor plus the spare shared up to each limit, SLO-sensitive first
 *     (slot-level reading of Algorithm 2, s3.4.1) -- the gang
 *     minima of training jobs (barrel effect) and the metric fold.
 * All quantities are integers (R1-R8 in DESIGN.md s3); outputs are bit-exact and
 * independent of launch shape, device count and run.
 *
 * Conventions
 *   - Every call returns dilu_status; no C++ exception crosses this boundary.
 *   - "d_" pointers are device memory on the handle's device; "h_" pointers are
 *     host memory read only during the call.  dilu_metrics accepts either kind.
 *   - The workspace is caller-owned (e.g. a torch uint8 tensor) of at least
 *     dilu_workspace_bytes(cfg) bytes, 256-byte aligned; the handle borrows it until
 *     dilu_sim_destroy.  The stream is caller-owned (cudaStream_t, may be 0).
 *   - A handle is not thread-safe; handles are independent of each other.
 *   - Capacity exhaustion of a placement is a per-request result (-1), not an error.
 *   - Launches are stream-ordered and asynchronous except dilu_metrics and
 *     dilu_snapshot, which synchronise the stream and surface deferred errors.
 */
#ifndef DILU_H
#define DILU_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t dilu_status;
enum {
  DILU_OK = 0,
  DILU_E_USAGE = 1,      /* invalid argument / validation failure (SPEC exit 1)      */
  DILU_E_INVARIANT = 2,  /* debug invariant check failed (SPEC exit 2)                      */
  DILU_E_IO = 3,         /* reserved (SPEC exit 3)                                          */
  DILU_E_CUDA = 4,       /* CUDA launch / runtime error                                     */
  DILU_E_STATE = 5,      /* call out of order, or handle already failed                     */
  DILU_E_CAPACITY = 6    /* live instances of a scenario exceeded cfg.max_instances         */
};

#define DILU_NT 17  /* tally vector length */
enum {
  DILU_T_GPU_SLOTS_ACTIVE = 0,  /* sum over slots of #active GPUs (Eq.1 g_i)        */
  DILU_T_SM_UNUSED = 1,         /* sum over active GPU-slots of T_slot - executed tokens    */
  DILU_T_MEM_UNUSED = 2,        /* sum over active GPU-slots of M - U_g (MiB)               */
  DILU_T_REQ_TOTAL = 3,
  DILU_T_REQ_SERVED = 4,
  DILU_T_REQ_VIOLATED = 5,      /* capacity-SVR numerator (Q17)                             */
  DILU_T_INF_EXEC = 6,          /* executed inference tokens                                */
  DILU_T_TRAIN_PROGRESS = 7,    /* n_workers * gang minimum, summed (Q22)                   */
  DILU_T_PLACEMENTS_OK = 8,
  DILU_T_PLACEMENT_FAILURES = 9,
  DILU_T_COLD_STARTS = 10,      /* CSC (Q20)                                                */
  DILU_T_SCALE_OUT = 11,
  DILU_T_SCALE_IN = 12,
  DILU_T_LLM_SPLIT = 13,
  DILU_T_ALLOC_HASH = 14,       /* uint64 wrap-sum of mix(scn,t,i,g,a) over warm residents  */
  DILU_T_GPU_ROW_SLOTS = 15,    /* G * slots = simulated GPU-slot decisions                 */
  DILU_T_MAX_ACTIVE = 16        /* per-scenario max #active; the scenario sum adds maxima   */
};

/* Scenario-independent configuration, all integer units (R1-R5). */
typedef struct {
  int32_t n_scenarios;        /* scenarios in this handle (>= 1)                           */
  int32_t gpus_per_scenario;  /* G, 1..32767 on this implementation                        */
  int32_t max_funcs;          /* F: profile-table rows per scenario                        */
  int32_t max_instances;      /* live (placed + pending) instances per scenario            */
  int32_t q_pm;               /* SM_total in per-mille; must be 1000 (R1)                  */
  int32_t mem_mib;            /* M, memory per GPU in MiB (R2), <= 2^20                    */
  int32_t omega_pm, gamma_pm; /* defaults for Omega, gamma when scen == NULL       */
  int32_t alpha_w, beta_w;    /* integer score weights a:b = alpha:beta (R6), 0..255       */
  int32_t slot_ms;            /* slot length; divides 1000. T_slot = 1000*slot_ms tokens   */
  int32_t window_s, phi_out, phi_in, min_instances; /* 40, 20, 30, 1           */
  int32_t max_residents;      /* must be 32                                                */
  int32_t max_llm_stages;     /* 1..4                                             */
  int32_t n_patterns, pattern_len;
  int32_t flags;              /* bit0: LLM worst-fit split enabled; bit2: literal Alg.2 at */
                              /* 5 ms periods (D8) instead of   */
                              /* the slot-level grant; needs slot_ms % 5 == 0; bit3: request- */
                              /* level latency (dilu_latency, D10); bit1: device state      */
                              /* invariants I1-I3, I7 checked after every scale_step /       */
                              /* place_batch, I6 in dilu_metrics; */
                              /* a violation is reported as DILU_E_INVARIANT by dilu_metrics */
} dilu_config;

/* Per-scenario parameters (the C4 sweep varies gamma per scenario). */
typedef struct {
  int32_t scenario_id;        /* global id, feeds alloc_hash so shards sum identically     */
  int32_t omega_pm, gamma_pm;
  int32_t mode;               /* DILU_MODE_*: Dilu or a baseline      */
} dilu_scenario;

/* Baseline modes, applied per scenario to the same profile table:
 * EXCLUSIVE: every instance on its own GPU, whole-GPU grant (pass-through);
 * STATIC_LIMIT: MPS-l, request := limit, no spare sharing;
 * STATIC_REQUEST: MPS-r, limit := request;
 * EAGER_HORIZONTAL: FaST-GS+-like, MPS-l quotas and scale-out/in on the latest 1 s
 * sample instead of the lazy 40 s window.  Limit-quota modes
 * require limit <= Omega (DILU_E_USAGE otherwise). */
enum { DILU_MODE_DILU = 0, DILU_MODE_EXCLUSIVE = 1, DILU_MODE_STATIC_LIMIT = 2,
       DILU_MODE_STATIC_REQUEST = 3, DILU_MODE_EAGER_HORIZONTAL = 4 };

/* One quantised profile-table row <IBS, request, limit, memory> plus lifecycle
 * (Table 1).  kind -1 marks an unused row. */
typedef struct {
  int32_t kind;            /* 0 inference, 1 LLM inference, 2 training, -1 unused          */
  int32_t prio;            /* 0 SLO-sensitive, 1 best-effort (Alg.2 Type)           */
  int32_t ibs, req_pm, lim_pm, mem_mib;
  int32_t work_per_batch;  /* c_b tokens = req_pm * SLO_ms / 2 (R4); 0 for training        */
  int32_t n_workers;       /* n_j GPUs of a training job (Alg.1)                    */
  int32_t duty_pm;         /* training compute duty (comm idle)                     */
  int32_t cold_slots, affinity_class, arrive_sec, depart_sec;
  int32_t pattern, scale_q10, phase_slots;  /* A_f(t) = pat[p][(t+phase)%T] * scale >> 10 */
} dilu_func;

typedef struct dilu_sim dilu_sim;

/* Bytes of device workspace a handle needs for cfg (0 if cfg is invalid). */
size_t dilu_workspace_bytes(const dilu_config* cfg);

/* Create the simulated clusters: the synthetic counterpart of the paper's large-scale
 * simulation setup (s4.1: a cluster of GPUs, DL instances of training / LLM
 * inference / non-LLM inference types, one profile-table row per function).
 * Validate the inputs (first violation named in *out's last error, or on stderr if
 * *out cannot be created), copy them H->D into the workspace on the stream, and
 * initialise every scenario at slot 0 (no function registered, all GPUs inactive).
 *   cfg      host, read during the call
 *   h_scen   host [n_scenarios] or NULL (then ids 0.. and cfg's Omega/gamma)
 *   h_funcs  host [n_scenarios * max_funcs]
 *   h_patterns host int32 [n_patterns * pattern_len]
 * Errors: DILU_E_USAGE (validation, workspace too small/misaligned), DILU_E_CUDA. */
dilu_status dilu_sim_create(const dilu_config* cfg, const dilu_scenario* h_scen,
                            const dilu_func* h_funcs, const int32_t* h_patterns,
                            void* d_workspace, size_t ws_bytes, void* cuda_stream,
                            dilu_sim** out);

/* Return every scenario to slot 0 with the inputs already resident (no H->D copy). */
dilu_status dilu_sim_reset(dilu_sim* s);

/* Explicit deployment requests at the current slot (Alg.1 "Accept the deployment
 * request for F_j"): request j deploys one request of function
 * d_req_func[j] in scenario d_req_scenario[j] (a gang of n_workers for training,
 * one instance otherwise), registering the function if needed; requests are
 * enqueued in array order per scenario, then one FIFO placement pass runs over every
 * scenario's whole queue.  Outputs per request: GPU of its first instance or -1 if
 * it stays queued ("-1"), and its first instance id.  All four arrays are
 * device int32 [n_req]; n_req may be 0 (just run the pass).                        */
dilu_status dilu_place_batch(dilu_sim* s, int32_t n_req, const int32_t* d_req_scenario,
                             const int32_t* d_req_func, int32_t* d_out_gpu, int32_t* d_out_iid);

/* Advance all scenarios by n_slots slots (boundary work included): per second the lazy
 * horizontal scaler over the sliding window (s3.4.2) and Alg.1
 * placement of the queue; per slot the token-based vertical scaling
 * (Alg.2 slot reading, or the literal 5 ms periods with cfg.flags bit2) and
 * the metric fold.  Stream-ordered, no host synchronisation.  Errors: DILU_E_USAGE for
 * n_slots < 0, DILU_E_STATE after a failed call, DILU_E_CUDA on a launch error (deferred
 * DILU_E_CAPACITY surfaces at dilu_metrics). */
dilu_status dilu_scale_step(dilu_sim* s, int32_t n_slots);

/* The paper's metrics as integer tallies (PAPER.md:1147 s4.1 "Metrics": SVR, CSC,
 * throughput; P:1379 aggregate throughput = served work over occupied resources;
 * P:1436 / Fig. 13 SM and memory fragments of the active GPUs): the ratios are
 * formed on the host from these exact sums (SURVEY s8(c) "Final ratios").
 * Reduce tallies: per-scenario int64 [n_scenarios][DILU_NT] (may be NULL) and the
 * scenario sum int64 [DILU_NT] (uint64 wrap-sum for the hash, may be NULL).  Pointers
 * may be host or device (copied with cudaMemcpyDefault).  Synchronises the stream and
 * returns any deferred DILU_E_CAPACITY / DILU_E_CUDA, and with cfg.flags bit1 a failed
 * device state invariant (I1-I3, I7, checked after every scale_step / place_batch) or
 * I6 on the tallies as DILU_E_INVARIANT. */
dilu_status dilu_metrics(dilu_sim* s, int64_t* per_scenario, int64_t* sum);

/* Parity helper (off the timed path): device outputs
 *   d_gpu  int32 [n_scenarios][G][4]        = R_g, L_g, U_g, |res_g|
 *   d_inst int32 [n_scenarios][id_cap][12]  = per instance id: func, status
 *          (0 pending, 1 placed, 2 terminated, -1 never issued), n_stages,
 *          ready_slot, gpu[4], mem_share[4] (-1 / 0 when not placed).
 * Synchronises the stream. */
dilu_status dilu_snapshot(dilu_sim* s, int32_t id_cap, int32_t* d_gpu, int32_t* d_inst);

/* Diagnostics (tracing; off the timed path): per-scenario int64 [n_scenarios][24] (may
 * be NULL) and their sum [24] (may be NULL) of kernel counters accumulated since the
 * last create/reset: full placement attempts, retry-skip checks, row repacks, boundary
 * events, queue scans, slots simulated, warm resident-slots allocated, inference
 * function-slots dispatched, then 16 per-phase cycle timers (leader thread; nonzero only
 * in a -DDILU_PHASE_TIMING build).  Host or device pointers.
 * Synchronises the stream. */
dilu_status dilu_kernel_stats(dilu_sim* s, int64_t* per_scenario, int64_t* sum);

/* Request-level latency (cfg.flags bit3; "latency (e.g.,
 * p50/p95) and SLO violation rate"; D10).  Per scenario DILU_NLAT int64:
 * [0, 79) request-latency histogram in microseconds, 4 log buckets per octave (L < 4 ->
 * bucket L, else 4*floor(log2 L) + next two bits - 4, capped at 78); [79] requests not
 * served in their slot; [80] latency-SLO violations (latency > SLO = 2 * t_exec at the
 * profiled request, plus every unserved request); [81] sum of served latencies.
 * per_scenario [S][DILU_NLAT] and/or sum [DILU_NLAT], host or device pointers; syncs
 * the stream.  DILU_E_USAGE if the handle was created without bit3. */
#define DILU_NLAT 82
dilu_status dilu_latency(dilu_sim* s, int64_t* per_scenario, int64_t* sum);

/* Current slot (number of slots simulated so far). */
int32_t dilu_current_slot(const dilu_sim* s);

/* Last error message, owned by the handle, valid until the next call. */
const char* dilu_last_error(const dilu_sim* s);

/* Release the handle (not the caller-owned workspace or stream). */
void dilu_sim_destroy(dilu_sim* s);

/* ---- batched profiler: the step before the loop ------------------
 * Multi-factor profiling of PAPER.md s3.2 over SPEC's synthetic perfmodel
 * (the paper measures real GPUs): training quotas by bisection,
 * inference <IBS, SMR> by the Hybrid Growth Search, one thread per session.
 * fp64 with plain IEEE operations (no contraction); readings DESIGN.md D9.  The output
 * rows carry the Q25-rounded per-mille quotas the loop's dilu_func rows take. */
typedef struct {
  int32_t kind;        /* 0 inference (Hybrid Growth Search), 2 training (bisection)     */
  int32_t workers;     /* training: data-parallel workers (>= 1)                          */
  int32_t ibs_max;     /* inference: largest IBS of the doubling grid, 1..1024 (32 = 6 levels) */
  int32_t reserved;    /* 0 */
  double a_ms, b_ms, knee_c;   /* inference t_exec = (a + b*IBS)*knee/min(SMR, knee),     */
                               /* knee = min(100, knee_c*sqrt(IBS))            */
  double knee_t, t_max, idle;  /* training throughput = workers*t_max*min(1, SMR/knee_t)*(1-idle) */
  double slo_ms, smr_step;     /* inference: SLO (t_exec budget SLO/2), SMR step (10) */
  double p_req, p_lim, tol;    /* training: 0.8, 1.0, 0.02                     */
} dilu_prof_session;           /* 104 bytes */
typedef struct {
  double request_smr, limit_smr;   /* percent                                             */
  double t_exec_ms;                /* inference: t_exec at <IBS, request>; training: T1    */
  int32_t ibs, trials;             /* chosen IBS (0 for training); perfmodel evaluations   */
  int32_t req_pm, lim_pm;          /* ceil(10*percent), limit capped at 1000 (Q25)         */
  int32_t status, reserved;        /* 0 ok, 1 SLO unattainable, 2 non-monotone throughput  */
} dilu_prof_out;                   /* 48 bytes */

/* Profile n sessions: d_sessions[n] in, d_out[n] out (device memory, 8-byte aligned),
 * stream-ordered and asynchronous on cuda_stream.  Returns DILU_E_USAGE for n < 0 or
 * null pointers with n > 0, DILU_E_CUDA on a launch error; per-session failures are
 * d_out[i].status, not call errors.  No handle needed. */
dilu_status dilu_profile(const dilu_prof_session* d_sessions, int32_t n, dilu_prof_out* d_out,
                         void* cuda_stream);

/* ---- profile-table loader: profiled tuples -> quantised rows --------
 * PAPER.md s3.2 (Table 1 <IBS, request, limit, memory>; P:628 training
 * request/limit at 80 % / 100 % of full throughput; P:634-637 inference request = the
 * profiled SMR meeting SLO/2, limit = 2 x request).  One catalogue row per function plus
 * the dilu_prof_out of its profiling session give one dilu_func row; readings Q25 and R4
 * (DESIGN.md s3): req_pm / lim_pm are the session's Q25-rounded quotas, ibs the profiled
 * IBS (inference), mem_mib = ceil(1024 * mem_gb), cold_slots = ceil(cold_ms / slot_ms),
 * c_b = floor(req_pm * slo_ms / 2) tokens (R4; 0 for training), each ceil taken of the
 * fp64 value minus 1e-9 (so exact decimal inputs are not pushed up by representation
 * error).  The remaining fields are copied.  The rows then go to dilu_sim_create, which
 * validates them (R1, R4, Q12, Q23, lifecycle). */
typedef struct {
  int32_t kind;            /* 0 inference, 1 LLM inference, 2 training                     */
  int32_t prio;            /* 0 SLO-sensitive, 1 best-effort                               */
  int32_t n_workers;       /* training: data-parallel workers; inference: ignored (1)     */
  int32_t duty_pm;         /* training compute duty; inference: ignored            */
  int32_t affinity_class, arrive_sec, depart_sec;
  int32_t pattern, scale_q10, phase_slots;
  int32_t reserved[2];     /* 0 */
  double mem_gb;           /* memory footprint in GB (Table 1 "memory")                    */
  double cold_ms;          /* cold-start latency in ms                                      */
  double slo_ms;           /* inference SLO in ms; training: ignored                        */
} dilu_catalog_row;        /* 72 bytes */

/* Load n rows: d_cat[n] and d_prof[n] (the dilu_profile output of row i's session) in,
 * d_out[n] rows and d_status[n] out, all device memory; stream-ordered and asynchronous.
 * d_status[i]: 0 loaded; 1 the session's profile failed (status != 0) -> row written as
 * unused (kind -1); 2 catalogue row invalid (kind out of range, kind and session disagree
 * (inference vs training), non-finite or negative mem/cold/slo) -> unused.  Returns
 * DILU_E_USAGE for n < 0, slot_ms outside 1..1000 or null pointers with n > 0,
 * DILU_E_CUDA on a launch error. */
dilu_status dilu_load_profiles(const dilu_catalog_row* d_cat, const dilu_prof_out* d_prof,
                               int32_t n, int32_t slot_ms, dilu_func* d_out, int32_t* d_status,
                               void* cuda_stream);

#ifdef __cplusplus
}
#endif
#endif /* DILU_H */
