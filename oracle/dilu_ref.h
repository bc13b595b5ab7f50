/*
 * dilu_ref.h -- CPU ORACLE for the Dilu introspective-elasticity provisioning loop.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2503_05130_b200/, include/dilu.h) never links, imports or calls it, and
 * shares no code, header, table or helper with it.
 *
 * What it computes: SURVEY.md s8(c) steps 1-10, which restate the paper's
 *   - Algorithm 1 ScheduleInstances / SelectOptGPU   (s3.3)
 *   - Principle 1-3 (affinity first, best-fit / LLM worst-fit, Omega/gamma caps)
 *                                                     (s3.3)
 *   - slot-level reading of Algorithm 2 IssueToken    (s3.4.1)
 *   - lazy scale-out/in on a 40 s window              (s3.4.2)
 *   - the SVR / CSC / fragmentation / throughput tallies
 * in integer quota units, one plain loop per step, in the
 * paper's order.  Readings of silent/ambiguous passages are DESIGN.md s3 (Q1-Q27).
 *
 * Struct layouts are declared here independently of include/dilu.h: both are a flat
 * sequence of int32 fields in the order the seeded input generator (dilu_inputs/)
 * writes, so the same numpy buffers feed both sides.
 */
#ifndef DILU_REF_H
#define DILU_REF_H
#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  REF_OK = 0, REF_E_USAGE = 1, REF_E_INVARIANT = 2, REF_E_IO = 3,
  REF_E_CUDA = 4, REF_E_STATE = 5, REF_E_CAPACITY = 6
};

#define REF_NT 17  /* tally vector length */

typedef struct {
  int32_t n_scenarios, gpus_per_scenario, max_funcs, max_instances;
  int32_t q_pm, mem_mib, omega_pm, gamma_pm, alpha_w, beta_w, slot_ms;
  int32_t window_s, phi_out, phi_in, min_instances, max_residents, max_llm_stages;
  int32_t n_patterns, pattern_len, flags;  /* bit0 LLM split, bit1 invariants, bit2 Alg.2 5 ms, bit3 latency */
} ref_config;

/* mode: 0 Dilu, 1 Exclusive, 2 StaticLimit (MPS-l), 3 StaticRequest (MPS-r),
 * 4 EagerHorizontal (FaST-GS+-like) -- baseline modes */
typedef struct { int32_t scenario_id, omega_pm, gamma_pm, mode; } ref_scenario;

typedef struct {
  int32_t kind, prio, ibs, req_pm, lim_pm, mem_mib, work_per_batch, n_workers;
  int32_t duty_pm, cold_slots, affinity_class, arrive_sec, depart_sec;
  int32_t pattern, scale_q10, phase_slots;
} ref_func;

typedef struct ref_sim ref_sim;

/* whole-loop API (mirrors the product C-ABI shape under a dilu_ref_ prefix) */
int32_t dilu_ref_create(const ref_config* cfg, const ref_scenario* scen /* [S] or NULL */,
                        const ref_func* funcs /* [S*F] */, const int32_t* patterns,
                        ref_sim** out);
int32_t dilu_ref_place_batch(ref_sim* s, int32_t n_req, const int32_t* req_scenario,
                             const int32_t* req_func, int32_t* out_gpu, int32_t* out_iid);
int32_t dilu_ref_scale_step(ref_sim* s, int32_t n_slots, int32_t n_threads);
int32_t dilu_ref_metrics(ref_sim* s, int64_t* per_scenario /* [S][17] or NULL */, int64_t* sum /* [17] */);
int32_t dilu_ref_snapshot(ref_sim* s, int32_t id_cap, int32_t* gpu /* [S][G][4] */,
                          int32_t* inst /* [S][id_cap][12] */);
int32_t dilu_ref_slot(const ref_sim* s);
/* last simulated slot of one scenario: a[id][stage] allocated tokens, r[id]
 * dispatched requests, exec[g] executed tokens (0 for cold / idle). */
int32_t dilu_ref_slot_detail(ref_sim* s, int32_t scenario, int32_t id_cap, int64_t* a,
                             int32_t* r, int64_t* exec);
const char* dilu_ref_last_error(const ref_sim* s);
void dilu_ref_destroy(ref_sim* s);

/* ---- request-level latency (cfg.flags bit3) ----
 * Per scenario a latency vector of REF_NLAT int64: [0, 79) log-spaced histogram of
 * request latencies in microseconds (bucket of L: L < 4 -> L; else 4*h + next two
 * bits - 4, h = floor(log2 L), capped at 78), [79] requests never served in their slot
 * (no warm instance, or beyond the executed batches), [80] latency-SLO violations
 * (latency > SLO, plus every unserved request), [81] sum of served latencies
 * (us).  Readings DESIGN.md D10. */
#define REF_NLAT 82
#define REF_LAT_UNSERVED 79
int32_t dilu_ref_latency(ref_sim* s, int64_t* per_scenario /* [S][82] or NULL */,
                         int64_t* sum /* [82] */);
int32_t dilu_ref_lat_bucket(int64_t L);
/* one instance-slot: r requests arriving at floor(j*T/r), ceil(r/IBS) batches of which
 * the first b execute back to back, each taking e us from max(its last member's
 * arrival, the previous completion); adds into lat[REF_NLAT]. */
void dilu_ref_instance_latency(int64_t r, int64_t ibs, int64_t b, int64_t e, int64_t slo_us,
                               int64_t T_us, int64_t* lat);

/* ---- literal Algorithm 2 at 5 ms periods (cfg.flags bit2) ----
 * Alg.2 IssueToken run per GPU every period ("periodically
 * (e.g., 5ms)"), with SPEC's vscaler drain and divisor clamp.
 * Readings (D8): tokens = kernel blocks = per-mille-ms; MaxTokens = 5000 per
 * 5 ms period; eta_violation = 300 per-mille, eta_increase = 5/4 with a ceiling and a
 * floor of 1 token, RW = 20 periods; KLC T in microseconds. */
#define REF_A2_PERIOD_MS 5
#define REF_A2_MAX_TOKENS 5000
#define REF_A2_ETA_V 300
#define REF_A2_RW 20
enum { REF_A2_NONE = 0, REF_A2_EMERGENCY = 1, REF_A2_RECOVERY = 2, REF_A2_CONTENTION = 3 };
typedef struct {             /* one stage resident's Alg.2 inputs that persist */
  int32_t t_cur, t_min;      /* T_current, T_min: last / minimum recorded KLC (us), 0 = none */
  int32_t r_last;            /* R_last: tokens issued in the previous period */
  int32_t last_exec;         /* last absolute period with R_current > 0 (sum RW == 0 test) */
} ref_a2_res;
typedef struct { int32_t state, owner, owner_dt; } ref_a2_gpu;   /* per-GPU "state" */
/* NP periods of one GPU row for one slot.  Inputs per warm resident (any order):
 * prio (0 SLO-sensitive), instance id, per-period request / limit tokens, the slot's
 * demand d (queued at the slot start), batch size cst (SLO residents; 0 = no KLC).
 * p0 = absolute index of the slot's first period.  exec_out[k] = tokens executed in
 * the slot; grant_trace[p*n + k] (optional) = R_issue per period. */
void dilu_ref_alg2_row(int32_t n, const int32_t* prio, const int32_t* id, const int32_t* req_p,
                       const int32_t* lim_p, const int64_t* d, const int32_t* cst, int32_t NP,
                       int32_t p0, ref_a2_res* rs, ref_a2_gpu* gs, int64_t* exec_out,
                       int32_t* grant_trace);

/* unit steps, exported so tests can pin each one on its own; the loop above calls
 * exactly these functions */
uint64_t dilu_ref_mix(uint64_t scn, uint64_t t, uint64_t i, uint64_t g, uint64_t a);
int64_t dilu_ref_cap1(int32_t slot_ms, int32_t req_pm, int32_t c_b, int32_t ibs);
int32_t dilu_ref_select_opt_gpu(int32_t n_cand, const int32_t* cand, const int32_t* R,
                                const int32_t* L, const int32_t* U, const int32_t* nres,
                                int32_t req, int32_t lim, int32_t mem, int32_t omega_u,
                                int32_t gamma_u, int32_t M, int32_t Q, int32_t a, int32_t b);
void dilu_ref_vertical_row(int32_t n, const int32_t* prio, const int32_t* id,
                           const int64_t* req_tok, const int64_t* lim_tok, const int64_t* d,
                           int64_t T_slot, int64_t* a_out);
int32_t dilu_ref_scaling_decision(int32_t W, const int32_t* window, int32_t n, int64_t cap1,
                                  int32_t phi_out, int32_t phi_in, int32_t min_instances,
                                  int32_t* k_out);
int32_t dilu_ref_llm_split(int32_t n_gpu, const int32_t* active, const int32_t* R,
                           const int32_t* L, const int32_t* U, const int32_t* nres,
                           const int32_t* excluded, int32_t req, int32_t lim, int32_t mem,
                           int32_t omega_u, int32_t gamma_u, int32_t M, int32_t max_stages,
                           int32_t* out_g, int32_t* out_share);

/* ---- batched profiler (PAPER.md:604-639 s3.2) ----
 * dilu_ref_profile.c.  fp64 throughout (the paper fixes no precision); no FMA
 * contraction (built with -ffp-contract=off) so every rounding is the plain IEEE one. */
typedef struct {
  int32_t kind;        /* 0 inference (Hybrid Growth Search), 2 training (bisection)     */
  int32_t workers;     /* training: data-parallel workers                                 */
  int32_t ibs_max;     /* inference: largest IBS of the doubling grid (32: 6 levels)      */
  int32_t reserved;
  double a_ms, b_ms, knee_c;   /* inference latency model                    */
  double knee_t, t_max, idle;  /* training throughput model                  */
  double slo_ms, smr_step;     /* inference: SLO (t_exec budget SLO/2), SMR growth */
  double p_req, p_lim, tol;    /* training: p = 0.8 / 1.0, +-2 %              */
} ref_prof_session;
typedef struct {
  double request_smr, limit_smr;   /* SM rate in percent                                 */
  double t_exec_ms;                /* inference: exec time at <IBS, request>; training: T1 */
  int32_t ibs, trials;             /* chosen IBS (inference), perfmodel evaluations        */
  int32_t req_pm, lim_pm;          /* Q25 loader rounding of the two quotas                */
  int32_t status, reserved;        /* 0 ok, 1 SLO unattainable, 2 non-monotone oracle      */
} ref_prof_out;
double dilu_ref_infer_exec_ms(const ref_prof_session* m, int32_t ibs, double smr);
double dilu_ref_train_tput(const ref_prof_session* m, double smr);
void dilu_ref_profile_one(const ref_prof_session* in, ref_prof_out* out);
void dilu_ref_profile_batch(int32_t n, const ref_prof_session* in, ref_prof_out* out);

/* ---- profile-table loader ----------
 * dilu_ref_load.c.  One catalogue row + its profiling result -> one 16-int32 function row
 * (field order of dilu_inputs.FUNC_FIELDS), readings Q25 and R4 of DESIGN.md s3. */
typedef struct {
  int32_t kind, prio, n_workers, duty_pm;
  int32_t affinity_class, arrive_sec, depart_sec;
  int32_t pattern, scale_q10, phase_slots;
  int32_t reserved[2];
  double mem_gb, cold_ms, slo_ms;
} ref_catalog_row;
int32_t dilu_ref_load_one(const ref_catalog_row* c, const ref_prof_out* p, int32_t slot_ms,
                          int32_t* row16);
void dilu_ref_load_batch(int32_t n, const ref_catalog_row* c, const ref_prof_out* p,
                         int32_t slot_ms, int32_t* rows16, int32_t* status);

#ifdef __cplusplus
}
#endif
#endif
