/*
 * dilu_ref.c -- CPU ORACLE (test infrastructure only; see dilu_ref.h).
 *
 * A plain, slow, literal implementation of SURVEY.md s8(c) steps 0-10.  Every
 * function cites the passage it follows: P:n = /root/reference/PAPER.md line n,
 * S:n = SPEC.md line n, Rn / Qn = the unit rules and readings restated in
 * DESIGN.md s3.  No blocking, fusion or reordering: each step is a loop over the
 * objects the paper names, in the paper's order.  One scenario runs on one thread;
 * independent scenarios may run on a pthread pool ("Multiple independent
 * runs ... may execute in parallel").
 *
 * Parity pins live in tests/test_oracle_*.py (Appendix A worked example, SPEC
 * examples, exact-rational brute force, lexicographic-max brute force, invariants).
 */
#include "dilu_ref.h"

#include <pthread.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

enum { K_UNUSED = -1, K_INF = 0, K_LLM = 1, K_TRAIN = 2 };
enum { ST_PENDING = 0, ST_PLACED = 1, ST_TERMINATED = 2 };
enum { M_DILU = 0, M_EXCLUSIVE = 1, M_STATIC_LIMIT = 2, M_STATIC_REQUEST = 3, M_EAGER = 4 };
enum {
  T_GPU_SLOTS_ACTIVE = 0, T_SM_UNUSED, T_MEM_UNUSED, T_REQ_TOTAL, T_REQ_SERVED,
  T_REQ_VIOLATED, T_INF_EXEC, T_TRAIN_PROGRESS, T_PLACEMENTS_OK, T_PLACEMENT_FAILURES,
  T_COLD_STARTS, T_SCALE_OUT, T_SCALE_IN, T_LLM_SPLIT, T_ALLOC_HASH, T_GPU_ROW_SLOTS,
  T_MAX_ACTIVE
};
#define MAX_STAGES 4
#define RES_CAP 32

/* ------------------------------------------------------------------ state */

typedef struct {              /* instance i (SURVEY s8(c) "State") */
  int32_t func, status, nst, ready, r;
  int32_t g[MAX_STAGES], share[MAX_STAGES];
  int64_t a[MAX_STAGES];      /* tokens allocated this slot, per stage (step 7) */
  int64_t loc[MAX_STAGES];    /* row-local capacity: b_g (INF/LLM) or x (TRAIN)   */
  int32_t warm;               /* placed && ready <= t, evaluated this slot        */
  ref_a2_res a2[MAX_STAGES];  /* Alg.2 per-stage state (flags bit2), from commit */
} RInst;

typedef struct {              /* GPU g: R_g, L_g, U_g, res_g (Alg.1)   */
  int32_t R, L, U, nres;
  int32_t res[RES_CAP];       /* instance ids (stage residents); unsorted set    */
  int64_t exec;               /* sum of executed tokens this slot (step 8)       */
  ref_a2_gpu a2;              /* Alg.2 "state" of this GPU (flags bit2)          */
} RGpu;

typedef struct {              /* function f: registration, window, live list     */
  int32_t registered, nsamp, rps_acc, head;
  int32_t* ring;              /* W per-second samples ("sliding window")   */
  int32_t* live;              /* ascending live instance ids                     */
  int32_t nlive, cap_live;
} RFunc;

typedef struct { int32_t func, first, n; } RReq;  /* request: gang of n ids      */

typedef struct {
  const ref_config* cfg;
  const ref_func* fn;          /* this scenario's function rows [F]              */
  const int32_t* pat;
  int32_t scn_id, omega_u, gamma_u, mode;
  RGpu* gpu;                   /* [G] */
  RFunc* fs;                   /* [F] */
  RInst* inst;                 /* indexed by instance id */
  int32_t n_ids, cap_ids, n_live;
  RReq* q; int32_t nq, cap_q;  /* FIFO queue (Q9) */
  int64_t tally[REF_NT];
  int64_t lat[REF_NLAT];       /* request-level latency vector (flags bit3) */
  int64_t* slo_us;             /* [F] SLO of each inference function (D10) */
  int32_t err;
  char msg[200];
} RScen;

struct ref_sim {
  ref_config cfg;
  int32_t S, t;
  ref_func* funcs;
  int32_t* patterns;
  RScen* sc;
  int32_t status;
  char err[256];
};

static void* xcalloc(size_t n, size_t sz) {
  void* p = calloc(n ? n : 1, sz);
  if (!p) { fprintf(stderr, "dilu_ref: out of memory\n"); abort(); }
  return p;
}

static int is_inf(int32_t kind) { return kind == K_INF || kind == K_LLM; }

/* ------------------------------------------------------------- unit rules */

/* R8: splitmix64 finaliser chain; alloc_hash is the mod-2^64 sum of these. */
static uint64_t sm64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
uint64_t dilu_ref_mix(uint64_t scn, uint64_t t, uint64_t i, uint64_t g, uint64_t a) {
  uint64_t h = sm64(scn);
  h = sm64(h ^ t);
  h = sm64(h ^ i);
  return sm64(h ^ ((g << 32) | (a & 0xFFFFFFFFull)));
}

/* R5: capacity of one instance at its request quota, in RPS:
 * (1000/slot_ms) * floor(req_tok / c_b) * IBS, req_tok = req_pm*slot_ms (R3),
 * i.e. "n*ibs/t_exec at <ibs, request>" with t_exec = SLO/2. */
int64_t dilu_ref_cap1(int32_t slot_ms, int32_t req_pm, int32_t c_b, int32_t ibs) {
  int64_t req_tok = (int64_t)req_pm * slot_ms;
  int64_t batches_per_slot = req_tok / c_b;
  return (int64_t)(1000 / slot_ms) * batches_per_slot * ibs;
}

/* ------------------------------------------------- Algorithm 1 SelectOptGPU */

/* SelectOptGPU.  For each candidate in the given (ascending) order:
 *   newReqSum = R + req, newLimSum = L + lim, newMemUsage = U + mem
 *   score = alpha(1 - newReqSum/SM_total) + beta(1 - newMemUsage/M)
 *   accept if newReqSum <= Omega and newLimSum <= gamma and newMem <= M
 *          and score < bestScore
 * plus the resident cap |res| < 32 (Q23; never binds for validated inputs).
 * The score is compared exactly (Q4, R6): with alpha:beta = a:b and SM_total = Q,
 *   score(x) < score(y)  <=>  K(x) > K(y),  K = a*newReqSum*M + b*newMemUsage*Q,
 * because score = (alpha+beta) - K/((a+b)*Q*M).  Strict comparison keeps the
 * earliest (lowest-id) candidate on ties (Q3).  Returns the GPU or -1.        */
static int32_t select_opt_gpu(int32_t n_cand, const int32_t* cand, const int32_t* R,
                              const int32_t* L, const int32_t* U, const int32_t* nres,
                              int32_t req, int32_t lim, int32_t mem, int32_t omega_u,
                              int32_t gamma_u, int32_t M, int32_t Q, int32_t a, int32_t b) {
  int32_t best = -1;
  int64_t bestK = -1;  /* score = +inf */
  for (int32_t c = 0; c < n_cand; ++c) {
    int32_t i = cand[c];
    int64_t newReqSum = (int64_t)R[i] + req;
    int64_t newLimSum = (int64_t)L[i] + lim;
    int64_t newMemUsage = (int64_t)U[i] + mem;
    int64_t K = (int64_t)a * newReqSum * M + (int64_t)b * newMemUsage * Q;
    if (newReqSum <= omega_u && newLimSum <= gamma_u && newMemUsage <= M &&
        nres[i] < RES_CAP && K > bestK) {
      bestK = K;
      best = i;
    }
  }
  return best;
}
int32_t dilu_ref_select_opt_gpu(int32_t n_cand, const int32_t* cand, const int32_t* R,
                                const int32_t* L, const int32_t* U, const int32_t* nres,
                                int32_t req, int32_t lim, int32_t mem, int32_t omega_u,
                                int32_t gamma_u, int32_t M, int32_t Q, int32_t a, int32_t b) {
  return select_opt_gpu(n_cand, cand, R, L, U, nres, req, lim, mem, omega_u, gamma_u, M, Q, a, b);
}

/* Principle 2, LLM memory worst-fit split (Q11).
 * Candidates: active GPUs not excluded with R+req <= Omega, L+lim <= gamma,
 * |res| < 32 and free memory M-U > 0.  Order them by free memory descending, then
 * id ascending ("prioritizes choosing GPUs with the most remaining memory").  Take
 * the smallest k <= max_stages whose top-k free memory covers mem ("to minimize
 * pipeline stages"); shares are a greedy fill.  Returns k, or 0 if none.       */
int32_t dilu_ref_llm_split(int32_t n_gpu, const int32_t* active, const int32_t* R,
                           const int32_t* L, const int32_t* U, const int32_t* nres,
                           const int32_t* excluded, int32_t req, int32_t lim, int32_t mem,
                           int32_t omega_u, int32_t gamma_u, int32_t M, int32_t max_stages,
                           int32_t* out_g, int32_t* out_share) {
  int32_t* cand = (int32_t*)xcalloc((size_t)n_gpu, sizeof(int32_t));
  int32_t nc = 0;
  for (int32_t g = 0; g < n_gpu; ++g) {
    if (!active[g] || (excluded && excluded[g])) continue;
    if ((int64_t)R[g] + req <= omega_u && (int64_t)L[g] + lim <= gamma_u &&
        nres[g] < RES_CAP && M - U[g] > 0)
      cand[nc++] = g;
  }
  /* plain insertion sort by (free desc, id asc) */
  for (int32_t x = 1; x < nc; ++x) {
    int32_t v = cand[x], y = x - 1;
    while (y >= 0 && ((M - U[cand[y]]) < (M - U[v]) ||
                      ((M - U[cand[y]]) == (M - U[v]) && cand[y] > v))) {
      cand[y + 1] = cand[y];
      --y;
    }
    cand[y + 1] = v;
  }
  int32_t k = 0;
  int64_t sum = 0;
  for (int32_t j = 0; j < nc && j < max_stages; ++j) {
    sum += M - U[cand[j]];
    if (sum >= mem) { k = j + 1; break; }
  }
  if (k > 0) {
    int32_t left = mem;
    for (int32_t j = 0; j < k; ++j) {
      int32_t fr = M - U[cand[j]];
      int32_t sh = fr < left ? fr : left;
      out_g[j] = cand[j];
      out_share[j] = sh;
      left -= sh;
    }
  }
  free(cand);
  return k;
}

/* ------------------------------------------- slot-level Algorithm 2 reading */

/* Vertical token allocation on one GPU row (Q13).
 * The n warm residents are visited in (prio, id) order -- SLO-sensitive (prio 0)
 * first, matching Alg. 2's protection of SLO instances -- and
 *   S_g    = T_slot - sum req_tok                 (request floor for everybody)
 *   want_i = max(0, min(d_i, lim_tok_i) - req_tok_i)
 *   s_i    = min(want_i, max(0, S_g - P_i)),  P_i = sum of want over earlier ones
 *   a_i    = req_tok_i + s_i.
 * a_out[k] is written for input position k.                                  */
void dilu_ref_vertical_row(int32_t n, const int32_t* prio, const int32_t* id,
                           const int64_t* req_tok, const int64_t* lim_tok, const int64_t* d,
                           int64_t T_slot, int64_t* a_out) {
  int32_t* ord = (int32_t*)xcalloc((size_t)n, sizeof(int32_t));
  for (int32_t k = 0; k < n; ++k) ord[k] = k;
  for (int32_t x = 1; x < n; ++x) {  /* insertion sort by (prio, id) */
    int32_t v = ord[x], y = x - 1;
    while (y >= 0 && (prio[ord[y]] > prio[v] || (prio[ord[y]] == prio[v] && id[ord[y]] > id[v]))) {
      ord[y + 1] = ord[y];
      --y;
    }
    ord[y + 1] = v;
  }
  int64_t S_g = T_slot;
  for (int32_t k = 0; k < n; ++k) S_g -= req_tok[k];
  int64_t P = 0;
  for (int32_t x = 0; x < n; ++x) {
    int32_t k = ord[x];
    int64_t cap = d[k] < lim_tok[k] ? d[k] : lim_tok[k];
    int64_t want = cap - req_tok[k];
    if (want < 0) want = 0;
    int64_t room = S_g - P;
    if (room < 0) room = 0;
    int64_t s = want < room ? want : room;
    a_out[k] = req_tok[k] + s;
    P += want;
  }
  free(ord);
}

/* ------------------------------------- literal Algorithm 2 at 5 ms periods */

/* eta_increase = 1.25 on integer tokens: ceil(max(R_last, 1) * 5 / 4) (D8: the ceiling
 * and the floor of 1 keep "gradually increased" from sticking at small R). */
static int32_t a2_grow(int32_t r_last) {
  int64_t r = r_last < 1 ? 1 : r_last;
  return (int32_t)((r * 5 + 3) / 4);
}

/* One GPU row, NP periods (Algorithm 2; P:885-902 workflow).
 * Each period, in this order:
 *  0. state bookkeeping (D8): an EMERGENCY whose owner is not a warm resident any more,
 *     or a row without SLO-sensitive residents, is NONE ("Without collocation").
 *  1. IssueToken for every SLO-sensitive resident in (prio, id) order (lines 12-24):
 *     dT = (T_current - T_min) / T_min                                    (line 13)
 *     dT > eta_violation        -> EMERGENCY, R = MaxTokens * limit        (14-15)
 *     sum(RW[current]) == 0     -> RECOVERY,  R = MaxTokens * request      (16-17)
 *     sum(RW[others]) == 0      -> RECOVERY,  R = min(R_last * eta_inc, MaxTokens * limit)
 *                                                                  (18-19; S:382 min)
 *     else                      -> CONTENTION, R = MaxTokens * request      (20-21)
 *     "Only the current instance can reset or modify the EMERGENCY state":
 *     a non-owner leaves an EMERGENCY in place; a second SLO resident tripping line
 *     14 takes ownership only with a larger dT.
 *  2. IssueToken for every best-effort resident in (prio, id) order (lines 25-38):
 *     NONE -> MaxTokens*limit; EMERGENCY -> min(MaxTokens*request, R_last) / max(dT, 1)
 *     (S:397 clamp); RECOVERY -> min(R_last*eta_inc, MaxTokens*limit); CONTENTION -> R_last.
 *  3. Kernel Redirect / drain in (prio, id) order:
 *     executed = min(pending, R_issue, MaxTokens - executed by earlier residents).
 *     RW: R_current = executed.  KLC (footnote P:899): a batch's span from the
 *     start of its first block to the end of its last block, blocks running at the
 *     resident's rate y = min(R_issue, capacity left) per 5 ms period.
 *  4. R_last = R_issue.                                                            */
void dilu_ref_alg2_row(int32_t n, const int32_t* prio, const int32_t* id, const int32_t* req_p,
                       const int32_t* lim_p, const int64_t* d, const int32_t* cst, int32_t NP,
                       int32_t p0, ref_a2_res* rs, ref_a2_gpu* gs, int64_t* exec_out,
                       int32_t* grant_trace) {
  const int64_t PT = (int64_t)REF_A2_PERIOD_MS * 1000;       /* period length in us */
  int32_t* ord = (int32_t*)xcalloc((size_t)(n ? n : 1), sizeof(int32_t));
  int64_t* pending = (int64_t*)xcalloc((size_t)(n ? n : 1), sizeof(int64_t));
  int64_t* done = (int64_t*)xcalloc((size_t)(n ? n : 1), sizeof(int64_t));
  int64_t* bstart = (int64_t*)xcalloc((size_t)(n ? n : 1), sizeof(int64_t));
  int32_t* grant = (int32_t*)xcalloc((size_t)(n ? n : 1), sizeof(int32_t));
  for (int32_t k = 0; k < n; ++k) {
    ord[k] = k;
    pending[k] = d[k];        /* the slot's kernels are queued at its start (D8) */
    done[k] = 0;              /* tokens executed in this slot */
    bstart[k] = -1;           /* start time (us, slot-relative) of the batch in progress */
  }
  for (int32_t x = 1; x < n; ++x) {  /* insertion sort by (prio, id) */
    int32_t v = ord[x], y = x - 1;
    while (y >= 0 && (prio[ord[y]] > prio[v] || (prio[ord[y]] == prio[v] && id[ord[y]] > id[v]))) {
      ord[y + 1] = ord[y];
      --y;
    }
    ord[y + 1] = v;
  }
  for (int32_t p = 0; p < NP; ++p) {
    const int32_t P = p0 + p;                                /* absolute period */
    /* 0. state bookkeeping */
    int32_t any_slo = 0, owner_here = 0;
    for (int32_t k = 0; k < n; ++k) {
      if (prio[k] == 0) any_slo = 1;
      if (id[k] == gs->owner) owner_here = 1;
    }
    if (!any_slo || (gs->state == REF_A2_EMERGENCY && !owner_here)) {
      gs->state = REF_A2_NONE;
      gs->owner = -1;
      gs->owner_dt = 0;
    }
    /* 1. SLO-sensitive residents */
    for (int32_t x = 0; x < n; ++x) {
      int32_t k = ord[x];
      if (prio[k] != 0) continue;
      ref_a2_res* r = &rs[k];
      int64_t dT = r->t_min > 0 ? ((int64_t)r->t_cur - r->t_min) * 1000 / r->t_min : 0;
      int32_t idle_self = r->last_exec < P - REF_A2_RW;
      int32_t idle_others = 1;
      for (int32_t j = 0; j < n; ++j)
        if (j != k && rs[j].last_exec >= P - REF_A2_RW) idle_others = 0;
      if (dT > REF_A2_ETA_V) {
        grant[k] = lim_p[k];
        if (gs->state != REF_A2_EMERGENCY || gs->owner == id[k] || dT > gs->owner_dt) {
          gs->state = REF_A2_EMERGENCY;
          gs->owner = id[k];
          gs->owner_dt = (int32_t)dT;
        }
      } else {
        int32_t ns;
        if (idle_self) {
          ns = REF_A2_RECOVERY;
          grant[k] = req_p[k];
        } else if (idle_others) {
          ns = REF_A2_RECOVERY;
          int32_t g2 = a2_grow(r->r_last);
          grant[k] = g2 < lim_p[k] ? g2 : lim_p[k];
        } else {
          ns = REF_A2_CONTENTION;
          grant[k] = req_p[k];
        }
        if (gs->state != REF_A2_EMERGENCY || gs->owner == id[k]) {
          gs->state = ns;
          gs->owner = -1;
          gs->owner_dt = 0;
        }
      }
    }
    /* 2. best-effort residents */
    for (int32_t x = 0; x < n; ++x) {
      int32_t k = ord[x];
      if (prio[k] == 0) continue;
      ref_a2_res* r = &rs[k];
      switch (gs->state) {
        case REF_A2_NONE: grant[k] = lim_p[k]; break;
        case REF_A2_EMERGENCY: {
          int64_t m = req_p[k] < r->r_last ? req_p[k] : r->r_last;
          int64_t div = gs->owner_dt > 1000 ? gs->owner_dt : 1000;   /* max(dT, 1) */
          grant[k] = (int32_t)(m * 1000 / div);
          break;
        }
        case REF_A2_RECOVERY: {
          int32_t g2 = a2_grow(r->r_last);
          grant[k] = g2 < lim_p[k] ? g2 : lim_p[k];
          break;
        }
        default: grant[k] = r->r_last; break;                      /* CONTENTION */
      }
    }
    if (grant_trace)
      for (int32_t k = 0; k < n; ++k) grant_trace[(int64_t)p * n + k] = grant[k];
    /* 3. drain with the physical capacity clamp, KLC */
    int64_t cap = REF_A2_MAX_TOKENS;
    for (int32_t x = 0; x < n; ++x) {
      int32_t k = ord[x];
      ref_a2_res* r = &rs[k];
      int64_t y = grant[k] < cap ? grant[k] : cap;   /* this period's rate */
      if (y < 0) y = 0;
      int64_t ex = pending[k] < y ? pending[k] : y;
      cap -= ex;
      if (ex > 0) {
        r->last_exec = P;
        if (cst[k] > 0) {
          /* tokens [a, b) of the slot run this period; token a + j occupies
           * [p*PT + j*PT/y, p*PT + ceil((j+1)*PT/y)).  Visit every batch m that has a
           * token here, in order: its start (token m*cst) and its end (token (m+1)*cst-1). */
          const int64_t a = done[k], b = done[k] + ex, c = cst[k];
          for (int64_t m = a / c; m * c < b; ++m) {
            const int64_t first = m * c, last = (m + 1) * c - 1;
            if (first >= a) bstart[k] = p * PT + (first - a) * PT / y;
            if (last < b) {
              const int64_t end = p * PT + ((last - a + 1) * PT + y - 1) / y;
              const int64_t T = end - bstart[k];
              r->t_cur = T > INT32_MAX ? INT32_MAX : (int32_t)T;     /* T_current */
              if (r->t_min == 0 || r->t_cur < r->t_min) r->t_min = r->t_cur;   /* T_min */
            }
          }
        }
      }
      pending[k] -= ex;
      done[k] += ex;
    }
    /* 4. */
    for (int32_t k = 0; k < n; ++k) rs[k].r_last = grant[k];
  }
  for (int32_t k = 0; k < n; ++k) exec_out[k] = done[k];
  free(ord); free(pending); free(done); free(bstart); free(grant);
}

/* ------------------------------------------------ request-level latency */

/* Log-spaced latency buckets, 4 per octave (D10). */
int32_t dilu_ref_lat_bucket(int64_t L) {
  if (L < 4) return (int32_t)(L < 0 ? 0 : L);
  int32_t h = 0;
  while ((L >> (h + 1)) != 0) ++h;               /* floor(log2 L) */
  int64_t b = 4 * (int64_t)h + ((L >> (h - 2)) & 3) - 4;
  return (int32_t)(b < 78 ? b : 78);
}

/* Request-level dispatch and batching inside one slot (
 * P:1147 "latency (e.g., p50/p95) and SLO violation rate"; D10):
 *   requests arrive evenly over the slot: request j at tau_j = floor(j*T/r) us;
 *   batch k holds requests [k*IBS, min((k+1)*IBS, r)) -- the slot model's ceil(r/IBS)
 *     batches (step 5) -- and is ready when its last member arrives (no SLO/2 timeout:
 *     SPEC S:513's early firing would change the batch count the capacity model fixes);
 *   the first b batches (the slot's executed batches, step 8) run back to back, each for
 *     e us: start = max(ready, previous completion), completion = start + e;
 *   a served request's latency = its batch's completion - its arrival; requests of
 *     batches >= b are unserved.                                                     */
void dilu_ref_instance_latency(int64_t r, int64_t ibs, int64_t b, int64_t e, int64_t slo_us,
                               int64_t T_us, int64_t* lat) {
  const int64_t need = (r + ibs - 1) / ibs;
  int64_t prev = 0;
  for (int64_t k = 0; k < need; ++k) {
    const int64_t j0 = k * ibs, j1 = (k + 1) * ibs < r ? (k + 1) * ibs : r;
    if (k >= b) {                                 /* not executed in this slot */
      lat[REF_LAT_UNSERVED] += j1 - j0;
      lat[80] += j1 - j0;
      continue;
    }
    const int64_t ready = (j1 - 1) * T_us / r;    /* the last member's arrival */
    const int64_t start = ready > prev ? ready : prev;
    const int64_t done = start + e;
    for (int64_t j = j0; j < j1; ++j) {
      const int64_t L = done - j * T_us / r;
      lat[dilu_ref_lat_bucket(L)] += 1;
      lat[81] += L;
      if (L > slo_us) lat[80] += 1;
    }
    prev = done;
  }
}

/* ------------------------------------------------ lazy horizontal scaling */

/* Lazy scale-out/in decision on a full window (Q18, Q19).
 *   up   = #{w > capacity(n)},   capacity(n) = n * cap1
 *   down = #{w < capacity(n-1)}
 *   "at least phi_out RPS values ... exceed"      -> up >= phi_out: ScaleOut(k),
 *        k = ceil(max w / cap1) - n, only if k >= 1
 *   "more than phi_in RPS values ... fall below"  -> down > phi_in and n > min: ScaleIn(1)
 * Returns 0 Hold, 1 ScaleOut (k in *k_out), 2 ScaleIn.                        */
int32_t dilu_ref_scaling_decision(int32_t W, const int32_t* window, int32_t n, int64_t cap1,
                                  int32_t phi_out, int32_t phi_in, int32_t min_instances,
                                  int32_t* k_out) {
  int64_t cap_n = (int64_t)n * cap1;
  int64_t cap_n1 = (int64_t)(n - 1) * cap1;
  int32_t up = 0, down = 0;
  int64_t mx = 0;
  for (int32_t j = 0; j < W; ++j) {
    if (window[j] > cap_n) ++up;
    if (window[j] < cap_n1) ++down;
    if (window[j] > mx) mx = window[j];
  }
  *k_out = 0;
  if (up >= phi_out) {
    int64_t k = (mx + cap1 - 1) / cap1 - n;
    if (k >= 1) { *k_out = (int32_t)k; return 1; }
    return 0;
  } else if (down > phi_in && n > min_instances) {
    return 2;
  }
  return 0;
}

/* ---------------------------------------------------------- bookkeeping */

static void fail(RScen* s, int32_t code, const char* fmt, ...) {
  if (s->err) return;
  s->err = code;
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(s->msg, sizeof s->msg, fmt, ap);
  va_end(ap);
}

static void live_add(RFunc* F, int32_t id) {  /* ids arrive in ascending order */
  if (F->nlive == F->cap_live) {
    F->cap_live = F->cap_live ? 2 * F->cap_live : 8;
    F->live = (int32_t*)realloc(F->live, (size_t)F->cap_live * sizeof(int32_t));
  }
  F->live[F->nlive++] = id;
}
static void live_remove(RFunc* F, int32_t id) {
  int32_t j = 0;
  while (j < F->nlive && F->live[j] != id) ++j;
  for (; j + 1 < F->nlive; ++j) F->live[j] = F->live[j + 1];
  if (F->nlive) --F->nlive;
}

/* Enqueue one request of n new instances of f; ids assigned at enqueue (Q19). */
static void enqueue(RScen* s, int32_t f, int32_t n) {
  if (s->n_live + n > s->cfg->max_instances) {
    fail(s, REF_E_CAPACITY, "scenario %d: live instances exceed max_instances=%d", s->scn_id,
         s->cfg->max_instances);
    return;
  }
  if (s->n_ids + n > s->cap_ids) {
    while (s->n_ids + n > s->cap_ids) s->cap_ids = s->cap_ids ? 2 * s->cap_ids : 256;
    s->inst = (RInst*)realloc(s->inst, (size_t)s->cap_ids * sizeof(RInst));
  }
  if (s->nq == s->cap_q) {
    s->cap_q = s->cap_q ? 2 * s->cap_q : 64;
    s->q = (RReq*)realloc(s->q, (size_t)s->cap_q * sizeof(RReq));
  }
  RReq r = {f, s->n_ids, n};
  s->q[s->nq++] = r;
  for (int32_t j = 0; j < n; ++j) {
    RInst* I = &s->inst[s->n_ids];
    memset(I, 0, sizeof *I);
    I->func = f;
    I->status = ST_PENDING;
    for (int32_t k = 0; k < MAX_STAGES; ++k) I->g[k] = -1;
    live_add(&s->fs[f], s->n_ids);
    ++s->n_ids;
    ++s->n_live;
  }
}

/* Commit one stage of instance id on GPU g (Alg.1 "Update resource info"). */
static void commit(RScen* s, int32_t id, int32_t g, int32_t share) {
  const ref_func* F = &s->fn[s->inst[id].func];
  RGpu* G = &s->gpu[g];
  G->R += F->req_pm;
  G->L += F->lim_pm;
  G->U += share;
  G->res[G->nres++] = id;
  RInst* I = &s->inst[id];
  I->g[I->nst] = g;
  I->share[I->nst] = share;
  ref_a2_res fresh = {0, 0, 0, -(1 << 30)};   /* no KLC recorded, never executed */
  I->a2[I->nst] = fresh;
  I->nst++;
}

/* release(i): undo every stage; g_i = 0 when emptied (Eq.5). */
static void release(RScen* s, int32_t id) {
  RInst* I = &s->inst[id];
  const ref_func* F = &s->fn[I->func];
  for (int32_t k = 0; k < I->nst; ++k) {
    RGpu* G = &s->gpu[I->g[k]];
    G->R -= F->req_pm;
    G->L -= F->lim_pm;
    G->U -= I->share[k];
    int32_t j = 0;
    while (j < G->nres && G->res[j] != id) ++j;
    for (; j + 1 < G->nres; ++j) G->res[j] = G->res[j + 1];
    --G->nres;
    I->g[k] = -1;
    I->share[k] = 0;
  }
  I->nst = 0;
}

static void terminate(RScen* s, int32_t id) {
  RInst* I = &s->inst[id];
  if (I->status == ST_PLACED) release(s, id);
  I->status = ST_TERMINATED;
  live_remove(&s->fs[I->func], id);
  --s->n_live;
}

/* -------------------------------------------- Algorithm 1 for one instance */

/* place(i, I*) -- ScheduleInstances body for one of the n_j GPUs
 * with Principle 2's LLM worst-fit between "no active GPU" and "start a
 * new GPU" (Q11).  Returns 1 on success (commits), 0 on failure (no change).   */
static int32_t place_one(RScen* s, int32_t id, const int32_t* Istar, int32_t nI) {
  const ref_config* c = s->cfg;
  const int32_t G = c->gpus_per_scenario;
  const ref_func* F = &s->fn[s->inst[id].func];
  int32_t *R = (int32_t*)xcalloc((size_t)G, 4), *L = (int32_t*)xcalloc((size_t)G, 4);
  int32_t *U = (int32_t*)xcalloc((size_t)G, 4), *nres = (int32_t*)xcalloc((size_t)G, 4);
  int32_t *wa = (int32_t*)xcalloc((size_t)G, 4), *other = (int32_t*)xcalloc((size_t)G, 4);
  int32_t *active = (int32_t*)xcalloc((size_t)G, 4), *excl = (int32_t*)xcalloc((size_t)G, 4);
  int32_t nwa = 0, nother = 0, ok = 0;
  for (int32_t g = 0; g < G; ++g) {
    R[g] = s->gpu[g].R; L[g] = s->gpu[g].L; U[g] = s->gpu[g].U; nres[g] = s->gpu[g].nres;
    active[g] = s->gpu[g].nres > 0;                      /* g_i, Eq.5 */
  }
  for (int32_t j = 0; j < nI; ++j) excl[Istar[j]] = 1;   /* Q7: workers on distinct GPUs */
  /* G_WA: active GPUs hosting an instance of the same affinity class (Q6) */
  for (int32_t g = 0; g < G; ++g) {
    if (!active[g] || excl[g]) continue;
    int32_t aff = 0;
    for (int32_t j = 0; j < s->gpu[g].nres; ++j)
      if (s->fn[s->inst[s->gpu[g].res[j]].func].affinity_class == F->affinity_class) aff = 1;
    if (aff) wa[nwa++] = g; else other[nother++] = g;
  }
  /* Exclusive baseline: "All GPUs are allocated exclusively to DL function instances via
   * pass-through" -- no sharing, so only a new GPU qualifies. */
  const int exclusive = s->mode == M_EXCLUSIVE;
  int32_t istar = exclusive ? -1 :
      select_opt_gpu(nwa, wa, R, L, U, nres, F->req_pm, F->lim_pm, F->mem_mib,
                     s->omega_u, s->gamma_u, c->mem_mib, c->q_pm, c->alpha_w, c->beta_w);
  if (istar == -1 && !exclusive)  /* "Select from the GPUs without WA" */
    istar = select_opt_gpu(nother, other, R, L, U, nres, F->req_pm, F->lim_pm, F->mem_mib,
                           s->omega_u, s->gamma_u, c->mem_mib, c->q_pm, c->alpha_w, c->beta_w);
  if (istar != -1) {
    commit(s, id, istar, F->mem_mib);
    ok = 1;
  } else {
    if (F->kind == K_LLM && (c->flags & 1) && !exclusive) {  /* Principle 2 worst-fit split */
      int32_t sg[MAX_STAGES], sh[MAX_STAGES];
      int32_t k = dilu_ref_llm_split(G, active, R, L, U, nres, excl, F->req_pm, F->lim_pm,
                                     F->mem_mib, s->omega_u, s->gamma_u, c->mem_mib,
                                     c->max_llm_stages, sg, sh);
      if (k > 0) {
        for (int32_t j = 0; j < k; ++j) commit(s, id, sg[j], sh[j]);
        s->tally[T_LLM_SPLIT] += 1;
        ok = 1;
      }
    }
    if (!ok) {  /* "Start a new GPU instance": lowest-id inactive (Q10) */
      for (int32_t g = 0; g < G; ++g) {
        if (active[g] || excl[g]) continue;
        if (F->req_pm <= s->omega_u && F->lim_pm <= s->gamma_u && F->mem_mib <= c->mem_mib) {
          commit(s, id, g, F->mem_mib);
          ok = 1;
        }
        break;
      }
    }
  }
  free(R); free(L); free(U); free(nres); free(wa); free(other); free(active); free(excl);
  return ok;
}

/* Placement pass, SURVEY s8(c) step 5 (Q8 all-or-nothing gangs, Q9 FIFO, no
 * head-of-line blocking).  Returns nothing; updates queue, tallies, instances.  */
static void placement_pass(RScen* s, int32_t t, int32_t* out_gpu_of_first /* per queue entry or NULL */) {
  int32_t nkeep = 0;
  for (int32_t qi = 0; qi < s->nq; ++qi) {
    RReq r = s->q[qi];
    const ref_func* F = &s->fn[r.func];
    int32_t Istar[64 + RES_CAP * MAX_STAGES];
    int32_t nI = 0, placed = 0;
    for (int32_t j = 0; j < r.n; ++j) {
      int32_t id = r.first + j;
      if (!place_one(s, id, Istar, nI)) break;
      for (int32_t k = 0; k < s->inst[id].nst; ++k) Istar[nI++] = s->inst[id].g[k];
      ++placed;
    }
    if (placed == r.n) {
      for (int32_t j = 0; j < r.n; ++j) {
        RInst* I = &s->inst[r.first + j];
        I->status = ST_PLACED;
        I->ready = t + F->cold_slots;
        s->tally[T_PLACEMENTS_OK] += 1;
        if (is_inf(F->kind) && F->cold_slots > 0) s->tally[T_COLD_STARTS] += 1;  /* Q20 */
      }
      if (out_gpu_of_first) out_gpu_of_first[qi] = s->inst[r.first].g[0];
    } else {
      for (int32_t j = 0; j < placed; ++j) release(s, r.first + j);  /* rollback */
      s->tally[T_PLACEMENT_FAILURES] += 1;
      if (out_gpu_of_first) out_gpu_of_first[qi] = -1;
      s->q[nkeep++] = r;
    }
  }
  s->nq = nkeep;
}

/* ---------------------------------------------------------- per-slot loop */

static int32_t arrivals(const RScen* s, int32_t f, int32_t t) {
  /* a1: A_f(t) = (pat[p_f][(t + phase_f) mod T_pat] * scale_f) >> 10 */
  const ref_func* F = &s->fn[f];
  int32_t Tp = s->cfg->pattern_len;
  int64_t v = s->pat[(int64_t)F->pattern * Tp + ((int64_t)t + F->phase_slots) % Tp];
  return (int32_t)((v * F->scale_q10) >> 10);
}

static void register_func(RScen* s, int32_t f) {
  RFunc* Fs = &s->fs[f];
  if (Fs->registered) return;
  Fs->registered = 1;
  Fs->nsamp = 0;
  Fs->rps_acc = 0;
  Fs->head = 0;
  memset(Fs->ring, 0, (size_t)s->cfg->window_s * sizeof(int32_t));
}

static void arrive(RScen* s, int32_t f) {  /* step 4 */
  const ref_func* F = &s->fn[f];
  register_func(s, f);
  if (F->kind == K_TRAIN) enqueue(s, f, F->n_workers);           /* a gang of n_j */
  else for (int32_t j = 0; j < s->cfg->min_instances; ++j) enqueue(s, f, 1);
}

static void depart(RScen* s, int32_t f) {  /* step 2 */
  int32_t nkeep = 0;
  for (int32_t qi = 0; qi < s->nq; ++qi)
    if (s->q[qi].func != f) s->q[nkeep++] = s->q[qi];
  s->nq = nkeep;
  RFunc* Fs = &s->fs[f];
  while (Fs->nlive > 0) terminate(s, Fs->live[0]);
  Fs->registered = 0;
}

/* Boundary work at t mod SPS == 0 (Q26 order). */
static void boundary(RScen* s, int32_t t, int32_t sec) {
  const ref_config* c = s->cfg;
  const int32_t F = c->max_funcs, W = c->window_s;
  /* 1. window push of last second's count (P:963 sliding window) */
  if (sec >= 1)
    for (int32_t f = 0; f < F; ++f) {
      RFunc* Fs = &s->fs[f];
      if (!Fs->registered || !is_inf(s->fn[f].kind)) continue;
      Fs->ring[Fs->head] = Fs->rps_acc;
      Fs->head = (Fs->head + 1) % W;
      Fs->nsamp += 1;
      Fs->rps_acc = 0;
    }
  /* 2. departures */
  for (int32_t f = 0; f < F; ++f)
    if (s->fs[f].registered && s->fn[f].depart_sec == sec) depart(s, f);
  /* 3. hscaler; training is never horizontally scaled */
  for (int32_t f = 0; f < F; ++f) {
    RFunc* Fs = &s->fs[f];
    const ref_func* Fn = &s->fn[f];
    if (!Fs->registered || !is_inf(Fn->kind) || Fs->nsamp < (s->mode == M_EAGER ? 1 : W)) continue;
    int32_t k = 0;
    int64_t cap1 = dilu_ref_cap1(c->slot_ms, Fn->req_pm, Fn->work_per_batch, Fn->ibs);
    int32_t dec;
    if (s->mode == M_EAGER) {
      /* FaST-GS+-like reactive scaling: decide on the latest one-second sample alone,
       * i.e. the same rule with a window of 1 and phi_out = 1, phi_in = 0. */
      int32_t last = Fs->ring[(Fs->head + W - 1) % W];
      dec = dilu_ref_scaling_decision(1, &last, Fs->nlive, cap1, 1, 0, c->min_instances, &k);
    } else {
      dec = dilu_ref_scaling_decision(W, Fs->ring, Fs->nlive, cap1, c->phi_out, c->phi_in,
                                      c->min_instances, &k);
    }
    if (dec == 1) {
      for (int32_t j = 0; j < k; ++j) enqueue(s, f, 1);
      s->tally[T_SCALE_OUT] += 1;
    } else if (dec == 2) {
      int32_t victim = Fs->live[Fs->nlive - 1];  /* highest live id (Q19) */
      if (s->inst[victim].status == ST_PENDING) {
        int32_t nkeep = 0;
        for (int32_t qi = 0; qi < s->nq; ++qi)
          if (!(s->q[qi].first <= victim && victim < s->q[qi].first + s->q[qi].n))
            s->q[nkeep++] = s->q[qi];
        s->nq = nkeep;
      }
      terminate(s, victim);
      s->tally[T_SCALE_IN] += 1;
    }
  }
  /* 4. function arrivals */
  for (int32_t f = 0; f < F; ++f)
    if (s->fn[f].kind != K_UNUSED && s->fn[f].arrive_sec == sec) arrive(s, f);
  /* 5. placement pass */
  placement_pass(s, t, NULL);
}

static int cmp_i32(const void* x, const void* y) {
  int32_t a = *(const int32_t*)x, b = *(const int32_t*)y;
  return (a > b) - (a < b);
}

/* Invariants I1-I7; checked when cfg.flags bit1 is set. */
static void check_invariants(RScen* s, int32_t t) {
  const ref_config* c = s->cfg;
  const int32_t G = c->gpus_per_scenario;
  for (int32_t g = 0; g < G; ++g) {
    RGpu* Gp = &s->gpu[g];
    int64_t R = 0, L = 0, U = 0;
    if (Gp->R > s->omega_u || Gp->L > s->gamma_u || Gp->U > c->mem_mib || Gp->nres > RES_CAP)
      fail(s, REF_E_INVARIANT, "I1 violated: scenario %d gpu %d slot %d", s->scn_id, g, t);
    for (int32_t j = 0; j < Gp->nres; ++j) {
      RInst* I = &s->inst[Gp->res[j]];
      const ref_func* F = &s->fn[I->func];
      R += F->req_pm; L += F->lim_pm;
      for (int32_t k = 0; k < I->nst; ++k) if (I->g[k] == g) U += I->share[k];
    }
    if (R != Gp->R || L != Gp->L || U != Gp->U)
      fail(s, REF_E_INVARIANT, "I3 violated: scenario %d gpu %d slot %d", s->scn_id, g, t);
  }
  for (int32_t id = 0; id < s->n_ids; ++id) {
    RInst* I = &s->inst[id];
    if (I->status != ST_PLACED) continue;
    if (I->nst < 1) fail(s, REF_E_INVARIANT, "I7 violated: instance %d unplaced", id);
    const ref_func* F = &s->fn[I->func];
    if (I->warm)
      for (int32_t k = 0; k < I->nst; ++k) {
        int64_t rq = (int64_t)F->req_pm * c->slot_ms, lm = (int64_t)F->lim_pm * c->slot_ms;
        if (s->mode == M_EXCLUSIVE) lm = 1000LL * c->slot_ms;   /* pass-through ceiling */
        if (I->a[k] < ((c->flags & 4) ? 0 : rq) || I->a[k] > lm)   /* Alg.2: no floor */
          fail(s, REF_E_INVARIANT, "I4 violated: instance %d slot %d", id, t);
      }
  }
}

/* One slot, SURVEY s8(c) steps 6-9. */
static void slot(RScen* s, int32_t t) {
  const ref_config* c = s->cfg;
  const int32_t G = c->gpus_per_scenario, F = c->max_funcs;
  const int64_t T_slot = 1000LL * c->slot_ms;   /* MaxTokens per slot, R3 */
  /* warm flags and per-slot scratch */
  for (int32_t id = 0; id < s->n_ids; ++id) {
    RInst* I = &s->inst[id];
    I->warm = (I->status == ST_PLACED && I->ready <= t);
    I->r = 0;
    for (int32_t k = 0; k < MAX_STAGES; ++k) { I->a[k] = 0; I->loc[k] = 0; }
  }
  /* 6. arrivals + dispatch: even split over warm instances, remainder to lowest ids (Q16) */
  for (int32_t f = 0; f < F; ++f) {
    RFunc* Fs = &s->fs[f];
    if (!Fs->registered || !is_inf(s->fn[f].kind)) continue;
    int32_t A = arrivals(s, f, t);
    Fs->rps_acc += A;
    s->tally[T_REQ_TOTAL] += A;
    int32_t nw = 0;
    for (int32_t j = 0; j < Fs->nlive; ++j) nw += s->inst[Fs->live[j]].warm;
    if (nw == 0) {                                               /* Q17 */
      s->tally[T_REQ_VIOLATED] += A;
      if (c->flags & 8) { s->lat[REF_LAT_UNSERVED] += A; s->lat[80] += A; }
      continue;
    }
    int32_t rank = 0;
    for (int32_t j = 0; j < Fs->nlive; ++j) {
      RInst* I = &s->inst[Fs->live[j]];
      if (!I->warm) continue;
      I->r = A / nw + (rank < A % nw ? 1 : 0);
      ++rank;
    }
  }
  /* 7. vertical token allocation on every active GPU row */
  for (int32_t g = 0; g < G; ++g) {
    RGpu* Gp = &s->gpu[g];
    Gp->exec = 0;
    if (Gp->nres == 0) continue;
    int32_t n = 0, prio[RES_CAP], ids[RES_CAP], stg[RES_CAP];
    int64_t rq[RES_CAP], lm[RES_CAP], d[RES_CAP], a[RES_CAP];
    for (int32_t j = 0; j < Gp->nres; ++j) {
      int32_t id = Gp->res[j];
      RInst* I = &s->inst[id];
      if (!I->warm) continue;                                    /* Q14 */
      const ref_func* Fn = &s->fn[I->func];
      int32_t k = 0;
      while (I->g[k] != g) ++k;
      prio[n] = Fn->prio;
      ids[n] = id;
      stg[n] = k;
      rq[n] = (int64_t)Fn->req_pm * c->slot_ms;                  /* R3 */
      lm[n] = (int64_t)Fn->lim_pm * c->slot_ms;
      if (s->mode == M_EXCLUSIVE) lm[n] = T_slot;               /* pass-through: whole GPU */
      if (Fn->kind == K_TRAIN) {
        d[n] = lm[n] * Fn->duty_pm / 1000;                        /* comm idle */
      } else {
        int64_t cst = (Fn->work_per_batch + I->nst - 1) / I->nst; /* c_stage = ceil(c_b/k) */
        d[n] = (((int64_t)I->r + Fn->ibs - 1) / Fn->ibs) * cst;  /* ceil(r/IBS) batches */
      }
      ++n;
    }
    if (c->flags & 4) {
      /* literal Algorithm 2, slot_ms / 5 periods of 5 ms */
      int32_t rp[RES_CAP], lp[RES_CAP], cs[RES_CAP];
      ref_a2_res st[RES_CAP];
      for (int32_t x = 0; x < n; ++x) {
        RInst* I = &s->inst[ids[x]];
        const ref_func* Fn = &s->fn[I->func];
        rp[x] = (int32_t)(rq[x] / c->slot_ms * REF_A2_PERIOD_MS);   /* req_pm * 5 */
        lp[x] = (int32_t)(lm[x] / c->slot_ms * REF_A2_PERIOD_MS);   /* lim_pm * 5 (Excl: 5000) */
        cs[x] = Fn->kind == K_TRAIN ? 0 : (Fn->work_per_batch + I->nst - 1) / I->nst;
        if (Fn->prio != 0) cs[x] = 0;                           /* KLC only drives SLO residents */
        st[x] = I->a2[stg[x]];
      }
      const int32_t NP = c->slot_ms / REF_A2_PERIOD_MS;
      dilu_ref_alg2_row(n, prio, ids, rp, lp, d, cs, NP, t * NP, st, &Gp->a2, a, NULL);
      for (int32_t x = 0; x < n; ++x) s->inst[ids[x]].a2[stg[x]] = st[x];
    } else {
      dilu_ref_vertical_row(n, prio, ids, rq, lm, d, T_slot, a);
    }
    for (int32_t x = 0; x < n; ++x) {
      RInst* I = &s->inst[ids[x]];
      const ref_func* Fn = &s->fn[I->func];
      int32_t k = stg[x];
      I->a[k] = a[x];
      if (Fn->kind == K_TRAIN) {
        I->loc[k] = d[x] < a[x] ? d[x] : a[x];                    /* x = min(d, a) */
      } else {
        int64_t cst = (Fn->work_per_batch + I->nst - 1) / I->nst;
        int64_t need = ((int64_t)I->r + Fn->ibs - 1) / Fn->ibs;
        int64_t fit = a[x] / cst;                                 /* whole batches */
        I->loc[k] = need < fit ? need : fit;
      }
      s->tally[T_ALLOC_HASH] = (int64_t)((uint64_t)s->tally[T_ALLOC_HASH] +
          dilu_ref_mix((uint64_t)(uint32_t)s->scn_id, (uint64_t)(uint32_t)t,
                       (uint64_t)(uint32_t)ids[x], (uint64_t)(uint32_t)g, (uint64_t)a[x]));
    }
  }
  /* 8. gang minima and executed tokens */
  for (int32_t id = 0; id < s->n_ids; ++id) {            /* inference (single + LLM stages) */
    RInst* I = &s->inst[id];
    const ref_func* Fn = &s->fn[I->func];
    if (!I->warm || Fn->kind == K_TRAIN) continue;
    int64_t b = I->loc[0];
    for (int32_t k = 1; k < I->nst; ++k) if (I->loc[k] < b) b = I->loc[k];
    int64_t cst = (Fn->work_per_batch + I->nst - 1) / I->nst;
    int64_t served = (int64_t)b * Fn->ibs;
    if (served > I->r) served = I->r;
    s->tally[T_REQ_SERVED] += served;
    s->tally[T_REQ_VIOLATED] += I->r - served;
    for (int32_t k = 0; k < I->nst; ++k) {
      s->gpu[I->g[k]].exec += b * cst;
      s->tally[T_INF_EXEC] += b * cst;
    }
    if (c->flags & 8) {
      /* a batch runs at the slowest stage's rate: e = max_k ceil(c_stage * T / a_k) us */
      const int64_t T_us = 1000LL * c->slot_ms;
      int64_t e = 0;
      for (int32_t k = 0; k < I->nst; ++k) {
        const int64_t ek = I->a[k] > 0 ? (cst * T_us + I->a[k] - 1) / I->a[k] : 0;
        if (ek > e) e = ek;
      }
      dilu_ref_instance_latency(I->r, Fn->ibs, b, e, s->slo_us[I->func], T_us, s->lat);
    }
  }
  for (int32_t f = 0; f < F; ++f) {                      /* training jobs: barrel effect (Q22) */
    RFunc* Fs = &s->fs[f];
    const ref_func* Fn = &s->fn[f];
    if (!Fs->registered || Fn->kind != K_TRAIN || Fs->nlive == 0) continue;
    int64_t gang = -1;
    int32_t all_warm = 1;
    for (int32_t j = 0; j < Fs->nlive; ++j) {
      RInst* I = &s->inst[Fs->live[j]];
      if (!I->warm) { all_warm = 0; break; }
      if (gang < 0 || I->loc[0] < gang) gang = I->loc[0];
    }
    if (!all_warm) gang = 0;
    for (int32_t j = 0; j < Fs->nlive; ++j) {
      RInst* I = &s->inst[Fs->live[j]];
      if (I->warm) s->gpu[I->g[0]].exec += gang;
    }
    s->tally[T_TRAIN_PROGRESS] += (int64_t)Fn->n_workers * gang;
  }
  /* 9. fold */
  int64_t nact = 0;
  for (int32_t g = 0; g < G; ++g) {
    RGpu* Gp = &s->gpu[g];
    if (Gp->nres == 0) continue;
    ++nact;
    s->tally[T_SM_UNUSED] += T_slot - Gp->exec;
    s->tally[T_MEM_UNUSED] += c->mem_mib - Gp->U;
    if (Gp->exec > T_slot) fail(s, REF_E_INVARIANT, "I5 violated: gpu %d slot %d", g, t);
  }
  s->tally[T_GPU_SLOTS_ACTIVE] += nact;
  if (nact > s->tally[T_MAX_ACTIVE]) s->tally[T_MAX_ACTIVE] = nact;
  s->tally[T_GPU_ROW_SLOTS] += G;
  if (c->flags & 2) check_invariants(s, t);
  (void)cmp_i32;
}

/* ------------------------------------------------------------- public API */

static int32_t set_err(ref_sim* s, int32_t code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(s->err, sizeof s->err, fmt, ap);
  va_end(ap);
  s->status = code;
  return code;
}

static int32_t validate(const ref_config* c, const ref_scenario* scen, const ref_func* fn,
                        const int32_t* pat, char* msg, size_t n) {
#define BAD(...) do { snprintf(msg, n, __VA_ARGS__); return REF_E_USAGE; } while (0)
  if (c->n_scenarios < 1 || c->gpus_per_scenario < 1 || c->max_funcs < 1 || c->max_instances < 1)
    BAD("config: sizes must be positive");
  if (c->gpus_per_scenario >= (1 << 22)) BAD("config: G must be < 2^22 (R7)");
  if (c->q_pm != 1000) BAD("config: q_pm must be 1000 (R1)");
  if (c->mem_mib < 1 || c->mem_mib > (1 << 20)) BAD("config: mem_mib out of range (R7)");
  if (c->alpha_w < 0 || c->beta_w < 0 || c->alpha_w > 255 || c->beta_w > 255 ||
      c->alpha_w + c->beta_w == 0) BAD("config: alpha_w/beta_w must be in [0,255], not both 0");
  if (c->slot_ms < 1 || c->slot_ms > 1000 || 1000 % c->slot_ms) BAD("config: slot_ms must divide 1000");
  if ((c->flags & 4) && c->slot_ms % REF_A2_PERIOD_MS) BAD("config: Alg.2 periods need slot_ms %% 5 == 0");
  if (c->window_s < 1 || c->phi_out < 1 || c->phi_out > c->window_s || c->phi_in < 0 ||
      c->phi_in >= c->window_s || c->phi_out + c->phi_in <= c->window_s)
    BAD("config: need 1<=phi_out<=W, 0<=phi_in<W, phi_out+phi_in>W (S:455)");
  if (c->min_instances < 1) BAD("config: min_instances must be >= 1");
  if (c->max_residents != RES_CAP) BAD("config: max_residents must be 32");
  if (c->max_llm_stages < 1 || c->max_llm_stages > MAX_STAGES) BAD("config: max_llm_stages in [1,4]");
  if (c->n_patterns < 0 || c->pattern_len < 1) BAD("config: pattern table shape");
  for (int32_t p = 0; p < c->n_patterns; ++p)
    for (int32_t x = 0; x < c->pattern_len; ++x)
      if (pat[(int64_t)p * c->pattern_len + x] < 0) BAD("pattern %d: negative arrivals", p);
  for (int32_t sc = 0; sc < c->n_scenarios; ++sc) {
    int32_t om = scen ? scen[sc].omega_pm : c->omega_pm;
    int32_t ga = scen ? scen[sc].gamma_pm : c->gamma_pm;
    if (om < 1 || om > c->q_pm) BAD("scenario %d: omega_pm must be in [1, q_pm] (Q12)", sc);
    if (ga < om) BAD("scenario %d: gamma_pm < omega_pm (S:242)", sc);
    const int32_t mode = scen ? scen[sc].mode : 0;
    if (mode < 0 || mode > 4) BAD("scenario %d: mode must be in [0, 4]", sc);
    for (int32_t f = 0; f < c->max_funcs; ++f) {
      const ref_func* F = &fn[(int64_t)sc * c->max_funcs + f];
      if (F->kind == K_UNUSED) continue;
      if (F->kind < K_INF || F->kind > K_TRAIN) BAD("scenario %d func %d: kind", sc, f);
      if (F->prio != 0 && F->prio != 1) BAD("scenario %d func %d: prio", sc, f);
      if (F->req_pm < 1 || F->req_pm > F->lim_pm || F->lim_pm > c->q_pm)
        BAD("scenario %d func %d: need 1 <= req_pm <= lim_pm <= q_pm", sc, f);
      if (F->req_pm * 32 < om) BAD("scenario %d func %d: req_pm < ceil(omega/32) (Q23)", sc, f);
      if (F->req_pm > om || F->lim_pm > ga) BAD("scenario %d func %d: quota exceeds Omega/gamma", sc, f);
      if ((mode == 2 || mode == 4) && F->lim_pm > om)
        BAD("scenario %d func %d: limit above Omega (limit-quota baseline)", sc, f);
      if (F->mem_mib < 1 || F->mem_mib > c->mem_mib) BAD("scenario %d func %d: mem_mib", sc, f);
      if (F->cold_slots < 0) BAD("scenario %d func %d: cold_slots", sc, f);
      if (F->arrive_sec < 0 || F->depart_sec <= F->arrive_sec) BAD("scenario %d func %d: lifecycle", sc, f);
      if (F->kind == K_TRAIN) {
        if (F->n_workers < 1 || F->n_workers > c->gpus_per_scenario || F->n_workers > 64)
          BAD("scenario %d func %d: n_workers", sc, f);
        if (F->duty_pm < 0 || F->duty_pm > 1000) BAD("scenario %d func %d: duty_pm", sc, f);
      } else {
        if (F->ibs < 1) BAD("scenario %d func %d: ibs", sc, f);
        int64_t req_tok = (int64_t)F->req_pm * c->slot_ms;
        if (F->work_per_batch < 1 || F->work_per_batch > req_tok)
          BAD("scenario %d func %d: need 1 <= c_b <= req_tok (R4)", sc, f);
        if (F->pattern < 0 || F->pattern >= c->n_patterns) BAD("scenario %d func %d: pattern", sc, f);
        if (F->scale_q10 < 0 || F->phase_slots < 0) BAD("scenario %d func %d: scale/phase", sc, f);
      }
    }
  }
  return REF_OK;
#undef BAD
}

int32_t dilu_ref_create(const ref_config* cfg, const ref_scenario* scen, const ref_func* funcs,
                        const int32_t* patterns, ref_sim** out) {
  if (!cfg || !funcs || !out) return REF_E_USAGE;
  char msg[256];
  int32_t rc = validate(cfg, scen, funcs, patterns, msg, sizeof msg);
  if (rc != REF_OK) { fprintf(stderr, "dilu_ref_create: %s\n", msg); *out = NULL; return rc; }
  ref_sim* s = (ref_sim*)xcalloc(1, sizeof *s);
  s->cfg = *cfg;
  s->S = cfg->n_scenarios;
  size_t nf = (size_t)cfg->n_scenarios * cfg->max_funcs;
  s->funcs = (ref_func*)xcalloc(nf, sizeof(ref_func));
  memcpy(s->funcs, funcs, nf * sizeof(ref_func));
  size_t np = (size_t)cfg->n_patterns * cfg->pattern_len;
  s->patterns = (int32_t*)xcalloc(np, sizeof(int32_t));
  if (np) memcpy(s->patterns, patterns, np * sizeof(int32_t));
  s->sc = (RScen*)xcalloc((size_t)s->S, sizeof(RScen));
  for (int32_t i = 0; i < s->S; ++i) {
    RScen* sc = &s->sc[i];
    sc->cfg = &s->cfg;
    sc->fn = s->funcs + (size_t)i * cfg->max_funcs;
    sc->pat = s->patterns;
    sc->scn_id = scen ? scen[i].scenario_id : i;
    sc->omega_u = scen ? scen[i].omega_pm : cfg->omega_pm;
    sc->gamma_u = scen ? scen[i].gamma_pm : cfg->gamma_pm;
    sc->mode = scen ? scen[i].mode : M_DILU;
    /* quota transforms of the baselines: MPS-l and FaST-GS+ run at the
     * limit quota, MPS-r at the request quota -- both without vertical scaling */
    sc->slo_us = (int64_t*)xcalloc((size_t)cfg->max_funcs, sizeof(int64_t));
    for (int32_t f = 0; f < cfg->max_funcs; ++f) {
      ref_func* F = &s->funcs[(size_t)i * cfg->max_funcs + f];
      if (F->kind == K_UNUSED) continue;
      /* SLO = 2 * t_exec at the profiled request (P:634 footnote, R4): c_b = req * SLO/2 */
      if (is_inf(F->kind)) sc->slo_us[f] = 2000LL * F->work_per_batch / F->req_pm;
      if (sc->mode == M_STATIC_LIMIT || sc->mode == M_EAGER) F->req_pm = F->lim_pm;
      if (sc->mode == M_STATIC_REQUEST) F->lim_pm = F->req_pm;
    }
    sc->gpu = (RGpu*)xcalloc((size_t)cfg->gpus_per_scenario, sizeof(RGpu));
    for (int32_t g = 0; g < cfg->gpus_per_scenario; ++g) sc->gpu[g].a2.owner = -1;   /* NONE */
    sc->fs = (RFunc*)xcalloc((size_t)cfg->max_funcs, sizeof(RFunc));
    for (int32_t f = 0; f < cfg->max_funcs; ++f)
      sc->fs[f].ring = (int32_t*)xcalloc((size_t)cfg->window_s, sizeof(int32_t));
  }
  *out = s;
  return REF_OK;
}

void dilu_ref_destroy(ref_sim* s) {
  if (!s) return;
  for (int32_t i = 0; i < s->S; ++i) {
    RScen* sc = &s->sc[i];
    for (int32_t f = 0; f < s->cfg.max_funcs; ++f) { free(sc->fs[f].ring); free(sc->fs[f].live); }
    free(sc->fs); free(sc->gpu); free(sc->inst); free(sc->q); free(sc->slo_us);
  }
  free(s->sc); free(s->funcs); free(s->patterns); free(s);
}

const char* dilu_ref_last_error(const ref_sim* s) { return s ? s->err : "null handle"; }
int32_t dilu_ref_slot(const ref_sim* s) { return s ? s->t : -1; }

static int32_t collect_errors(ref_sim* s) {
  for (int32_t i = 0; i < s->S; ++i)
    if (s->sc[i].err) return set_err(s, s->sc[i].err, "%s", s->sc[i].msg);
  return REF_OK;
}

int32_t dilu_ref_place_batch(ref_sim* s, int32_t n_req, const int32_t* req_scenario,
                             const int32_t* req_func, int32_t* out_gpu, int32_t* out_iid) {
  if (!s) return REF_E_USAGE;
  if (s->status) return REF_E_STATE;
  for (int32_t j = 0; j < n_req; ++j) {
    if (req_scenario[j] < 0 || req_scenario[j] >= s->S || req_func[j] < 0 ||
        req_func[j] >= s->cfg.max_funcs ||
        s->sc[req_scenario[j]].fn[req_func[j]].kind == K_UNUSED)
      return set_err(s, REF_E_USAGE, "place_batch: request %d names an invalid scenario/function", j);
  }
  for (int32_t i = 0; i < s->S; ++i) {
    RScen* sc = &s->sc[i];
    int32_t nq0 = sc->nq;
    /* enqueue this scenario's explicit requests in array order (an arrival of f, one request) */
    int32_t* qpos = (int32_t*)xcalloc((size_t)(n_req ? n_req : 1), sizeof(int32_t));
    for (int32_t j = 0; j < n_req; ++j) {
      qpos[j] = -1;
      if (req_scenario[j] != i) continue;
      int32_t f = req_func[j];
      register_func(sc, f);
      qpos[j] = sc->nq;
      if (out_iid) out_iid[j] = sc->n_ids;
      enqueue(sc, f, sc->fn[f].kind == K_TRAIN ? sc->fn[f].n_workers : 1);
    }
    if (sc->err) { free(qpos); break; }
    int32_t* gof = (int32_t*)xcalloc((size_t)sc->nq + 1, sizeof(int32_t));
    placement_pass(sc, s->t, gof);
    for (int32_t j = 0; j < n_req; ++j)
      if (qpos[j] >= 0 && out_gpu) out_gpu[j] = gof[qpos[j]];
    (void)nq0;
    free(gof);
    free(qpos);
  }
  return collect_errors(s);
}

typedef struct { ref_sim* s; int32_t lo, hi, n_slots; } Job;

static void* run_job(void* p) {
  Job* J = (Job*)p;
  const int32_t SPS = 1000 / J->s->cfg.slot_ms;
  for (int32_t i = J->lo; i < J->hi; ++i) {
    RScen* sc = &J->s->sc[i];
    for (int32_t k = 0; k < J->n_slots && !sc->err; ++k) {
      int32_t t = J->s->t + k;
      if (t % SPS == 0) boundary(sc, t, t / SPS);
      slot(sc, t);
    }
  }
  return NULL;
}

int32_t dilu_ref_scale_step(ref_sim* s, int32_t n_slots, int32_t n_threads) {
  if (!s) return REF_E_USAGE;
  if (s->status) return REF_E_STATE;
  if (n_slots < 0) return set_err(s, REF_E_USAGE, "scale_step: n_slots < 0");
  if (n_threads < 1) n_threads = 1;
  if (n_threads > s->S) n_threads = s->S;
  pthread_t* th = (pthread_t*)xcalloc((size_t)n_threads, sizeof(pthread_t));
  Job* jobs = (Job*)xcalloc((size_t)n_threads, sizeof(Job));
  for (int32_t k = 0; k < n_threads; ++k) {
    jobs[k].s = s;
    jobs[k].lo = (int32_t)((int64_t)s->S * k / n_threads);
    jobs[k].hi = (int32_t)((int64_t)s->S * (k + 1) / n_threads);
    jobs[k].n_slots = n_slots;
    if (n_threads == 1) run_job(&jobs[k]);
    else pthread_create(&th[k], NULL, run_job, &jobs[k]);
  }
  if (n_threads > 1)
    for (int32_t k = 0; k < n_threads; ++k) pthread_join(th[k], NULL);
  free(th);
  free(jobs);
  s->t += n_slots;
  return collect_errors(s);
}

int32_t dilu_ref_metrics(ref_sim* s, int64_t* per_scenario, int64_t* sum) {
  if (!s) return REF_E_USAGE;
  int64_t acc[REF_NT];
  memset(acc, 0, sizeof acc);
  for (int32_t i = 0; i < s->S; ++i) {
    for (int32_t k = 0; k < REF_NT; ++k) {
      if (per_scenario) per_scenario[(int64_t)i * REF_NT + k] = s->sc[i].tally[k];
      acc[k] = (int64_t)((uint64_t)acc[k] + (uint64_t)s->sc[i].tally[k]);
    }
  }
  if (sum) memcpy(sum, acc, sizeof acc);
  return s->status;
}

int32_t dilu_ref_latency(ref_sim* s, int64_t* per_scenario, int64_t* sum) {
  if (!s) return REF_E_USAGE;
  int64_t acc[REF_NLAT];
  memset(acc, 0, sizeof acc);
  for (int32_t i = 0; i < s->S; ++i)
    for (int32_t k = 0; k < REF_NLAT; ++k) {
      if (per_scenario) per_scenario[(int64_t)i * REF_NLAT + k] = s->sc[i].lat[k];
      acc[k] += s->sc[i].lat[k];
    }
  if (sum) memcpy(sum, acc, sizeof acc);
  return s->status;
}

int32_t dilu_ref_slot_detail(ref_sim* s, int32_t scenario, int32_t id_cap, int64_t* a,
                             int32_t* r, int64_t* exec) {
  if (!s || scenario < 0 || scenario >= s->S) return REF_E_USAGE;
  RScen* sc = &s->sc[scenario];
  for (int32_t id = 0; id < id_cap; ++id) {
    for (int32_t k = 0; k < MAX_STAGES; ++k)
      a[(int64_t)id * MAX_STAGES + k] = id < sc->n_ids ? sc->inst[id].a[k] : 0;
    r[id] = id < sc->n_ids ? sc->inst[id].r : 0;
  }
  for (int32_t g = 0; g < s->cfg.gpus_per_scenario; ++g) exec[g] = sc->gpu[g].exec;
  return REF_OK;
}

int32_t dilu_ref_snapshot(ref_sim* s, int32_t id_cap, int32_t* gpu, int32_t* inst) {
  if (!s) return REF_E_USAGE;
  const int32_t G = s->cfg.gpus_per_scenario;
  for (int32_t i = 0; i < s->S; ++i) {
    RScen* sc = &s->sc[i];
    if (gpu)
      for (int32_t g = 0; g < G; ++g) {
        int32_t* o = gpu + ((int64_t)i * G + g) * 4;
        o[0] = sc->gpu[g].R; o[1] = sc->gpu[g].L; o[2] = sc->gpu[g].U; o[3] = sc->gpu[g].nres;
      }
    if (inst)
      for (int32_t id = 0; id < id_cap; ++id) {
        int32_t* o = inst + ((int64_t)i * id_cap + id) * 12;
        if (id >= sc->n_ids) {
          for (int32_t k = 0; k < 12; ++k) o[k] = -1;
          continue;
        }
        RInst* I = &sc->inst[id];
        o[0] = I->status == ST_TERMINATED ? -1 : I->func;   /* ABI: -1 once terminated */
        o[1] = I->status;
        o[2] = I->status == ST_PLACED ? I->nst : 0;
        o[3] = I->status == ST_PLACED ? I->ready : -1;
        for (int32_t k = 0; k < MAX_STAGES; ++k) {
          int on = I->status == ST_PLACED && k < I->nst;
          o[4 + k] = on ? I->g[k] : -1;
          o[8 + k] = on ? I->share[k] : 0;
        }
      }
  }
  return REF_OK;
}
