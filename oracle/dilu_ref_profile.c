/*
 * dilu_ref_profile.c -- CPU ORACLE of the multi-factor profiler (test infrastructure
 * only; see dilu_ref.h).  SURVEY s8(f) #3: the step before the path -- it produces the
 * <IBS, request, limit> rows the provisioning loop consumes (step a0).
 *
 * Follows PAPER.md s3.2 "Multi-Factor Profiling" in the paper's order, over
 * SPEC's synthetic perfmodel because the paper measures real GPUs.  Readings
 * (D9): the paper's stop rule "ends until the T_i satisfies T1*p +- 2%" is
 * taken literally; the Hybrid Growth Search doubles IBS from 1 and grows SMR by 10 from
 * the previous level's point, stopping at the first level without a feasible SMR or
 * whose TE is lower than the best so far (SPEC S:225 one-level lookahead).
 * fp64, plain IEEE operations, no contraction (-ffp-contract=off).
 */
#include "dilu_ref.h"

#include <math.h>

/* t_exec = (a + b*IBS) * knee / min(SMR, knee), knee = min(100, c*sqrt(IBS)):
 * the latency falls with SMR up to the knee and is flat beyond it (Figure 4's marginal
 * effect, "merely a 2% throughput boost"). */
double dilu_ref_infer_exec_ms(const ref_prof_session* m, int32_t ibs, double smr) {
  double knee = m->knee_c * sqrt((double)ibs);
  if (knee > 100.0) knee = 100.0;
  double den = smr < knee ? smr : knee;
  return (m->a_ms + m->b_ms * (double)ibs) * knee / den;
}

/* throughput = workers * T_max * min(1, SMR/knee_t) * (1 - idle). */
double dilu_ref_train_tput(const ref_prof_session* m, double smr) {
  double frac = smr / m->knee_t;
  if (frac > 1.0) frac = 1.0;
  return (double)m->workers * m->t_max * frac * (1.0 - m->idle);
}

/* Q25 loader rounding: ceil(10 * percent) per-mille, the limit capped at 1000. */
static int32_t to_pm(double pct) { return (int32_t)ceil(10.0 * pct - 1e-9); }

/* Training profiling: "records exclusive throughput T1 with high (=100%,
 * firstly) SMR and T2 with mid (=50%) SMR ... If T2 is less than T1*p ... low = mid.
 * Otherwise, the high value is set to mid.  The profiling ends until the T_i satisfies
 * T1*p +- 2%."  Request at p = 80 %, limit at p = 100 %.  A bracket narrower than one SMR
 * unit also ends the search, returning high.  A probe whose throughput is more
 * than tol below (above) the previous probe's at a higher (lower) SMR flags a
 * non-monotone oracle; the search still completes. */
static void profile_training(const ref_prof_session* m, ref_prof_out* o) {
  const double T1 = dilu_ref_train_tput(m, 100.0);
  int32_t trials = 1;
  double res[2];
  const double ps[2] = {m->p_req, m->p_lim};
  o->status = 0;
  for (int k = 0; k < 2; ++k) {
    const double target = T1 * ps[k];
    double low = 0.0, high = 100.0, prev_smr = 100.0, prev_T = T1;
    res[k] = high;
    for (;;) {
      const double mid = (low + high) / 2.0;
      const double T = dilu_ref_train_tput(m, mid);
      ++trials;
      if ((mid > prev_smr && T < prev_T * (1.0 - m->tol)) ||
          (mid < prev_smr && T > prev_T * (1.0 + m->tol)))
        o->status = 2;
      prev_smr = mid;
      prev_T = T;
      if (fabs(T - target) <= m->tol * target) { res[k] = mid; break; }
      if (T < target) low = mid; else high = mid;
      if (high - low < 1.0) { res[k] = high; break; }
    }
  }
  o->request_smr = res[0];
  o->limit_smr = res[1];
  o->t_exec_ms = T1;
  o->ibs = 0;
  o->trials = trials;
}

/* Inference profiling, Hybrid Growth Search: "IBS iteratively increases by
 * doubling during profiling, while SMR increases linearly by a fixed rate (i.e., 10
 * units)"; feasible iff t_exec <= SLO/2 (footnote P:634); TE = IBS / (t_exec * SMR)
 * (P:633); the best TE point is the request, "limit quota at twice of request". */
static void profile_inference(const ref_prof_session* m, ref_prof_out* o) {
  const double budget = m->slo_ms / 2.0;
  double best_te = -1.0, best_s = 0.0, best_t = 0.0;
  int32_t best_ibs = 0, trials = 0;
  double s = m->smr_step;
  for (int32_t ibs = 1; ibs <= m->ibs_max; ibs *= 2) {
    double t = 0.0;
    int feasible = 0;
    while (s <= 100.0) {                       /* grow SMR from the previous point */
      t = dilu_ref_infer_exec_ms(m, ibs, s);
      ++trials;
      if (t <= budget) { feasible = 1; break; }
      s += m->smr_step;
    }
    if (!feasible) break;                      /* blocked path (Figure 4) */
    const double te = (double)ibs / (t * s);
    if (best_te >= 0.0 && te < best_te) break; /* TE stopped improving */
    if (te > best_te) { best_te = te; best_s = s; best_t = t; best_ibs = ibs; }
  }
  o->trials = trials;
  if (best_te < 0.0) {                         /* no feasible point at IBS 1 */
    o->status = 1;
    o->request_smr = o->limit_smr = o->t_exec_ms = 0.0;
    o->ibs = 0;
    return;
  }
  o->status = 0;
  o->request_smr = best_s;
  o->limit_smr = 2.0 * best_s < 100.0 ? 2.0 * best_s : 100.0;
  o->t_exec_ms = best_t;
  o->ibs = best_ibs;
}

void dilu_ref_profile_one(const ref_prof_session* in, ref_prof_out* out) {
  if (in->kind == 2) profile_training(in, out);
  else profile_inference(in, out);
  out->req_pm = out->status == 1 ? 0 : to_pm(out->request_smr);
  int32_t lp = out->status == 1 ? 0 : to_pm(out->limit_smr);
  out->lim_pm = lp < 1000 ? lp : 1000;
  out->reserved = 0;
}

void dilu_ref_profile_batch(int32_t n, const ref_prof_session* in, ref_prof_out* out) {
  for (int32_t i = 0; i < n; ++i) dilu_ref_profile_one(&in[i], &out[i]);
}
