// profile.cuh -- batched multi-factor profiler, one thread per session.
//
// PAPER.md s3.2: training quotas by bisection on throughput and
// inference <IBS, SMR> by the Hybrid Growth Search, over SPEC's synthetic
// perfmodel.  Readings: DESIGN.md D9.  fp64 with explicitly rounded IEEE
// operations (__dadd_rn / __dmul_rn / __ddiv_rn / __dsqrt_rn): nvcc may not contract them
// into FMAs, so every result is the plain IEEE one.  Sessions are tiny (<= ~20 perfmodel
// evaluations), so the kernel is a grid-stride loop sized to the SM count; a warp reads
// its 32 x 104-byte rows as one contiguous 3.3 KB span.
#pragma once
#include <stdint.h>

#include "../../include/dilu.h"

namespace dilu {
namespace prof {

static_assert(sizeof(dilu_prof_session) == 104, "session layout");
static_assert(sizeof(dilu_prof_out) == 48, "output layout");

// t_exec = (a + b*IBS) * knee / min(SMR, knee), knee = min(100, c*sqrt(IBS))
__device__ __forceinline__ double infer_exec_ms(const dilu_prof_session& m, int32_t ibs, double smr) {
  double knee = __dmul_rn(m.knee_c, __dsqrt_rn((double)ibs));
  if (knee > 100.0) knee = 100.0;
  const double den = smr < knee ? smr : knee;
  return __ddiv_rn(__dmul_rn(__dadd_rn(m.a_ms, __dmul_rn(m.b_ms, (double)ibs)), knee), den);
}

// throughput = workers * T_max * min(1, SMR/knee_t) * (1 - idle)
__device__ __forceinline__ double train_tput(const dilu_prof_session& m, double smr) {
  double frac = __ddiv_rn(smr, m.knee_t);
  if (frac > 1.0) frac = 1.0;
  return __dmul_rn(__dmul_rn(__dmul_rn((double)m.workers, m.t_max), frac), __dsub_rn(1.0, m.idle));
}

__device__ __forceinline__ int32_t to_pm(double pct) {             // Q25: ceil(10 * percent)
  return (int32_t)ceil(__dsub_rn(__dmul_rn(10.0, pct), 1e-9));
}

// Training: T1 at SMR 100, then per p a bisection that ends at the first probe
// within T1*p +- tol (the paper's stop rule) or when the bracket is narrower than 1.
__device__ void profile_training(const dilu_prof_session& m, dilu_prof_out& o) {
  const double T1 = train_tput(m, 100.0);
  int32_t trials = 1, status = 0;
  double res[2];
  const double ps[2] = {m.p_req, m.p_lim};
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const double target = __dmul_rn(T1, ps[k]);
    const double band = __dmul_rn(m.tol, target);
    double low = 0.0, high = 100.0, prev_smr = 100.0, prev_T = T1;
    res[k] = high;
    for (;;) {
      const double mid = __ddiv_rn(__dadd_rn(low, high), 2.0);
      const double T = train_tput(m, mid);
      ++trials;
      if ((mid > prev_smr && T < __dmul_rn(prev_T, __dsub_rn(1.0, m.tol))) ||
          (mid < prev_smr && T > __dmul_rn(prev_T, __dadd_rn(1.0, m.tol))))
        status = 2;                                      // non-monotone oracle
      prev_smr = mid;
      prev_T = T;
      if (fabs(__dsub_rn(T, target)) <= band) { res[k] = mid; break; }
      if (T < target) low = mid; else high = mid;
      if (__dsub_rn(high, low) < 1.0) { res[k] = high; break; }
    }
  }
  o.request_smr = res[0];
  o.limit_smr = res[1];
  o.t_exec_ms = T1;
  o.ibs = 0;
  o.trials = trials;
  o.status = status;
}

// Inference, Hybrid Growth Search: IBS doubles, SMR grows by smr_step from the
// previous level's point until t_exec <= SLO/2; stop at a blocked level or a TE drop.
__device__ void profile_inference(const dilu_prof_session& m, dilu_prof_out& o) {
  const double budget = __ddiv_rn(m.slo_ms, 2.0);
  double best_te = -1.0, best_s = 0.0, best_t = 0.0;
  int32_t best_ibs = 0, trials = 0;
  double s = m.smr_step;
  for (int32_t ibs = 1; ibs <= m.ibs_max; ibs *= 2) {
    double t = 0.0;
    bool feasible = false;
    while (s <= 100.0) {
      t = infer_exec_ms(m, ibs, s);
      ++trials;
      if (t <= budget) { feasible = true; break; }
      s = __dadd_rn(s, m.smr_step);
    }
    if (!feasible) break;
    const double te = __ddiv_rn((double)ibs, __dmul_rn(t, s));
    if (best_te >= 0.0 && te < best_te) break;
    if (te > best_te) { best_te = te; best_s = s; best_t = t; best_ibs = ibs; }
  }
  o.trials = trials;
  if (best_te < 0.0) {                                   // SLO unattainable
    o.status = 1;
    o.request_smr = o.limit_smr = o.t_exec_ms = 0.0;
    o.ibs = 0;
    return;
  }
  o.status = 0;
  o.request_smr = best_s;
  const double two = __dmul_rn(2.0, best_s);
  o.limit_smr = two < 100.0 ? two : 100.0;
  o.t_exec_ms = best_t;
  o.ibs = best_ibs;
}

__global__ void __launch_bounds__(256) k_profile(const dilu_prof_session* __restrict__ in, int32_t n,
                                                 dilu_prof_out* __restrict__ out) {
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const dilu_prof_session m = in[i];
    dilu_prof_out o;
    if (m.kind == 2) profile_training(m, o);
    else profile_inference(m, o);
    o.req_pm = o.status == 1 ? 0 : to_pm(o.request_smr);
    const int32_t lp = o.status == 1 ? 0 : to_pm(o.limit_smr);
    o.lim_pm = lp < 1000 ? lp : 1000;
    o.reserved = 0;
    out[i] = o;
  }
}

}  // namespace prof
}  // namespace dilu

namespace dilu {
namespace prof {

static_assert(sizeof(dilu_catalog_row) == 72, "catalogue row layout");
static_assert(sizeof(dilu_func) == 64, "function row layout");

// Q25 ceiling of a non-negative fp64 quantity (ceil(x - 1e-9)), int32-saturated
__device__ __forceinline__ int32_t q25_ceil(double x) {
  const double y = ceil(__dsub_rn(x, 1e-9));
  return y >= 2147483647.0 ? 2147483647 : (int32_t)y;
}

// a0: one thread per row (include/dilu.h dilu_load_profiles)
__global__ void k_load(const dilu_catalog_row* __restrict__ cat, const dilu_prof_out* __restrict__ pr,
                       int32_t n, int32_t slot_ms, dilu_func* __restrict__ out, int32_t* __restrict__ st) {
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const dilu_catalog_row c = cat[i];
    const dilu_prof_out p = pr[i];
    dilu_func r;
    r.kind = -1; r.prio = c.prio; r.ibs = 0; r.req_pm = 0; r.lim_pm = 0; r.mem_mib = 0;
    r.work_per_batch = 0; r.n_workers = 1; r.duty_pm = 0; r.cold_slots = 0;
    r.affinity_class = c.affinity_class; r.arrive_sec = c.arrive_sec; r.depart_sec = c.depart_sec;
    r.pattern = c.pattern; r.scale_q10 = c.scale_q10; r.phase_slots = c.phase_slots;
    const bool train = c.kind == 2, inf = c.kind == 0 || c.kind == 1;
    int32_t status = 0;
    if (!(train || inf) || !(c.mem_gb >= 0.0) || !(c.cold_ms >= 0.0) || (inf && !(c.slo_ms >= 0.0)) ||
        !isfinite(c.mem_gb) || !isfinite(c.cold_ms) || (inf && !isfinite(c.slo_ms)))
      status = 2;
    else if (p.status != 0)
      status = 1;
    else if (train != (p.ibs == 0))                 // training session <-> training row
      status = 2;
    if (status == 0) {
      r.kind = c.kind;
      r.req_pm = p.req_pm;                                        // Q25 (profiler)
      r.lim_pm = p.lim_pm;
      r.mem_mib = q25_ceil(__dmul_rn(1024.0, c.mem_gb));           // Q25
      r.cold_slots = q25_ceil(__ddiv_rn(c.cold_ms, (double)slot_ms));
      if (train) {
        r.n_workers = c.n_workers;
        r.duty_pm = c.duty_pm;
      } else {
        r.ibs = p.ibs;
        const double cb = floor(__ddiv_rn(__dmul_rn((double)p.req_pm, c.slo_ms), 2.0));   // R4
        r.work_per_batch = cb >= 2147483647.0 ? 2147483647 : (int32_t)cb;
      }
    }
    out[i] = r;
    st[i] = status;
  }
}

}  // namespace prof
}  // namespace dilu
