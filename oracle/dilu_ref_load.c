/* dilu_ref_load.c -- oracle of the profile-table loader.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Plain C, one row at a time, in the
 * order the readings state them:
 *   PAPER.md s3.2: a function is profiled into <IBS, request, limit, memory> (P:606-610,
 *   Table 1); training request / limit = the SM rates reaching 80 % / 100 % of full
 *   throughput; inference request = the profiled SMR meeting SLO/2 at the chosen
 *   IBS, limit = 2 x request.  The profiler (dilu_ref_profile.c) already
 *   returns the Q25-rounded per-mille quotas; the loader adds
 *   Q25  mem_mib = ceil(1024 * GB), cold_slots = ceil(cold_ms / slot_ms)  (each the ceiling of
 *        the value minus 1e-9),
 *   R4   c_b = req_pm * SLO_ms / 2 tokens, rounded down (0 for training),
 * and copies the remaining fields.  Status 0 loaded, 1 profile failed, 2 catalogue row
 * invalid (both leave an unused row, kind -1). */
#include <math.h>
#include <string.h>

#include "dilu_ref.h"

enum { F_KIND, F_PRIO, F_IBS, F_REQ, F_LIM, F_MEM, F_CB, F_NW, F_DUTY, F_COLD, F_CLS, F_ARR,
       F_DEP, F_PAT, F_SCALE, F_PHASE };

static int32_t ceil_q25(double x) {
  double y = ceil(x - 1e-9);
  return y >= 2147483647.0 ? 2147483647 : (int32_t)y;
}

int32_t dilu_ref_load_one(const ref_catalog_row* c, const ref_prof_out* p, int32_t slot_ms,
                          int32_t* r) {
  int train = c->kind == 2;
  int inf = c->kind == 0 || c->kind == 1;
  int32_t status = 0;
  memset(r, 0, 16 * sizeof(int32_t));
  r[F_KIND] = -1;
  r[F_PRIO] = c->prio;
  r[F_NW] = 1;
  r[F_CLS] = c->affinity_class;
  r[F_ARR] = c->arrive_sec;
  r[F_DEP] = c->depart_sec;
  r[F_PAT] = c->pattern;
  r[F_SCALE] = c->scale_q10;
  r[F_PHASE] = c->phase_slots;
  if (!(train || inf) || !(c->mem_gb >= 0.0) || !(c->cold_ms >= 0.0) || !isfinite(c->mem_gb) ||
      !isfinite(c->cold_ms) || (inf && (!(c->slo_ms >= 0.0) || !isfinite(c->slo_ms))))
    status = 2;
  else if (p->status != 0)
    status = 1;
  else if (train != (p->ibs == 0))
    status = 2;
  if (status != 0) return status;
  r[F_KIND] = c->kind;
  r[F_REQ] = p->req_pm;
  r[F_LIM] = p->lim_pm;
  r[F_MEM] = ceil_q25(1024.0 * c->mem_gb);
  r[F_COLD] = ceil_q25(c->cold_ms / (double)slot_ms);
  if (train) {
    r[F_NW] = c->n_workers;
    r[F_DUTY] = c->duty_pm;
  } else {
    double cb = floor((double)p->req_pm * c->slo_ms / 2.0);
    r[F_IBS] = p->ibs;
    r[F_CB] = cb >= 2147483647.0 ? 2147483647 : (int32_t)cb;
  }
  return 0;
}

void dilu_ref_load_batch(int32_t n, const ref_catalog_row* c, const ref_prof_out* p,
                         int32_t slot_ms, int32_t* rows16, int32_t* status) {
  for (int32_t i = 0; i < n; ++i) status[i] = dilu_ref_load_one(&c[i], &p[i], slot_ms, rows16 + 16 * (size_t)i);
}
