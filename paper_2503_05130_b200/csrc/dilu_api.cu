// dilu_api.cu -- extern "C" boundary of libdilu.so (declared in include/dilu.h).
//
// Host responsibilities only: validate inputs, carve the caller's workspace, copy the
// inputs H->D on the caller's stream, pick the launch shape, launch the kernels of
// sim_kernel.cuh, surface deferred errors.  Every step of the provisioning loop runs
// on the device.
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "../../include/dilu.h"
#include "sim_kernel.cuh"
#include "profile.cuh"
#include "variants.h"

using namespace dilu;

struct dilu_sim {
  dilu_config cfg;
  int engine;          // 0: CTA per scenario, 2: cluster per scenario
  int K;               // cluster engine: CTAs per scenario group
  int Kc;              // cluster engine: CTAs per hardware cluster (K = m * Kc)
  Layout L;
  Params P;
  cudaStream_t stream;
  uint8_t* ws;
  size_t ws_bytes;
  int64_t* d_sum;      // [NT + 1] scratch (last word: max error code)
  int32_t* d_next;     // persistent-CTA scenario counter
  int grid;            // persistent CTAs per launch
  int32_t t;
  int32_t status;
  bool use_smem;
  int threads;
  std::vector<int8_t> kind;   // host copy of every function row's kind (place_batch validation)
  char err[512];
};

namespace {

constexpr size_t ALIGN = 256;
inline size_t up(size_t x) { return (x + ALIGN - 1) & ~(ALIGN - 1); }

struct Carve {
  size_t funcs, pat, scen, state, ring, tally, stats, gscr, lat, sum, total;
};

bool check_cfg(const dilu_config* c, char* msg, size_t n) {
#define BAD(...) do { snprintf(msg, n, __VA_ARGS__); return false; } while (0)
  if (!c) BAD("config is NULL");
  if (c->n_scenarios < 1) BAD("n_scenarios must be >= 1");
  if (c->gpus_per_scenario < 1 || c->gpus_per_scenario > 32767)
    BAD("gpus_per_scenario must be in [1, 32767] on this implementation");
  if (c->max_funcs < 1) BAD("max_funcs must be >= 1");
  if (c->max_instances < 1 || c->max_instances > (1 << 24)) BAD("max_instances out of range");
  if (c->q_pm != 1000) BAD("q_pm must be 1000 (R1)");
  if (c->mem_mib < 1 || c->mem_mib > (1 << 20)) BAD("mem_mib must be in [1, 2^20] (R7)");
  if (c->alpha_w < 0 || c->alpha_w > 255 || c->beta_w < 0 || c->beta_w > 255 ||
      c->alpha_w + c->beta_w == 0)
    BAD("alpha_w, beta_w must be in [0, 255] and not both 0 (R7)");
  if (c->slot_ms < 1 || c->slot_ms > 1000 || 1000 % c->slot_ms != 0) BAD("slot_ms must divide 1000");
  if ((c->flags & 4) && c->slot_ms % 5 != 0) BAD("Alg.2 periods (flags bit2) need slot_ms %% 5 == 0");
  if (c->window_s < 1 || c->phi_out < 1 || c->phi_out > c->window_s || c->phi_in < 0 ||
      c->phi_in >= c->window_s || c->phi_out + c->phi_in <= c->window_s)
    BAD("window: need 1<=phi_out<=W, 0<=phi_in<W, phi_out+phi_in>W (S:455)");
  if (c->min_instances < 1) BAD("min_instances must be >= 1");
  if (c->max_residents != RES) BAD("max_residents must be 32");
  if (c->max_llm_stages < 1 || c->max_llm_stages > MAXST) BAD("max_llm_stages must be in [1, 4]");
  if (c->n_patterns < 0 || c->pattern_len < 1) BAD("pattern table shape invalid");
  return true;
#undef BAD
}

bool check_inputs(const dilu_config* c, const dilu_scenario* scen, const dilu_func* fn,
                  const int32_t* pat, char* msg, size_t n) {
#define BAD(...) do { snprintf(msg, n, __VA_ARGS__); return false; } while (0)
  const size_t np = (size_t)c->n_patterns * c->pattern_len;
  if (np && !pat) BAD("patterns is NULL");
  for (size_t k = 0; k < np; ++k) if (pat[k] < 0) BAD("pattern %zu: negative arrivals", k / c->pattern_len);
  if (!fn) BAD("funcs is NULL");
  for (int32_t s = 0; s < c->n_scenarios; ++s) {
    const int32_t om = scen ? scen[s].omega_pm : c->omega_pm;
    const int32_t ga = scen ? scen[s].gamma_pm : c->gamma_pm;
    if (om < 1 || om > c->q_pm) BAD("scenario %d: omega_pm must be in [1, q_pm] (Q12)", s);
    if (ga < om) BAD("scenario %d: gamma_pm < omega_pm", s);
    const int32_t mode = scen ? scen[s].mode : 0;
    if (mode < 0 || mode > 4) BAD("scenario %d: mode must be in [0, 4]", s);
    for (int32_t f = 0; f < c->max_funcs; ++f) {
      const dilu_func& F = fn[(size_t)s * c->max_funcs + f];
      if (F.kind == K_UNUSED) continue;
      if (F.kind < K_INF || F.kind > K_TRAIN) BAD("scenario %d func %d: kind", s, f);
      if (F.prio != 0 && F.prio != 1) BAD("scenario %d func %d: prio", s, f);
      if (F.req_pm < 1 || F.lim_pm < F.req_pm || F.lim_pm > c->q_pm)
        BAD("scenario %d func %d: need 1 <= req_pm <= lim_pm <= q_pm", s, f);
      if ((int64_t)F.req_pm * RES < om) BAD("scenario %d func %d: req_pm < ceil(omega/32) (Q23)", s, f);
      if (F.req_pm > om || F.lim_pm > ga) BAD("scenario %d func %d: quota above Omega/gamma", s, f);
      if ((mode == 2 || mode == 4) && F.lim_pm > om)
        BAD("scenario %d func %d: limit above Omega (limit-quota baseline mode)", s, f);
      if (F.mem_mib < 1 || F.mem_mib > c->mem_mib) BAD("scenario %d func %d: mem_mib", s, f);
      if (F.cold_slots < 0) BAD("scenario %d func %d: cold_slots", s, f);
      if (F.arrive_sec < 0 || F.depart_sec <= F.arrive_sec) BAD("scenario %d func %d: lifecycle", s, f);
      if (F.kind == K_TRAIN) {
        if (F.n_workers < 1 || F.n_workers > c->gpus_per_scenario || F.n_workers > 64)
          BAD("scenario %d func %d: n_workers", s, f);
        if (F.duty_pm < 0 || F.duty_pm > 1000) BAD("scenario %d func %d: duty_pm", s, f);
      } else {
        if (F.ibs < 1) BAD("scenario %d func %d: ibs", s, f);
        const int64_t req_tok = (int64_t)F.req_pm * c->slot_ms;
        if (F.work_per_batch < 1 || F.work_per_batch > req_tok)
          BAD("scenario %d func %d: need 1 <= c_b <= req_tok (R4)", s, f);
        if (F.pattern < 0 || F.pattern >= c->n_patterns) BAD("scenario %d func %d: pattern", s, f);
        if (F.scale_q10 < 0 || F.phase_slots < 0) BAD("scenario %d func %d: scale/phase", s, f);
      }
    }
  }
  return true;
#undef BAD
}

// Engine choice (a pure function of the config and the DILU_ENGINE hook): one CTA per
// scenario for G <= 256 (state staged in shared memory), a thread-block cluster per
// scenario above.
int choose_engine(const dilu_config* c) {
  int e = c->gpus_per_scenario > 256 ? 2 : 0;   // large scenarios: a cluster each
  if (const char* v = getenv("DILU_ENGINE")) {
    if (!strcmp(v, "cta")) e = 0;
    if (!strcmp(v, "cluster")) e = 2;
  }
  return e;
}
// Fused-batch length: with sub-second slots the SPS slots between two
// second boundaries share one placement state, so P0/P1/P2 run once per batch of up to
// 16 slots.  DILU_BATCH=n (1..16) is a tuning/test hook; 1 runs every slot separately.
int choose_batch(const dilu_config* c) {
  const int sps = 1000 / c->slot_ms;
  int b = sps < 16 ? sps : 16;
  if (const char* v = getenv("DILU_BATCH")) {
    const int x = atoi(v);
    if (x >= 1 && x <= 16) b = x < sps ? x : sps;
  }
  return b < 1 ? 1 : b;
}

// Kernel variant for a handle: bit0 fused sub-second batches, bit1 literal Alg.2 periods,
// bit2 request-level latency (instantiated in run_variants.cu, see variants.h).
int variant_of(const dilu_config* c, const Layout& L) {
  return (L.B > 1 ? 1 : 0) | ((c->flags & 4) ? 2 : 0) | ((c->flags & 8) ? 4 : 0);
}
RunFn run_fn(bool smem, int var) {
  switch ((var & 7) >> 1) {
    case 0: return smem ? run_fn_smem_group0(var) : run_fn_gmem_group0(var);
    case 1: return smem ? run_fn_smem_group1(var) : run_fn_gmem_group1(var);
    case 2: return smem ? run_fn_smem_group2(var) : run_fn_gmem_group2(var);
    default: return smem ? run_fn_smem_group3(var) : run_fn_gmem_group3(var);
  }
}
ClusterFn cluster_fn(int var) {
  switch ((var & 7) >> 1) {
    case 0: return cluster_fn_group0(var);
    case 1: return cluster_fn_group1(var);
    case 2: return cluster_fn_group2(var);
    default: return cluster_fn_group3(var);
  }
}

Carve carve(const dilu_config* c, const Layout& L) {
  Carve k;
  size_t o = 0;
  const size_t S = c->n_scenarios, F = c->max_funcs;
  k.funcs = o; o = up(o + S * F * sizeof(dilu_func));
  k.pat = o; o = up(o + (size_t)c->n_patterns * c->pattern_len * 4);
  k.scen = o; o = up(o + S * 16);
  k.state = o; o = up(o + S * L.bytes);
  k.ring = o; o = up(o + S * F * c->window_s * 4);
  k.tally = o; o = up(o + S * NT * 8);
  k.stats = o; o = up(o + S * NSTAT * 8);
  k.gscr = o; o = up(o + S * GSCR * 8);
  k.lat = o; o = up(o + ((c->flags & 8) ? S * NLAT * 8 : 0));
  k.sum = o; o = up(o + (NT + 2) * 8);
  k.total = o;
  return k;
}

dilu_status fail(dilu_sim* s, dilu_status code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(s->err, sizeof s->err, fmt, ap);
  va_end(ap);
  if (code == DILU_E_CUDA || code == DILU_E_CAPACITY || code == DILU_E_INVARIANT) s->status = code;
  return code;
}

dilu_status cuda_check(dilu_sim* s, cudaError_t e, const char* what) {
  if (e == cudaSuccess) return DILU_OK;
  return fail(s, DILU_E_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

__global__ void k_sum_err(Params P, int64_t* out, int with_err) {
  const int k = threadIdx.x;
  if (k < NT) {
    unsigned long long s = 0;
    for (int32_t i = 0; i < P.S; ++i) s += (unsigned long long)P.tally[(size_t)i * NT + k];
    out[k] = (long long)s;
  } else if (k == NT && with_err) {
    int32_t e = 0;
    for (int32_t i = 0; i < P.S; ++i) {
      const int32_t x = reinterpret_cast<const int32_t*>(P.state + (size_t)i * P.L.bytes + P.L.hdr)[H_ERR];
      e = x > e ? x : e;
    }
    out[NT] = e;
  }
}

dilu_status launch_run(dilu_sim* s, int32_t n_slots, int32_t n_req, const int32_t* rs,
                       const int32_t* rf, int32_t* og, int32_t* oi) {
  dilu_status rc = cuda_check(s, cudaMemsetAsync(s->d_next, 0, sizeof(int32_t), s->stream), "counter reset");
  if (rc) return rc;
  const dim3 grid(s->grid), block(s->threads);
  if (s->engine == 2) {
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(s->cfg.n_scenarios * s->K);
    lc.blockDim = dim3(s->threads);
    lc.dynamicSmemBytes = 0;
    lc.stream = s->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = s->Kc;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    rc = cuda_check(s, cudaLaunchKernelEx(&lc, cluster_fn(variant_of(&s->cfg, s->L)), s->P, s->t, n_slots, n_req, rs, rf, og, oi),
                    "k_run_cluster launch");
    if (rc) return rc;
    return cuda_check(s, cudaGetLastError(), "k_run_cluster");
  }
  const RunFn fn = run_fn(s->use_smem, variant_of(&s->cfg, s->L));
  fn<<<grid, block, s->use_smem ? s->L.hot_bytes : 0, s->stream>>>(s->P, s->d_next, s->t, n_slots, n_req, rs, rf, og, oi);
  return cuda_check(s, cudaGetLastError(), "k_run launch");
}

}  // namespace

extern "C" {

size_t dilu_workspace_bytes(const dilu_config* cfg) {
  char msg[256];
  if (!check_cfg(cfg, msg, sizeof msg)) return 0;
  const Layout L = make_layout(cfg->gpus_per_scenario, cfg->max_funcs, cfg->max_instances,
                               cfg->window_s, choose_batch(cfg), (cfg->flags & 4) != 0,
                               (cfg->flags & 8) != 0);
  return carve(cfg, L).total;
}

dilu_status dilu_sim_create(const dilu_config* cfg, const dilu_scenario* h_scen,
                            const dilu_func* h_funcs, const int32_t* h_patterns,
                            void* d_workspace, size_t ws_bytes, void* cuda_stream,
                            dilu_sim** out) {
  if (!out) return DILU_E_USAGE;
  *out = nullptr;
  char msg[512];
  if (!check_cfg(cfg, msg, sizeof msg) || !check_inputs(cfg, h_scen, h_funcs, h_patterns, msg, sizeof msg)) {
    fprintf(stderr, "dilu_sim_create: %s\n", msg);
    return DILU_E_USAGE;
  }
  dilu_sim* s = new (std::nothrow) dilu_sim();
  if (!s) return DILU_E_USAGE;
  s->cfg = *cfg;
  s->stream = reinterpret_cast<cudaStream_t>(cuda_stream);
  s->L = make_layout(cfg->gpus_per_scenario, cfg->max_funcs, cfg->max_instances, cfg->window_s,
                     choose_batch(cfg), (cfg->flags & 4) != 0, (cfg->flags & 8) != 0);
  const Carve k = carve(cfg, s->L);
  if (!d_workspace || ws_bytes < k.total || (reinterpret_cast<uintptr_t>(d_workspace) % ALIGN)) {
    fprintf(stderr, "dilu_sim_create: workspace needs %zu bytes, 256-byte aligned (got %zu)\n",
            k.total, ws_bytes);
    delete s;
    return DILU_E_USAGE;
  }
  s->ws = reinterpret_cast<uint8_t*>(d_workspace);
  s->ws_bytes = ws_bytes;
  s->d_sum = reinterpret_cast<int64_t*>(s->ws + k.sum);
  s->d_next = reinterpret_cast<int32_t*>(s->d_sum + NT + 1);
  *out = s;

  const size_t S = cfg->n_scenarios, F = cfg->max_funcs;
  try { s->kind.resize(S * F); } catch (...) { return fail(s, DILU_E_USAGE, "out of host memory"); }
  for (size_t i = 0; i < S * F; ++i) s->kind[i] = (int8_t)h_funcs[i].kind;
  // H->D copies of the inputs (caller's stream)
  dilu_status rc;
  if ((rc = cuda_check(s, cudaMemcpyAsync(s->ws + k.funcs, h_funcs, S * F * sizeof(dilu_func),
                                          cudaMemcpyHostToDevice, s->stream), "copy funcs")))
    return rc;
  const size_t np = (size_t)cfg->n_patterns * cfg->pattern_len;
  if (np && (rc = cuda_check(s, cudaMemcpyAsync(s->ws + k.pat, h_patterns, np * 4,
                                                cudaMemcpyHostToDevice, s->stream), "copy patterns")))
    return rc;
  // per-scenario parameters (host-side defaulting only)
  int32_t* hs = new (std::nothrow) int32_t[S * 4];
  if (!hs) return fail(s, DILU_E_USAGE, "out of host memory");
  for (size_t i = 0; i < S; ++i) {
    hs[i * 4 + 0] = h_scen ? h_scen[i].scenario_id : (int32_t)i;
    hs[i * 4 + 1] = h_scen ? h_scen[i].omega_pm : cfg->omega_pm;
    hs[i * 4 + 2] = h_scen ? h_scen[i].gamma_pm : cfg->gamma_pm;
    hs[i * 4 + 3] = h_scen ? h_scen[i].mode : 0;
  }
  rc = cuda_check(s, cudaMemcpyAsync(s->ws + k.scen, hs, S * 16, cudaMemcpyHostToDevice, s->stream),
                  "copy scenarios");
  cudaError_t se = cudaStreamSynchronize(s->stream);  // hs is pageable and freed next
  delete[] hs;
  if (rc) return rc;
  if ((rc = cuda_check(s, se, "sync after copies"))) return rc;

  Params& P = s->P;
  P.funcs = reinterpret_cast<const int32_t*>(s->ws + k.funcs);
  P.pat = reinterpret_cast<const int32_t*>(s->ws + k.pat);
  P.scen = reinterpret_cast<const int32_t*>(s->ws + k.scen);
  P.state = s->ws + k.state;
  P.ring = reinterpret_cast<int32_t*>(s->ws + k.ring);
  P.tally = reinterpret_cast<int64_t*>(s->ws + k.tally);
  P.stats = reinterpret_cast<int64_t*>(s->ws + k.stats);
  P.gscratch = reinterpret_cast<unsigned long long*>(s->ws + k.gscr);
  P.lat = (cfg->flags & 8) ? reinterpret_cast<int64_t*>(s->ws + k.lat) : nullptr;
  P.L = s->L;
  P.S = cfg->n_scenarios; P.G = cfg->gpus_per_scenario; P.F = cfg->max_funcs;
  P.I = cfg->max_instances; P.W = cfg->window_s; P.M = cfg->mem_mib; P.Q = cfg->q_pm;
  P.aw = cfg->alpha_w; P.bw = cfg->beta_w; P.slot_ms = cfg->slot_ms; P.SPS = 1000 / cfg->slot_ms;
  P.phi_out = cfg->phi_out; P.phi_in = cfg->phi_in; P.min_inst = cfg->min_instances;
  P.max_stages = cfg->max_llm_stages; P.flags = cfg->flags; P.Tp = cfg->pattern_len;
  P.T_slot = 1000LL * cfg->slot_ms;
  P.ovl = 0;
  P.covl = 0;
  P.gK = 1;

  s->engine = choose_engine(cfg);
  int dev = 0;
  cudaGetDevice(&dev);
  if (s->engine == 2) {
    s->threads = 1024;
    if (const char* e = getenv("DILU_CTHREADS")) {   // tuning hook: threads per cluster CTA
      const int v = atoi(e);
      if (v >= 128 && v <= 1024 && v % 32 == 0) s->threads = v;
    }
    s->use_smem = false;
    if ((rc = cuda_check(s, cudaFuncSetAttribute(cluster_fn(variant_of(cfg, s->L)),
                                                 cudaFuncAttributeNonPortableClusterSizeAllowed, 1),
                         "cluster attribute")))
      return rc;
    int n_sm = 0;
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    // Scenario groups of K = m x Kc CTAs (m hardware clusters of Kc): the largest K that
    // keeps every scenario's group resident in one wave (the groups spin on scenario-wide
    // barriers), preferring larger clusters at equal K (the placement pass runs in the
    // leader's cluster with hardware cluster barriers).  DILU_CLUSTER (Kc) / DILU_GROUP (K)
    // are tuning / test hooks; results never depend on the shape.
    const int S = cfg->n_scenarios > 0 ? cfg->n_scenarios : 1;
    int want_kc = 0, want_k = 0;
    if (const char* e = getenv("DILU_CLUSTER")) want_kc = atoi(e);
    if (const char* e = getenv("DILU_GROUP")) want_k = atoi(e);
    int K = 0, Kc = 0, best_waves = 0;
    for (int kc = 16; kc >= 1; --kc) {
      if (want_kc > 0 && kc != want_kc) continue;
      cudaLaunchConfig_t lc = {};
      lc.gridDim = dim3(kc);
      lc.blockDim = dim3(s->threads);
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = kc; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      lc.attrs = at;
      lc.numAttrs = 1;
      int nclusters = 0;
      if (cudaOccupancyMaxActiveClusters(&nclusters, cluster_fn(variant_of(cfg, s->L)), &lc) != cudaSuccess || nclusters < 1) {
        cudaGetLastError();
        continue;
      }
      const int m_res = nclusters / S;           // clusters per scenario with every group resident
      // groups beyond 32-64 CTAs lose on C5 (one C5 scenario: 1,229 / 1,199 / 1,399 / 1,747
      // ms per step at 32 / 64 / 96 / 144 CTAs; 32 and 64 within box-to-box noise, DESIGN.md
      // s5: scenario-wide barriers cost more than the extra SMs save), so at most 32 unless
      // DILU_KCAP / DILU_GROUP ask; never more than fit at once -- the groups spin
      int cap = 32;                               // CTAs per scenario (tuning hook DILU_KCAP)
      if (const char* e = getenv("DILU_KCAP")) cap = atoi(e) > 0 ? atoi(e) : cap;
      int m = m_res < cap / kc ? m_res : (cap / kc > 0 ? cap / kc : 1);
      if (want_k > 0) m = want_k / kc < m_res ? want_k / kc : m_res;
      if (m * kc > KMAX) m = KMAX / kc;
      int waves = 1;
      if (m < 1) {                                // more scenarios than resident clusters:
        m = 1;                                    // one cluster each, in waves
        waves = (S + nclusters - 1) / nclusters;
      }
      const int k = m * kc;
      if (want_k > 0 && k != want_k) continue;
      // fewest waves, then the most CTAs per scenario, then the largest cluster
      const bool better = K == 0 || waves < best_waves ||
                          (waves == best_waves && (k > K || (k == K && kc > Kc)));
      if (better) { K = k; Kc = kc; best_waves = waves; }
    }
    if (K < 1) return fail(s, DILU_E_CUDA, "no schedulable cluster size");
    if (K > Kc && best_waves > 1) { K = Kc; }     // multi-cluster groups need one wave
    s->K = K;
    s->Kc = Kc;
    s->P.gK = K;
    P.gK = K;
    s->grid = cfg->n_scenarios * K;
    // Overlapped batches: the leader's cluster places while the other CTAs
    // run the batch.  Exact only if nothing placed at a boundary turns warm inside that
    // batch, i.e. every cold start >= one batch of slots.
    {
      bool cold_ok = true;
      const size_t nf = (size_t)cfg->n_scenarios * cfg->max_funcs;
      for (size_t i = 0; i < nf && cold_ok; ++i)
        if (h_funcs[i].kind != -1 && h_funcs[i].cold_slots < s->L.B) cold_ok = false;
      const char* e = getenv("DILU_NO_OVL");
      P.covl = cold_ok && variant_of(cfg, s->L) == 1 && K > Kc && s->L.B > 1 && !(e && atoi(e));
    }
    if (getenv("DILU_VERBOSE"))
      fprintf(stderr, "dilu: cluster engine group K=%d (clusters of %d) waves=%d covl=%d\n", K, Kc,
              best_waves, P.covl);
    return dilu_sim_reset(s);
  }
  // CTA engine launch shape: one CTA per scenario; hot state in shared memory when it fits
  int max_optin = 0;
  cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const size_t static_smem = sizeof(Red) + sizeof(Params) + 64;
  s->use_smem = s->L.hot_bytes + static_smem <= (size_t)max_optin;
  const int32_t G = cfg->gpus_per_scenario;
  // Narrow state (ET<true>) for the shared-memory kernels when the sizes allow
  const bool nar = narrow_ok(G, cfg->max_funcs, cfg->max_instances, cfg->window_s);
  const Layout Ln = make_layout(G, cfg->max_funcs, cfg->max_instances, cfg->window_s, choose_batch(cfg),
                                (cfg->flags & 4) != 0, (cfg->flags & 8) != 0, true);
  if (nar) s->use_smem = Ln.hot_bytes + static_smem <= (size_t)max_optin;
  if (const char* e = getenv("DILU_NO_SMEM")) if (atoi(e)) s->use_smem = false;
  s->threads = G <= 256 && cfg->max_funcs <= 1024 ? 256 : (G <= 2048 ? 512 : 1024);
  if (s->use_smem && nar) {
    s->L = Ln;
    P.L = Ln;
  }
  // Shared-memory kernels: the thread count that maximises resident scenarios per SM over
  // per-scenario latency.  Latency per slot grows only slowly as threads shrink (C4:
  // 454 / 457 / 478 / 495 / 511 ms at 256 / 224 / 192 / 160 / 128 threads and 3 CTAs/SM,
  // DESIGN.md s7) while fewer threads and the narrow state let more scenarios share an SM.
  if (s->use_smem && G <= 256) {
    static const int cand[5] = {256, 224, 192, 160, 128};
    static const double lat[5] = {454, 457, 478, 495, 511};
    double best = 0.0;
    cudaFuncAttributes fa = {};
    if ((rc = cuda_check(s, cudaFuncGetAttributes(&fa, run_fn(true, variant_of(cfg, s->L))), "kernel attributes")))
      return rc;
    // (the one-slot-per-second kernel is compiled for 128 threads x 5 CTAs per SM)
    if (s->threads > fa.maxThreadsPerBlock) s->threads = fa.maxThreadsPerBlock & ~31;
    for (int k = 0; k < 5; ++k) {
      int per = 0;
      if (cand[k] > fa.maxThreadsPerBlock) continue;
      if ((rc = cuda_check(s, cudaFuncSetAttribute(run_fn(true, variant_of(cfg, s->L)),
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   (int)s->L.hot_bytes), "smem attribute")))
        return rc;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, run_fn(true, variant_of(cfg, s->L)), cand[k],
                                                        s->L.hot_bytes) != cudaSuccess) {
        cudaGetLastError();
        continue;
      }
      const double score = per / lat[k];
      if (score > best * 1.0001) { best = score; s->threads = cand[k]; }
    }
  }
  // test hooks: outputs must not depend on the launch shape
  if (const char* e = getenv("DILU_THREADS")) {
    const int v = atoi(e);
    if (v >= 32 && v <= 1024 && v % 32 == 0) s->threads = v;
  }
  if (s->threads > SMEM_MAX_THREADS) s->use_smem = false;
  if (!s->use_smem && s->L.N) {            // back to the wide state for the global kernels
    s->L = make_layout(G, cfg->max_funcs, cfg->max_instances, cfg->window_s, choose_batch(cfg),
                       (cfg->flags & 4) != 0, (cfg->flags & 8) != 0, false);
    P.L = s->L;
  }
  if (s->use_smem) {
    if ((rc = cuda_check(s, cudaFuncSetAttribute(run_fn(true, variant_of(cfg, s->L)),
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)s->L.hot_bytes), "smem attribute")))
      return rc;
  }
  // persistent grid: as many CTAs as can be co-resident, never more than scenarios
  int per_sm = 0, n_sm = 0;
  cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
  if (s->use_smem)
    rc = cuda_check(s, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, run_fn(true, variant_of(cfg, s->L)), s->threads,
                                                                     s->L.hot_bytes), "occupancy");
  else
    rc = cuda_check(s, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, run_fn(false, variant_of(cfg, s->L)), s->threads, 0),
                    "occupancy");
  if (rc) return rc;
  if (per_sm < 1) return fail(s, DILU_E_CUDA, "kernel cannot be resident with %d threads", s->threads);
  const long long cap = (long long)per_sm * n_sm;
  s->grid = (int)(cfg->n_scenarios < cap ? cfg->n_scenarios : cap);
  // Overlapped slots: warp 0 places while the other warps run P0/P1/P2.
  // Exact only if nothing placed in a slot is warm in it, i.e. every cold start >= 1 slot.
  {
    bool cold_ok = true;
    for (size_t i = 0; i < S * F && cold_ok; ++i)
      if (h_funcs[i].kind != -1 && h_funcs[i].cold_slots < 1) cold_ok = false;
    const char* e = getenv("DILU_NO_OVL");
    P.ovl = cold_ok && variant_of(cfg, s->L) == 0 && G <= WARP_PLACE_MAX && s->threads >= 64 &&
            !(e && atoi(e));

  }
  if (getenv("DILU_VERBOSE"))
    fprintf(stderr, "dilu: cta engine threads=%d smem=%d hot=%zu per_sm=%d grid=%d ovl=%d\n", s->threads,
            (int)s->use_smem, s->L.hot_bytes, per_sm, s->grid, P.ovl);
  if (const char* e = getenv("DILU_GRID")) {   // test/tuning hook: resident scenarios
    const int v = atoi(e);
    if (v >= 1 && v < s->grid) s->grid = v;
  }
  return dilu_sim_reset(s);
}

dilu_status dilu_sim_reset(dilu_sim* s) {
  if (!s) return DILU_E_USAGE;
  if (s->status == DILU_E_CUDA) return DILU_E_STATE;
  s->status = DILU_OK;
  s->t = 0;
  dilu_status rc = cuda_check(s, cudaMemsetAsync(s->P.state, 0, (size_t)s->cfg.n_scenarios * s->L.bytes, s->stream),
                              "state reset");
  if (rc) return rc;
  // the RPS rings too: the next-second evictee is prefetched before a window is full
  // (its value is only used once W samples exist) -- defined bytes for initcheck
  rc = cuda_check(s, cudaMemsetAsync(s->P.ring, 0, (size_t)s->cfg.n_scenarios * s->cfg.max_funcs * s->cfg.window_s * 4,
                                     s->stream), "ring reset");
  if (rc) return rc;
  // group scratch: the multi-cluster barrier counters start at zero
  rc = cuda_check(s, cudaMemsetAsync(s->P.gscratch, 0, (size_t)s->cfg.n_scenarios * GSCR * 8, s->stream),
                  "scratch reset");
  if (rc) return rc;
  if (s->L.N) k_init<true><<<s->cfg.n_scenarios, 256, 0, s->stream>>>(s->P);
  else k_init<false><<<s->cfg.n_scenarios, 256, 0, s->stream>>>(s->P);
  return cuda_check(s, cudaGetLastError(), "k_init launch");
}

// cfg.flags bit1: the state invariants after every call (k_check)
static dilu_status launch_check(dilu_sim* s) {
  if (!(s->cfg.flags & 2)) return DILU_OK;
  if (s->L.N)
    k_check<true><<<s->cfg.n_scenarios, 256, 0, s->stream>>>(s->P);
  else
    k_check<false><<<s->cfg.n_scenarios, 256, 0, s->stream>>>(s->P);
  return cuda_check(s, cudaGetLastError(), "k_check launch");
}

dilu_status dilu_place_batch(dilu_sim* s, int32_t n_req, const int32_t* d_req_scenario,
                             const int32_t* d_req_func, int32_t* d_out_gpu, int32_t* d_out_iid) {
  if (!s) return DILU_E_USAGE;
  if (s->status) return DILU_E_STATE;
  if (n_req < 0 || (n_req > 0 && (!d_req_scenario || !d_req_func || !d_out_gpu || !d_out_iid)))
    return fail(s, DILU_E_USAGE, "place_batch: bad request arrays");
  // request validation against the host copy of the function kinds kept at create: one
  // bulk copy of the two request arrays, one stream sync, no per-request round trips
  if (n_req > 0) {
    std::vector<int32_t> hs;
    try { hs.resize(2 * (size_t)n_req); } catch (...) { return fail(s, DILU_E_USAGE, "out of host memory"); }
    dilu_status rc = cuda_check(s, cudaMemcpyAsync(hs.data(), d_req_scenario, 4 * (size_t)n_req,
                                                   cudaMemcpyDeviceToHost, s->stream), "place_batch copy");
    if (!rc) rc = cuda_check(s, cudaMemcpyAsync(hs.data() + n_req, d_req_func, 4 * (size_t)n_req,
                                                cudaMemcpyDeviceToHost, s->stream), "place_batch copy");
    if (!rc) rc = cuda_check(s, cudaStreamSynchronize(s->stream), "place_batch sync");
    if (rc) return rc;
    for (int32_t j = 0; j < n_req; ++j) {
      const int32_t sc = hs[j], f = hs[n_req + j];
      const bool ok = sc >= 0 && sc < s->cfg.n_scenarios && f >= 0 && f < s->cfg.max_funcs &&
                      s->kind[(size_t)sc * s->cfg.max_funcs + f] != K_UNUSED;
      if (!ok) return fail(s, DILU_E_USAGE, "place_batch: request %d names an invalid scenario/function", j);
    }
  }
  const dilu_status rc = launch_run(s, 0, n_req, d_req_scenario, d_req_func, d_out_gpu, d_out_iid);
  return rc == DILU_OK ? launch_check(s) : rc;
}

dilu_status dilu_scale_step(dilu_sim* s, int32_t n_slots) {
  if (!s) return DILU_E_USAGE;
  if (s->status) return DILU_E_STATE;
  if (n_slots < 0) return fail(s, DILU_E_USAGE, "scale_step: n_slots < 0");
  if (n_slots == 0) return DILU_OK;
  dilu_status rc = launch_run(s, n_slots, -1, nullptr, nullptr, nullptr, nullptr);
  if (rc == DILU_OK) s->t += n_slots;
  if (rc == DILU_OK) rc = launch_check(s);
  return rc;
}

dilu_status dilu_metrics(dilu_sim* s, int64_t* per_scenario, int64_t* sum) {
  if (!s) return DILU_E_USAGE;
  if (s->status == DILU_E_CUDA) return DILU_E_STATE;
  k_sum_err<<<1, 32, 0, s->stream>>>(s->P, s->d_sum, 1);
  dilu_status rc = cuda_check(s, cudaGetLastError(), "k_sum launch");
  if (rc) return rc;
  int64_t host_sum[NT + 1];
  if ((rc = cuda_check(s, cudaMemcpyAsync(host_sum, s->d_sum, sizeof host_sum, cudaMemcpyDeviceToHost,
                                          s->stream), "copy sum")))
    return rc;
  if (per_scenario &&
      (rc = cuda_check(s, cudaMemcpyAsync(per_scenario, s->P.tally, (size_t)s->cfg.n_scenarios * NT * 8,
                                          cudaMemcpyDefault, s->stream), "copy per-scenario")))
    return rc;
  if ((rc = cuda_check(s, cudaStreamSynchronize(s->stream), "stream sync"))) return rc;
  if (sum && (rc = cuda_check(s, cudaMemcpy(sum, host_sum, NT * 8, cudaMemcpyDefault), "copy out")))
    return rc;
  if (host_sum[NT] == DILU_E_CAPACITY)
    return fail(s, DILU_E_CAPACITY, "a scenario exceeded max_instances=%d live instances",
                s->cfg.max_instances);
  if (host_sum[NT] == 2)
    return fail(s, DILU_E_INVARIANT, "a state invariant (I1/I2/I3/I7) failed on the device");
  if (host_sum[NT] != 0) return fail(s, DILU_E_INVARIANT, "scenario error code %lld", (long long)host_sum[NT]);
  if ((s->cfg.flags & 2) && host_sum[T_RTOT] != host_sum[T_RSRV] + host_sum[T_RVIO])   // I6
    return fail(s, DILU_E_INVARIANT, "I6: requests total != served + violated");
  return DILU_OK;
}

dilu_status dilu_snapshot(dilu_sim* s, int32_t id_cap, int32_t* d_gpu, int32_t* d_inst) {
  if (!s) return DILU_E_USAGE;
  if (s->status == DILU_E_CUDA) return DILU_E_STATE;
  if (id_cap < 0 || (id_cap > 0 && !d_inst && d_gpu == nullptr)) return fail(s, DILU_E_USAGE, "snapshot: bad args");
  if (s->L.N)
    k_snapshot<true><<<s->cfg.n_scenarios, 256, 0, s->stream>>>(s->P, id_cap, d_gpu, id_cap > 0 ? d_inst : nullptr);
  else
    k_snapshot<false><<<s->cfg.n_scenarios, 256, 0, s->stream>>>(s->P, id_cap, d_gpu, id_cap > 0 ? d_inst : nullptr);
  dilu_status rc = cuda_check(s, cudaGetLastError(), "k_snapshot launch");
  if (rc) return rc;
  return cuda_check(s, cudaStreamSynchronize(s->stream), "snapshot sync");
}

dilu_status dilu_kernel_stats(dilu_sim* s, int64_t* per_scenario, int64_t* sum) {
  if (!s) return DILU_E_USAGE;
  if (s->status == DILU_E_CUDA) return DILU_E_STATE;
  const size_t n = (size_t)s->cfg.n_scenarios * NSTAT;
  int64_t* h = new (std::nothrow) int64_t[n];
  if (!h) return fail(s, DILU_E_USAGE, "out of host memory");
  dilu_status rc = cuda_check(s, cudaMemcpyAsync(h, s->P.stats, n * 8, cudaMemcpyDeviceToHost, s->stream),
                              "copy stats");
  if (!rc) rc = cuda_check(s, cudaStreamSynchronize(s->stream), "stats sync");
  if (!rc) {
    int64_t acc[NSTAT] = {0};
    for (size_t i = 0; i < n; ++i) acc[i % NSTAT] += h[i];
    if (per_scenario) rc = cuda_check(s, cudaMemcpy(per_scenario, h, n * 8, cudaMemcpyDefault), "stats out");
    if (!rc && sum) rc = cuda_check(s, cudaMemcpy(sum, acc, sizeof acc, cudaMemcpyDefault), "stats sum");
  }
  delete[] h;
  return rc;
}

dilu_status dilu_latency(dilu_sim* s, int64_t* per_scenario, int64_t* sum) {
  if (!s) return DILU_E_USAGE;
  if (s->status == DILU_E_CUDA) return DILU_E_STATE;
  if (!(s->cfg.flags & 8)) return fail(s, DILU_E_USAGE, "latency: cfg.flags bit3 not set");
  const size_t n = (size_t)s->cfg.n_scenarios * NLAT;
  int64_t* h = new (std::nothrow) int64_t[n];
  if (!h) return fail(s, DILU_E_USAGE, "out of host memory");
  dilu_status rc = cuda_check(s, cudaMemcpyAsync(h, s->P.lat, n * 8, cudaMemcpyDeviceToHost, s->stream),
                              "copy latency");
  if (!rc) rc = cuda_check(s, cudaStreamSynchronize(s->stream), "latency sync");
  if (!rc) {
    int64_t acc[NLAT] = {0};
    for (size_t i = 0; i < n; ++i) acc[i % NLAT] += h[i];
    if (per_scenario) rc = cuda_check(s, cudaMemcpy(per_scenario, h, n * 8, cudaMemcpyDefault), "latency out");
    if (!rc && sum) rc = cuda_check(s, cudaMemcpy(sum, acc, sizeof acc, cudaMemcpyDefault), "latency sum");
  }
  delete[] h;
  return rc;
}

int32_t dilu_current_slot(const dilu_sim* s) { return s ? s->t : -1; }

const char* dilu_last_error(const dilu_sim* s) { return s ? s->err : "null handle"; }

void dilu_sim_destroy(dilu_sim* s) { delete s; }

dilu_status dilu_profile(const dilu_prof_session* d_sessions, int32_t n, dilu_prof_out* d_out,
                         void* cuda_stream) {
  if (n < 0 || (n > 0 && (!d_sessions || !d_out))) return DILU_E_USAGE;
  if ((reinterpret_cast<uintptr_t>(d_sessions) | reinterpret_cast<uintptr_t>(d_out)) & 7)
    return DILU_E_USAGE;
  if (n == 0) return DILU_OK;
  int dev = 0, n_sm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
  const int per = 8;                          // resident 256-thread CTAs per SM (regs permitting)
  long long blocks = (n + 255) / 256;
  if (blocks > (long long)n_sm * per) blocks = (long long)n_sm * per;
  prof::k_profile<<<(int)blocks, 256, 0, reinterpret_cast<cudaStream_t>(cuda_stream)>>>(d_sessions, n, d_out);
  return cudaGetLastError() == cudaSuccess ? DILU_OK : DILU_E_CUDA;
}

dilu_status dilu_load_profiles(const dilu_catalog_row* d_cat, const dilu_prof_out* d_prof,
                               int32_t n, int32_t slot_ms, dilu_func* d_out, int32_t* d_status,
                               void* cuda_stream) {
  if (n < 0 || slot_ms < 1 || slot_ms > 1000 || (n > 0 && (!d_cat || !d_prof || !d_out || !d_status)))
    return DILU_E_USAGE;
  if (n == 0) return DILU_OK;
  int dev = 0, n_sm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
  long long blocks = (n + 255) / 256;
  if (blocks > (long long)n_sm * 8) blocks = (long long)n_sm * 8;
  prof::k_load<<<(int)blocks, 256, 0, reinterpret_cast<cudaStream_t>(cuda_stream)>>>(d_cat, d_prof, n, slot_ms,
                                                                                    d_out, d_status);
  return cudaGetLastError() == cudaSuccess ? DILU_OK : DILU_E_CUDA;
}

}  // extern "C"
