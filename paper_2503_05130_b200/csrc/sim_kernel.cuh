// sim_kernel.cuh -- the B200 megakernel for the batched Dilu provisioning loop.
//
// Grid: one CTA per scenario (scenarios are independent); the CTA runs
// every slot of the call.  Per slot:
//   boundary (t % SPS == 0):
//     B1  function-parallel: window push + incremental lazy-scaling counts and
//         decisions, departure/arrival flags; ordered compaction of the
//         functions with an event
//     B3  thread 0 applies events in the paper's order: departures, ScaleOut/In,
//         arrivals (ids assigned at enqueue)
//     B4  FIFO placement pass, Alg.1: per instance, every thread scores a
//         stride of GPUs with a packed 64-bit key (tier | fit | id), block min, thread
//         0 commits.  LLM worst-fit split by <=4 block argmax rounds.
//     B5  repack GPU rows into warp chunks when the residency changed
//   P0  function-parallel: arrivals A_f(t), even dispatch over warm instances
//   P1  warp chunks of GPU rows (rows of width w in {1..32} lanes): slot-level Alg.2
//       allocation a = req + min(want, max(0, S_g - prefix)) with width-w segmented
//       shuffles, executed batches, hash, gang/stage minima via shared atomics
//   P2  function-parallel: training gangs (barrel effect) and LLM stage minima
// Tallies accumulate in registers and are block-reduced once per call.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "state.cuh"

namespace dilu {

// rare paths (capacity errors, LLM splits, lifecycle events, window recounts): laid out
// away from the per-slot code, whose instruction footprint matters
#define DILU_UNLIKELY(x) __builtin_expect(!!(x), 0)

#ifndef DILU_HOT_SMEM
#define DILU_HOT_SMEM 0
#endif
// the shared-memory CTA kernels use the narrow state (ET<true>); everything else the wide
typedef ViewT<DILU_HOT_SMEM != 0> View;

struct Params {
  const int32_t* funcs;      // [S][F][16] input rows
  const int32_t* pat;        // [P][Tp]
  const int32_t* scen;       // [S][4]
  uint8_t* state;            // [S][L.bytes]
  int32_t* ring;             // [S][F][W]
  int64_t* tally;            // [S][NT]
  int64_t* stats;            // [S][NSTAT] kernel statistics
  unsigned long long* gscratch;  // [S][GSCR] cluster-collective scratch
  int64_t* lat;              // [S][NLAT] request-level latency (cfg.flags bit3), else null
  Layout L;
  int32_t S, G, F, I, W, M, Q, aw, bw, slot_ms, SPS, phi_out, phi_in, min_inst, max_stages,
      flags, Tp;
  int32_t ovl;               // overlapped slots: CTA engine, VAR 0, G <= 256, cold >= 1
  int32_t covl;              // overlapped batches: cluster engine, VAR 1, K > Kc, every cold start >= one batch
  int32_t gK;                // cluster engine: CTAs per scenario group (a multiple of the cluster size)
  int64_t T_slot;
};

constexpr int KMAX = 160;    // CTAs per scenario group (multi-cluster groups)
constexpr int GSCR = 4 * KMAX + 48;   // u64 words of per-scenario group scratch

struct Acc0 {  // thread-0 tallies, kept in shared memory (not in every thread's registers)
  long long act, memu, rows, pok, pfail, cold, sout, sin, split, maxa;
  long long st[NSTAT];   // statistics: attempts, hope checks, relayouts, events, scanned, slots
  unsigned long long sum[9];   // end-of-call block sums of the per-thread tallies (Acc)
};
enum { S_ATTEMPT = 0, S_HOPE, S_LAYOUT, S_EVENT, S_SCAN, S_SLOT, S_RES, S_FUN };
struct Acc {   // per-thread tallies
  long long rtot, rsrv, rvio, iexe, tprg, etot;
  unsigned long long hash;
  int32_t nres, nfun;   // statistics: warm resident-slots (P1), inference function-slots (P0)
  Acc0* z;     // shared, written by thread 0 only
};

static __device__ __forceinline__ uint64_t sm64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static __device__ __forceinline__ uint64_t mix5(uint32_t scn, uint32_t t, uint32_t i, uint32_t g,
                                         uint32_t a) {
  uint64_t h = sm64(scn);
  h = sm64(h ^ t);
  h = sm64(h ^ i);
  return sm64(h ^ ((uint64_t(g) << 32) | a));
}

// ---------------------------------------------------------------- block helpers

struct Red {                 // reduction scratch (static shared)
  unsigned long long u64[2][32];
  int32_t i32[2][33];
  int32_t flag[2];           // [0] next queue entry / scenario counter, [1] queue length
  unsigned long long lat[NLAT];   // request-level latency of this call (cfg.flags bit3)
  int32_t members[64];       // gang member slots of the request being placed
  Acc0 z;
};

// One-sync block min; double-buffered so back-to-back calls do not race.
static __device__ __forceinline__ unsigned long long block_min_u64(unsigned long long v, Red& r,
                                                            int& phase) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long y = __shfl_xor_sync(0xffffffffu, v, o);
    v = y < v ? y : v;
  }
  unsigned long long* buf = r.u64[phase];
  phase ^= 1;
  if (lane == 0) buf[wid] = v;
  __syncthreads();
  unsigned long long m = lane < nw ? buf[lane] : ~0ull;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long y = __shfl_xor_sync(0xffffffffu, m, o);
    m = y < m ? y : m;
  }
  return m;
}

// One-sync block exclusive scan of int32; returns exclusive prefix, *total.
static __device__ __forceinline__ int32_t block_scan_i32(int32_t v, Red& r, int& phase,
                                                  int32_t* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  int32_t* buf = r.i32[phase];
  phase ^= 1;
  if (lane == 31) buf[wid] = x;
  __syncthreads();
  int32_t before = 0, tot = 0;
  for (int k = 0; k < nw; ++k) {
    if (k < wid) before += buf[k];
    tot += buf[k];
  }
  *total = tot;
  return before + x - v;
}

#ifdef DILU_BOUNDS
constexpr int DILU_ID_MEMBERS = 82;   // index of "members" in DILU_ARRAY_NAMES
static __device__ __noinline__ void dilu_oob(int id, long long j, long long n) {
  const char* names[] = {DILU_ARRAY_NAMES};
  printf("DILU_BOUNDS: %s[%lld] outside [0, %lld) (block %d thread %d)\n",
         id >= 0 && id <= DILU_ID_MEMBERS ? names[id] : "?", j, n, (int)blockIdx.x, (int)threadIdx.x);
  __trap();
}
#endif

// ------------------------------------------------------------------ groups
//
// The threads that run one scenario: one CTA (K = 1), or a thread-block cluster of K
// CTAs (large scenarios, state in HBM/L2).  Cluster-wide collectives are the CTA-level
// ones followed by one hardware cluster barrier (release/acquire, which also makes the
// other CTAs' global writes visible) over a small per-scenario global scratch.

static __device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
               ::: "memory");
}

// Scenario-wide barrier across several clusters (multi-cluster groups): one
// arrival per CTA on a per-scenario counter in global memory, the last arrival advances
// the generation; every thread then fences (acquire at GPU scope) so it observes the other
// CTAs' state writes -- the pattern of a cooperative grid sync, restricted to the scenario.
static __device__ __noinline__ void group_barrier(unsigned int* cnt, unsigned int* gen, int K) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int g;
    asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(g) : "l"(gen) : "memory");
    __threadfence();
    if (atomicAdd(cnt, 1u) == (unsigned)K - 1) {
      *cnt = 0;
      __threadfence();
      asm volatile("st.release.gpu.u32 [%0], %1;" :: "l"(gen), "r"(g + 1) : "memory");
    } else {
      unsigned int x;
      long long spins = 0;
      do {
        __nanosleep(64);
        asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(x) : "l"(gen) : "memory");
        if (++spins > (1ll << 24)) __trap();   // a group not resident as a whole: fail, do not hang
      } while (x == g);
    }
  }
  __syncthreads();
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
}

struct Grp {
  int K, crank, cph;
  int Kc;                    // CTAs per hardware cluster (K = m * Kc clusters of the scenario)
  int off;                   // threads [0, off) sit out (overlapped slots: warp 0 places)
  int sub;                   // > 0: the group minus its first `sub` CTAs (overlapped batches)
  unsigned long long* gu;    // [2][KMAX] group scratch (u64)
  int32_t* gi;               // [2][KMAX] group scratch (i32)
  unsigned int* bar;         // [2] multi-cluster barrier: arrivals, generation
  __device__ int rank() const { return crank * blockDim.x + threadIdx.x - off; }
  __device__ int size() const { return K * blockDim.x - off; }
  __device__ int wrank() const { return (crank * blockDim.x + threadIdx.x - off) >> 5; }
  __device__ int nwarps() const { return (K * blockDim.x - off) >> 5; }
  __device__ bool leader() const { return crank == 0 && threadIdx.x == 0; }
  __device__ bool lead_warp() const { return crank == 0 && threadIdx.x < 32; }
  __device__ void sync() const {
#if DILU_HOT_SMEM            // the shared-memory kernels run one CTA per scenario
    __syncthreads();
#else
    if (K == 1) __syncthreads();
    else if (K == Kc) cluster_sync_all();
    else if (sub) group_barrier(bar + 2, bar + 3, K - sub);   // own counter: runs beside the leader cluster
    else group_barrier(bar, bar + 1, K);
#endif
  }
  // the leader's hardware cluster alone (the placement pass of multi-cluster groups)
  __device__ Grp first_cluster() const { Grp g = *this; g.K = Kc; return g; }
};

// ------------------------------------------------------------------ scenario

struct Scn {
  const Params* P;           // the kernel's __grid_constant__ parameter (constant bank)
  uint8_t* gblock;           // this scenario's state block (cold region)
  uint8_t* hot;              // its hot region: the shared-memory copy or gblock
  int32_t* ring;             // this scenario's RPS rings [F][W]
  const View* sv;            // DILU_VMODE 1/2: the view built once per scenario in shared memory
  Grp g;
  DPN(int32_t) members;      // gang member slots of the request being placed (group-visible, [64])
  int32_t* flag;             // group-visible broadcast word
  Acc0* z;                   // leader tallies (shared)
  const int32_t* frow;       // this scenario's input function rows [F][16]
  unsigned long long* lat;   // request-level latency accumulator (shared, [NLAT])
  int32_t scn_id, om, ga, mode;   // mode: baseline (0 Dilu, 1 Exclusive, 2 MPS-l, 3 MPS-r, 4 eager)
  int32_t b1lo, b1hi;        // B1: this thread's contiguous function range (fixed per call)
  // The view of the state, rebuilt where it is used: every array address is the Layout's
  // offset (constant bank) from the dynamic shared memory (hot arrays, DILU_HOT_SMEM units)
  // or from gblock -- no loads, nothing kept in shared memory or local memory.
  __device__ __forceinline__ View view() const {
    View v = make_view<DILU_HOT_SMEM != 0>(hot, gblock, P->L);
#ifdef DILU_BOUNDS
    v.ring = Chk<int32_t>(ring, (long long)P->F * P->W, v.ring.id);
#else
    v.ring = ring;
#endif
    return v;
  }
};
enum : int32_t { M_DILU = 0, M_EXCLUSIVE = 1, M_STATIC_LIMIT = 2, M_STATIC_REQUEST = 3, M_EAGER = 4 };
// literal Algorithm 2 at 5 ms periods (cfg.flags bit2; D8)
enum : int32_t { A2_NONE = 0, A2_EMERGENCY = 1, A2_RECOVERY = 2, A2_CONTENTION = 3 };
constexpr int32_t A2_PERIOD_MS = 5, A2_MAX_TOKENS = 5000, A2_ETA_V = 300, A2_RW = 20;
constexpr int32_t A2_NEVER = -(1 << 30);

static __device__ __forceinline__ int st_of(int32_t meta) { return meta & 3; }
static __device__ __forceinline__ int nst_of(int32_t meta) { return (meta >> 4) & 7; }
static __device__ __forceinline__ bool is_inf(int32_t k) { return k == K_INF || k == K_LLM; }

// ---- group collectives (K = 1: CTA-level; K > 1: CTA-level then one cluster barrier) --

static __device__ unsigned long long g_min_u64(Scn& c, unsigned long long v, Red& red, int& ph) {
  v = block_min_u64(v, red, ph);
  if (c.g.K == 1) return v;
  unsigned long long* buf = c.g.gu + (c.g.cph & 1) * KMAX;
  if (threadIdx.x == 0) buf[c.g.crank] = v;
  c.g.cph ^= 1;
  c.g.sync();                    // cluster barrier, or the scenario-wide one
  unsigned long long m = ~0ull;
  for (int k = 0; k < c.g.K; ++k) { const unsigned long long x = __ldcg(buf + k); m = x < m ? x : m; }
  return m;
}
static __device__ int32_t g_sum_i32(Scn& c, int32_t cta_value) {   // cta_value uniform within the CTA
  if (c.g.K == 1) return cta_value;
  int32_t* buf = c.g.gi + (c.g.cph & 1) * KMAX;
  if (threadIdx.x == 0) buf[c.g.crank] = cta_value;
  c.g.cph ^= 1;
  c.g.sync();                    // cluster barrier, or the scenario-wide one
  int32_t r = 0;
  for (int k = 0; k < c.g.K; ++k) r += __ldcg(buf + k);
  return r;
}
static __device__ bool g_any(Scn& c, bool p) { return g_sum_i32(c, __syncthreads_or(p)) != 0; }
static __device__ int32_t g_count(Scn& c, int p) { return g_sum_i32(c, __syncthreads_count(p)); }
static __device__ int32_t g_scan(Scn& c, int32_t v, Red& red, int& ph, int32_t* total) {
  int32_t ctot;
  const int32_t pre = block_scan_i32(v, red, ph, &ctot);
  if (c.g.K == 1) { *total = ctot; return pre; }
  int32_t* buf = c.g.gi + (c.g.cph & 1) * KMAX;
  if (threadIdx.x == 0) buf[c.g.crank] = ctot;
  c.g.cph ^= 1;
  c.g.sync();                    // cluster barrier, or the scenario-wide one
  int32_t before = 0, tot = 0;
  for (int k = 0; k < c.g.K; ++k) {
    const int32_t x = __ldcg(buf + k);
    if (k < c.g.crank) before += x;
    tot += x;
  }
  *total = tot;
  return before + pre;
}

// ---- hot-region view ------------------------------------------------------------------
// In translation units compiled with DILU_HOT_SMEM=1 (the k_run<true, *> kernels: the hot
// region staged in shared memory) every hot-region array of the view is an SPtr
// (state.cuh) that asserts the shared window at each use, so the compiler emits
// LDS/STS/ATOMS.  Functions work through a reference to the one shared View.
#ifndef DILU_HOT_SMEM
#define DILU_HOT_SMEM 0
#endif
#if DILU_VMODE == 1 && DILU_HOT_SMEM && !defined(DILU_BOUNDS)
// mode 1: a register copy of the shared view whose hot pointers carry the shared-window
// assertion (LDS/STS); the pointers are shared addresses by construction (run_scenario).
static __device__ __forceinline__ View hot_view(const View& s) {
  View v = s;
#define DILU_A(p) __builtin_assume(__isShared(v.p))
  DILU_A(h); DILU_A(gR); DILU_A(gL); DILU_A(gU); DILU_A(gRel); DILU_A(rlG); DILU_A(rlE);
  DILU_A(gN); DILU_A(gNs); DILU_A(gExcl); DILU_A(gRes); DILU_A(gGrow); DILU_A(gMask); DILU_A(gChk);
  DILU_A(iId); DILU_A(iReady); DILU_A(iR); DILU_A(iFunc); DILU_A(iNext); DILU_A(fstack); DILU_A(iMeta);
  DILU_A(fKind); DILU_A(fPrio); DILU_A(fNw); DILU_A(fReq); DILU_A(fLim); DILU_A(fCb); DILU_A(fIbs);
  DILU_A(fCls); DILU_A(fDtr); DILU_A(fPat); DILU_A(fScale); DILU_A(fCap1); DILU_A(fReg); DILU_A(fNsamp);
  DILU_A(fHead); DILU_A(fUp); DILU_A(fDown); DILU_A(fFlag); DILU_A(fThrn); DILU_A(fNlive); DILU_A(fAcc);
  DILU_A(fOld); DILU_A(fPv); DILU_A(fGang); DILU_A(fK); DILU_A(fArr); DILU_A(fDep); DILU_A(fPidx);
  DILU_A(fLh); DILU_A(fLt); DILU_A(fList); DILU_A(fInfL); DILU_A(fDefL); DILU_A(qN); DILU_A(qFail);
  DILU_A(qSlot); DILU_A(iQ);
#undef DILU_A
  return v;
}
#else
static __device__ __forceinline__ const View& hot_view(const View& s) { return s; }
#endif
#if DILU_VMODE == 0        // rebuilt from the Layout in the kernel parameter
#define DILU_VIEW(v, c) const View v = (c).view()
#elif DILU_VMODE == 1      // register copy of the shared view, hot pointers asserted shared
#define DILU_VIEW(v, c) const View v = hot_view(*(c).sv)
#else                      // the shared view itself (SPtr offsets)
#define DILU_VIEW(v, c) const View& v = *(c).sv
#endif
typedef DPN(int32_t) GP32;   // a generic (shared or global) int32 array
#define DILU_CVIEW(v, c) DILU_VIEW(v, c)

// Asynchronous 4-byte global -> shared copies (no register staging): the next second's
// evicted ring sample (B1) and the next slot's pattern value (P0) land in the hot state
// while the slot runs, so neither global load sits on a phase's critical path.  Each thread
// consumes only what it issued (same function mapping every slot) after cp.async.wait_all.
static __device__ __forceinline__ void cp_async4(int32_t* sdst, const int32_t* gsrc) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" :: "r"(s), "l"(gsrc) : "memory");
}
static __device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;" ::: "memory");
}
static __device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N> static __device__ __forceinline__ void cp_async_wait_group() {
  asm volatile("cp.async.wait_group %0;" :: "n"(N) : "memory");
}


// Serial helpers the leader / warp 0 call from several places (event application,
// placement, rollback): one out-of-line copy each keeps the code the SM executes per
// slot small -- with several resident scenarios per SM at different points of the slot,
// inlined copies thrash the instruction cache (ncu "no_instruction" stalls).
#ifndef DILU_SERIAL_INLINE
#define DILU_SERIAL __forceinline__
#else
#define DILU_SERIAL __forceinline__
#endif
// ---- serial helpers (thread 0 only) ------------------------------------------------

static __device__ void list_append(const View& v, int32_t f, int32_t s) {
  v.iNext[s] = -1;
  __threadfence_block();   // pipelined slots: P0/P2 may walk the list meanwhile; the node
                           // (pending, next = -1) is complete before it becomes reachable
  if (v.fLt[f] < 0) v.fLh[f] = s; else v.iNext[v.fLt[f]] = s;
  v.fLt[f] = s;
}
static __device__ DILU_SERIAL void list_remove(Scn& c, int32_t f, int32_t s) {
  DILU_VIEW(v, c);
  int32_t prev = -1, cur = v.fLh[f];
  #pragma unroll 1
  while (cur >= 0 && cur != s) { prev = cur; cur = v.iNext[cur]; }
  if (cur < 0) return;
  int32_t nx = v.iNext[cur];
  if (prev < 0) v.fLh[f] = nx; else v.iNext[prev] = nx;
  if (v.fLt[f] == s) v.fLt[f] = prev;
}

// resident order key: (prio, id) -- SLO-sensitive first (Alg.2)
static __device__ __forceinline__ long long res_key(const View& v, int32_t s) {
  return ((long long)v.fPrio[v.iFunc[s]] << 32) | (uint32_t)v.iId[s];
}

static __device__ DILU_SERIAL void commit(Scn& c, int32_t s, int32_t g, int32_t share) {
  DILU_VIEW(v, c);
  // every value read before any write: the reads are independent, so they overlap (the
  // rows are in HBM/L2 on the cluster engine, where each dependent read is a round trip)
  const int32_t f = v.iFunc[s];
  const int32_t n0 = v.gN[g], R0 = v.gR[g], L0 = v.gL[g], U0 = v.gU[g];
  const unsigned long long m0 = v.gMask[g];
  const int32_t fr = v.fReq[f], fl = v.fLim[f], fc = v.fCls[f], meta = v.iMeta[s];
  const int32_t nact = v.h[H_NACT], sumu = v.h[H_SUMU];
  if (n0 == 0) v.h[H_NACT] = nact + 1;
  v.gMask[g] = m0 | (1ull << (fc & 63));
  v.gR[g] = R0 + fr;
  v.gL[g] = L0 + fl;
  v.gU[g] = U0 + share;
  v.h[H_SUMU] = sumu + share;
  const auto res = v.gRes + (size_t)g * RES;
  int pos = n0;
#if !DILU_HOT_SMEM
  const auto rcl = v.gRcl + (size_t)g * RES;   // (wide layout) classes beside the residents
#endif
  if (DILU_UNLIKELY(!(c.P->ovl | c.P->covl))) {   // keep (prio, id) order now ...
    const long long k = res_key(v, s);
    #pragma unroll 1
    while (pos > 0 && res_key(v, res[pos - 1]) > k) {
      res[pos] = res[pos - 1];
#if !DILU_HOT_SMEM
      rcl[pos] = rcl[pos - 1];
#endif
      --pos;
    }
  }                           // ... or append (overlapped slots: rows below gNs never move
  res[pos] = s;               // while P1 reads them; the next repack sorts the row)
#if !DILU_HOT_SMEM
  rcl[pos] = fc;
#endif
  v.gN[g] = n0 + 1;
  const int k0 = nst_of(meta);
  v.iG[s * MAXST + k0] = (int16_t)g;
  v.iShare[s * MAXST + k0] = share;
  if (k0 == 0) v.iSh0[s] = share;
  if (DILU_UNLIKELY(c.P->flags & 4)) {   // Alg.2 stage state starts fresh (D8)
    const int32_t e = s * MAXST + k0;
    v.aTc[e] = 0; v.aTm[e] = 0; v.aRl[e] = 0; v.aLe[e] = A2_NEVER;
  }
  v.iMeta[s] = (meta & ~(7 << 4)) | ((k0 + 1) << 4);
  v.gExcl[g] = 1;             // I* of the request in flight (Q7)
  v.h[H_DIRTY] = 1;
}

static __device__ DILU_SERIAL void release(Scn& c, int32_t s) {
  DILU_VIEW(v, c);
  const int32_t f = v.iFunc[s];
  const int32_t meta = v.iMeta[s];
  const int n = nst_of(meta);
  #pragma unroll 1
  for (int k = 0; k < n; ++k) {
    const int32_t g = v.iG[s * MAXST + k];
    const int32_t sh = k == 0 ? v.iSh0[s] : v.iShare[s * MAXST + k];
    v.gR[g] -= v.fReq[f];
    v.gL[g] -= v.fLim[f];
    v.gU[g] -= sh;
    v.h[H_SUMU] -= sh;
    const auto res = v.gRes + (size_t)g * RES;
    int j = 0;
    const int nr = v.gN[g];
    #pragma unroll 1
    while (j < nr && res[j] != s) ++j;
#if !DILU_HOT_SMEM
    const auto rcl = v.gRcl + (size_t)g * RES;
    #pragma unroll 1
    for (; j + 1 < nr; ++j) { res[j] = res[j + 1]; rcl[j] = rcl[j + 1]; }
#else
    #pragma unroll 1
    for (; j + 1 < nr; ++j) res[j] = res[j + 1];
#endif
    v.gN[g] = nr - 1;
    if (nr - 1 == 0) v.h[H_NACT] -= 1;
    unsigned long long m = 0;
#if !DILU_HOT_SMEM
    #pragma unroll 1
    for (int x = 0; x < nr - 1; ++x) m |= 1ull << (rcl[x] & 63);
#else
    #pragma unroll 1
    for (int x = 0; x < nr - 1; ++x) m |= 1ull << (v.fCls[v.iFunc[res[x]]] & 63);
#endif
    v.gMask[g] = m;
    v.iG[s * MAXST + k] = -1;
  }
  v.iMeta[s] = meta & ~(7 << 4);
  v.h[H_DIRTY] = 1;
}

// terminate a live instance (placed or pending); frees its slot
#if defined(DILU_PHASE_TIMING) && DILU_PHASE_TIMING != 2
#define TSTART long long _t0 = clock64()
#define TSTOP(k) do { if (c.g.leader()) c.z->st[k] += clock64() - _t0; } while (0)
#else
#define TSTART do { } while (0)
#define TSTOP(k) do { } while (0)
#endif
static __device__ DILU_SERIAL void terminate_impl(Scn& c, int32_t s);
static __device__ void terminate(Scn& c, int32_t s) {
  TSTART;
  terminate_impl(c, s);
  TSTOP(15);
}
static __device__ DILU_SERIAL void terminate_impl(Scn& c, int32_t s) {
  DILU_VIEW(v, c);
  const int32_t f = v.iFunc[s];
  if (st_of(v.iMeta[s]) == ST_PLACED) {
    const int32_t ep = ++v.h[H_EPOCH];   // room was freed: queued failures may now succeed
    const int ns = nst_of(v.iMeta[s]);
    #pragma unroll 1
    for (int k = 0; k < ns; ++k) {
      const int32_t g = v.iG[s * MAXST + k];
#ifdef DILU_TERM_PROBE
      if (g < 0 || g >= c.P->G)
        printf("TERM_PROBE scn %d s %d k %d ns %d g %d meta %d id %d func %d gRel %p iG %p iMeta %p sv.iG %p\n",
               c.scn_id, s, k, ns, g, v.iMeta[s], v.iId[s], v.iFunc[s], (void*)v.gRel, (void*)v.iG,
               (void*)v.iMeta, (void*)v.iG);
#endif
      v.gRel[g] = ep;
      const int32_t slot = v.h[H_RLN]++ % RLOG;
      v.rlG[slot] = g;
      v.rlE[slot] = ep;
    }
    release(c, s);
  }
  v.iMeta[s] = ST_FREE;
  list_remove(c, f, s);
  v.fNlive[f] -= 1;
  v.h[H_NLIVE] -= 1;
  v.fstack[v.h[H_FSTOP]++] = s;
}

static __device__ DILU_SERIAL void compact_queue(Scn& c) {
  DILU_VIEW(v, c);
  const int32_t n = v.h[H_QLEN];
  int32_t k = 0;
  #pragma unroll 1
  for (int32_t q = 0; q < n; ++q) {
    if (v.qN[q] == 0) continue;
    if (k != q) {
      v.qN[k] = v.qN[q]; v.qFail[k] = v.qFail[q];
      v.qSlot[k] = v.qSlot[q];
      v.iQ[v.qSlot[k]] = k;
    }
    ++k;
  }
  v.h[H_QLEN] = k;
}

// enqueue one request of n new instances of f; returns first id or -1 on capacity error
static __device__ DILU_SERIAL int32_t enqueue_impl(Scn& c, int32_t f, int32_t n);
static __device__ int32_t enqueue(Scn& c, int32_t f, int32_t n) {
  TSTART;
  const int32_t r = enqueue_impl(c, f, n);
  TSTOP(16);
  return r;
}
static __device__ DILU_SERIAL int32_t enqueue_impl(Scn& c, int32_t f, int32_t n) {
  DILU_VIEW(v, c);
  if (DILU_UNLIKELY(v.h[H_FSTOP] < n)) { v.h[H_ERR] = 6; return -1; }
  if (DILU_UNLIKELY(v.h[H_QLEN] == c.P->I)) {
    compact_queue(c);
    v.h[H_QNEWPOS] = 0;               // positions moved: the next pass scans everything
  }
  const int32_t first = v.h[H_NEXT_IID];
  const int32_t q = v.h[H_QLEN]++;
  v.h[H_QLIVE] += 1;
  if (v.h[H_QNEWPOS] < 0) v.h[H_QNEWPOS] = q;
  #pragma unroll 1
  for (int32_t j = 0; j < n; ++j) {
    const int32_t s = v.fstack[--v.h[H_FSTOP]];
    v.iId[s] = v.h[H_NEXT_IID]++;
    v.iFunc[s] = f;
    v.iMeta[s] = ST_PEND;
    v.iReady[s] = BIG;               // not ready until placed (read racily in overlapped slots)
    v.iQ[s] = q;                      // request index (single-instance kills are O(1))
    if (j == 0) v.qSlot[q] = s;
    #pragma unroll 1
    for (int k = 0; k < MAXST; ++k) v.iG[s * MAXST + k] = -1;
    if (c.P->SPS == 1) {
      v.iR[c.P->I + s] = BIG;         // stage-minimum half of iR (phase1); iBmin unused
    } else {
      v.iBmin[s] = BIG;
      v.iBmin[c.P->I + s] = BIG;
    }
    list_append(v, f, s);
    v.fNlive[f] += 1;
    v.h[H_NLIVE] += 1;
  }
  v.qN[q] = n; v.qFail[q] = -1;
  return first;
}

static __device__ DILU_SERIAL void register_func(Scn& c, int32_t f, int32_t t, int32_t Tp) {
  DILU_VIEW(v, c);
  if (v.fReg[f]) return;
  v.fReg[f] = 1;
  v.fNsamp[f] = 0; v.fAcc[f] = 0; v.fHead[f] = 0; v.fUp[f] = 0; v.fDown[f] = 0;
  v.fThrn[f] = -1;
  v.fPv[f] = -1;                     // no prefetched pattern value for the first slot
  v.fPidx[f] = (int32_t)(((long long)t + v.fPhase[f]) % Tp);   // arrivals index for slot t
}

static __device__ DILU_SERIAL void kill_queue_entries_of(Scn& c, int32_t f) {
  DILU_VIEW(v, c);
  const int32_t n = v.h[H_QLEN];
  #pragma unroll 1
  for (int32_t q = 0; q < n; ++q)
    if (v.qN[q] > 0 && v.iFunc[v.qSlot[q]] == f) { v.qN[q] = 0; v.h[H_QLIVE] -= 1; }
}

// ---- placement (collective) --------------------------------------------------------

// Placement primitives of the group (WARP = false: every thread of the CTA / cluster) or
// of warp 0 alone (WARP = true: CTA engine, G <= WARP_PLACE_MAX -- scoring 64..256 GPUs
// at 2..8 per lane beats three CTA barriers per attempt).
constexpr int WARP_PLACE_MAX = 256;
template <bool WARP> struct PlaceGrp;
template <> struct PlaceGrp<false> {
  static __device__ __forceinline__ int rank(const Scn& c) { return c.g.rank(); }
  static __device__ __forceinline__ int size(const Scn& c) { return c.g.size(); }
  static __device__ __forceinline__ bool leader(const Scn& c) { return c.g.leader(); }
  static __device__ __forceinline__ void sync(const Scn& c) { c.g.sync(); }
};
template <> struct PlaceGrp<true> {
  static __device__ __forceinline__ int rank(const Scn&) { return threadIdx.x; }
  static __device__ __forceinline__ int size(const Scn&) { return 32; }
  static __device__ __forceinline__ bool leader(const Scn&) { return threadIdx.x == 0; }
  static __device__ __forceinline__ void sync(const Scn&) { __syncwarp(); }
};
__device__ __forceinline__ unsigned long long warp_min_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long y = __shfl_xor_sync(0xffffffffu, v, o);
    v = y < v ? y : v;
  }
  return v;
}

// Algorithm 1 for one instance s with Principle 2's LLM split before a new
// GPU (Q11).  All threads of the placing group call; its leader commits.  Returns a
// uniform success flag.
template <bool WARP>
static __device__ bool place_one(Scn& c, Red& red, int& ph, int32_t s) {
  using PG = PlaceGrp<WARP>;
  DILU_VIEW(v, c);
  const Params& P = *c.P;
  const int32_t f = v.iFunc[s];
  const int32_t req = v.fReq[f], lim = v.fLim[f], mem = v.fMem[f], cls = v.fCls[f];
  const long long aM = (long long)P.aw * P.M, bQ = (long long)P.bw * P.Q;
  const unsigned long long MASK40 = (1ull << 40) - 1;
  unsigned long long best = ~0ull;
  #pragma unroll 1
  for (int32_t g = PG::rank(c); g < P.G; g += PG::size(c)) {
    if (v.gExcl[g]) continue;
    const int32_t n = v.gN[g];
    unsigned long long key;
    if (n == 0) {
      key = (2ull << 62) | (MASK40 << 22) | (unsigned long long)g;  // tier 2, K := 0
    } else if (c.mode == M_EXCLUSIVE) {
      continue;                          // pass-through: never share a GPU
    } else {
      const int32_t R = v.gR[g] + req, Lm = v.gL[g] + lim, U = v.gU[g] + mem;
      if (!(R <= c.om && Lm <= c.ga && U <= P.M && n < RES)) continue;
      // affinity: the class bitmask rules most GPUs out exactly; scan on a hit
      int aff = 0;
#if !DILU_HOT_SMEM
      const auto rcl = v.gRcl + (size_t)g * RES;   // one row of classes (wide layout)
      if ((v.gMask[g] >> (cls & 63)) & 1ull)
        #pragma unroll 1
        for (int j = 0; j < n && !aff; ++j) aff = (rcl[j] == cls);
#else
      const auto res = v.gRes + (size_t)g * RES;
      if ((v.gMask[g] >> (cls & 63)) & 1ull)
        #pragma unroll 1
        for (int j = 0; j < n && !aff; ++j) aff = (v.fCls[v.iFunc[res[j]]] == cls);
#endif
      const unsigned long long K = (unsigned long long)(aM * R + bQ * U);
      key = ((unsigned long long)(aff ? 0 : 1) << 62) | ((MASK40 - K) << 22) |
            (unsigned long long)g;
    }
    best = key < best ? key : best;
  }
  best = WARP ? warp_min_u64(best) : g_min_u64(c, best, red, ph);
  const int tier = best == ~0ull ? 3 : (int)(best >> 62);
  if (tier <= 1) {
    if (PG::leader(c)) commit(c, s, (int32_t)(best & 0x3FFFFF), mem);
    PG::sync(c);
    return true;
  }
  if (DILU_UNLIKELY(v.fKind[f] == K_LLM && (P.flags & 1) && c.mode != M_EXCLUSIVE)) {
    // worst-fit split: repeated argmax of free memory over active, cap-feasible GPUs
    int32_t picked[MAXST];
    int32_t pfree[MAXST];
    int k = 0;
    long long sum = 0;
    bool okk = false;
    #pragma unroll 1
    for (int r = 0; r < P.max_stages; ++r) {
      unsigned long long kk = ~0ull;
      #pragma unroll 1
      for (int32_t g = PG::rank(c); g < P.G; g += PG::size(c)) {
        const int32_t n = v.gN[g];
        if (n == 0 || v.gExcl[g] || n >= RES) continue;
        bool dup = false;
        #pragma unroll 1
        for (int j = 0; j < r; ++j) dup |= (picked[j] == g);
        if (dup) continue;
        if (v.gR[g] + req > c.om || v.gL[g] + lim > c.ga) continue;
        const int32_t fr = P.M - v.gU[g];
        if (fr <= 0) continue;
        const unsigned long long key =
            ((unsigned long long)(0xFFFFFFFFu - (uint32_t)fr) << 32) | (uint32_t)g;
        kk = key < kk ? key : kk;
      }
      kk = WARP ? warp_min_u64(kk) : g_min_u64(c, kk, red, ph);
      if (kk == ~0ull) break;
      picked[r] = (int32_t)(kk & 0xFFFFFFFFu);
      pfree[r] = (int32_t)(0xFFFFFFFFu - (uint32_t)(kk >> 32));
      sum += pfree[r];
      k = r + 1;
      if (sum >= mem) { okk = true; break; }
    }
    if (okk) {
      if (PG::leader(c)) {
        int32_t left = mem;
        #pragma unroll 1
        for (int j = 0; j < k; ++j) {
          const int32_t sh = pfree[j] < left ? pfree[j] : left;
          commit(c, s, picked[j], sh);
          left -= sh;
        }
      }
      PG::sync(c);
      return true;
    }
  }
  if (tier == 2) {
    if (PG::leader(c)) commit(c, s, (int32_t)(best & 0x3FFFFF), mem);
    PG::sync(c);
    return true;
  }
  return false;
}

// Can GPU g, released after a request of f last failed, now change that outcome?
// Non-LLM: g hosts one instance now (an emptied GPU always can).  LLM with split
// enabled: g is also a split candidate (caps hold, some free memory).
static __device__ __forceinline__ bool could_help(const Scn& c, int32_t g, int32_t f) {
  DILU_CVIEW(v, c);
  const Params& P = *c.P;
  const int32_t n = v.gN[g];
  if (n == 0) return true;
  if (n >= RES || v.gR[g] + v.fReq[f] > c.om || v.gL[g] + v.fLim[f] > c.ga) return false;
  if (v.gU[g] + v.fMem[f] <= P.M) return true;
  return v.fKind[f] == K_LLM && (P.flags & 1) && P.M - v.gU[g] > 0;
}

// Could any GPU released after epoch fe now host a request of f?  Walks the release
// log back to fe (usually 1-3 entries); falls back to scanning every GPU's last-release
// epoch when the log no longer covers fe.
static __device__ DILU_SERIAL bool hope_after(const Scn& c, int32_t fe, int32_t f) {
  DILU_CVIEW(v, c);
  const int32_t n = v.h[H_RLN];
  const int32_t lo = n > RLOG ? n - RLOG : 0;
  if (DILU_UNLIKELY(n > RLOG && v.rlE[lo % RLOG] > fe)) {
    #pragma unroll 1
    for (int32_t g = 0; g < c.P->G; ++g)
      if (v.gRel[g] > fe && could_help(c, g, f)) return true;
    return false;
  }
  #pragma unroll 1
  for (int32_t k = n - 1; k >= lo; --k) {
    if (v.rlE[k % RLOG] <= fe) break;
    if (could_help(c, v.rlG[k % RLOG], f)) return true;
  }
  return false;
}

// Warp 0 walks the queue from position q, 32 entries per step (lane per entry):
// requests that fail again by the skip rule are counted and stamped with the current
// epoch; returns the first entry that needs a real attempt, or qn.  Lane 0 is thread 0
// (owner of the thread-0 tallies).
static __device__ int32_t next_attempt(Scn& c, int32_t q, int32_t qn, Acc& acc) {
  DILU_VIEW(v, c);
  const int lane = threadIdx.x & 31;
  const int32_t ep = v.h[H_EPOCH];
  int32_t nfail = 0, found = qn, nhope = 0;
  #pragma unroll 1
  for (int32_t p = q; p < qn; p += 32) {
    const int32_t qq = p + lane;
    int cls = 0;                      // 0 dead/none, 1 fails again, 2 needs an attempt
    bool stamp = false;
    if (qq < qn && v.qN[qq] > 0) {
      const int32_t fe = v.qFail[qq];
      if (fe < 0) cls = 2;                       // never tried
      else if (fe == ep) cls = 1;                // nothing released since its failure
      else {
        ++nhope;
        cls = hope_after(c, fe, v.iFunc[v.qSlot[qq]]) ? 2 : 1;
        stamp = cls == 1;
      }
    }
    const unsigned m = __ballot_sync(0xffffffffu, cls == 2);
    const int first = m ? __ffs(m) - 1 : 32;
    const bool before = lane < first;
    nfail += __popc(__ballot_sync(0xffffffffu, cls == 1 && before));
    if (stamp && before) v.qFail[qq] = ep;
    if (m) { found = p + first; break; }
  }
  for (int o = 16; o > 0; o >>= 1) nhope += __shfl_xor_sync(0xffffffffu, nhope, o);
  if (lane == 0) {
    acc.z->pfail += nfail;
    acc.z->st[S_HOPE] += nhope;
    acc.z->st[S_SCAN] += 1;
  }
  return found;
}

// One FIFO pass over the queue (Q8, Q9).
// Retry skip (exact): a request that failed at release epoch E saw every
// GPU unable to host it (and no inactive GPU).  Afterwards, GPUs without a release only
// fill up, so the request can succeed again only through a GPU g released after E that
// could host it now (gang: the count of hosting GPUs only grows through such g; LLM:
// the top-4 free memory only grows through such g).  If no such g exists it fails
// again without rescoring, exactly as the oracle's full rescoring would.
// Entered without a group barrier after B3 (the leader's serial event pass): only warp 0
// (which contains the leader) reads the queue before the first barrier below, and it
// broadcasts the queue length with the first attempt index.
template <bool WARP>
static __device__ void placement_pass(Scn& c, Red& red, int& ph, int32_t t, Acc& acc) {
  using PG = PlaceGrp<WARP>;
  DILU_VIEW(v, c);
  int32_t qn = 0;
  bool removed = false;                 // leader only
  int32_t q = 0, prev = -1, prev_placed = 0;
  #pragma unroll 1
  for (;;) {
    // One warp-0 section per attempt: finish the previous request (leader), find the next
    // request needing a real attempt (warp 0, 32 entries per step), gather its members
    // (leader); then a single group barrier.
    TSTART;
    if (WARP || c.g.lead_warp()) {
      if (WARP && prev >= 0)                  // clear I* marks: every lane clears a stride
        #pragma unroll 1
        for (int32_t g = threadIdx.x; g < c.P->G; g += 32) v.gExcl[g] = 0;   // (no iG loads)
      if (PG::leader(c) && prev >= 0) {
        const int32_t n = v.qN[prev], f = v.iFunc[v.qSlot[prev]];
        if (!WARP)
          #pragma unroll 1
          for (int j = 0; j < prev_placed; ++j) {   // clear I* marks
            const int32_t s = c.members[j];
            const int ns = nst_of(v.iMeta[s]);
            #pragma unroll 1
            for (int k = 0; k < ns; ++k) v.gExcl[v.iG[s * MAXST + k]] = 0;
          }
        if (prev_placed == n) {
          const int32_t cold = v.fCold[f];
          #pragma unroll 1
          for (int j = 0; j < n; ++j) {
            const int32_t s = c.members[j];
            v.iMeta[s] = (v.iMeta[s] & ~3) | ST_PLACED;
            v.iReady[s] = t + cold;
            acc.z->pok += 1;
            if (is_inf(v.fKind[f]) && cold > 0) acc.z->cold += 1;
            if (nst_of(v.iMeta[s]) > 1) acc.z->split += 1;
          }
          v.qN[prev] = 0;
          v.h[H_QLIVE] -= 1;
          removed = true;
        } else {
          #pragma unroll 1
          for (int j = 0; j < prev_placed; ++j) release(c, c.members[j]);  // rollback
          acc.z->pfail += 1;
          v.qFail[prev] = v.h[H_EPOCH];
        }
      }
      __syncwarp();
      if (prev < 0) {                   // pass start, after B3 (same warp)
        qn = v.h[H_ERR] ? 0 : v.h[H_QLEN];
        // Every request still queued at the end of the last pass fails on that pass's
        // final state.  With no release since (same epoch) the state has only filled,
        // so those requests fail again without rescoring: count them and start at the
        // first request enqueued since (all of which are live).  Exact, DESIGN.md s5.
        if (v.h[H_LASTEP] == v.h[H_EPOCH]) {
          const int32_t np = v.h[H_QNEWPOS];
          q = np < 0 ? qn : np;             // np == 0: positions moved, scan all
          if (threadIdx.x == 0 && q > 0) acc.z->pfail += v.h[H_QLIVE] - (qn - q);
        }
      }
      const int32_t e = next_attempt(c, q, qn, acc);
      if (PG::leader(c)) {
        c.flag[0] = e;
        c.flag[1] = qn;
        if (e < qn) {                   // gang members, ascending id
          const int32_t n = v.qN[e], s0 = v.qSlot[e];
          if (n == 1) {
            c.members[0] = s0;          // a single instance: the queue holds its slot
          } else {
            const int32_t f = v.iFunc[s0], first = v.iId[s0];
            int j = 0;
            #pragma unroll 1
            for (int32_t s = v.fLh[f]; s >= 0 && j < n; s = v.iNext[s]) {
              const int32_t id = v.iId[s];
              if (id >= first && id < first + n) c.members[j++] = s;
            }
          }
          acc.z->st[S_ATTEMPT] += 1;
        }
      }
    }
    PG::sync(c);
    TSTOP(17);
    q = c.g.K == 1 ? c.flag[0] : __ldcg(c.flag);
    qn = c.g.K == 1 ? c.flag[1] : __ldcg(c.flag + 1);
    if (q >= qn) break;
    const int32_t n = v.qN[q];
    int placed = 0;
    {
      TSTART;
      #pragma unroll 1
      for (int j = 0; j < n; ++j) {
        if (!place_one<WARP>(c, red, ph, c.g.K == 1 ? c.members[j] : __ldcg(c.members + j))) break;
        ++placed;
      }
      TSTOP(18);
    }
    prev = q;
    prev_placed = placed;
    ++q;
  }
  if (PG::leader(c)) {
    if (removed) compact_queue(c);
    v.h[H_LASTEP] = v.h[H_EPOCH];
    v.h[H_QNEWPOS] = -1;
  }
}

// The placement pass by the cheapest group: warp 0 alone for CTA-engine scenarios with
// few GPUs (then one CTA barrier publishes its commits), else the whole group.
// Multi-cluster groups place within the leader's hardware cluster alone (fast cluster
// barriers per attempt); the other clusters wait at one scenario-wide barrier.
static __device__ void placement(Scn& c, Red& red, int& ph, int32_t t, Acc& acc) {
  if (c.g.K == 1 && c.P->G <= WARP_PLACE_MAX) {
    if (threadIdx.x < 32) placement_pass<true>(c, red, ph, t, acc);
    __syncthreads();
#if !DILU_HOT_SMEM
  } else if (c.g.K > c.g.Kc) {
    if (c.g.crank < c.g.Kc) {
      Scn cp = c;
      cp.g = c.g.first_cluster();
      placement_pass<false>(cp, red, ph, t, acc);
    }
    c.g.sync();
#endif
  } else {
    placement_pass<false>(c, red, ph, t, acc);
  }
}

// ---- B5: pack GPU rows into 32-lane warp chunks by width class (1..32 lanes) ----------

static __device__ __forceinline__ int width_class(int32_t n) {
  return n <= 1 ? 0 : 32 - __clz(n - 1);
}

static __device__ void rebuild_layout(Scn& c) {
  DILU_VIEW(v, c);
  const Params& P = *c.P;
  if (c.g.crank == 0 && threadIdx.x < 6) { v.h[H_CCNT + threadIdx.x] = 0; v.h[H_CCNT2 + threadIdx.x] = 0; }
  c.g.sync();
  #pragma unroll 1
  for (int32_t g = c.g.rank(); g < P.G; g += c.g.size()) {
    const int32_t n = v.gN[g];
    if ((P.ovl | P.covl) && n > 1) {   // overlapped slots / batches append commits: restore (prio, id) order
      const auto res = v.gRes + (size_t)g * RES;
      long long kp = res_key(v, res[0]);
      #pragma unroll 1
      for (int j = 1; j < n; ++j) {
        const int32_t s = res[j];
        const long long k = res_key(v, s);
        if (k > kp) { kp = k; continue; }
        int pos = j;
#if !DILU_HOT_SMEM
        const auto rcl = v.gRcl + (size_t)g * RES;
        const int32_t cj = rcl[j];
        #pragma unroll 1
        while (pos > 0 && res_key(v, res[pos - 1]) > k) { res[pos] = res[pos - 1]; rcl[pos] = rcl[pos - 1]; --pos; }
        rcl[pos] = cj;
#else
        #pragma unroll 1
        while (pos > 0 && res_key(v, res[pos - 1]) > k) { res[pos] = res[pos - 1]; --pos; }
#endif
        res[pos] = s;
      }
    }
    v.gNs[g] = n;
    if (n > 0) atomicAdd(&v.h[H_CCNT + width_class(n)], 1);
  }
  c.g.sync();
  if (c.g.leader()) {
    int32_t cb = 0, gb = 0;
    #pragma unroll 1
    for (int k = 0; k < 6; ++k) {
      v.h[H_CBASE + k] = cb;
      v.h[H_GBASE + k] = gb;
      const int32_t per = 32 >> k;
      cb += (v.h[H_CCNT + k] + per - 1) / per;
      gb += v.h[H_CCNT + k];
    }
    v.h[H_CBASE + 6] = cb;
    v.h[H_DIRTY] = 0;
  }
  c.g.sync();
  #pragma unroll 1
  for (int32_t g = c.g.rank(); g < P.G; g += c.g.size()) {
    const int32_t n = v.gN[g];
    if (n > 0) {
      const int k = width_class(n);
      const int32_t idx = atomicAdd(&v.h[H_CCNT2 + k], 1);
      v.gGrow[v.h[H_GBASE + k] + idx] = g;   // order inside a class is irrelevant
    }
  }
  // one descriptor per warp chunk: its first row in gGrow, its row count, its width class
  const int32_t nch = v.h[H_CBASE + 6];
  #pragma unroll 1
  for (int32_t ch = c.g.rank(); ch < nch; ch += c.g.size()) {
    int k = 0;
    #pragma unroll
    for (int x = 1; x < 6; ++x) k += (ch >= v.h[H_CBASE + x]);
    const int32_t per = 32 >> k, i0 = (ch - v.h[H_CBASE + k]) * per;
    const int32_t nv = min(per, v.h[H_CCNT + k] - i0);
    v.gChk[ch] = (v.h[H_GBASE + k] + i0) | (nv << 16) | (k << 24);
  }
  c.g.sync();
}

// ---- request-level latency (cfg.flags bit3; D10) ----------
static __device__ __forceinline__ int lat_bucket(long long L) {   // 4 log buckets per octave (us)
  if (L < 4) return L < 0 ? 0 : (int)L;
  const int h = 63 - __clzll(L);
  const int b = 4 * h + (int)((L >> (h - 2)) & 3) - 4;
  return b < 78 ? b : 78;
}

// One instance-slot: r requests arriving at floor(j*T/r) us, ceil(r/IBS) batches ready at
// their last arrival, the first b running back to back for e us each; per-request
// latencies go to the shared histogram (runs of equal buckets flushed once), unserved
// requests to bucket LAT_UNSERVED.  Arrival times advance by quotient/remainder steps, so
// only one division per batch remains.
static __device__ void lat_instance(unsigned long long* lat, int32_t r, int32_t ibs, int32_t b, long long e,
                             int32_t slo, long long T) {
  if (r <= 0) return;
  const int32_t served = (long long)b * ibs < r ? b * ibs : r;
  const long long q0 = T / r, r0 = T % r;
  long long sum = 0, viol = 0, tq = 0, tr = 0, prev = 0;   // tau_j = tq (+ tr/r)
  int cur = -1;
  unsigned long long cnt = 0;
  for (int32_t j0 = 0; j0 < served; j0 += ibs) {
    const int32_t j1 = j0 + ibs < r ? j0 + ibs : r;
    const long long ready = (long long)(j1 - 1) * T / r;
    const long long done = (ready > prev ? ready : prev) + e;
    for (int32_t j = j0; j < j1; ++j) {
      const long long L = done - tq;
      const int bk = lat_bucket(L);
      if (bk != cur) {
        if (cnt) atomicAdd(&lat[cur], cnt);
        cur = bk;
        cnt = 0;
      }
      ++cnt;
      sum += L;
      viol += L > slo;
      tq += q0;
      tr += r0;
      if (tr >= r) { tr -= r; ++tq; }
    }
    prev = done;
  }
  if (cnt) atomicAdd(&lat[cur], cnt);
  const int32_t uns = r - served;
  if (uns) atomicAdd(&lat[LAT_UNSERVED], (unsigned long long)uns);
  viol += uns;
  if (viol) atomicAdd(&lat[LAT_VIOL], (unsigned long long)viol);
  if (sum) atomicAdd(&lat[LAT_SUM], (unsigned long long)sum);
}

static __device__ __forceinline__ void lat_unserved(unsigned long long* lat, int32_t A) {
  if (A > 0) { atomicAdd(&lat[LAT_UNSERVED], (unsigned long long)A); atomicAdd(&lat[LAT_VIOL], (unsigned long long)A); }
}

// batch time of one stage: ceil(c_stage * T / a) us (<= T whenever a batch runs)
static __device__ __forceinline__ int32_t lat_e(int32_t cst, int32_t a, long long T) {
  if (a <= 0) return 0;
  const long long e = ((long long)cst * T + a - 1) / a;
  return e < 0x7fffffffLL ? (int32_t)e : 0x7fffffff;
}

// ---- per-slot phases ------------------------------------------------------------------


// P0: arrivals and even dispatch over warm instances (Q16, Q17).
// A_f(t) = (pat[p_f][(t + phase_f) mod T_pat] * scale_f) >> 10; the pattern index is
// advanced incrementally (set at registration), so no modulo runs per slot.
template <bool LAT>
static __device__ void phase0(Scn& c, int32_t t, Acc& acc) {
  DILU_VIEW(v, c);
  const Params& P = *c.P;
  const auto infl = v.fInfL;
  const auto reg = v.fReg;
  const auto fpat = v.fPat;
  const auto fscale = v.fScale;
  const auto pidx = v.fPidx;
  const auto facc = v.fAcc;
  const auto lh = v.fLh;
  const auto nxt = v.iNext;
  const auto meta = v.iMeta;
  const auto ready = v.iReady;
  const auto r = v.iR + (P.SPS == 1 ? 0 : (t & 1)) * P.I;   // see phase1
  const int32_t* __restrict__ gpat = P.pat;
  const int32_t Tp = P.Tp, ninf = v.h[H_NINF];
#if DILU_HOT_SMEM
  cp_async_wait_all();
#endif
  for (int32_t k = c.g.rank(); k < ninf; k += c.g.size()) {
    const int32_t f = infl[k];
    if (!reg[f]) continue;
    const int32_t idx = pidx[f];
    const int32_t nidx = idx + 1 == Tp ? 0 : idx + 1;
    pidx[f] = nidx;
    const int32_t* prow = gpat + (size_t)fpat[f] * Tp;
#if DILU_HOT_SMEM
    const int32_t pv = v.fPv[f];           // landed since the last slot (waited above)
    const long long x = pv >= 0 ? pv : __ldg(prow + idx);
    cp_async4(v.fPv + f, prow + nidx);      // next slot's value
#else
    const long long x = __ldg(prow + idx);
#endif
    const int32_t A = (int32_t)((x * fscale[f]) >> 10);
    acc.nfun += 1;
    facc[f] += A;
    acc.rtot += A;
    int32_t nw = 0, s1 = -1;
    for (int32_t s = lh[f]; s >= 0; s = nxt[s])
      if (st_of(meta[s]) == ST_PLACED && ready[s] <= t) { s1 = nw == 0 ? s : s1; ++nw; }
    if (nw == 0) {
      acc.rvio += A;
      if (LAT) lat_unserved(c.lat, A);
      continue;
    }
    if (nw == 1) { r[s1] = A; continue; }   // one warm instance (the common case): no second walk
    const int32_t q = A / nw, rem = A - q * nw;
    int32_t rank = 0;
    for (int32_t s = lh[f]; s >= 0; s = nxt[s]) {
      if (st_of(meta[s]) == ST_PLACED && ready[s] <= t) {
        r[s] = q + (rank < rem ? 1 : 0);
        ++rank;
      }
    }
  }
#if DILU_HOT_SMEM
  cp_async_commit();                       // this slot's fPv copies: one group
#endif
}

// P1: vertical token allocation per GPU row (Q13, Q14)
template <bool LAT>
static __device__ void phase1(Scn& c, int32_t t, Acc& acc) {
  DILU_VIEW(v, c);
  const Params& P = *c.P;
  const int lane = threadIdx.x & 31, wid = c.g.wrank(), nwarp = c.g.nwarps();
  const int par = t & 1;
  // With one slot per second every slot starts with B1's counting barrier (or an
  // overlapped slot's join), which orders P2(t) before P0/P1(t+1): r needs one buffer and
  // the LLM stage minima use the other half of iR (shared memory) instead of the cold
  // double buffer iBmin.
  const bool one = P.SPS == 1;
  const auto r = v.iR + (one ? 0 : par) * P.I;
  DPN(int32_t) bmin = one ? GP32(v.iR + P.I) : GP32(v.iBmin + par * P.I);
  const auto gang = v.fGang + par * P.F;
  const auto grow = v.gGrow;
  // row sizes as of the last repack: in overlapped slots warp 0 appends (cold) residents
  // beyond them while this runs; rows below gNs never move (commit)
  const auto gn = v.gNs;
  const auto gres = v.gRes;
  const auto meta_ = v.iMeta;
  const auto ready = v.iReady;
  const auto ifunc = v.iFunc;
  const auto iid = v.iId;
  const auto fkind = v.fKind;
  const auto freq = v.fReq;
  const auto flim = v.fLim;
  const auto fdtr = v.fDtr;
  const auto fibs = v.fIbs;
  const auto fcb = v.fCb;
  const auto chk = v.gChk;
  const int32_t nch = v.h[H_CBASE + 6];
  const int32_t T = (int32_t)P.T_slot, slot_ms = P.slot_ms;
  const uint64_t ht = sm64(sm64((uint32_t)c.scn_id) ^ (uint32_t)t);   // mix() prefix, per slot
  for (int32_t ch = wid; ch < nch; ch += nwarp) {
    const int32_t cd = chk[ch];
    const int k = cd >> 24;
    const int w = 1 << k;
    const int32_t gi = lane >> k;
    int32_t g = -1, s = -1;
    if (gi < ((cd >> 16) & 255)) {
      g = grow[(cd & 0xFFFF) + gi];
      const int j = lane & (w - 1);
      if (j < gn[g]) s = gres[(size_t)g * RES + j];
    }
    int32_t req = 0, want = 0, f = -1, kind = 0, nst = 1, cst = 1, ibs = 1, rr = 0, need = 0;
    int32_t d = 0;
    bool warm = false;
    if (s >= 0) {
      const int32_t meta = meta_[s];
      warm = st_of(meta) == ST_PLACED && ready[s] <= t;
      if (warm) {
        f = ifunc[s];
        kind = fkind[f];
        nst = nst_of(meta);
        req = freq[f] * slot_ms;
        const int32_t lim = c.mode == M_EXCLUSIVE ? T : flim[f] * slot_ms;  // whole GPU
        long long dd;
        if (kind == K_TRAIN) {
          dd = fdtr[f];
        } else {
          ibs = fibs[f];
          const int32_t cb = fcb[f];
          cst = nst == 1 ? cb : (cb + nst - 1) / nst;   // c_stage (R4)
          rr = r[s];
          need = rr / ibs + (rr % ibs != 0);             // ceil(r / IBS) batches
          dd = (long long)need * cst;
        }
        d = dd < lim ? (int32_t)dd : lim;                // min(d, limit) (want only uses this)
        want = d > req ? d - req : 0;
        if (kind == K_TRAIN) d = (int32_t)dd;            // training keeps x = min(d, a)
      }
    }
    // width-w segmented inclusive scan of want, and row sum of req
    int32_t incl = want, sreq = req;
    for (int o = 1; o < w; o <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, incl, o, w);
      if ((lane & (w - 1)) >= o) incl += y;
    }
    for (int o = w >> 1; o > 0; o >>= 1) sreq += __shfl_xor_sync(0xffffffffu, sreq, o, w);
    if (warm) {
      const int32_t room = T - sreq - (incl - want);
      const int32_t sp = want < room ? want : (room > 0 ? room : 0);
      const int32_t a = req + sp;
      acc.nres += 1;
      acc.hash += sm64(sm64(ht ^ (uint32_t)iid[s]) ^ ((uint64_t((uint32_t)g) << 32) | (uint32_t)a));
      if (kind == K_TRAIN) {
        atomicMin(&gang[f], d < a ? d : a);              // x = min(d, a)
      } else {
        const int32_t fit = a / cst;
        const int32_t b = need < fit ? need : fit;
        if (nst == 1) {
          const long long cap = (long long)b * ibs;
          const int32_t served = cap < rr ? (int32_t)cap : rr;
          acc.rsrv += served;
          acc.rvio += rr - served;
          const long long e = (long long)b * cst;
          acc.iexe += e;
          acc.etot += e;
          if (LAT) lat_instance(c.lat, rr, ibs, b, lat_e(cst, a, T), v.fSlo[f], T);
        } else {
          atomicMin(&bmin[s], b);
          if (LAT) atomicMax(&v.iEmax[par * P.I + s], lat_e(cst, a, T));
        }
      }
    }
  }
}

// P2: cross-row minima -- training gang (Q22) and LLM pipeline stages (Q11); only the
// training and LLM functions (static list fDefL) are visited.
template <bool LAT>
static __device__ void phase2(Scn& c, int32_t t, Acc& acc) {
  DILU_VIEW(v, c);
  const Params& P = *c.P;
  const int par = t & 1;
  const bool one = P.SPS == 1;          // buffers as in phase1
  const auto r = v.iR + (one ? 0 : par) * P.I;
  DPN(int32_t) bmin = one ? GP32(v.iR + P.I) : GP32(v.iBmin + par * P.I);
  const auto gang = v.fGang + par * P.F;
  const auto defl = v.fDefL;
  const auto reg = v.fReg;
  const auto lh = v.fLh;
  const auto nxt = v.iNext;
  const auto meta = v.iMeta;
  const int32_t ndef = v.h[H_NDEF];
  for (int32_t k = c.g.rank(); k < ndef; k += c.g.size()) {
    const int32_t f = defl[k];
    if (!reg[f]) continue;
    if (v.fKind[f] == K_TRAIN) {
      // the job is the function: gang = min x over its live workers, 0 unless all are
      // warm; every warm worker executes the gang, progress = n_workers * gang (Q22)
      const int32_t gm = gang[f];
      if (gm != BIG) {
        gang[f] = BIG;
        int32_t nlive = 0;
        bool all_warm = true;
        for (int32_t s = lh[f]; s >= 0; s = nxt[s]) {
          ++nlive;
          all_warm &= st_of(meta[s]) == ST_PLACED && v.iReady[s] <= t;
        }
        if (all_warm) {
          acc.tprg += (long long)v.fNw[f] * gm;
          acc.etot += (long long)nlive * gm;
        }
      }
    } else {
      for (int32_t s = lh[f]; s >= 0; s = nxt[s]) {
        const int32_t nst = nst_of(meta[s]);
        if (__builtin_expect(nst <= 1, 1)) continue;   // unsplit: finished in P1
        const int32_t b = bmin[s];
        if (b == BIG) continue;
        bmin[s] = BIG;
        const int32_t ibs = v.fIbs[f];
        const int32_t cst = (v.fCb[f] + nst - 1) / nst;
        const int32_t rr = r[s];
        const long long cap = (long long)b * ibs;
        const int32_t served = cap < rr ? (int32_t)cap : rr;
        acc.rsrv += served;
        acc.rvio += rr - served;
        const long long e = (long long)nst * b * cst;
        acc.iexe += e;
        acc.etot += e;
        if (LAT) {
          int32_t* em = &v.iEmax[par * P.I + s];
          lat_instance(c.lat, rr, ibs, b, *em, v.fSlo[f], (long long)P.T_slot);
          *em = 0;
        }
      }
    }
  }
}

// ---- fused batches (sub-second slots) ---------------------------------------------------
// Between two second boundaries nothing mutates the placement (scaling and
// placement run at t mod SPS == 0 only), so the slots t..t+B-1 of one batch see the same
// residents, rows and functions; only the arrivals A_f(u) and the warm set (ready <= u)
// change.  P0b/P1b/P2b load each function / resident once and loop over the batch's slots,
// writing the per-slot r, stage minimum and gang into the [B][I] / [B][F] buffers.  The
// arithmetic per slot is exactly that of phase0/1/2 (same expressions, same order of the
// integer operations), so results are bit-identical; only the hash summation order moves
// (it is a mod-2^64 sum, order-free by construction, R8).

template <bool LAT>
static __device__ void phase0_b(Scn& c, int32_t t, int32_t B, Acc& acc) {
  DILU_VIEW(v, c);
  const Params& P = *c.P;
  const auto infl = v.fInfL;
  const auto reg = v.fReg;
  const auto pidx = v.fPidx;
  const auto lh = v.fLh;
  const auto nxt = v.iNext;
  const auto meta = v.iMeta;
  const auto ready = v.iReady;
  const auto rb = v.rB;
  const int32_t Tp = P.Tp, ninf = v.h[H_NINF], I = P.I;
  for (int32_t k = c.g.rank(); k < ninf; k += c.g.size()) {
    const int32_t f = infl[k];
    if (!reg[f]) continue;
    const int32_t* __restrict__ prow = P.pat + (size_t)v.fPat[f] * Tp;
    const long long scale = v.fScale[f];
    const int32_t s0 = lh[f];
    int32_t idx = pidx[f];
    // warm set over the batch: instances placed and ready by t, plus those turning warm
    // inside it (cold starts finishing mid-batch)
    int32_t nw0 = 0, rmin = BIG;
    for (int32_t s = s0; s >= 0; s = nxt[s]) {
      if (st_of(meta[s]) != ST_PLACED) continue;
      const int32_t rd = ready[s];
      if (rd <= t) ++nw0; else rmin = rd < rmin ? rd : rmin;
    }
    int32_t asum = 0;
    for (int32_t u = 0; u < B; ++u) {
      const int32_t tu = t + u;
      const long long x = __ldg(prow + idx);
      idx = idx + 1 == Tp ? 0 : idx + 1;
      const int32_t A = (int32_t)((x * scale) >> 10);
      acc.nfun += 1;
      asum += A;
      acc.rtot += A;
      int32_t nw = nw0;
      if (rmin <= tu) {
        nw = 0;
        for (int32_t s = s0; s >= 0; s = nxt[s]) nw += (st_of(meta[s]) == ST_PLACED && ready[s] <= tu);
      }
      if (nw == 0) {
        acc.rvio += A;
        if (LAT) lat_unserved(c.lat, A);
        continue;
      }
      const int32_t q = A / nw, rem = A - q * nw;
      int32_t rank = 0;
      const auto ru = rb + (size_t)u * I;
      for (int32_t s = s0; s >= 0; s = nxt[s]) {
        if (st_of(meta[s]) == ST_PLACED && ready[s] <= tu) {
          ru[s] = q + (rank < rem ? 1 : 0);
          ++rank;
        }
      }
    }
    pidx[f] = idx;
    v.fAcc[f] += asum;
  }
}

template <bool LAT>
static __device__ void phase1_b(Scn& c, int32_t t, int32_t B, Acc& acc) {
  DILU_VIEW(v, c);
  const Params& P = *c.P;
  const int lane = threadIdx.x & 31, wid = c.g.wrank(), nwarp = c.g.nwarps();
  const auto chk = v.gChk;
  const int32_t nch = v.h[H_CBASE + 6];
  const int32_t T = (int32_t)P.T_slot, slot_ms = P.slot_ms, I = P.I, F = P.F;
  const uint64_t hs = sm64((uint32_t)c.scn_id);
  for (int32_t ch = wid; ch < nch; ch += nwarp) {
    const int32_t cd = v.gChk[ch];
    const int k = cd >> 24;
    const int w = 1 << k;
    const int32_t gi = lane >> k;
    int32_t g = -1, s = -1;
    if (gi < ((cd >> 16) & 255)) {
      g = v.gGrow[(cd & 0xFFFF) + gi];
      const int j = lane & (w - 1);
      if (j < (P.covl ? v.gNs[g] : v.gN[g])) s = v.gRes[(size_t)g * RES + j];   // gNs: see covl
    }
    // batch-invariant resident fields
    bool placed = false;
    int32_t rd = BIG, f = -1, kind = 0, nst = 1, cst = 1, ibs = 1, req0 = 0, lim = 0, id = 0;
    long long dtr = 0;
    if (s >= 0) {
      const int32_t meta = v.iMeta[s];
      placed = st_of(meta) == ST_PLACED;
      if (placed) {
        rd = v.iReady[s];
        f = v.iFunc[s];
        id = v.iId[s];
        kind = v.fKind[f];
        nst = nst_of(meta);
        req0 = v.fReq[f] * slot_ms;
        lim = c.mode == M_EXCLUSIVE ? T : v.fLim[f] * slot_ms;
        if (kind == K_TRAIN) {
          dtr = v.fDtr[f];
        } else {
          ibs = v.fIbs[f];
          const int32_t cb = v.fCb[f];
          cst = nst == 1 ? cb : (cb + nst - 1) / nst;
        }
      }
    }
    const uint64_t gk = uint64_t((uint32_t)g) << 32;
    for (int32_t u = 0; u < B; ++u) {
      const int32_t tu = t + u;
      const bool warm = placed && rd <= tu;
      int32_t req = 0, want = 0, rr = 0, need = 0, d = 0;
      if (warm) {
        req = req0;
        long long dd;
        if (kind == K_TRAIN) {
          dd = dtr;
        } else {
          rr = v.rB[(size_t)u * I + s];
          need = rr / ibs + (rr % ibs != 0);
          dd = (long long)need * cst;
        }
        d = dd < lim ? (int32_t)dd : lim;
        want = d > req ? d - req : 0;
        if (kind == K_TRAIN) d = (int32_t)dd;
      }
      int32_t incl = want, sreq = req;
      for (int o = 1; o < w; o <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, incl, o, w);
        if ((lane & (w - 1)) >= o) incl += y;
      }
      for (int o = w >> 1; o > 0; o >>= 1) sreq += __shfl_xor_sync(0xffffffffu, sreq, o, w);
      if (warm) {
        const int32_t room = T - sreq - (incl - want);
        const int32_t sp = want < room ? want : (room > 0 ? room : 0);
        const int32_t a = req + sp;
        acc.nres += 1;
        const uint64_t ht = sm64(hs ^ (uint32_t)tu);
        acc.hash += sm64(sm64(ht ^ (uint32_t)id) ^ (gk | (uint32_t)a));
        if (kind == K_TRAIN) {
          atomicMin(&v.gB[(size_t)u * F + f], d < a ? d : a);
        } else {
          const int32_t fit = a / cst;
          const int32_t b = need < fit ? need : fit;
          if (nst == 1) {
            const long long cap = (long long)b * ibs;
            const int32_t served = cap < rr ? (int32_t)cap : rr;
            acc.rsrv += served;
            acc.rvio += rr - served;
            const long long e = (long long)b * cst;
            acc.iexe += e;
            acc.etot += e;
            if (LAT) lat_instance(c.lat, rr, ibs, b, lat_e(cst, a, T), v.fSlo[f], T);
          } else {
            atomicMin(&v.bB[(size_t)u * I + s], b);
            if (LAT) atomicMax(&v.eB[(size_t)u * I + s], lat_e(cst, a, T));
          }
        }
      }
    }
  }
}

template <bool LAT>
static __device__ void phase2_b(Scn& c, int32_t t, int32_t B, Acc& acc) {
  DILU_VIEW(v, c);
  const Params& P = *c.P;
  const auto defl = v.fDefL;
  const auto lh = v.fLh;
  const auto nxt = v.iNext;
  const auto meta = v.iMeta;
  const int32_t ndef = v.h[H_NDEF], I = P.I, F = P.F;
  for (int32_t k = c.g.rank(); k < ndef; k += c.g.size()) {
    const int32_t f = defl[k];
    if (!v.fReg[f]) continue;
    if (v.fKind[f] == K_TRAIN) {
      int32_t nlive = 0, rmax = 0;
      bool placed = true;
      for (int32_t s = lh[f]; s >= 0; s = nxt[s]) {
        ++nlive;
        placed &= st_of(meta[s]) == ST_PLACED;
        const int32_t rd = v.iReady[s];
        rmax = rd > rmax ? rd : rmax;
      }
      const long long nwk = v.fNw[f];
      for (int32_t u = 0; u < B; ++u) {
        int32_t* gp = &v.gB[(size_t)u * F + f];
        const int32_t gm = *gp;
        if (gm == BIG) continue;
        *gp = BIG;
        if (placed && rmax <= t + u) {
          acc.tprg += nwk * gm;
          acc.etot += (long long)nlive * gm;
        }
      }
    } else {
      const int32_t ibs = v.fIbs[f], cb = v.fCb[f];
      for (int32_t s = lh[f]; s >= 0; s = nxt[s]) {
        const int32_t nst = nst_of(meta[s]);
        if (nst <= 1) continue;
        const int32_t cst = (cb + nst - 1) / nst;
        for (int32_t u = 0; u < B; ++u) {
          int32_t* bp = &v.bB[(size_t)u * I + s];
          const int32_t b = *bp;
          if (b == BIG) continue;
          *bp = BIG;
          const int32_t rr = v.rB[(size_t)u * I + s];
          const long long cap = (long long)b * ibs;
          const int32_t served = cap < rr ? (int32_t)cap : rr;
          acc.rsrv += served;
          acc.rvio += rr - served;
          const long long e = (long long)nst * b * cst;
          acc.iexe += e;
          acc.etot += e;
          if (LAT) {
            int32_t* em = &v.eB[(size_t)u * I + s];
            lat_instance(c.lat, rr, ibs, b, *em, v.fSlo[f], (long long)P.T_slot);
            *em = 0;
          }
        }
      }
    }
  }
}

// ---- literal Algorithm 2 at 5 ms periods (cfg.flags bit2) -------------
// Replaces P1's one-shot grant: per GPU row (a width-w lane segment, residents in (prio,
// id) order), slot_ms/5 periods of IssueToken and the drain with the
// physical capacity clamp, readings DESIGN.md D8.  All per-resident and per-row
// state stays in registers across the periods; the sequential parts of one period (the
// per-GPU "state" fold over the SLO residents, the capacity clamp) are segment shuffles.
// B slots (fused batch) or one slot; r, stage minima and gangs come through base/stride.

static __device__ __forceinline__ int32_t a2_grow(int32_t r_last) {   // ceil(max(R_last,1) * 5/4)
  const long long r = r_last < 1 ? 1 : r_last;
  return (int32_t)((r * 5 + 3) / 4);
}

template <bool LAT>
static __device__ void phase1_alg2(Scn& c, int32_t t, int32_t B, DPN(const int32_t) rbase, size_t rstride,
                            DPN(int32_t) bminb, size_t bstride, DPN(int32_t) gangb, size_t gstride,
                            DPN(int32_t) emaxb, Acc& acc) {
  DILU_VIEW(v, c);
  const Params& P = *c.P;
  const int lane = threadIdx.x & 31, wid = c.g.wrank(), nwarp = c.g.nwarps();
  const unsigned FULL = 0xffffffffu;
  const auto chk = v.gChk;
  const int32_t nch = v.h[H_CBASE + 6];
  const int32_t NP = P.slot_ms / A2_PERIOD_MS;
  const long long PT = (long long)A2_PERIOD_MS * 1000;          // period in us
  const uint64_t hs = sm64((uint32_t)c.scn_id);
  for (int32_t ch = wid; ch < nch; ch += nwarp) {
    const int32_t cd = v.gChk[ch];
    const int k = cd >> 24;
    const int w = 1 << k;
    const int j = lane & (w - 1);
    const int32_t gi = lane >> k;
    int32_t g = -1, s = -1;
    if (gi < ((cd >> 16) & 255)) {
      g = v.gGrow[(cd & 0xFFFF) + gi];
      if (j < v.gN[g]) s = v.gRes[(size_t)g * RES + j];
    }
    // batch-invariant resident fields and its stage's Alg.2 state
    bool placed = false;
    int32_t rd = BIG, f = -1, kind = 0, nst = 1, cst = 1, ibs = 1, id = -1, prio = 1;
    int32_t req_p = 0, lim_p = 0, e = -1;
    long long dtr = 0;
    int32_t tc = 0, tm = 0, rl = 0, le = A2_NEVER;
    if (s >= 0) {
      const int32_t meta = v.iMeta[s];
      placed = st_of(meta) == ST_PLACED;
      if (placed) {
        rd = v.iReady[s];
        f = v.iFunc[s];
        id = v.iId[s];
        kind = v.fKind[f];
        prio = v.fPrio[f];
        nst = nst_of(meta);
        req_p = v.fReq[f] * A2_PERIOD_MS;
        lim_p = c.mode == M_EXCLUSIVE ? A2_MAX_TOKENS : v.fLim[f] * A2_PERIOD_MS;
        if (kind == K_TRAIN) {
          dtr = v.fDtr[f];
        } else {
          ibs = v.fIbs[f];
          const int32_t cb = v.fCb[f];
          cst = nst == 1 ? cb : (cb + nst - 1) / nst;
        }
        int32_t kst = 0;
        if (nst > 1) while (v.iG[s * MAXST + kst] != g) ++kst;
        e = s * MAXST + kst;
        tc = v.aTc[e]; tm = v.aTm[e]; rl = v.aRl[e]; le = v.aLe[e];
      }
    }
    int32_t st = A2_NONE, ow = -1, odt = 0;          // this row's "state" (replicated)
    if (g >= 0) { st = v.aSt[g]; ow = v.aOw[g]; odt = v.aDt[g]; }
    const uint64_t gk = uint64_t((uint32_t)g) << 32;
    for (int32_t u = 0; u < B; ++u) {
      const int32_t tu = t + u;
      const bool warm = placed && rd <= tu;
      int32_t rr = 0, need = 0;
      long long dem = 0;                              // the slot's demand, queued at its start
      if (warm) {
        if (kind == K_TRAIN) {
          dem = dtr;
        } else {
          rr = rbase[(size_t)u * rstride + s];
          need = rr / ibs + (rr % ibs != 0);
          dem = (long long)need * cst;
        }
      }
      const bool slo = warm && prio == 0;
      const int32_t cklc = slo && kind != K_TRAIN ? cst : 0;
      long long pend = dem;
      int32_t done = 0, bst = -1;                     // slot-relative: <= slot_ms * 1000
      long long dT = tm > 0 ? ((long long)tc - tm) * 1000 / tm : 0;   // changes with tc, tm only
      for (int32_t p = 0; p < NP; ++p) {
        const int32_t Pa = tu * NP + p;
        // 0. bookkeeping: no SLO resident, or the EMERGENCY owner left -> NONE.  One
        // segment sum of three packed counts (each <= 32): SLO, owner, busy (RW != 0)
        const int32_t busy = warm && le >= Pa - A2_RW;
        int32_t cnt = (int32_t)slo | ((int32_t)(warm && id == ow) << 8) | (busy << 16);
        for (int o = w >> 1; o > 0; o >>= 1) cnt += __shfl_xor_sync(FULL, cnt, o, w);
        const int32_t nslo = cnt & 0xff, nown = (cnt >> 8) & 0xff, nbusy = cnt >> 16;
        if (nslo == 0 || (st == A2_EMERGENCY && nown == 0)) { st = A2_NONE; ow = -1; odt = 0; }
        // 1. SLO-sensitive residents (lines 12-24): own grant, proposed state
        int32_t grant = 0, act = -1, dtv = 0;
        if (slo) {
          if (dT > A2_ETA_V) {
            grant = lim_p; act = A2_EMERGENCY; dtv = (int32_t)dT;
          } else if (le < Pa - A2_RW) {
            grant = req_p; act = A2_RECOVERY;
          } else if (nbusy - busy == 0) {
            const int32_t g2 = a2_grow(rl);
            grant = g2 < lim_p ? g2 : lim_p; act = A2_RECOVERY;
          } else {
            grant = req_p; act = A2_CONTENTION;
          }
        }
        // ... the state, folded over them in row order (P:1003 ownership): visit
        // the segment's SLO lanes in order (the warp iterates max-over-segments times)
        const unsigned seg = (w == 32 ? FULL : ((1u << w) - 1)) << (lane & ~(w - 1));
        unsigned todo = __ballot_sync(FULL, act >= 0) & seg;
        const int nrounds = __reduce_max_sync(FULL, __popc(todo));
        for (int x = 0; x < nrounds; ++x) {
          const bool have = todo != 0;              // this segment still has an SLO lane
          const int src = have ? __ffs(todo) - 1 : lane;
          todo &= todo - 1;
          const int32_t axs = __shfl_sync(FULL, act, src);
          const int32_t ax = have ? axs : -1;
          const int32_t ix = __shfl_sync(FULL, id, src);
          const int32_t dx = __shfl_sync(FULL, dtv, src);
          if (ax == A2_EMERGENCY) {
            if (st != A2_EMERGENCY || ow == ix || dx > odt) { st = A2_EMERGENCY; ow = ix; odt = dx; }
          } else if (ax >= 0) {
            if (st != A2_EMERGENCY || ow == ix) { st = ax; ow = -1; odt = 0; }
          }
        }
        // 2. best-effort residents (lines 25-38)
        if (warm && prio != 0) {
          if (st == A2_NONE) {
            grant = lim_p;
          } else if (st == A2_EMERGENCY) {
            const long long m = req_p < rl ? req_p : rl;
            grant = (int32_t)(m * 1000 / (odt > 1000 ? odt : 1000));   // max(dT, 1)
          } else if (st == A2_RECOVERY) {
            const int32_t g2 = a2_grow(rl);
            grant = g2 < lim_p ? g2 : lim_p;
          } else {
            grant = rl;
          }
        }
        // 3. drain: rate y = min(R_issue, capacity left by earlier residents)
        const long long q = warm ? (pend < grant ? pend : grant) : 0;
        long long incl = q;
        for (int o = 1; o < w; o <<= 1) {
          const long long yq = __shfl_up_sync(FULL, incl, o, w);
          if (j >= o) incl += yq;
        }
        long long cap = A2_MAX_TOKENS - (incl - q);
        if (cap < 0) cap = 0;
        const long long y = grant < cap ? grant : cap;
        const long long ex = q < cap ? q : cap;
        if (ex > 0) {
          le = Pa;
          if (cklc > 0) {   // KLC: batch spans at rate y (footnote P:899); 32-bit: spans and
                            // offsets are within the slot, (token offset) * 5000 <= 2.5e7
            const int32_t a0 = done, b0 = done + (int32_t)ex, yy = (int32_t)y, pt = (int32_t)PT;
            bool upd = false;
            for (int32_t m = a0 / cklc; m * cklc < b0; ++m) {
              const int32_t first = m * cklc, last = first + cklc - 1;
              if (first >= a0) bst = p * pt + (first - a0) * pt / yy;
              if (last < b0) {
                tc = p * pt + ((last - a0 + 1) * pt + yy - 1) / yy - bst;
                if (tm == 0 || tc < tm) tm = tc;
                upd = true;
              }
            }
            if (upd) dT = ((long long)tc - tm) * 1000 / tm;
          }
        }
        pend -= ex;
        done += (int32_t)ex;
        if (warm) rl = grant;                         // 4. R_last
      }
      // the slot's results exactly as P1, with a = executed tokens
      if (warm) {
        const int32_t a = (int32_t)done;
        acc.nres += 1;
        const uint64_t ht = sm64(hs ^ (uint32_t)tu);
        acc.hash += sm64(sm64(ht ^ (uint32_t)id) ^ (gk | (uint32_t)a));
        if (kind == K_TRAIN) {
          const int32_t d = (int32_t)dtr;
          atomicMin(&gangb[(size_t)u * gstride + f], d < a ? d : a);
        } else {
          const int32_t fit = a / cst;
          const int32_t b = need < fit ? need : fit;
          if (nst == 1) {
            const long long capb = (long long)b * ibs;
            const int32_t served = capb < rr ? (int32_t)capb : rr;
            acc.rsrv += served;
            acc.rvio += rr - served;
            const long long ee = (long long)b * cst;
            acc.iexe += ee;
            acc.etot += ee;
            if (LAT) lat_instance(c.lat, rr, ibs, b, lat_e(cst, a, (long long)P.T_slot), v.fSlo[f],
                                  (long long)P.T_slot);
          } else {
            atomicMin(&bminb[(size_t)u * bstride + s], b);
            if (LAT) atomicMax(&emaxb[(size_t)u * bstride + s], lat_e(cst, a, (long long)P.T_slot));
          }
        }
      }
    }
    if (e >= 0) { v.aTc[e] = tc; v.aTm[e] = tm; v.aRl[e] = rl; v.aLe[e] = le; }
    if (g >= 0 && j == 0) { v.aSt[g] = st; v.aOw[g] = ow; v.aDt[g] = odt; }
  }
}

// ---- boundary -----------------------------------------------------------------------

enum : int32_t { EV_DEP = 1, EV_OUT = 2, EV_IN = 4, EV_ARR = 8 };

// B1 for one function f at the boundary of second `sec`: window push of second sec-1,
// incremental up/down counts, the lazy (or eager) scaling decision, departure / arrival
// flags.  Writes fFlag[f]; returns the flags.  The
// fOld prefetch is issued and consumed by the same thread (fixed f -> thread mapping).
static __device__ int32_t b1_func(Scn& c, int32_t f, int32_t sec) {
  DILU_VIEW(v, c);
  const Params& P = *c.P;
  const int32_t W = P.W;
  const int32_t kind = v.fKind[f];
  int32_t ev = 0;
  if (kind != K_UNUSED) {
    if (v.fReg[f]) {
      const bool inf = is_inf(kind);
      const auto ring = v.ring + (size_t)f * W;
      const long long cap1 = v.fCap1[f];
      int32_t last = 0;
      if (inf && sec >= 1) {                      // step 1: push second sec-1
        const int32_t val = v.fAcc[f];
        last = val;
        const int32_t head = v.fHead[f];
        const int32_t ns = v.fNsamp[f];
        const int32_t thr = v.fThrn[f];
        if (thr >= 0) {
          const long long cu = (long long)thr * cap1, cd = (long long)(thr - 1) * cap1;
          int32_t du = val > cu, dd = val < cd;
          if (ns >= W) {
#if DILU_HOT_SMEM
            const int32_t old = W > 1 ? v.fOld[f] : ring[head];   // prefetched last second
#else
            const int32_t old = ring[head];
#endif
            du -= old > cu; dd -= old < cd;
          }
          v.fUp[f] += du;
          v.fDown[f] += dd;
        }
        ring[head] = val;
        const int32_t nhead = head + 1 == W ? 0 : head + 1;
        v.fHead[f] = nhead;
#if DILU_HOT_SMEM
        if (W > 1) cp_async4(v.fOld + f, ring + nhead);        // next second's evictee
#endif
        v.fNsamp[f] = ns < W ? ns + 1 : W;     // saturating: only >= W / >= 1 matter
        v.fAcc[f] = 0;
      }
      if (DILU_UNLIKELY(v.fDep[f] == sec)) {      // step 2: departure
        ev = EV_DEP;
      } else if (DILU_UNLIKELY(inf && c.mode == M_EAGER)) {   // reactive scaling on the last sample
        if (v.fNsamp[f] >= 1) {
          const int32_t n = v.fNlive[f];
          if ((long long)last > (long long)n * cap1) {
            const long long k = ((long long)last + cap1 - 1) / cap1 - n;
            if (k >= 1) { ev = EV_OUT; v.fK[f] = (int32_t)k; }
          } else if ((long long)last < (long long)(n - 1) * cap1 && n > P.min_inst) {
            ev = EV_IN;
          }
        }
      } else if (inf && v.fNsamp[f] >= W) {       // step 3: lazy scaling decision
        const int32_t n = v.fNlive[f];
        const long long cu = (long long)n * cap1, cd = (long long)(n - 1) * cap1;
        if (DILU_UNLIKELY(v.fThrn[f] != n)) {
          int32_t up = 0, dn = 0;
          for (int j = 0; j < W; ++j) { const int32_t w = ring[j]; up += w > cu; dn += w < cd; }
          v.fUp[f] = up; v.fDown[f] = dn; v.fThrn[f] = n;
        }
        if (DILU_UNLIKELY(v.fUp[f] >= P.phi_out)) {
          int32_t mx = 0;
          for (int j = 0; j < W; ++j) mx = max(mx, ring[j]);
          const long long k = ((long long)mx + cap1 - 1) / cap1 - n;
          if (k >= 1) { ev = EV_OUT; v.fK[f] = (int32_t)k; }
        } else if (v.fDown[f] > P.phi_in && n > P.min_inst) {
          ev = EV_IN;
        }
      }
    }
    if (DILU_UNLIKELY(v.fArr[f] == sec)) ev |= EV_ARR;   // step 4: arrival
  }
  v.fFlag[f] = ev;
  return ev;
}

// Overlapped slots: after its placement pass warp 0 recounts the windows
// of the functions whose live count n B3 just changed (ScaleOut / ScaleIn), against the
// new thresholds n*cap1 and (n-1)*cap1, so that B1 of the next boundary -- where the whole
// CTA waits for its slowest thread -- finds fThrn == n and only updates incrementally.
// Exact: the counts cover the valid samples (ring[0, ns) before the ring first fills),
// nothing but B1 writes the ring, and n cannot change before that B1 (placement does not
// change live counts).  Counting before the ring is full only starts the incremental
// counts earlier; at the first decision (ns >= W) they equal a full recount.
static __device__ void prerecount_warp(Scn& c) {
  DILU_VIEW(v, c);
  __syncwarp();
  const int lane = threadIdx.x & 31;
  const int32_t ne = v.h[H_NEV], W = c.P->W;
  if (c.mode == M_EAGER) return;                   // (reactive: no window counts)
  #pragma unroll 1
  for (int32_t e = 0; e < ne; ++e) {
    const int32_t f = v.fList[e];
    if (!(v.fFlag[f] & (EV_OUT | EV_IN)) || !v.fReg[f]) continue;
    const int32_t n = v.fNlive[f];
    if (v.fThrn[f] == n) continue;
    const int32_t ns = v.fNsamp[f], cnt = ns < W ? ns : W;
    const long long cap1 = v.fCap1[f], cu = (long long)n * cap1, cd = (long long)(n - 1) * cap1;
    const auto ring = v.ring + (size_t)f * W;
    int32_t up = 0, dn = 0;
    #pragma unroll 1
    for (int32_t j = lane; j < cnt; j += 32) { const int32_t w = ring[j]; up += w > cu; dn += w < cd; }
    up = __reduce_add_sync(0xffffffffu, up);
    dn = __reduce_add_sync(0xffffffffu, dn);
    if (lane == 0) { v.fUp[f] = up; v.fDown[f] = dn; v.fThrn[f] = n; }
  }
  __syncwarp();
}

// Returns whether a placement pass is due.  ovl (overlapped slots): the pass is left to
// the caller, which runs it in warp 0 beside P0/P1/P2.
static __device__ bool boundary(Scn& c, Red& red, int& ph, int32_t t, Acc& acc, bool ovl = false) {
  DILU_VIEW(v, c);
  const Params& P = *c.P;
  const int32_t sec = P.SPS == 1 ? t : t / P.SPS;
  // B1 (function-parallel): window push, incremental counts, decisions, event flags.
  // Contiguous function ranges per thread keep the event list in ascending order.
  const int32_t lo = c.b1lo, hi = c.b1hi;   // this thread's contiguous function range
  const auto fflag = v.fFlag;
  int32_t cnt = 0;
#if defined(DILU_PHASE_TIMING) && DILU_PHASE_TIMING == 2
  const long long fa = clock64();
#endif
#if DILU_HOT_SMEM
  cp_async_wait_all();                              // this thread's fOld / fPv copies landed
#endif
  for (int32_t f = lo; f < hi; ++f) cnt += b1_func(c, f, sec) != 0;
#if DILU_HOT_SMEM
  cp_async_commit();
#endif
#ifdef DILU_PHASE_TIMING
  const long long cb0 = clock64();   // st[22]: B1 count barrier -> end of compaction (leader)
#if DILU_PHASE_TIMING == 2
  if (c.g.leader()) acc.z->st[15] += cb0 - fa;
#endif
#endif
  const int32_t any = g_count(c, cnt);
#if defined(DILU_PHASE_TIMING) && DILU_PHASE_TIMING == 2
  const long long fc = clock64();
  if (c.g.leader()) acc.z->st[16] += fc - cb0;
#endif
  int32_t total = 0;
  if (any) {                                        // ordered compaction of the events
    int32_t pos = g_scan(c, cnt, red, ph, &total);
    for (int32_t f = lo; f < hi && cnt; ++f)
      if (fflag[f]) { v.fList[pos++] = f; --cnt; }
    c.g.sync();                                     // the event list is complete before B3
#if defined(DILU_PHASE_TIMING) && DILU_PHASE_TIMING == 2
    if (c.g.leader()) acc.z->st[17] += clock64() - fc;
#endif
  }
#if defined(DILU_PHASE_TIMING) && DILU_PHASE_TIMING != 2
  if (c.g.leader()) acc.z->st[22] += clock64() - cb0;
#endif
  if (c.g.leader()) v.h[H_NEV] = total;            // (overlapped slots: prerecount_warp)
  const int32_t need_pass = total > 0 || v.h[H_QLEN] > 0;   // uniform: QLEN only changes in B3/placement
#ifdef DILU_PHASE_TIMING
  long long bt0 = clock64();
  if (c.g.leader()) acc.z->st[14] -= bt0;   // st[14] += (end of B3) - (end of B1)
#endif
  if (!need_pass) {
#ifdef DILU_PHASE_TIMING
    if (c.g.leader()) acc.z->st[14] += bt0;
#endif
    return false;
  }
  // B3: apply in the paper's order (steps 2, 3, 4), thread 0
  if (c.g.leader() && total > 0) {
    acc.z->st[S_EVENT] += total;
    for (int32_t e = 0; e < total; ++e) {     // step 2: departures
      const int32_t f = v.fList[e];
      if (!(v.fFlag[f] & EV_DEP)) continue;
      // a live queue entry holds pending instances of its function: scan the queue only if
      // f has one (its list is short, the queue is not)
      bool pend = false;
      #pragma unroll 1
      for (int32_t s = v.fLh[f]; s >= 0 && !pend; s = v.iNext[s]) pend = st_of(v.iMeta[s]) == ST_PEND;
      if (pend) kill_queue_entries_of(c, f);
      while (v.fLh[f] >= 0) terminate(c, v.fLh[f]);
      v.fReg[f] = 0;
    }
    for (int32_t e = 0; e < total && !v.h[H_ERR]; ++e) {     // step 3: hscaler actions
      const int32_t f = v.fList[e];
      const int32_t ev = v.fFlag[f];
      if (ev & EV_OUT) {
        for (int32_t j = 0; j < v.fK[f] && !v.h[H_ERR]; ++j) enqueue(c, f, 1);
        acc.z->sout += 1;
      } else if (ev & EV_IN) {
        const int32_t victim = v.fLt[f];        // highest live id (Q19)
        if (st_of(v.iMeta[victim]) == ST_PEND) {     // its own request
          v.qN[v.iQ[victim]] = 0;
          v.h[H_QLIVE] -= 1;
        }
        terminate(c, victim);
        acc.z->sin += 1;
      }
    }
    for (int32_t e = 0; e < total && !v.h[H_ERR]; ++e) {     // step 4: arrivals
      const int32_t f = v.fList[e];
      if (!(v.fFlag[f] & EV_ARR)) continue;
      register_func(c, f, t, P.Tp);
      if (v.fKind[f] == K_TRAIN) enqueue(c, f, v.fNw[f]);
      else for (int32_t j = 0; j < P.min_inst && !v.h[H_ERR]; ++j) enqueue(c, f, 1);
    }
  }
  if (ovl && total > 0) c.g.sync();   // B3's state changes before P0/P1/P2 and the repack
#ifdef DILU_PHASE_TIMING
  if (c.g.leader()) acc.z->st[14] += clock64();
#endif
  if (ovl) return true;
  // step 5.  No barrier between: the pass starts with a warp-0 section (see there).  It
  // ends with a group barrier after the last commit; what follows it (the leader's queue
  // compaction) touches only the queue, which nothing reads before the next boundary.
  placement(c, red, ph, t, acc);
  return true;
}

// ---------------------------------------------------------------------------- kernels

// One scenario for one call (scale_step: n_req < 0; place_batch: n_req >= 0), run by a
// group of K CTAs (K = 1: the calling CTA; K > 1: the calling cluster, crank = CTA rank).
// VAR bit0: sub-second slots run as fused batches (L.B > 1); bit1: literal Alg.2 periods
// (cfg.flags bit2).  Separate instantiations, so the one-slot-per-second slot-model kernels
// (C1-C4) carry neither the batch nor the period code.
template <bool SMEM, int VAR>
static __device__ void run_scenario(const Params& P, Red& red, View* sv, uint8_t* smem, int32_t sc, int32_t t0,
                             int32_t n_slots, int32_t n_req, const int32_t* req_scn,
                             const int32_t* req_func, int32_t* out_gpu, int32_t* out_iid,
                             int K = 1, int crank = 0, int Kc = 1) {
  uint8_t* gblock = P.state + (size_t)sc * P.L.bytes;
  uint8_t* hot = gblock;
  if (SMEM) {
    const int4* src = reinterpret_cast<const int4*>(gblock);
    int4* dst = reinterpret_cast<int4*>(smem);
    for (size_t k = threadIdx.x; k < P.L.hot_bytes / 16; k += blockDim.x) dst[k] = src[k];
    hot = smem;
  }
  Scn c;
  c.gblock = gblock;
  c.hot = hot;
  c.sv = sv;
#if DILU_VMODE != 0
  if (threadIdx.x == 0) {
    *sv = make_view<DILU_HOT_SMEM != 0>(hot, gblock, P.L);
#ifdef DILU_BOUNDS
    sv->ring = Chk<int32_t>(P.ring + (size_t)sc * P.F * P.W, (long long)P.F * P.W, sv->ring.id);
#else
    sv->ring = P.ring + (size_t)sc * P.F * P.W;
#endif
  }
#endif
  c.ring = P.ring + (size_t)sc * P.F * P.W;
  c.P = &P;
  c.g.K = K;
  c.g.crank = crank;
  c.g.cph = 0;
  c.g.off = 0;
  c.g.sub = 0;
  c.g.Kc = Kc;
  c.g.gu = P.gscratch + (size_t)sc * GSCR;
  c.g.gi = reinterpret_cast<int32_t*>(c.g.gu + 2 * KMAX);
  c.g.bar = reinterpret_cast<unsigned int*>(c.g.gu + 3 * KMAX);
  int32_t* const mem = K == 1 ? red.members : reinterpret_cast<int32_t*>(c.g.gu + 3 * KMAX + 8);
#ifdef DILU_BOUNDS
  c.members = Chk<int32_t>(mem, 64, DILU_ID_MEMBERS);
#else
  c.members = mem;
#endif
  c.flag = K == 1 ? red.flag : reinterpret_cast<int32_t*>(c.g.gu + 3 * KMAX + 40);
  c.frow = P.funcs + (size_t)sc * P.F * 16;
  {
    const int32_t per = (P.F + c.g.size() - 1) / c.g.size();
    c.b1lo = min(P.F, c.g.rank() * per);
    c.b1hi = min(P.F, c.b1lo + per);
  }
  c.scn_id = P.scen[sc * 4 + 0];
  c.om = P.scen[sc * 4 + 1];
  c.ga = P.scen[sc * 4 + 2];
  c.mode = P.scen[sc * 4 + 3];
  Acc acc = {};
  acc.z = &red.z;
  c.z = &red.z;
  if (threadIdx.x == 0) red.z = Acc0{};
  c.lat = red.lat;
  if (VAR & 4)
    for (int k = threadIdx.x; k < NLAT; k += blockDim.x) red.lat[k] = 0;
  int ph = 0;
  __syncthreads();
  DILU_VIEW(v, c);
  if (v.h[H_ERR]) return;     // uniform: nobody has written since the group started

  if (n_req >= 0) {
    // ---- dilu_place_batch: enqueue this scenario's requests in array order, one pass
    if (c.g.leader()) {
      for (int32_t j = 0; j < n_req && !v.h[H_ERR]; ++j) {
        if (req_scn[j] != sc) continue;
        const int32_t f = req_func[j];
        register_func(c, f, t0, P.Tp);
        out_iid[j] = enqueue(c, f, v.fKind[f] == K_TRAIN ? v.fNw[f] : 1);
      }
    }
    c.g.sync();
    if (!v.h[H_ERR]) placement(c, red, ph, t0, acc);
    c.g.sync();
    for (int32_t j = c.g.rank(); j < n_req; j += c.g.size()) {
      if (req_scn[j] != sc) continue;
      const int32_t id = out_iid[j];
      int32_t g = -1;
      for (int32_t s = v.fLh[req_func[j]]; s >= 0; s = v.iNext[s])
        if (v.iId[s] == id) { if (st_of(v.iMeta[s]) == ST_PLACED) g = v.iG[s * MAXST]; break; }
      out_gpu[j] = g;
    }
  } else {
    // ---- dilu_scale_step: the slot loop
    for (int32_t t = t0; t < t0 + n_slots; ++t) {
      constexpr bool fused = (VAR & 1) != 0;
      constexpr bool alg2 = (VAR & 2) != 0;
      constexpr bool lat = (VAR & 4) != 0;
#ifdef DILU_PHASE_TIMING
      long long tk0 = clock64(), tk1;
#define TICK(slot) do { tk1 = clock64(); if (c.g.leader()) acc.z->st[8 + (slot)] += tk1 - tk0; tk0 = tk1; } while (0)
#else
#define TICK(slot) do { } while (0)
#endif
      // (no cross-phase prefetch of the B1 ring word or the P0 pattern value: holding them
      // in registers across the boundary cost 8.5 % of C4's step)
      // overlapped slot: warp 0 runs the placement pass while warps 1.. run
      // P0/P1/P2 over the state after B3.  Exact when every cold start is >= 1 slot (the
      // host's P.ovl): what the pass commits is cold in this slot, so P0/P1/P2 never count
      // it; pending instances read as not ready (iReady = BIG), rows only grow past gNs.
      const bool ovl = !fused && !alg2 && !lat && P.ovl;
      if (ovl) {
        bool pass = false;
        TICK(0);
        if (P.SPS == 1 || t % P.SPS == 0) {
          pass = boundary(c, red, ph, t, acc, true);   // B1 + B3 (+ barrier)
          if (v.h[H_ERR]) break;                                  // uniform after B3's barrier
        }
        TICK(1);
        if (v.h[H_DIRTY]) {
          rebuild_layout(c);
          if (c.g.leader()) acc.z->st[S_LAYOUT] += 1;
        }
        TICK(2);
        if (threadIdx.x < 32) {
          if (pass) placement_pass<true>(c, red, ph, t, acc);
          if (pass) prerecount_warp(c);
          if (c.g.leader()) {        // after the pass: this slot's active set
            const long long na = v.h[H_NACT];
            acc.z->act += na;
            acc.z->memu += na * P.M - v.h[H_SUMU];
            acc.z->rows += P.G;
            acc.z->maxa = na > acc.z->maxa ? na : acc.z->maxa;
            acc.z->st[S_SLOT] += 1;
          }
          TICK(3);
        } else {
          Scn cw = c;
          cw.g.off = 32;
          const int nb = (int)blockDim.x - 32;
#ifdef DILU_PHASE_TIMING
          long long w0 = clock64(), w1;   // worker arm, first worker thread: st[19..21]
          const long long w_arm0 = w0;
#define WTICK(k) do { w1 = clock64(); if (threadIdx.x == 32) acc.z->st[k] += w1 - w0; w0 = w1; } while (0)
#else
#define WTICK(k) do { } while (0)
#endif
          phase0<false>(cw, t, acc);
          asm volatile("bar.sync 1, %0;" :: "r"(nb) : "memory");
          WTICK(19);
          phase1<false>(cw, t, acc);
          asm volatile("bar.sync 1, %0;" :: "r"(nb) : "memory");
          WTICK(20);
          phase2<false>(cw, t, acc);
          WTICK(21);
#ifdef DILU_PHASE_TIMING
          {
            const long long mine = clock64() - w_arm0;
            atomicMax(reinterpret_cast<unsigned long long*>(&acc.z->st[22]), (unsigned long long)mine);
          }
#endif
#undef WTICK
        }
        __syncthreads();     // join: B1(t+1) resets the window fields P0(t) accumulates
#ifdef DILU_PHASE_TIMING
        if (c.g.leader()) { acc.z->st[23] += acc.z->st[22]; acc.z->st[22] = 0; }
#endif
        TICK(5);
        continue;
      }
#if !DILU_HOT_SMEM
      if (fused && !alg2 && !lat && P.covl) {
        // overlapped batch (cluster engine): the leader's hardware cluster runs
        // the placement pass while the other CTAs of the group run P0b/P1b/P2b over the
        // state after B3.  Exact when every cold start is at least one batch (the host's
        // P.covl): what the pass commits is cold for the whole batch, so the batch never
        // counts it; rows only grow past gNs (commits append, the next repack sorts).
        bool pass = false;
        TICK(0);
        if (P.SPS == 1 || t % P.SPS == 0) {
          pass = boundary(c, red, ph, t, acc, true);   // B1 + B3 (+ barrier)
          if (v.h[H_ERR]) break;                       // uniform after B3's barrier
        }
        TICK(1);
        if (v.h[H_DIRTY]) {
          rebuild_layout(c);
          if (c.g.leader()) acc.z->st[S_LAYOUT] += 1;
        }
        TICK(2);
        int32_t B = P.SPS - t % P.SPS;
        if (B > t0 + n_slots - t) B = t0 + n_slots - t;
        if (B > P.L.B) B = P.L.B;
        if (t % P.SPS != 0) c.g.sync();   // previous batch's P2 has read rB / bB
        if (c.g.crank < c.g.Kc) {
          if (pass) {
            Scn cp = c;
            cp.g = c.g.first_cluster();
            placement_pass<false>(cp, red, ph, t, acc);
          }
          if (c.g.leader()) {        // after the pass: this batch's active set
            const long long na = v.h[H_NACT];
            acc.z->act += na * B;
            acc.z->memu += (na * P.M - v.h[H_SUMU]) * B;
            acc.z->rows += (long long)P.G * B;
            acc.z->maxa = na > acc.z->maxa ? na : acc.z->maxa;
            acc.z->st[S_SLOT] += B;
          }
          TICK(3);
        } else {
          Scn cw = c;
          cw.g.off = c.g.Kc * (int)blockDim.x;
          cw.g.sub = c.g.Kc;
          phase0_b<false>(cw, t, B, acc);
          cw.g.sync();
          phase1_b<false>(cw, t, B, acc);
          cw.g.sync();
          phase2_b<false>(cw, t, B, acc);
        }
        c.g.sync();                  // join
        TICK(5);
        t += B - 1;
        continue;
      }
#endif
      if (P.SPS == 1 || t % P.SPS == 0) {
        // no barrier here: B1 touches only the per-function window fields, which P2(t-1)
        // never reads, and B1's own count barrier orders P2(t-1) before B3 mutates state
        TICK(0);
        boundary(c, red, ph, t, acc);
        TICK(1);
        if (v.h[H_ERR]) break;
      }
      if (v.h[H_DIRTY]) {       // set only by boundary work, after >= 1 barrier since P1(t-1)
        rebuild_layout(c);
        if (c.g.leader()) acc.z->st[S_LAYOUT] += 1;
      }
      TICK(2);
      if (fused) {
        // one fused batch: the slots up to the next second boundary (<= L.B of them)
        int32_t B = P.SPS - t % P.SPS;
        if (B > t0 + n_slots - t) B = t0 + n_slots - t;
        if (B > P.L.B) B = P.L.B;
        if (t % P.SPS != 0) c.g.sync();   // previous batch's P2 has read rB / bB
        phase0_b<lat>(c, t, B, acc);
        if (c.g.leader()) {
          const long long na = v.h[H_NACT];
          acc.z->act += na * B;
          acc.z->memu += (na * P.M - v.h[H_SUMU]) * B;
          acc.z->rows += (long long)P.G * B;
          acc.z->maxa = na > acc.z->maxa ? na : acc.z->maxa;
          acc.z->st[S_SLOT] += B;
        }
        c.g.sync();
        TICK(3);
        if (alg2) phase1_alg2<lat>(c, t, B, v.rB, P.I, v.bB, P.I, v.gB, P.F, v.eB, acc);
        else phase1_b<lat>(c, t, B, acc);
        c.g.sync();
        TICK(4);
        phase2_b<lat>(c, t, B, acc);
        TICK(5);
        t += B - 1;
        continue;
      }
      phase0<lat>(c, t, acc);
      if (c.g.leader()) {
        const long long na = v.h[H_NACT];
        acc.z->act += na;
        acc.z->memu += na * P.M - v.h[H_SUMU];
        acc.z->rows += P.G;
        acc.z->maxa = na > acc.z->maxa ? na : acc.z->maxa;
        acc.z->st[S_SLOT] += 1;
      }
      c.g.sync();
      TICK(3);
      if (alg2) {
        const int par = t & 1;
        const bool one = P.SPS == 1;         // buffers as in phase1
        phase1_alg2<lat>(c, t, 1, v.iR + (one ? 0 : par) * P.I, 0, one ? GP32(v.iR + P.I) : GP32(v.iBmin + par * P.I), 0,
                         v.fGang + par * P.F, 0,
                         v.iEmax + par * P.I, acc);
      } else {
        phase1<lat>(c, t, acc);
      }
      c.g.sync();
      TICK(4);
      phase2<lat>(c, t, acc);
      TICK(5);
#undef TICK
    }
  }
  c.g.sync();

  // ---- block-reduce the tallies once per call; cluster CTAs merge with atomics
  {
    const int lane = threadIdx.x & 31;
    long long vals[9] = {acc.rtot, acc.rsrv, acc.rvio, acc.iexe, acc.tprg, acc.etot,
                         (long long)acc.hash, acc.nres, acc.nfun};
#pragma unroll
    for (int q = 0; q < 9; ++q) {
      long long x = vals[q];
      for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      if (lane == 0) atomicAdd(&acc.z->sum[q], (unsigned long long)x);   // mod 2^64 (R8)
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      long long s7[9];
      for (int q = 0; q < 9; ++q) s7[q] = (long long)acc.z->sum[q];
      long long d[NT];
      d[T_ACT] = acc.z->act;
      d[T_SMU] = acc.z->act * P.T_slot - s7[5];
      d[T_MEMU] = acc.z->memu;
      d[T_RTOT] = s7[0]; d[T_RSRV] = s7[1]; d[T_RVIO] = s7[2]; d[T_IEXE] = s7[3]; d[T_TPRG] = s7[4];
      d[T_POK] = acc.z->pok; d[T_PFAIL] = acc.z->pfail; d[T_COLD] = acc.z->cold;
      d[T_SOUT] = acc.z->sout; d[T_SIN] = acc.z->sin; d[T_SPLIT] = acc.z->split;
      d[T_HASH] = s7[6]; d[T_ROWS] = acc.z->rows; d[T_MAXA] = acc.z->maxa;
      acc.z->st[S_RES] += s7[7];
      acc.z->st[S_FUN] += s7[8];
      unsigned long long* T = reinterpret_cast<unsigned long long*>(P.tally) + (size_t)sc * NT;
      unsigned long long* ST = reinterpret_cast<unsigned long long*>(P.stats) + (size_t)sc * NSTAT;
      if (K == 1) {
        for (int k = 0; k < NT; ++k)
          if (k != T_MAXA) T[k] += (unsigned long long)d[k];
        if ((unsigned long long)d[T_MAXA] > T[T_MAXA]) T[T_MAXA] = (unsigned long long)d[T_MAXA];
        for (int k = 0; k < NSTAT; ++k) ST[k] += (unsigned long long)acc.z->st[k];
      } else {
        for (int k = 0; k < NT; ++k)
          if (k != T_MAXA) atomicAdd(T + k, (unsigned long long)d[k]);
        atomicMax(T + T_MAXA, (unsigned long long)d[T_MAXA]);
        for (int k = 0; k < NSTAT; ++k) atomicAdd(ST + k, (unsigned long long)acc.z->st[k]);
      }
    }
  }
  if (VAR & 4) {                       // request-level latency of this call
    __syncthreads();
    unsigned long long* LT = reinterpret_cast<unsigned long long*>(P.lat) + (size_t)sc * NLAT;
    for (int k = threadIdx.x; k < NLAT; k += blockDim.x)
      if (red.lat[k]) {
        if (K == 1) LT[k] += red.lat[k];
        else atomicAdd(LT + k, red.lat[k]);
      }
  }
  if (SMEM) {
#if DILU_HOT_SMEM
    cp_async_wait_all();             // in-flight prefetches land before the write-back
#endif
    __syncthreads();
    const int4* src = reinterpret_cast<const int4*>(smem);
    int4* dst = reinterpret_cast<int4*>(gblock);
    for (size_t k = threadIdx.x; k < P.L.hot_bytes / 16; k += blockDim.x) dst[k] = src[k];
  }
  c.g.sync();
}

#ifndef DILU_MINB
#define DILU_MINB 3
#endif
#ifndef DILU_SMEM_THREADS
#define DILU_SMEM_THREADS 256
#endif
constexpr int SMEM_MAX_THREADS = DILU_SMEM_THREADS;   // shared-memory variant: <= this many threads, DILU_MINB CTAs/SM

// The one-slot-per-second shared-memory kernel (C4's) runs 128 threads x 5 scenarios per
// SM (what the hot state allows): 96 registers per thread instead of 80 (no spills).
template <bool SMEM, int VAR>
__global__ void __launch_bounds__(SMEM ? (VAR == 0 ? 128 : SMEM_MAX_THREADS) : 1024,
                                  SMEM ? (VAR == 0 ? 5 : DILU_MINB) : 1)
k_run(const __grid_constant__ Params Pin, int32_t* next_scn, int32_t t0,
                                              int32_t n_slots, int32_t n_req,
                                              const int32_t* req_scn, const int32_t* req_func,
                                              int32_t* out_gpu, int32_t* out_iid) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ Red red;
  __shared__ View sv;
  for (;;) {
    if (threadIdx.x == 0) red.flag[0] = atomicAdd(next_scn, 1);
    __syncthreads();
    const int32_t sc = red.flag[0];
    __syncthreads();
    if (sc >= Pin.S) break;
    run_scenario<SMEM, VAR>(Pin, red, &sv, smem, sc, t0, n_slots, n_req, req_scn, req_func, out_gpu, out_iid);
  }
}

// Large scenarios (C3/C5): one thread-block cluster of K CTAs per scenario (cluster
// dims set at launch, K <= 16), state in HBM/L2; clusters beyond the resident capacity
// run in waves.  Same device code as k_run through the group abstraction.
template <int VAR>
__global__ void __launch_bounds__(1024, 1)
k_run_cluster(const __grid_constant__ Params Pin, int32_t t0, int32_t n_slots, int32_t n_req, const int32_t* req_scn,
              const int32_t* req_func, int32_t* out_gpu, int32_t* out_iid) {
  __shared__ Red red;
  __shared__ View sv;
  unsigned int csize;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(csize));
  // a scenario's group: Pin.gK consecutive CTAs = Pin.gK / csize whole hardware clusters
  const int32_t K = Pin.gK;
  const int32_t sc = blockIdx.x / K;
  if (sc >= Pin.S) return;   // whole groups only: uniform across the group
  run_scenario<false, VAR>(Pin, red, &sv, nullptr, sc, t0, n_slots, n_req, req_scn, req_func, out_gpu,
                      out_iid, (int)K, (int)(blockIdx.x % K), (int)csize);
}

#ifndef DILU_VARIANT_TU   // the init / snapshot kernels live in dilu_api.cu's unit only
// Initialise every scenario's block at slot 0 (one CTA per scenario).
template <bool N>
__global__ void k_init(Params P) {
  const int32_t sc = blockIdx.x;
  uint8_t* b = P.state + (size_t)sc * P.L.bytes;
  const ViewT<N> v = make_view<N>(b, b, P.L);
  const int32_t* rows = P.funcs + (size_t)sc * P.F * 16;
  // (dilu_sim_reset zeroes the whole state area first: alignment gaps are defined bytes
  // when the run kernel stages the hot region -- compute-sanitizer initcheck clean)
  for (int k = threadIdx.x; k < H_WORDS; k += blockDim.x) v.h[k] = 0;
  __syncthreads();
  if (threadIdx.x == 0) { v.h[H_FSTOP] = P.I; v.h[H_DIRTY] = 1; v.h[H_LASTEP] = -1; v.h[H_QNEWPOS] = -1; }
  for (int32_t g = threadIdx.x; g < P.G; g += blockDim.x) {
    v.gR[g] = 0; v.gL[g] = 0; v.gU[g] = 0; v.gN[g] = 0; v.gNs[g] = 0; v.gExcl[g] = 0; v.gGrow[g] = 0;
    v.gRel[g] = 0;
    v.gMask[g] = 0;
  }
  for (int32_t k = threadIdx.x; k < P.G * RES; k += blockDim.x) v.gRes[k] = -1;
  for (int32_t s = threadIdx.x; s < P.I; s += blockDim.x) {
    v.iId[s] = -1; v.iFunc[s] = -1; v.iMeta[s] = ST_FREE; v.iReady[s] = 0; v.iNext[s] = -1;
    for (int k = 0; k < MAXST; ++k) { v.iG[s * MAXST + k] = -1; v.iShare[s * MAXST + k] = 0; }
    v.iSh0[s] = 0;
    v.iR[s] = 0; v.iR[P.I + s] = P.SPS == 1 ? BIG : 0; v.iBmin[s] = BIG; v.iBmin[P.I + s] = BIG;
    v.fstack[s] = P.I - 1 - s;
  }
  const int32_t mode = P.scen[sc * 4 + 3];
  for (int32_t f = threadIdx.x; f < P.F; f += blockDim.x) {
    const int32_t* r = rows + (size_t)f * 16;
    const int32_t kind = r[0];
    // baseline quota transforms: limit-quota modes run at lim, MPS-r at req
    const int32_t req = (mode == M_STATIC_LIMIT || mode == M_EAGER) ? r[4] : r[3];
    const int32_t limq = mode == M_STATIC_REQUEST ? r[3] : r[4];
    v.fKind[f] = kind; v.fPrio[f] = r[1]; v.fIbs[f] = r[2] > 0 ? r[2] : 1; v.fReq[f] = req;
    v.fLim[f] = limq; v.fMem[f] = r[5]; v.fCb[f] = r[6] > 0 ? r[6] : 1; v.fNw[f] = r[7];
    v.fCold[f] = r[9]; v.fCls[f] = r[10]; v.fPat[f] = r[13]; v.fScale[f] = r[14];
    v.fPhase[f] = r[15];
    // training demand d = lim * duty; Exclusive owns the whole GPU (lim = T_slot, D7)
    const long long lim_tok = (long long)(mode == M_EXCLUSIVE ? 1000 : limq) * P.slot_ms;
    v.fDtr[f] = kind == K_TRAIN ? (int32_t)(lim_tok * r[8] / 1000) : 0;
    // R5: cap1 = (1000/slot_ms) * floor(req_tok / c_b) * IBS
    v.fCap1[f] = is_inf(kind) ? (long long)P.SPS * (((long long)req * P.slot_ms) / r[6]) * r[2] : 0;
    v.fReg[f] = 0; v.fNsamp[f] = 0; v.fAcc[f] = 0; v.fHead[f] = 0; v.fUp[f] = 0; v.fDown[f] = 0;
    v.fThrn[f] = -1; v.fOld[f] = 0; v.fPv[f] = -1; v.fNlive[f] = 0; v.fLh[f] = -1; v.fLt[f] = -1;
    v.fGang[f] = BIG; v.fGang[P.F + f] = BIG; v.fFlag[f] = 0; v.fK[f] = 0; v.fList[f] = 0;
    v.fArr[f] = r[11]; v.fDep[f] = r[12]; v.fPidx[f] = 0;
  }
  if (P.flags & 4)
    for (int32_t g = threadIdx.x; g < P.G; g += blockDim.x) { v.aSt[g] = A2_NONE; v.aOw[g] = -1; v.aDt[g] = 0; }
  if (P.flags & 8) {                   // request-level latency (D10)
    for (int k = threadIdx.x; k < NLAT; k += blockDim.x) P.lat[(size_t)sc * NLAT + k] = 0;
    for (int32_t f = threadIdx.x; f < P.F; f += blockDim.x) {
      const int32_t* r = rows + (size_t)f * 16;
      // SLO = 2 * t_exec at the profiled request (R4): c_b = req * SLO / 2
      v.fSlo[f] = is_inf(r[0]) ? (int32_t)(2000LL * r[6] / r[3]) : 0;
    }
    for (size_t k = threadIdx.x; k < 2 * (size_t)P.I; k += blockDim.x) v.iEmax[k] = 0;
    if (P.L.B > 1)
      for (size_t k = threadIdx.x; k < (size_t)P.L.B * P.I; k += blockDim.x) v.eB[k] = 0;
  }
  if (P.L.B > 1) {
    for (size_t k = threadIdx.x; k < (size_t)P.L.B * P.I; k += blockDim.x) v.bB[k] = BIG;
    for (size_t k = threadIdx.x; k < (size_t)P.L.B * P.F; k += blockDim.x) v.gB[k] = BIG;
  }
  if (threadIdx.x == 0) {   // static lists: inference functions (P0), training + LLM (P2)
    int32_t ni = 0, nd = 0;
    for (int32_t f = 0; f < P.F; ++f) {
      const int32_t kind = rows[(size_t)f * 16];
      if (is_inf(kind)) v.fInfL[ni++] = f;
      if (kind == K_TRAIN || kind == K_LLM) v.fDefL[nd++] = f;
    }
    v.h[H_NINF] = ni;
    v.h[H_NDEF] = nd;
  }
  for (int32_t q = threadIdx.x; q < P.I; q += blockDim.x) {
    v.qN[q] = 0; v.qFail[q] = -1; v.qSlot[q] = 0;
  }
  for (int k = threadIdx.x; k < NT; k += blockDim.x) P.tally[(size_t)sc * NT + k] = 0;
  for (int k = threadIdx.x; k < NSTAT; k += blockDim.x) P.stats[(size_t)sc * NSTAT + k] = 0;
  for (int k = threadIdx.x; k < RLOG; k += blockDim.x) { v.rlG[k] = 0; v.rlE[k] = 0; }
}

// Snapshot for parity tests (off the timed path).
// State invariants (cfg.flags bit1), checked on the device
// at the end of every dilu_scale_step / dilu_place_batch call, one CTA per scenario:
//   I1  R_g <= Omega_u, L_g <= gamma_u, U_g <= M, |res_g| <= 32 (Eq.4)
//   I2  the active count equals #{g : res_g != {}}, the memory total equals sum_g U_g (Eq.5)
//   I3  R_g, L_g, U_g equal the sums over the residents of g (their stage shares)
//   I7  a placed instance has 1..4 stage GPUs, distinct, each listing it (Eq.2)
// A violation sets the scenario's error word to DILU_E_INVARIANT (2), which dilu_metrics
// reports; I6 (requests total = served + violated) is checked there on the tallies.
template <bool N>
__global__ void k_check(Params P) {
  const int32_t sc = blockIdx.x;
  uint8_t* blk = P.state + (size_t)sc * P.L.bytes;
  const ViewT<N> v = make_view<N>(blk, blk, P.L);
  const int32_t om = P.scen[sc * 4 + 1], ga = P.scen[sc * 4 + 2];
  __shared__ int bad;
  __shared__ unsigned long long act, sumu;
  if (threadIdx.x == 0) { bad = 0; act = 0; sumu = 0; }
  __syncthreads();
  if (v.h[H_ERR]) return;                        // an earlier error stands
  for (int32_t g = threadIdx.x; g < P.G; g += blockDim.x) {
    const int32_t n = v.gN[g];
    long long R = 0, L = 0, U = 0;
    bool ok = n >= 0 && n <= RES && v.gR[g] <= om && v.gL[g] <= ga && v.gU[g] <= P.M;   // I1
    for (int32_t j = 0; ok && j < n; ++j) {
      const int32_t s = v.gRes[(size_t)g * RES + j];
      if (s < 0 || s >= P.I || st_of(v.iMeta[s]) != ST_PLACED) { ok = false; break; }
      const int32_t f = v.iFunc[s], ns = nst_of(v.iMeta[s]);
      R += v.fReq[f]; L += v.fLim[f];
      int hits = 0;
      for (int k = 0; k < ns; ++k)
        if (v.iG[s * MAXST + k] == g) { U += k == 0 ? v.iSh0[s] : v.iShare[s * MAXST + k]; ++hits; }
      ok &= hits == 1;                           // listed on g exactly once among its stages
    }
    ok &= R == v.gR[g] && L == v.gL[g] && U == v.gU[g];                                   // I3
    if (!ok) atomicOr(&bad, 1);
    if (n > 0) atomicAdd(&act, 1ull);
    atomicAdd(&sumu, (unsigned long long)(long long)v.gU[g]);
  }
  for (int32_t s = threadIdx.x; s < P.I; s += blockDim.x) {                              // I7
    const int32_t meta = v.iMeta[s];
    if (st_of(meta) != ST_PLACED) continue;
    const int32_t ns = nst_of(meta);
    bool ok = ns >= 1 && ns <= MAXST;
    for (int k = 0; ok && k < ns; ++k) {
      const int32_t g = v.iG[s * MAXST + k];
      ok = g >= 0 && g < P.G;
      for (int k2 = 0; ok && k2 < k; ++k2) ok = v.iG[s * MAXST + k2] != g;
      bool listed = false;
      for (int32_t j = 0; ok && j < v.gN[g] && !listed; ++j) listed = v.gRes[(size_t)g * RES + j] == s;
      ok &= listed;
    }
    if (!ok) atomicOr(&bad, 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (act != (unsigned long long)v.h[H_NACT] || (long long)sumu != (long long)v.h[H_SUMU]) bad = 1;   // I2
    if (bad) v.h[H_ERR] = 2;
  }
}

template <bool N>
__global__ void k_snapshot(Params P, int32_t id_cap, int32_t* out_gpu, int32_t* out_inst) {
  const int32_t sc = blockIdx.x;
  const ViewT<N> v = make_view<N>(P.state + (size_t)sc * P.L.bytes, P.state + (size_t)sc * P.L.bytes, P.L);
  if (out_gpu)
    for (int32_t g = threadIdx.x; g < P.G; g += blockDim.x) {
      int32_t* o = out_gpu + ((size_t)sc * P.G + g) * 4;
      o[0] = v.gR[g]; o[1] = v.gL[g]; o[2] = v.gU[g]; o[3] = v.gN[g];
    }
  if (!out_inst) return;
  const int32_t issued = v.h[H_NEXT_IID];
  for (int32_t id = threadIdx.x; id < id_cap; id += blockDim.x) {
    int32_t* o = out_inst + ((size_t)sc * id_cap + id) * 12;
    if (id >= issued) { for (int k = 0; k < 12; ++k) o[k] = -1; continue; }
    // terminated unless a live slot overwrites it below
    o[0] = -1; o[1] = 2; o[2] = 0; o[3] = -1;
    for (int k = 0; k < MAXST; ++k) { o[4 + k] = -1; o[8 + k] = 0; }
  }
  __syncthreads();
  for (int32_t s = threadIdx.x; s < P.I; s += blockDim.x) {
    const int32_t meta = v.iMeta[s];
    if (st_of(meta) == ST_FREE) continue;
    const int32_t id = v.iId[s];
    if (id >= id_cap) continue;
    int32_t* o = out_inst + ((size_t)sc * id_cap + id) * 12;
    const bool pl = st_of(meta) == ST_PLACED;
    o[0] = v.iFunc[s];
    o[1] = pl ? 1 : 0;
    o[2] = pl ? nst_of(meta) : 0;
    o[3] = pl ? v.iReady[s] : -1;
    for (int k = 0; k < MAXST; ++k) {
      const bool on = pl && k < nst_of(meta);
      o[4 + k] = on ? v.iG[s * MAXST + k] : -1;
      o[8 + k] = on ? v.iShare[s * MAXST + k] : 0;
    }
  }
}
#endif  // DILU_VARIANT_TU

}  // namespace dilu
