// state.cuh -- per-scenario state layout of the B200 Dilu provisioning loop.
//
// Every scenario owns one contiguous, 16-byte-aligned state block of SoA int32
// arrays (plus one int64 array), split into a hot region (read or written every slot)
// and a cold region (placement / release / scaling events only).  The run kernel
// stages the hot region into shared memory when it fits (the 64-GPU scenarios of
// C1/C2/C4: ~45 KB) and otherwise works in place in HBM/L2 through the same generic
// pointers (C3/C5); the cold region always stays in global memory (L1/L2-cached).  Per-function RPS
// rings (W ints per function, touched once per simulated second) always live in
// global memory.  See DESIGN.md s5 "Data layout".
#pragma once
#include <stddef.h>
#include <stdint.h>

namespace dilu {

constexpr int RES = 32;    // residents per GPU row (Q23; one lane each)
constexpr int MAXST = 4;   // LLM pipeline stages
constexpr int NT = 17;     // tally vector length
constexpr int32_t BIG = 0x7fffffff;
constexpr int RLOG = 64;   // release log ring (GPU, epoch) for the placement retry skip
constexpr int NSTAT = 24;  // kernel statistics per scenario (dilu_kernel_stats): 8 counters + 16 timers
constexpr int NLAT = 82;   // request-level latency vector: 80 buckets, violations, latency sum
constexpr int LAT_UNSERVED = 79, LAT_VIOL = 80, LAT_SUM = 81;

enum : int32_t { K_UNUSED = -1, K_INF = 0, K_LLM = 1, K_TRAIN = 2 };
enum : int32_t { ST_FREE = 0, ST_PEND = 1, ST_PLACED = 2 };

// header slots (int32)
enum : int {
  H_NEXT_IID = 0, H_NLIVE, H_QLEN, H_NACT, H_SUMU, H_EPOCH, H_DIRTY, H_FSTOP, H_ERR,
  H_NEV /* events of the current boundary (prerecount_warp) */, H_CCNT = 10 /*6*/, H_CBASE = 16 /*7*/, H_GBASE = 23 /*6*/, H_CCNT2 = 29 /*6*/,
  H_RLN = 35 /* release-log entries appended */, H_NINF = 36, H_NDEF = 37,
  H_QLIVE = 38 /* live queue requests */, H_LASTEP = 39 /* release epoch at the last pass's end */,
  H_QNEWPOS = 40 /* first request enqueued since the last pass, -1 if none */,
  H_SPARE = 41 /* unused */, H_WORDS = 44
};

// tally indices (match include/dilu.h)
enum : int {
  T_ACT = 0, T_SMU, T_MEMU, T_RTOT, T_RSRV, T_RVIO, T_IEXE, T_TPRG, T_POK, T_PFAIL,
  T_COLD, T_SOUT, T_SIN, T_SPLIT, T_HASH, T_ROWS, T_MAXA
};

// Element types of the state arrays.  Wide (ET<false>): int32 everywhere -- the cluster
// engine and the global-memory CTA kernels.  Narrow (ET<true>): the shared-memory CTA
// kernels when I, F, G <= 32767 and W <= 127: slot / function / GPU indices in int16,
// flags, small counts and window counters in int8 -- the hot region of a C4 scenario
// shrinks so more scenarios are resident per SM (DESIGN.md s5 "Narrow state").
template <bool B, class A, class C> struct Sel { typedef A T; };
template <class A, class C> struct Sel<false, A, C> { typedef C T; };
template <bool N> struct ET {
  typedef typename Sel<N, int16_t, int32_t>::T idx;    // slot, function, GPU index (or -1)
  typedef typename Sel<N, int8_t, int32_t>::T small;   // flags, metas, counts <= 127
  typedef typename Sel<N, int16_t, int32_t>::T quota;  // per-mille quotas, live counts
};
inline bool narrow_ok(int32_t G, int32_t F, int32_t I, int32_t W) {
  return G <= 32767 && F <= 32767 && I <= 32767 && W <= 127;
}

struct Layout {
  int32_t G, F, I, W, B;   // B: slots per fused batch between second boundaries (1 = unfused)
  int32_t A2, LT;          // literal Alg.2 / request-level latency arrays present
  int32_t N;               // narrow element types (ET<true>): CTA engine, hot region in smem
  // byte offsets inside one block
  size_t hdr;
  size_t gR, gL, gU, gN, gNs, gRes, gExcl, gGrow, gMask, gChk, gRel, rlG, rlE;
  size_t iId, iFunc, iMeta, iReady, iG, iSh0, iShare, iNext, iR, iBmin, fstack;
  size_t fKind, fPrio, fReq, fLim, fMem, fCb, fIbs, fNw, fCold, fCls, fDtr, fPat, fScale,
      fPhase, fCap1;
  size_t fReg, fNsamp, fAcc, fHead, fUp, fDown, fThrn, fOld, fPv, fNlive, fLh, fLt, fGang, fFlag, fK,
      fList, fArr, fDep, fPidx, fInfL, fDefL;
  size_t qN, qFail, qSlot, iQ;
  size_t rB, bB, gB;       // per-batch-slot r, LLM stage minimum, training gang (B > 1 only)
  size_t aTc, aTm, aRl, aLe, aSt, aOw, aDt;   // literal Alg.2 state (cfg.flags bit2 only)
  size_t fSlo, iEmax, eB;  // request-level latency (cfg.flags bit3 only)
  size_t gRcl;             // wide layout: each resident's affinity class, beside gRes
  size_t hot_bytes, bytes;
};

inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

inline Layout make_layout(int32_t G, int32_t F, int32_t I, int32_t W, int32_t B = 1,
                          bool alg2 = false, bool lat = false, bool narrow = false) {
  Layout L;
  L.G = G; L.F = F; L.I = I; L.W = W; L.B = B; L.A2 = alg2; L.LT = lat; L.N = narrow;
  const size_t X = narrow ? 2 : 4;      // index arrays
  const size_t S1 = narrow ? 1 : 4;     // small arrays
  const size_t Q = narrow ? 2 : 4;      // quota / count arrays
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t at = o; o = align16(o + bytes); return at; };
  // hot region: touched every slot -> staged in shared memory when it fits
  L.hdr = take(H_WORDS * 4);
  L.gR = take(4 * (size_t)G); L.gL = take(4 * (size_t)G); L.gU = take(4 * (size_t)G);
  L.gN = take(S1 * (size_t)G);
  L.gNs = take(S1 * (size_t)G);         // row sizes at the last repack (overlapped slots, s5)
  L.gRes = take(X * (size_t)G * RES);
  L.gExcl = take(S1 * (size_t)G); L.gGrow = take(X * (size_t)G);
  L.gMask = take(8 * (size_t)G);        // bit (affinity_class & 63) per resident class
  L.gChk = take(4 * ((size_t)G + 8));   // P1 warp-chunk descriptors (first row | rows << 16 | class << 24)
  L.rlG = take(4 * RLOG); L.rlE = take(4 * RLOG);
  L.iId = take(4 * (size_t)I); L.iFunc = take(X * (size_t)I); L.iMeta = take(S1 * (size_t)I);
  L.iReady = take(4 * (size_t)I); L.iNext = take(X * (size_t)I); L.iR = take(4 * 2 * (size_t)I);
#ifdef DILU_HOT_PAD
  take(DILU_HOT_PAD);                   // layout-sensitivity parity variant
#endif
  L.fKind = take(S1 * (size_t)F); L.fReq = take(Q * (size_t)F); L.fLim = take(Q * (size_t)F);
  L.fCb = take(4 * (size_t)F); L.fIbs = take(4 * (size_t)F);
  L.fNw = take(S1 * (size_t)F); L.fCls = take(4 * (size_t)F); L.fDtr = take(4 * (size_t)F);
  L.fPat = take(4 * (size_t)F); L.fScale = take(4 * (size_t)F);
  L.fCap1 = take(8 * (size_t)F);
  L.fReg = take(S1 * (size_t)F); L.fNsamp = take(S1 * (size_t)F); L.fAcc = take(4 * (size_t)F);
  L.fHead = take(S1 * (size_t)F); L.fUp = take(S1 * (size_t)F); L.fDown = take(S1 * (size_t)F);
  L.fThrn = take(Q * (size_t)F);
  L.fOld = take(4 * (size_t)F); L.fPv = take(4 * (size_t)F);   // cp.async landing slots
  L.fNlive = take(Q * (size_t)F); L.fLh = take(X * (size_t)F);
  L.fGang = take(4 * 2 * (size_t)F); L.fFlag = take(S1 * (size_t)F);
  L.fArr = take(4 * (size_t)F); L.fDep = take(4 * (size_t)F); L.fPidx = take(4 * (size_t)F);
  L.fInfL = take(X * (size_t)F); L.fDefL = take(X * (size_t)F);
  // serial-path structures the leader walks every boundary (queue, free stack, ...)
  L.gRel = take(4 * (size_t)G);
  L.fLt = take(X * (size_t)F); L.fK = take(4 * (size_t)F); L.fList = take(X * (size_t)F);
  L.fstack = take(X * (size_t)I);
  L.fPrio = take(S1 * (size_t)F);
  // queue of pending requests: first member's slot (its function and first id are that
  // instance's), member count, failure epoch; per instance its request index
  L.qN = take(S1 * (size_t)I); L.qFail = take(4 * (size_t)I); L.qSlot = take(X * (size_t)I);
  L.iQ = take(X * (size_t)I);
  L.hot_bytes = align16(o);
  // cold region: stage placements and LLM stage minima, per-function constants read only
  // by placement / registration -> stays in HBM/L2 (L1-cached)
  L.fMem = take(4 * (size_t)F); L.fCold = take(4 * (size_t)F); L.fPhase = take(4 * (size_t)F);
  L.iG = take(2 * (size_t)I * MAXST);   // int16 stage GPUs (G <= 32767)
  L.iSh0 = take(4 * (size_t)I);         // stage-0 memory share
  L.iShare = take(4 * (size_t)I * MAXST);
  L.iBmin = take(4 * 2 * (size_t)I);
  // fused-batch buffers [B][I] / [B][F] (slot-major): the slots between two second
  // boundaries share one placement state, so P0/P1/P2 run once per batch
  const size_t bb = B > 1 ? (size_t)B : 0;
  L.rB = take(4 * bb * I); L.bB = take(4 * bb * I); L.gB = take(4 * bb * F);
  // literal Algorithm 2 (D8): per stage resident T_current, T_min, R_last,
  // last executing period [I][MAXST]; per GPU state, owner id, owner dT [G]
  const size_t ai = alg2 ? (size_t)I * MAXST : 0, ag = alg2 ? (size_t)G : 0;
  L.aTc = take(4 * ai); L.aTm = take(4 * ai); L.aRl = take(4 * ai); L.aLe = take(4 * ai);
  L.aSt = take(4 * ag); L.aOw = take(4 * ag); L.aDt = take(4 * ag);
  // request-level latency (D10): per-function SLO (us), per split instance the
  // slowest stage's batch time, per slot parity [2][I] or per batch slot [B][I]
  L.fSlo = take(lat ? 4 * (size_t)F : 0);
  L.iEmax = take(lat ? 4 * 2 * (size_t)I : 0);
  L.eB = take(lat && B > 1 ? 4 * (size_t)B * I : 0);
  // wide layout (state in HBM/L2): the affinity class of each row position, kept beside
  // gRes so the placement's affinity test reads one row instead of res -> func -> class
  L.gRcl = take(narrow ? 0 : 4 * (size_t)G * RES);
  L.bytes = align16(o);
  return L;
}


// ---- element pointers of the view ----------------------------------------------------
// Normal builds: raw pointers.  -DDILU_BOUNDS (debug side library): every
// array of the view is a checked pointer {base, offset, length, array id}; an index
// outside [0, length) of its array prints the array, the index and the thread and traps.
// Phase code declares its local aliases through DP()/DPN() so they stay checked too.
#ifdef DILU_BOUNDS
#ifdef __CUDACC__
static __device__ __noinline__ void dilu_oob(int id, long long j, long long n);
#endif
template <class T> struct Chk {
  T* b; long long o, n; int id;
  __host__ __device__ Chk() : b(nullptr), o(0), n(0), id(-1) {}
  __host__ __device__ Chk(T* b_, long long n_, int id_) : b(b_), o(0), n(n_), id(id_) {}
  template <class U> __host__ __device__ Chk(const Chk<U>& x) : b(x.b), o(x.o), n(x.n), id(x.id) {}
#ifdef __CUDACC__
  template <class Ix> __device__ __forceinline__ T& operator[](Ix i) const {
    const long long j = o + (long long)i;
    if (j < 0 || j >= n) dilu_oob(id, j, n);
    return b[j];
  }
#endif
  template <class Ix> __host__ __device__ Chk operator+(Ix k) const { Chk r = *this; r.o += (long long)k; return r; }
  __host__ __device__ operator T*() const { return b + o; }
};
#define VP(T) ::dilu::Chk<T>
#define HP(T) ::dilu::Chk<T>
#define DP(T) ::dilu::Chk<T>
#define DPN(T) ::dilu::Chk<T>
#else
#define VP(T) T*
#define DP(T) T* __restrict__
#define DPN(T) T*
#ifndef DILU_VMODE
#define DILU_VMODE 1
#endif
#if defined(__CUDACC__) && defined(DILU_HOT_SMEM) && DILU_HOT_SMEM && DILU_VMODE != 1
// Hot-region arrays of the shared-memory kernels (run_variants.cu units compiled with
// DILU_HOT_SMEM=1): a 32-bit byte offset into the kernel's dynamic shared memory.  Every
// access forms its address from the __shared__ symbol itself, so NVVM's address-space
// inference emits LDS/STS/ATOMS (28 vs 33 cycles per dependent load against generic
// LD/ST, tools/ubench/smem_chase.cu) with no __builtin_assume (whose false assumptions
// would be undefined behaviour the optimiser may exploit) and half-size view fields.
extern __shared__ __align__(16) uint8_t dilu_dsmem[];
template <class T> struct SPtr {
  uint32_t o;
  SPtr() = default;
  static __host__ __device__ SPtr at(size_t off) { SPtr r; r.o = (uint32_t)off; return r; }
  __device__ __forceinline__ T* ptr() const { return reinterpret_cast<T*>(dilu_dsmem + o); }
  template <class Ix> __device__ __forceinline__ T& operator[](Ix i) const { return ptr()[i]; }
  template <class Ix> __device__ __forceinline__ SPtr operator+(Ix k) const {
    return at(o + (size_t)(long long)k * sizeof(T));
  }
  __device__ __forceinline__ operator T*() const { return ptr(); }
};
#define HP(T) ::dilu::SPtr<T>
#else
#define HP(T) T*
#endif
#endif

// Typed view of one scenario's block (pointers into smem or global).
template <bool N> struct ViewT {
  typedef typename ET<N>::idx X;
  typedef typename ET<N>::small S1;
  typedef typename ET<N>::quota Q;
  typedef VP(int32_t) PI;   // cold region / global arrays
  typedef HP(int32_t) HI;   // hot region (shared memory in the DILU_HOT_SMEM kernels)
  typedef HP(X) HX;
  typedef HP(S1) HS;
  typedef HP(Q) HQ;
  HI h;
  HI gR, gL, gU, gRel, rlG, rlE;
  HS gN, gNs, gExcl;
  HX gRes, gGrow;
  HP(unsigned long long) gMask;
  HI gChk;
  HI iId, iReady, iR;
  HX iFunc, iNext, fstack;
  HS iMeta;
  PI iSh0, iShare, iBmin;
  VP(int16_t) iG;
  HS fKind, fPrio, fNw;
  HQ fReq, fLim;
  HI fCb, fIbs, fCls, fDtr, fPat, fScale;
  PI fMem, fCold, fPhase;
  HP(int64_t) fCap1;
  HS fReg, fNsamp, fHead, fUp, fDown, fFlag;
  HQ fThrn, fNlive;
  HI fAcc, fOld, fPv, fGang, fK, fArr, fDep, fPidx;
  HX fLh, fLt, fList, fInfL, fDefL;
  HS qN;
  HI qFail;
  HX qSlot, iQ;
  PI rB, bB, gB;
  PI aTc, aTm, aRl, aLe, aSt, aOw, aDt;
  PI fSlo, iEmax, eB;
  PI gRcl;
  PI ring;  // global [F][W]
};

#if defined(__CUDACC__) && defined(DILU_HOT_SMEM) && DILU_HOT_SMEM && !defined(DILU_BOUNDS) && DILU_VMODE != 1
template <class T> __host__ __device__ inline void dilu_set(SPtr<T>& f, uint8_t*, uint8_t*, size_t off, size_t) {
  f = SPtr<T>::at(off);   // hot arrays always precede hot_bytes (make_layout)
}
template <class T> __host__ __device__ inline void dilu_set(T*& f, uint8_t* hot, uint8_t* b, size_t off, size_t hb) {
  f = reinterpret_cast<T*>((off < hb ? hot : b) + off);
}
#endif
template <bool N>
#ifdef __CUDACC__
__host__ __device__
#endif
inline ViewT<N> make_view(uint8_t* hot, uint8_t* b, const Layout& L) {
  // arrays in the hot region resolve against `hot` (smem copy or b), the rest against b
  typedef typename ET<N>::idx X;
  typedef typename ET<N>::small S1;
  typedef typename ET<N>::quota Q;
  ViewT<N> v;
  const long long G = L.G, F = L.F, I = L.I, BB = L.B > 1 ? L.B : 0;
  const long long AI = L.A2 ? I * MAXST : 0, AG = L.A2 ? G : 0;
#ifdef DILU_BOUNDS
  int id = 0;
#define PT(T, name, cnt) v.name = Chk<T>(reinterpret_cast<T*>((L.name < L.hot_bytes ? hot : b) + L.name), (cnt), id++)
#elif defined(__CUDACC__) && defined(DILU_HOT_SMEM) && DILU_HOT_SMEM && DILU_VMODE != 1
  // shared-memory kernels: hot arrays are offsets into dynamic shared memory (SPtr), the
  // cold ones generic pointers into the global block
#define PT(T, name, cnt) dilu_set(v.name, hot, b, L.name, L.hot_bytes)
#else
#define PT(T, name, cnt) v.name = reinterpret_cast<T*>((L.name < L.hot_bytes ? hot : b) + L.name)
#endif
  // (order = DILU_ARRAY_NAMES below)
#ifdef DILU_BOUNDS
  v.h = Chk<int32_t>(reinterpret_cast<int32_t*>(hot + L.hdr), H_WORDS, id++);
#elif defined(__CUDACC__) && defined(DILU_HOT_SMEM) && DILU_HOT_SMEM && DILU_VMODE != 1
  v.h = SPtr<int32_t>::at(L.hdr);
#else
  v.h = reinterpret_cast<int32_t*>(hot + L.hdr);
#endif
  PT(int32_t, gR, G); PT(int32_t, gL, G); PT(int32_t, gU, G); PT(S1, gN, G); PT(S1, gNs, G);
  PT(X, gRes, G * RES); PT(S1, gExcl, G); PT(X, gGrow, G); PT(int32_t, gRel, G);
  PT(int32_t, rlG, RLOG); PT(int32_t, rlE, RLOG);
  PT(unsigned long long, gMask, G);
  PT(int32_t, gChk, G + 8);
  PT(int32_t, iId, I); PT(X, iFunc, I); PT(S1, iMeta, I); PT(int32_t, iReady, I);
  PT(int32_t, iSh0, I); PT(int32_t, iShare, I * MAXST); PT(X, iNext, I); PT(int32_t, iR, 2 * I);
  PT(int32_t, iBmin, 2 * I); PT(X, fstack, I);
  PT(int16_t, iG, I * MAXST);
  PT(S1, fKind, F); PT(S1, fPrio, F); PT(Q, fReq, F); PT(Q, fLim, F);
  PT(int32_t, fMem, F); PT(int32_t, fCb, F); PT(int32_t, fIbs, F); PT(S1, fNw, F);
  PT(int32_t, fCold, F); PT(int32_t, fCls, F); PT(int32_t, fDtr, F); PT(int32_t, fPat, F);
  PT(int32_t, fScale, F); PT(int32_t, fPhase, F);
  PT(int64_t, fCap1, F);
  PT(S1, fReg, F); PT(S1, fNsamp, F); PT(int32_t, fAcc, F); PT(S1, fHead, F);
  PT(S1, fUp, F); PT(S1, fDown, F); PT(Q, fThrn, F); PT(int32_t, fOld, F);
  PT(int32_t, fPv, F); PT(Q, fNlive, F); PT(X, fLh, F); PT(X, fLt, F);
  PT(int32_t, fGang, 2 * F); PT(S1, fFlag, F); PT(int32_t, fK, F); PT(X, fList, F);
  PT(int32_t, fArr, F); PT(int32_t, fDep, F); PT(int32_t, fPidx, F); PT(X, fInfL, F);
  PT(X, fDefL, F);
  PT(S1, qN, I); PT(int32_t, qFail, I);
  PT(X, qSlot, I); PT(X, iQ, I);
  PT(int32_t, rB, BB * I); PT(int32_t, bB, BB * I); PT(int32_t, gB, BB * F);
  PT(int32_t, aTc, AI); PT(int32_t, aTm, AI); PT(int32_t, aRl, AI); PT(int32_t, aLe, AI);
  PT(int32_t, aSt, AG); PT(int32_t, aOw, AG); PT(int32_t, aDt, AG);
  PT(int32_t, fSlo, L.LT ? F : 0); PT(int32_t, iEmax, L.LT ? 2 * I : 0);
  PT(int32_t, eB, L.LT ? BB * I : 0);
  PT(int32_t, gRcl, L.N ? 0 : G * RES);
#undef PT
#ifdef DILU_BOUNDS
  v.ring = Chk<int32_t>(nullptr, 0, id);   // set by the kernel (ring)
#else
  v.ring = nullptr;
#endif
  (void)G; (void)F; (void)I; (void)BB; (void)AI; (void)AG;
  return v;
}

#define DILU_ARRAY_NAMES                                                                     \
  "h", "gR", "gL", "gU", "gN", "gNs", "gRes", "gExcl", "gGrow", "gRel", "rlG", "rlE", "gMask", "gChk", \
  "iId", "iFunc", "iMeta", "iReady", "iSh0", "iShare", "iNext", "iR", "iBmin", "fstack", "iG",  \
  "fKind", "fPrio", "fReq", "fLim", "fMem", "fCb", "fIbs", "fNw", "fCold", "fCls", "fDtr",     \
  "fPat", "fScale", "fPhase", "fCap1", "fReg", "fNsamp", "fAcc", "fHead", "fUp", "fDown",      \
  "fThrn", "fOld", "fPv", "fNlive", "fLh", "fLt", "fGang", "fFlag", "fK", "fList", "fArr",     \
  "fDep", "fPidx", "fInfL", "fDefL", "qN", "qFail", "qSlot", "iQ", "rB",    \
  "bB", "gB", "aTc", "aTm", "aRl", "aLe", "aSt", "aOw", "aDt", "fSlo", "iEmax", "eB", "gRcl", "ring",  \
  "members"

}  // namespace dilu
