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
  H_NEV, H_CCNT = 10 /*6*/, H_CBASE = 16 /*7*/, H_GBASE = 23 /*6*/, H_CCNT2 = 29 /*6*/,
  H_RLN = 35 /* release-log entries appended */, H_NINF = 36, H_NDEF = 37,
  H_QLIVE = 38 /* live queue requests */, H_LASTEP = 39 /* release epoch at the last pass's end */,
  H_QNEWPOS = 40 /* first request enqueued since the last pass, -1 if none */, H_WORDS = 44
};

// tally indices (match include/dilu.h)
enum : int {
  T_ACT = 0, T_SMU, T_MEMU, T_RTOT, T_RSRV, T_RVIO, T_IEXE, T_TPRG, T_POK, T_PFAIL,
  T_COLD, T_SOUT, T_SIN, T_SPLIT, T_HASH, T_ROWS, T_MAXA
};

struct Layout {
  int32_t G, F, I, W, B;   // B: slots per fused batch between second boundaries (1 = unfused)
  // byte offsets inside one block
  size_t hdr;
  size_t gR, gL, gU, gN, gNs, gRes, gExcl, gGrow, gMask, gRel, rlG, rlE;
  size_t iId, iFunc, iMeta, iReady, iG, iSh0, iShare, iNext, iR, iBmin, fstack;
  size_t fKind, fPrio, fReq, fLim, fMem, fCb, fIbs, fNw, fCold, fCls, fDtr, fPat, fScale,
      fPhase, fCap1;
  size_t fReg, fNsamp, fAcc, fHead, fUp, fDown, fThrn, fOld, fPv, fNlive, fLh, fLt, fGang, fFlag, fK,
      fList, fArr, fDep, fPidx, fInfL, fDefL;
  size_t qFunc, qFirst, qN, qFail, qSlot, iQ;
  size_t rB, bB, gB;       // per-batch-slot r, LLM stage minimum, training gang (B > 1 only)
  size_t aTc, aTm, aRl, aLe, aSt, aOw, aDt;   // literal Alg.2 state (cfg.flags bit2 only)
  size_t fSlo, iEmax, eB;  // request-level latency (cfg.flags bit3 only)
  size_t hot_bytes, bytes;
};

inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

inline Layout make_layout(int32_t G, int32_t F, int32_t I, int32_t W, int32_t B = 1,
                          bool alg2 = false, bool lat = false) {
  Layout L;
  L.G = G; L.F = F; L.I = I; L.W = W; L.B = B;
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t at = o; o = align16(o + bytes); return at; };
  // hot region: touched every slot -> staged in shared memory when it fits
  L.hdr = take(H_WORDS * 4);
  L.gR = take(4 * (size_t)G); L.gL = take(4 * (size_t)G); L.gU = take(4 * (size_t)G);
  L.gN = take(4 * (size_t)G);
  L.gNs = take(4 * (size_t)G);          // row sizes at the last repack (overlapped slots, s5)
  L.gRes = take(4 * (size_t)G * RES);
  L.gExcl = take(4 * (size_t)G); L.gGrow = take(4 * (size_t)G);
  L.gMask = take(8 * (size_t)G);        // bit (affinity_class & 63) per resident class
  L.rlG = take(4 * RLOG); L.rlE = take(4 * RLOG);
  L.iId = take(4 * (size_t)I); L.iFunc = take(4 * (size_t)I); L.iMeta = take(4 * (size_t)I);
  L.iReady = take(4 * (size_t)I); L.iNext = take(4 * (size_t)I); L.iR = take(4 * 2 * (size_t)I);
  L.fKind = take(4 * (size_t)F); L.fReq = take(4 * (size_t)F); L.fLim = take(4 * (size_t)F);
  L.fMem = take(4 * (size_t)F); L.fCb = take(4 * (size_t)F); L.fIbs = take(4 * (size_t)F);
  L.fNw = take(4 * (size_t)F); L.fCls = take(4 * (size_t)F); L.fDtr = take(4 * (size_t)F);
  L.fPat = take(4 * (size_t)F); L.fScale = take(4 * (size_t)F); L.fPhase = take(4 * (size_t)F);
  L.fCap1 = take(8 * (size_t)F);
  L.fReg = take(4 * (size_t)F); L.fNsamp = take(4 * (size_t)F); L.fAcc = take(4 * (size_t)F);
  L.fHead = take(4 * (size_t)F); L.fUp = take(4 * (size_t)F); L.fDown = take(4 * (size_t)F);
  L.fThrn = take(4 * (size_t)F);
  L.fOld = take(4 * (size_t)F); L.fPv = take(4 * (size_t)F);   // cp.async landing slots
  L.fNlive = take(4 * (size_t)F); L.fLh = take(4 * (size_t)F);
  L.fGang = take(4 * 2 * (size_t)F); L.fFlag = take(4 * (size_t)F);
  L.fArr = take(4 * (size_t)F); L.fDep = take(4 * (size_t)F); L.fPidx = take(4 * (size_t)F);
  L.fInfL = take(4 * (size_t)F); L.fDefL = take(4 * (size_t)F);
  // serial-path structures the leader walks every boundary (queue, free stack, ...)
  L.gRel = take(4 * (size_t)G);
  L.fLt = take(4 * (size_t)F); L.fK = take(4 * (size_t)F); L.fList = take(4 * (size_t)F);
  L.fstack = take(4 * (size_t)I);
  L.fPrio = take(4 * (size_t)F); L.fCold = take(4 * (size_t)F);
  L.qFunc = take(4 * (size_t)I); L.qFirst = take(4 * (size_t)I); L.qN = take(4 * (size_t)I);
  L.qFail = take(4 * (size_t)I); L.qSlot = take(4 * (size_t)I); L.iQ = take(4 * (size_t)I);
  L.hot_bytes = align16(o);
  // cold region: stage placements and LLM stage minima -> stays in HBM/L2
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
  L.bytes = align16(o);
  return L;
}

// Typed view of one scenario's block (pointers into smem or global).
struct View {
  int32_t* h;
  int32_t *gR, *gL, *gU, *gN, *gNs, *gRes, *gExcl, *gGrow, *gRel, *rlG, *rlE;
  unsigned long long* gMask;
  int32_t *iId, *iFunc, *iMeta, *iReady, *iSh0, *iShare, *iNext, *iR, *iBmin, *fstack;
  int16_t* iG;
  int32_t *fKind, *fPrio, *fReq, *fLim, *fMem, *fCb, *fIbs, *fNw, *fCold, *fCls, *fDtr, *fPat,
      *fScale, *fPhase;
  int64_t* fCap1;
  int32_t *fReg, *fNsamp, *fAcc, *fHead, *fUp, *fDown, *fThrn, *fOld, *fPv, *fNlive, *fLh, *fLt, *fGang,
      *fFlag, *fK, *fList, *fArr, *fDep, *fPidx, *fInfL, *fDefL;
  int32_t *qFunc, *qFirst, *qN, *qFail, *qSlot, *iQ;
  int32_t *rB, *bB, *gB;
  int32_t *aTc, *aTm, *aRl, *aLe, *aSt, *aOw, *aDt;
  int32_t *fSlo, *iEmax, *eB;
  int32_t* ring;  // global [F][W]
};

#ifdef __CUDACC__
__host__ __device__
#endif
inline View make_view(uint8_t* hot, uint8_t* b, const Layout& L) {
  // arrays in the hot region resolve against `hot` (smem copy or b), the rest against b
  View v;
#define P32(name) v.name = reinterpret_cast<int32_t*>((L.name < L.hot_bytes ? hot : b) + L.name)
  v.h = reinterpret_cast<int32_t*>(hot + L.hdr);
  P32(gR); P32(gL); P32(gU); P32(gN); P32(gNs); P32(gRes); P32(gExcl); P32(gGrow); P32(gRel); P32(rlG); P32(rlE);
  v.gMask = reinterpret_cast<unsigned long long*>((L.gMask < L.hot_bytes ? hot : b) + L.gMask);
  P32(iId); P32(iFunc); P32(iMeta); P32(iReady); P32(iSh0); P32(iShare); P32(iNext); P32(iR);
  v.iG = reinterpret_cast<int16_t*>((L.iG < L.hot_bytes ? hot : b) + L.iG);
  P32(iBmin); P32(fstack);
  P32(fKind); P32(fPrio); P32(fReq); P32(fLim); P32(fMem); P32(fCb); P32(fIbs); P32(fNw);
  P32(fCold); P32(fCls); P32(fDtr); P32(fPat); P32(fScale); P32(fPhase);
  v.fCap1 = reinterpret_cast<int64_t*>(hot + L.fCap1);
  P32(fReg); P32(fNsamp); P32(fAcc); P32(fHead); P32(fUp); P32(fDown); P32(fThrn); P32(fOld); P32(fPv); P32(fNlive);
  P32(fLh); P32(fLt); P32(fGang); P32(fFlag); P32(fK); P32(fList); P32(fArr); P32(fDep);
  P32(fPidx); P32(fInfL); P32(fDefL);
  P32(qFunc); P32(qFirst); P32(qN); P32(qFail); P32(qSlot); P32(iQ);
  P32(rB); P32(bB); P32(gB);
  P32(aTc); P32(aTm); P32(aRl); P32(aLe); P32(aSt); P32(aOw); P32(aDt);
  P32(fSlo); P32(iEmax); P32(eB);
#undef P32
  v.ring = nullptr;
  return v;
}

}  // namespace dilu
