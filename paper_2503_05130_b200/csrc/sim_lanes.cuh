// sim_lanes.cuh -- "lanes" engine for many small scenarios (C1/C2/C4: G <= 256).
//
// A CTA of 32*P threads owns a group of 32 scenarios: lane L of every warp works on
// scenario L of the group, warp k is "part" k of that scenario.  All per-scenario state
// is interleaved [element][32 lanes] in global memory, so the common-path loops (over
// functions, GPU rows, residents) issue one coalesced 128-byte transaction per warp for
// 32 scenarios.  The P parts split each scenario's parallel loops (function ranges, GPU
// row ranges); the sequential steps of the method (events in f order, FIFO queue,
// commits, releases) run in part 0 -- warp 0 -- SIMT across the 32 scenarios, and every
// __syncthreads is shared by 32 scenarios.  Steps and readings are the same as the CTA
// engine (sim_kernel.cuh) and the oracle: SURVEY s8(c), DESIGN.md s2-s3.
//
// GPU rows keep their residents as (prio, id)-sorted records that carry the per-slot
// fields the token allocator needs (ready slot, request/limit tokens, c_stage, IBS,
// training demand, kind|stages, instance id, function, requests r), so the allocator
// streams records instead of chasing instance/function indices; the dispatcher writes r
// straight into the records through each instance's record positions.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "sim_kernel.cuh"

namespace dilu {
namespace lanes {

constexpr int LN = 32;  // scenarios per group (lanes)

// header words (per lane)
enum : int {
  LH_NEXT_IID = 0, LH_NLIVE, LH_QLEN, LH_NACT, LH_SUMU, LH_EPOCH, LH_FSTOP, LH_ERR, LH_RLN,
  LH_REMOVED, LH_EVN = 16 /* P words */, LH_WORDS = 48
};

struct LLayout {
  int32_t G, F, I, W, P;
  size_t hdr;
  size_t gR, gL, gU, gN, gExcl, gRel, gRes;
  size_t rId, rReady, rFunc, rReq, rLim, rCst, rIbs, rDtr, rInfo, rStage, rR;
  size_t iId, iFunc, iMeta, iReady, iNext, iG, iShare, iPos, iBmin, fstack, mList;
  size_t fKind, fPrio, fReq, fLim, fMem, fCb, fIbs, fNw, fCold, fCls, fDtr, fPat, fScale,
      fCap1, fArr, fDep;
  size_t fReg, fNsamp, fAcc, fHead, fUp, fDown, fThrn, fNlive, fLh, fLt, fGang, fFlag, fK,
      fPidx, fEvl;
  size_t qFunc, qFirst, qN, qFail;
  size_t rlG, rlE;
  size_t ring;
  size_t bytes;  // per group of 32 scenarios
};

inline LLayout make_llayout(int32_t G, int32_t F, int32_t I, int32_t W, int32_t P) {
  LLayout L;
  L.G = G; L.F = F; L.I = I; L.W = W; L.P = P;
  size_t o = 0;
  // n elements of esize bytes, times 32 lanes, 128-byte aligned
  auto take = [&](size_t n, size_t esize) {
    size_t at = o;
    o = (o + n * esize * LN + 127) & ~size_t(127);
    return at;
  };
  const size_t GR = (size_t)G * RES;
  L.hdr = take(LH_WORDS, 4);
  L.gR = take(G, 4); L.gL = take(G, 4); L.gU = take(G, 4); L.gN = take(G, 4);
  L.gExcl = take(G, 4); L.gRel = take(G, 4); L.gRes = take(GR, 4);
  L.rId = take(GR, 4); L.rReady = take(GR, 4); L.rFunc = take(GR, 4); L.rReq = take(GR, 4);
  L.rLim = take(GR, 4); L.rCst = take(GR, 4); L.rIbs = take(GR, 4); L.rDtr = take(GR, 4);
  L.rInfo = take(GR, 4); L.rStage = take(GR, 4); L.rR = take(2 * GR, 4);
  L.iId = take(I, 4); L.iFunc = take(I, 4); L.iMeta = take(I, 4); L.iReady = take(I, 4);
  L.iNext = take(I, 4); L.iG = take((size_t)I * MAXST, 4); L.iShare = take((size_t)I * MAXST, 4);
  L.iPos = take((size_t)I * MAXST, 4); L.iBmin = take(2 * (size_t)I, 4); L.fstack = take(I, 4);
  L.mList = take(64, 4);
  L.fKind = take(F, 4); L.fPrio = take(F, 4); L.fReq = take(F, 4); L.fLim = take(F, 4);
  L.fMem = take(F, 4); L.fCb = take(F, 4); L.fIbs = take(F, 4); L.fNw = take(F, 4);
  L.fCold = take(F, 4); L.fCls = take(F, 4); L.fDtr = take(F, 4); L.fPat = take(F, 4);
  L.fScale = take(F, 4); L.fCap1 = take(F, 8); L.fArr = take(F, 4); L.fDep = take(F, 4);
  L.fReg = take(F, 4); L.fNsamp = take(F, 4); L.fAcc = take(F, 4); L.fHead = take(F, 4);
  L.fUp = take(F, 4); L.fDown = take(F, 4); L.fThrn = take(F, 4); L.fNlive = take(F, 4);
  L.fLh = take(F, 4); L.fLt = take(F, 4); L.fGang = take(2 * (size_t)F, 4); L.fFlag = take(F, 4);
  L.fK = take(F, 4); L.fPidx = take(F, 4); L.fEvl = take(F, 4);
  L.qFunc = take(I, 4); L.qFirst = take(I, 4); L.qN = take(I, 4); L.qFail = take(I, 4);
  L.rlG = take(RLOG, 4); L.rlE = take(RLOG, 4);
  L.ring = take((size_t)F * W, 4);
  L.bytes = o;
  return L;
}

struct LParams {
  const int32_t* funcs;   // [S][F][16]
  const int32_t* pat;     // [P][Tp]
  const int32_t* scen;    // [S][4]
  uint8_t* state;         // [groups][L.bytes]
  int64_t* tally;         // [S][NT]
  int64_t* stats;         // [S][NSTAT]
  LLayout L;
  int32_t S, ngroups, G, F, I, W, M, Q, aw, bw, slot_ms, SPS, phi_out, phi_in, min_inst,
      max_stages, flags, Tp;
  int64_t T_slot;
};

// Group view (one per CTA, in shared memory): element e of array X for lane L is
// X[(e << 5) + L].
struct LV {
  int32_t* h;
  int32_t *gR, *gL, *gU, *gN, *gExcl, *gRel, *gRes;
  int32_t *rId, *rReady, *rFunc, *rReq, *rLim, *rCst, *rIbs, *rDtr, *rInfo, *rStage, *rR;
  int32_t *iId, *iFunc, *iMeta, *iReady, *iNext, *iG, *iShare, *iPos, *iBmin, *fstack, *mList;
  int32_t *fKind, *fPrio, *fReq, *fLim, *fMem, *fCb, *fIbs, *fNw, *fCold, *fCls, *fDtr, *fPat,
      *fScale, *fArr, *fDep;
  long long* fCap1;
  int32_t *fReg, *fNsamp, *fAcc, *fHead, *fUp, *fDown, *fThrn, *fNlive, *fLh, *fLt, *fGang,
      *fFlag, *fK, *fPidx, *fEvl;
  int32_t *qFunc, *qFirst, *qN, *qFail;
  int32_t *rlG, *rlE;
  int32_t* ring;
};

__host__ __device__ inline LV make_lv(uint8_t* b, const LLayout& L) {
  LV v;
#define LP(name) v.name = reinterpret_cast<int32_t*>(b + L.name)
  v.h = reinterpret_cast<int32_t*>(b + L.hdr);
  LP(gR); LP(gL); LP(gU); LP(gN); LP(gExcl); LP(gRel); LP(gRes);
  LP(rId); LP(rReady); LP(rFunc); LP(rReq); LP(rLim); LP(rCst); LP(rIbs); LP(rDtr); LP(rInfo);
  LP(rStage); LP(rR);
  LP(iId); LP(iFunc); LP(iMeta); LP(iReady); LP(iNext); LP(iG); LP(iShare); LP(iPos); LP(iBmin);
  LP(fstack); LP(mList);
  LP(fKind); LP(fPrio); LP(fReq); LP(fLim); LP(fMem); LP(fCb); LP(fIbs); LP(fNw); LP(fCold);
  LP(fCls); LP(fDtr); LP(fPat); LP(fScale); LP(fArr); LP(fDep);
  v.fCap1 = reinterpret_cast<long long*>(b + L.fCap1);
  LP(fReg); LP(fNsamp); LP(fAcc); LP(fHead); LP(fUp); LP(fDown); LP(fThrn); LP(fNlive); LP(fLh);
  LP(fLt); LP(fGang); LP(fFlag); LP(fK); LP(fPidx); LP(fEvl);
  LP(qFunc); LP(qFirst); LP(qN); LP(qFail); LP(rlG); LP(rlE); LP(ring);
#undef LP
  return v;
}

#define AT(p, e) (p)[((size_t)(e) << 5) + LANE]

__device__ __forceinline__ int st_l(int32_t meta) { return meta & 3; }
__device__ __forceinline__ int nst_l(int32_t meta) { return (meta >> 4) & 7; }
__device__ __forceinline__ bool inf_l(int32_t k) { return k == K_INF || k == K_LLM; }

// per-thread context
struct Ctx {
  const LV* vp;         // shared
  const LParams* P;
  const int32_t* frow;  // this scenario's input rows
  int32_t scn_id, om, ga, mode, k, lane;
  bool active;
};

struct Tl {   // tallies of one thread for its scenario
  long long rtot, rsrv, rvio, iexe, tprg, etot;
  unsigned long long hash;
  long long nres, nfun;
  // part 0 only
  long long act, memu, rows, pok, pfail, cold, sout, sin, split, maxa;
  long long st[NSTAT];
};

template <int P>
struct Shr {
  unsigned long long key[P][LN];
  long long acc[9][P][LN];
  int32_t grp;
  int32_t ev_off[P][LN];
  // placement state per lane (part 0 writes, all read)
  int32_t mode[LN];       // 0 idle, 1 attempting a member, 2 split rounds
  int32_t inst[LN];       // instance slot being placed
  int32_t tier2[LN];      // tier-2 GPU of the current member or -1
  int32_t pick[MAXST][LN];
  int32_t pfree[MAXST][LN];
  int32_t nsplit[LN];
  int32_t sdone[LN];
};

// ------------------------------------------------------------------ serial helpers
// (called by part 0 for its lane's scenario)

__device__ void l_list_append(Ctx& c, int32_t f, int32_t s) {
  const LV& v = *c.vp;
  const int LANE = c.lane;
  AT(v.iNext, s) = -1;
  const int32_t lt = AT(v.fLt, f);
  if (lt < 0) AT(v.fLh, f) = s; else AT(v.iNext, lt) = s;
  AT(v.fLt, f) = s;
}
__device__ void l_list_remove(Ctx& c, int32_t f, int32_t s) {
  const LV& v = *c.vp;
  const int LANE = c.lane;
  int32_t prev = -1, cur = AT(v.fLh, f);
  while (cur >= 0 && cur != s) { prev = cur; cur = AT(v.iNext, cur); }
  if (cur < 0) return;
  const int32_t nx = AT(v.iNext, cur);
  if (prev < 0) AT(v.fLh, f) = nx; else AT(v.iNext, prev) = nx;
  if (AT(v.fLt, f) == s) AT(v.fLt, f) = prev;
}

// write record j of row g from instance s (stage k)
__device__ void put_rec(Ctx& c, int32_t g, int32_t j, int32_t s, int32_t k) {
  const LV& v = *c.vp;
  const int LANE = c.lane;
  const LParams& P = *c.P;
  const int32_t e = g * RES + j;
  const int32_t f = AT(v.iFunc, s);
  const int32_t meta = AT(v.iMeta, s);
  const int32_t nst = nst_l(meta);
  const int32_t kind = AT(v.fKind, f);
  AT(v.gRes, e) = s;
  AT(v.rId, e) = AT(v.iId, s);
  AT(v.rReady, e) = AT(v.iReady, s);
  AT(v.rFunc, e) = f;
  AT(v.rReq, e) = AT(v.fReq, f) * P.slot_ms;
  AT(v.rLim, e) = AT(v.fLim, f) * P.slot_ms;
  const int32_t cb = AT(v.fCb, f);
  AT(v.rCst, e) = nst <= 1 ? cb : (cb + nst - 1) / nst;
  AT(v.rIbs, e) = AT(v.fIbs, f);
  AT(v.rDtr, e) = AT(v.fDtr, f);
  AT(v.rInfo, e) = kind | (nst << 4) | (AT(v.fPrio, f) << 8);
  AT(v.rStage, e) = k;
  AT(v.iPos, s * MAXST + k) = e;
}

__device__ void copy_rec(Ctx& c, int32_t g, int32_t jd, int32_t js) {
  const LV& v = *c.vp;
  const int LANE = c.lane;
  const int32_t d = g * RES + jd, s0 = g * RES + js;
  AT(v.gRes, d) = AT(v.gRes, s0); AT(v.rId, d) = AT(v.rId, s0);
  AT(v.rReady, d) = AT(v.rReady, s0); AT(v.rFunc, d) = AT(v.rFunc, s0);
  AT(v.rReq, d) = AT(v.rReq, s0); AT(v.rLim, d) = AT(v.rLim, s0);
  AT(v.rCst, d) = AT(v.rCst, s0); AT(v.rIbs, d) = AT(v.rIbs, s0);
  AT(v.rDtr, d) = AT(v.rDtr, s0); AT(v.rInfo, d) = AT(v.rInfo, s0);
  AT(v.rStage, d) = AT(v.rStage, s0);
  AT(v.iPos, AT(v.gRes, d) * MAXST + AT(v.rStage, d)) = d;
}

__device__ void l_commit(Ctx& c, int32_t s, int32_t g, int32_t share) {
  const LV& v = *c.vp;
  const int LANE = c.lane;
  const int32_t f = AT(v.iFunc, s);
  const int32_t n = AT(v.gN, g);
  if (n == 0) AT(v.h, LH_NACT) += 1;
  AT(v.gR, g) += AT(v.fReq, f);
  AT(v.gL, g) += AT(v.fLim, f);
  AT(v.gU, g) += share;
  AT(v.h, LH_SUMU) += share;
  const int32_t meta = AT(v.iMeta, s);
  const int k0 = nst_l(meta);
  AT(v.iG, s * MAXST + k0) = g;
  AT(v.iShare, s * MAXST + k0) = share;
  AT(v.iMeta, s) = (meta & ~(7 << 4)) | ((k0 + 1) << 4);
  // insert into the row keeping (prio, id) order (SLO-sensitive first, Alg.2)
  const long long key = ((long long)AT(v.fPrio, f) << 32) | (uint32_t)AT(v.iId, s);
  int pos = n;
  while (pos > 0) {
    const int32_t e = g * RES + pos - 1;
    const long long kp = ((long long)(AT(v.rInfo, e) >> 8) << 32) | (uint32_t)AT(v.rId, e);
    if (kp <= key) break;
    copy_rec(c, g, pos, pos - 1);
    --pos;
  }
  put_rec(c, g, pos, s, k0);
  AT(v.gN, g) = n + 1;
  AT(v.gExcl, g) = 1;
}

// placement succeeded or stages changed: refresh c_stage / stage count in the records
__device__ void refresh_rec_stages(Ctx& c, int32_t s) {
  const LV& v = *c.vp;
  const int LANE = c.lane;
  const int32_t meta = AT(v.iMeta, s);
  const int32_t nst = nst_l(meta);
  const int32_t f = AT(v.iFunc, s);
  const int32_t cb = AT(v.fCb, f);
  const int32_t cst = nst <= 1 ? cb : (cb + nst - 1) / nst;
  for (int k = 0; k < nst; ++k) {
    const int32_t e = AT(v.iPos, s * MAXST + k);
    AT(v.rCst, e) = cst;
    AT(v.rInfo, e) = (AT(v.rInfo, e) & ~(7 << 4)) | (nst << 4);
    AT(v.rReady, e) = AT(v.iReady, s);
  }
}

__device__ void l_release(Ctx& c, int32_t s) {
  const LV& v = *c.vp;
  const int LANE = c.lane;
  const int32_t f = AT(v.iFunc, s);
  const int32_t meta = AT(v.iMeta, s);
  const int n = nst_l(meta);
  for (int k = 0; k < n; ++k) {
    const int32_t g = AT(v.iG, s * MAXST + k);
    const int32_t sh = AT(v.iShare, s * MAXST + k);
    AT(v.gR, g) -= AT(v.fReq, f);
    AT(v.gL, g) -= AT(v.fLim, f);
    AT(v.gU, g) -= sh;
    AT(v.h, LH_SUMU) -= sh;
    const int32_t nr = AT(v.gN, g);
    int32_t j = AT(v.iPos, s * MAXST + k) - g * RES;
    for (; j + 1 < nr; ++j) copy_rec(c, g, j, j + 1);
    AT(v.gN, g) = nr - 1;
    if (nr - 1 == 0) AT(v.h, LH_NACT) -= 1;
    AT(v.iG, s * MAXST + k) = -1;
    AT(v.iShare, s * MAXST + k) = 0;
    AT(v.iPos, s * MAXST + k) = -1;
  }
  AT(v.iMeta, s) = meta & ~(7 << 4);
}

__device__ void l_terminate(Ctx& c, int32_t s) {
  const LV& v = *c.vp;
  const int LANE = c.lane;
  const int32_t f = AT(v.iFunc, s);
  if (st_l(AT(v.iMeta, s)) == ST_PLACED) {
    const int32_t ep = ++AT(v.h, LH_EPOCH);
    const int ns = nst_l(AT(v.iMeta, s));
    for (int k = 0; k < ns; ++k) {
      const int32_t g = AT(v.iG, s * MAXST + k);
      AT(v.gRel, g) = ep;
      const int32_t slot = AT(v.h, LH_RLN)++ % RLOG;
      AT(v.rlG, slot) = g;
      AT(v.rlE, slot) = ep;
    }
    l_release(c, s);
  }
  AT(v.iMeta, s) = ST_FREE;
  l_list_remove(c, f, s);
  AT(v.fNlive, f) -= 1;
  AT(v.h, LH_NLIVE) -= 1;
  AT(v.fstack, AT(v.h, LH_FSTOP)++) = s;
}

__device__ void l_compact_queue(Ctx& c) {
  const LV& v = *c.vp;
  const int LANE = c.lane;
  const int32_t n = AT(v.h, LH_QLEN);
  int32_t k = 0;
  for (int32_t q = 0; q < n; ++q) {
    if (AT(v.qN, q) == 0) continue;
    if (k != q) {
      AT(v.qFunc, k) = AT(v.qFunc, q); AT(v.qFirst, k) = AT(v.qFirst, q);
      AT(v.qN, k) = AT(v.qN, q); AT(v.qFail, k) = AT(v.qFail, q);
    }
    ++k;
  }
  AT(v.h, LH_QLEN) = k;
}

__device__ int32_t l_enqueue(Ctx& c, int32_t f, int32_t n) {
  const LV& v = *c.vp;
  const int LANE = c.lane;
  if (AT(v.h, LH_FSTOP) < n) { AT(v.h, LH_ERR) = 6; return -1; }
  if (AT(v.h, LH_QLEN) == c.P->I) l_compact_queue(c);
  const int32_t first = AT(v.h, LH_NEXT_IID);
  for (int32_t j = 0; j < n; ++j) {
    const int32_t s = AT(v.fstack, --AT(v.h, LH_FSTOP));
    AT(v.iId, s) = AT(v.h, LH_NEXT_IID)++;
    AT(v.iFunc, s) = f;
    AT(v.iMeta, s) = ST_PEND;
    AT(v.iReady, s) = 0;
    for (int k = 0; k < MAXST; ++k) {
      AT(v.iG, s * MAXST + k) = -1; AT(v.iShare, s * MAXST + k) = 0; AT(v.iPos, s * MAXST + k) = -1;
    }
    AT(v.iBmin, s) = BIG;
    AT(v.iBmin, c.P->I + s) = BIG;
    l_list_append(c, f, s);
    AT(v.fNlive, f) += 1;
    AT(v.h, LH_NLIVE) += 1;
  }
  const int32_t q = AT(v.h, LH_QLEN)++;
  AT(v.qFunc, q) = f; AT(v.qFirst, q) = first; AT(v.qN, q) = n; AT(v.qFail, q) = -1;
  return first;
}

__device__ void l_register(Ctx& c, int32_t f, int32_t t) {
  const LV& v = *c.vp;
  const int LANE = c.lane;
  if (AT(v.fReg, f)) return;
  AT(v.fReg, f) = 1;
  AT(v.fNsamp, f) = 0; AT(v.fAcc, f) = 0; AT(v.fHead, f) = 0; AT(v.fUp, f) = 0;
  AT(v.fDown, f) = 0; AT(v.fThrn, f) = -1;
  const int32_t phase = __ldg(c.frow + (size_t)f * 16 + 15);
  AT(v.fPidx, f) = (int32_t)(((long long)t + phase) % c.P->Tp);
}

__device__ bool l_could_help(const Ctx& c, int32_t g, int32_t f) {
  const LV& v = *c.vp;
  const int LANE = c.lane;
  const int32_t n = AT(v.gN, g);
  if (n == 0) return true;
  if (n >= RES || AT(v.gR, g) + AT(v.fReq, f) > c.om || AT(v.gL, g) + AT(v.fLim, f) > c.ga)
    return false;
  if (AT(v.gU, g) + AT(v.fMem, f) <= c.P->M) return true;
  return AT(v.fKind, f) == K_LLM && (c.P->flags & 1) && c.P->M - AT(v.gU, g) > 0;
}

// release log check (see sim_kernel.cuh hope_after)
__device__ bool l_hope(const Ctx& c, int32_t fe, int32_t f) {
  const LV& v = *c.vp;
  const int LANE = c.lane;
  const int32_t n = AT(v.h, LH_RLN);
  const int32_t lo = n > RLOG ? n - RLOG : 0;
  if (n > RLOG && AT(v.rlE, lo % RLOG) > fe) {
    for (int32_t g = 0; g < c.P->G; ++g)
      if (AT(v.gRel, g) > fe && l_could_help(c, g, f)) return true;
    return false;
  }
  for (int32_t k = n - 1; k >= lo; --k) {
    if (AT(v.rlE, k % RLOG) <= fe) break;
    if (l_could_help(c, AT(v.rlG, k % RLOG), f)) return true;
  }
  return false;
}

// next queue entry needing a real attempt, from q (part 0).  Exact retry skip: see
// sim_kernel.cuh placement_pass.
__device__ int32_t l_next_attempt(Ctx& c, int32_t q, Tl& tl) {
  const LV& v = *c.vp;
  const int LANE = c.lane;
  const int32_t qn = AT(v.h, LH_QLEN), ep = AT(v.h, LH_EPOCH);
  for (; q < qn; ++q) {
    if (AT(v.qN, q) == 0) continue;
    const int32_t fe = AT(v.qFail, q);
    if (fe < 0) return q;
    if (fe == ep) { tl.pfail += 1; continue; }
    tl.st[S_HOPE] += 1;
    if (l_hope(c, fe, AT(v.qFunc, q))) return q;
    tl.pfail += 1;
    AT(v.qFail, q) = ep;
  }
  return qn;
}

// ------------------------------------------------------------------------- kernel

template <int P>
struct Engine {
  // score this part's GPU range for instance s of lane: min packed key (R7)
  static __device__ unsigned long long score(Ctx& c, int32_t s) {
    const LV& v = *c.vp;
  const int LANE = c.lane;
    const LParams& Pm = *c.P;
    const int32_t f = AT(v.iFunc, s);
    const int32_t req = AT(v.fReq, f), lim = AT(v.fLim, f), mem = AT(v.fMem, f), cls = AT(v.fCls, f);
    const long long aM = (long long)Pm.aw * Pm.M, bQ = (long long)Pm.bw * Pm.Q;
    const unsigned long long MASK40 = (1ull << 40) - 1;
    unsigned long long best = ~0ull;
    const int32_t lo = Pm.G * c.k / P, hi = Pm.G * (c.k + 1) / P;
    for (int32_t g = lo; g < hi; ++g) {
      if (AT(v.gExcl, g)) continue;
      const int32_t n = AT(v.gN, g);
      unsigned long long key;
      if (n == 0) {
        key = (2ull << 62) | (MASK40 << 22) | (unsigned long long)g;
      } else if (c.mode == M_EXCLUSIVE) {
        continue;
      } else {
        const int32_t R = AT(v.gR, g) + req, Lm = AT(v.gL, g) + lim, U = AT(v.gU, g) + mem;
        if (!(R <= c.om && Lm <= c.ga && U <= Pm.M && n < RES)) continue;
        int aff = 0;
        for (int j = 0; j < n && !aff; ++j) aff = AT(v.fCls, AT(v.rFunc, g * RES + j)) == cls;
        const unsigned long long K = (unsigned long long)(aM * R + bQ * U);
        key = ((unsigned long long)(aff ? 0 : 1) << 62) | ((MASK40 - K) << 22) | (unsigned long long)g;
      }
      best = key < best ? key : best;
    }
    return best;
  }

  // split round: this part's best (max free memory, lowest id) candidate excluding picks
  static __device__ unsigned long long split_pick(Ctx& c, int32_t s, const int32_t* picked, int np) {
    const LV& v = *c.vp;
  const int LANE = c.lane;
    const LParams& Pm = *c.P;
    const int32_t f = AT(v.iFunc, s);
    const int32_t req = AT(v.fReq, f), lim = AT(v.fLim, f);
    unsigned long long best = ~0ull;
    const int32_t lo = Pm.G * c.k / P, hi = Pm.G * (c.k + 1) / P;
    for (int32_t g = lo; g < hi; ++g) {
      const int32_t n = AT(v.gN, g);
      if (n == 0 || AT(v.gExcl, g) || n >= RES) continue;
      bool dup = false;
      for (int j = 0; j < np; ++j) dup |= picked[j * LN] == g;
      if (dup) continue;
      if (AT(v.gR, g) + req > c.om || AT(v.gL, g) + lim > c.ga) continue;
      const int32_t fr = Pm.M - AT(v.gU, g);
      if (fr <= 0) continue;
      const unsigned long long key = ((unsigned long long)(0xFFFFFFFFu - (uint32_t)fr) << 32) | (uint32_t)g;
      best = key < best ? key : best;
    }
    return best;
  }

  // One FIFO placement pass for all 32 scenarios of the group.
  static __device__ void pass(Ctx& c, Shr<P>& sh, int32_t t, Tl& tl) {
    const LV& v = *c.vp;
  const int LANE = c.lane;
    const LParams& Pm = *c.P;
    const int L = c.lane;
    const bool lead = c.k == 0;
    int32_t q = 0, qe = 0, nmem = 0, j = 0, placed = 0;
    bool removed = false;
    bool done = !c.active;
    // part 0 drives; all parts loop while any lane has an attempt in flight
    for (;;) {
      if (lead) {
        sh.mode[L] = 0;
        if (!done) {
          qe = l_next_attempt(c, q, tl);
          if (qe >= AT(v.h, LH_QLEN)) {
            done = true;
          } else {
            const int32_t f = AT(v.qFunc, qe), first = AT(v.qFirst, qe);
            nmem = AT(v.qN, qe);
            int jj = 0;
            for (int32_t s = AT(v.fLh, f); s >= 0 && jj < nmem; s = AT(v.iNext, s)) {
              const int32_t id = AT(v.iId, s);
              if (id >= first && id < first + nmem) AT(v.mList, jj++) = s;
            }
            j = 0; placed = 0;
            sh.mode[L] = 1;
            sh.inst[L] = AT(v.mList, 0);
            tl.st[S_ATTEMPT] += 1;
          }
        }
      }
      if (!__syncthreads_or(lead && sh.mode[L] != 0)) break;
      // members of the current request, one per round (lanes with fewer members idle)
      for (;;) {
        const bool mine = c.active && sh.mode[L] == 1;
        if (mine) sh.key[c.k][L] = score(c, sh.inst[L]);
        __syncthreads();
        bool split_needed = false;
        if (lead && mine) {
          unsigned long long best = ~0ull;
#pragma unroll
          for (int x = 0; x < P; ++x) best = sh.key[x][L] < best ? sh.key[x][L] : best;
          const int tier = best == ~0ull ? 3 : (int)(best >> 62);
          const int32_t s = sh.inst[L];
          const int32_t f = AT(v.iFunc, s);
          sh.tier2[L] = tier == 2 ? (int32_t)(best & 0x3FFFFF) : -1;
          if (tier <= 1) {
            l_commit(c, s, (int32_t)(best & 0x3FFFFF), AT(v.fMem, f));
            sh.mode[L] = 3;  // member placed
          } else if (AT(v.fKind, f) == K_LLM && (Pm.flags & 1) && c.mode != M_EXCLUSIVE) {
            sh.mode[L] = 2;  // worst-fit split rounds
            sh.nsplit[L] = 0;
            sh.sdone[L] = 0;
            split_needed = true;
          } else if (tier == 2) {
            l_commit(c, s, sh.tier2[L], AT(v.fMem, f));
            sh.mode[L] = 3;
          } else {
            sh.mode[L] = 4;  // member failed
          }
        }
        if (__syncthreads_or(split_needed)) {
          long long sum = 0;   // part 0 only
          for (int r = 0; r < Pm.max_stages; ++r) {
            const bool sp = c.active && sh.mode[L] == 2 && !sh.sdone[L];
            if (sp) sh.key[c.k][L] = split_pick(c, sh.inst[L], &sh.pick[0][L], r);
            __syncthreads();
            if (lead && sp) {
              unsigned long long best = ~0ull;
#pragma unroll
              for (int x = 0; x < P; ++x) best = sh.key[x][L] < best ? sh.key[x][L] : best;
              if (best == ~0ull) {
                sh.sdone[L] = 2;   // no candidate: split impossible
              } else {
                sh.pick[r][L] = (int32_t)(best & 0xFFFFFFFFu);
                sh.pfree[r][L] = (int32_t)(0xFFFFFFFFu - (uint32_t)(best >> 32));
                sum += sh.pfree[r][L];
                sh.nsplit[L] = r + 1;
                if (sum >= AT(v.fMem, AT(v.iFunc, sh.inst[L]))) sh.sdone[L] = 1;
              }
            }
            __syncthreads();
          }
          if (lead && c.active && sh.mode[L] == 2) {
            const int32_t s = sh.inst[L];
            const int32_t f = AT(v.iFunc, s);
            if (sh.sdone[L] == 1) {
              int32_t left = AT(v.fMem, f);
              for (int x = 0; x < sh.nsplit[L]; ++x) {
                const int32_t shv = sh.pfree[x][L] < left ? sh.pfree[x][L] : left;
                l_commit(c, s, sh.pick[x][L], shv);
                left -= shv;
              }
              sh.mode[L] = 3;
            } else if (sh.tier2[L] >= 0) {
              l_commit(c, s, sh.tier2[L], AT(v.fMem, f));
              sh.mode[L] = 3;
            } else {
              sh.mode[L] = 4;
            }
          }
        }
        // part 0: advance the request of this lane
        bool more = false;
        if (lead && c.active && (sh.mode[L] == 3 || sh.mode[L] == 4)) {
          const int32_t f = AT(v.qFunc, qe);
          if (sh.mode[L] == 3) { ++placed; ++j; }
          if (sh.mode[L] == 3 && j < nmem) {
            sh.inst[L] = AT(v.mList, j);
            sh.mode[L] = 1;
            more = true;
          } else {
            for (int x = 0; x < placed; ++x) {          // clear I* marks
              const int32_t s = AT(v.mList, x);
              const int ns = nst_l(AT(v.iMeta, s));
              for (int y = 0; y < ns; ++y) AT(v.gExcl, AT(v.iG, s * MAXST + y)) = 0;
            }
            if (placed == nmem) {
              const int32_t cold = AT(v.fCold, f);
              for (int x = 0; x < nmem; ++x) {
                const int32_t s = AT(v.mList, x);
                AT(v.iMeta, s) = (AT(v.iMeta, s) & ~3) | ST_PLACED;
                AT(v.iReady, s) = t + cold;
                refresh_rec_stages(c, s);
                tl.pok += 1;
                if (inf_l(AT(v.fKind, f)) && cold > 0) tl.cold += 1;
                if (nst_l(AT(v.iMeta, s)) > 1) tl.split += 1;
              }
              AT(v.qN, qe) = 0;
              removed = true;
            } else {
              for (int x = 0; x < placed; ++x) l_release(c, AT(v.mList, x));
              tl.pfail += 1;
              AT(v.qFail, qe) = AT(v.h, LH_EPOCH);
            }
            sh.mode[L] = 0;
            q = qe + 1;
          }
        }
        if (!__syncthreads_or(more)) break;
      }
    }
    if (lead && c.active && removed) l_compact_queue(c);
    __syncthreads();
  }

  enum : int32_t { EV_DEP = 1, EV_OUT = 2, EV_IN = 4, EV_ARR = 8 };

  static __device__ void boundary(Ctx& c, Shr<P>& sh, int32_t t, Tl& tl) {
    const LV& v = *c.vp;
  const int LANE = c.lane;
    const LParams& Pm = *c.P;
    const int32_t sec = t / Pm.SPS;
    const int32_t W = Pm.W;
    const int32_t lo = Pm.F * c.k / P, hi = Pm.F * (c.k + 1) / P;
    int32_t cnt = 0;
    if (c.active) {
      for (int32_t f = lo; f < hi; ++f) {
        const int32_t kind = AT(v.fKind, f);
        int32_t ev = 0;
        if (kind != K_UNUSED) {
          if (AT(v.fReg, f)) {
            const bool inf = inf_l(kind);
            int32_t* ring = v.ring + ((size_t)f * W << 5);
            const long long cap1 = AT(v.fCap1, f);
            int32_t last = 0;
            if (inf && sec >= 1) {                    // step 1: push second sec-1
              const int32_t val = AT(v.fAcc, f);
              last = val;
              const int32_t head = AT(v.fHead, f);
              const int32_t ns = AT(v.fNsamp, f);
              const int32_t thr = AT(v.fThrn, f);
              if (thr >= 0) {
                const long long cu = (long long)thr * cap1, cd = (long long)(thr - 1) * cap1;
                int32_t du = val > cu, dd = val < cd;
                if (ns >= W) { const int32_t old = AT(ring, head); du -= old > cu; dd -= old < cd; }
                AT(v.fUp, f) += du;
                AT(v.fDown, f) += dd;
              }
              AT(ring, head) = val;
              AT(v.fHead, f) = head + 1 == W ? 0 : head + 1;
              AT(v.fNsamp, f) = ns + 1;
              AT(v.fAcc, f) = 0;
            }
            if (AT(v.fDep, f) == sec) {               // step 2: departure
              ev = EV_DEP;
            } else if (inf && c.mode == M_EAGER) {
              if (AT(v.fNsamp, f) >= 1) {
                const int32_t n = AT(v.fNlive, f);
                if ((long long)last > (long long)n * cap1) {
                  const long long kk = ((long long)last + cap1 - 1) / cap1 - n;
                  if (kk >= 1) { ev = EV_OUT; AT(v.fK, f) = (int32_t)kk; }
                } else if ((long long)last < (long long)(n - 1) * cap1 && n > Pm.min_inst) {
                  ev = EV_IN;
                }
              }
            } else if (inf && AT(v.fNsamp, f) >= W) { // step 3: lazy scaling decision
              const int32_t n = AT(v.fNlive, f);
              const long long cu = (long long)n * cap1, cd = (long long)(n - 1) * cap1;
              if (AT(v.fThrn, f) != n) {
                int32_t up = 0, dn = 0;
                for (int x = 0; x < W; ++x) { const int32_t w = AT(ring, x); up += w > cu; dn += w < cd; }
                AT(v.fUp, f) = up; AT(v.fDown, f) = dn; AT(v.fThrn, f) = n;
              }
              if (AT(v.fUp, f) >= Pm.phi_out) {
                int32_t mx = 0;
                for (int x = 0; x < W; ++x) mx = max(mx, AT(ring, x));
                const long long kk = ((long long)mx + cap1 - 1) / cap1 - n;
                if (kk >= 1) { ev = EV_OUT; AT(v.fK, f) = (int32_t)kk; }
              } else if (AT(v.fDown, f) > Pm.phi_in && n > Pm.min_inst) {
                ev = EV_IN;
              }
            }
          }
          if (AT(v.fArr, f) == sec) ev |= EV_ARR;    // step 4: arrival
        }
        if (ev) { AT(v.fFlag, f) = ev; AT(v.fEvl, lo + cnt) = f; ++cnt; }
      }
    }
    AT(v.h, LH_EVN + c.k) = cnt;
    __syncthreads();
    if (c.k == 0 && c.active) {
      int32_t total = 0;
      for (int x = 0; x < P; ++x) total += AT(v.h, LH_EVN + x);
      tl.st[S_EVENT] += total;
      if (total) {
        // step 2: departures (ascending f: part segments are ascending ranges)
        for (int x = 0; x < P; ++x) {
          const int32_t base = Pm.F * x / P, n = AT(v.h, LH_EVN + x);
          for (int32_t e = 0; e < n; ++e) {
            const int32_t f = AT(v.fEvl, base + e);
            if (!(AT(v.fFlag, f) & EV_DEP)) continue;
            const int32_t qn = AT(v.h, LH_QLEN);
            for (int32_t q = 0; q < qn; ++q) if (AT(v.qN, q) > 0 && AT(v.qFunc, q) == f) AT(v.qN, q) = 0;
            while (AT(v.fLh, f) >= 0) l_terminate(c, AT(v.fLh, f));
            AT(v.fReg, f) = 0;
          }
        }
        // step 3: lazy scaling actions
        for (int x = 0; x < P && !AT(v.h, LH_ERR); ++x) {
          const int32_t base = Pm.F * x / P, n = AT(v.h, LH_EVN + x);
          for (int32_t e = 0; e < n && !AT(v.h, LH_ERR); ++e) {
            const int32_t f = AT(v.fEvl, base + e);
            const int32_t ev = AT(v.fFlag, f);
            if (ev & EV_OUT) {
              for (int32_t y = 0; y < AT(v.fK, f) && !AT(v.h, LH_ERR); ++y) l_enqueue(c, f, 1);
              tl.sout += 1;
            } else if (ev & EV_IN) {
              const int32_t victim = AT(v.fLt, f);     // highest live id (Q19)
              if (st_l(AT(v.iMeta, victim)) == ST_PEND) {
                const int32_t id = AT(v.iId, victim), qn = AT(v.h, LH_QLEN);
                for (int32_t q = 0; q < qn; ++q)
                  if (AT(v.qN, q) > 0 && AT(v.qFirst, q) <= id && id < AT(v.qFirst, q) + AT(v.qN, q)) {
                    AT(v.qN, q) = 0;
                    break;
                  }
              }
              l_terminate(c, victim);
              tl.sin += 1;
            }
          }
        }
        // step 4: arrivals
        for (int x = 0; x < P && !AT(v.h, LH_ERR); ++x) {
          const int32_t base = Pm.F * x / P, n = AT(v.h, LH_EVN + x);
          for (int32_t e = 0; e < n && !AT(v.h, LH_ERR); ++e) {
            const int32_t f = AT(v.fEvl, base + e);
            if (!(AT(v.fFlag, f) & EV_ARR)) continue;
            l_register(c, f, t);
            if (AT(v.fKind, f) == K_TRAIN) l_enqueue(c, f, AT(v.fNw, f));
            else for (int32_t y = 0; y < Pm.min_inst && !AT(v.h, LH_ERR); ++y) l_enqueue(c, f, 1);
          }
        }
        for (int x = 0; x < P; ++x) {
          const int32_t base = Pm.F * x / P, n = AT(v.h, LH_EVN + x);
          for (int32_t e = 0; e < n; ++e) AT(v.fFlag, AT(v.fEvl, base + e)) = 0;
        }
      }
    }
    __syncthreads();
    pass(c, sh, t, tl);
  }

  // P0: arrivals and dispatch into the resident records (step 6)
  static __device__ void phase0(Ctx& c, int32_t t, Tl& tl) {
    const LV& v = *c.vp;
  const int LANE = c.lane;
    const LParams& Pm = *c.P;
    if (!c.active) return;
    int32_t* rR = v.rR + ((size_t)(t & 1) * Pm.G * RES << 5);
    const int32_t lo = Pm.F * c.k / P, hi = Pm.F * (c.k + 1) / P;
    for (int32_t f = lo; f < hi; ++f) {
      if (!AT(v.fReg, f) || !inf_l(AT(v.fKind, f))) continue;
      const int32_t idx = AT(v.fPidx, f);
      AT(v.fPidx, f) = idx + 1 == Pm.Tp ? 0 : idx + 1;
      const long long x = __ldg(Pm.pat + (size_t)AT(v.fPat, f) * Pm.Tp + idx);
      const int32_t A = (int32_t)((x * AT(v.fScale, f)) >> 10);
      tl.nfun += 1;
      AT(v.fAcc, f) += A;
      tl.rtot += A;
      int32_t nw = 0;
      for (int32_t s = AT(v.fLh, f); s >= 0; s = AT(v.iNext, s))
        nw += st_l(AT(v.iMeta, s)) == ST_PLACED && AT(v.iReady, s) <= t;
      if (nw == 0) { tl.rvio += A; continue; }
      const int32_t qv = A / nw, rem = A - qv * nw;
      int32_t rank = 0;
      for (int32_t s = AT(v.fLh, f); s >= 0; s = AT(v.iNext, s)) {
        const int32_t meta = AT(v.iMeta, s);
        if (st_l(meta) == ST_PLACED && AT(v.iReady, s) <= t) {
          const int32_t r = qv + (rank < rem ? 1 : 0);
          const int ns = nst_l(meta);
          for (int k = 0; k < ns; ++k) AT(rR, AT(v.iPos, s * MAXST + k)) = r;
          ++rank;
        }
      }
    }
  }

  // P1: token allocation over this part's GPU rows (step 7) + local capacity
  static __device__ void phase1(Ctx& c, int32_t t, Tl& tl) {
    const LV& v = *c.vp;
  const int LANE = c.lane;
    const LParams& Pm = *c.P;
    if (!c.active) return;
    const int par = t & 1;
    const int32_t* rR = v.rR + ((size_t)par * Pm.G * RES << 5);
    int32_t* gang = v.fGang + ((size_t)par * Pm.F << 5);
    int32_t* bmin = v.iBmin + ((size_t)par * Pm.I << 5);
    const int32_t T = (int32_t)Pm.T_slot;
    const uint64_t ht = sm64(sm64((uint32_t)c.scn_id) ^ (uint32_t)t);
    const int32_t lo = Pm.G * c.k / P, hi = Pm.G * (c.k + 1) / P;
    for (int32_t g = lo; g < hi; ++g) {
      const int32_t n = AT(v.gN, g);
      if (n == 0) continue;
      const int32_t e0 = g * RES;
      int32_t sreq = 0;
      for (int32_t j = 0; j < n; ++j)
        if (AT(v.rReady, e0 + j) <= t) sreq += AT(v.rReq, e0 + j);
      const int32_t Sg = T - sreq;
      int32_t pref = 0;
      for (int32_t j = 0; j < n; ++j) {
        const int32_t e = e0 + j;
        if (AT(v.rReady, e) > t) continue;                 // cold: a = e = 0 (Q14)
        const int32_t info = AT(v.rInfo, e);
        const int32_t kind = info & 15, nst = (info >> 4) & 7;
        const int32_t req = AT(v.rReq, e), lim = c.mode == M_EXCLUSIVE ? T : AT(v.rLim, e);
        int32_t d, need = 0, rr = 0, cst = 1, ibs = 1;
        if (kind == K_TRAIN) {
          d = AT(v.rDtr, e);
        } else {
          rr = AT(rR, e);
          ibs = AT(v.rIbs, e);
          cst = AT(v.rCst, e);
          need = rr / ibs + (rr % ibs != 0);
          const long long dd = (long long)need * cst;
          d = dd < lim ? (int32_t)dd : lim;
        }
        const int32_t cap = d < lim ? d : lim;
        const int32_t want = cap > req ? cap - req : 0;
        const int32_t room = Sg - pref;
        const int32_t sp = want < room ? want : (room > 0 ? room : 0);
        pref += want;
        const int32_t a = req + sp;
        tl.nres += 1;
        tl.hash += sm64(sm64(ht ^ (uint32_t)AT(v.rId, e)) ^ ((uint64_t((uint32_t)g) << 32) | (uint32_t)a));
        if (kind == K_TRAIN) {
          atomicMin(&AT(gang, AT(v.rFunc, e)), d < a ? d : a);
        } else {
          const int32_t fit = a / cst;
          const int32_t b = need < fit ? need : fit;
          if (nst == 1) {
            const long long capb = (long long)b * ibs;
            const int32_t served = capb < rr ? (int32_t)capb : rr;
            tl.rsrv += served;
            tl.rvio += rr - served;
            const long long ex = (long long)b * cst;
            tl.iexe += ex;
            tl.etot += ex;
          } else {
            atomicMin(&AT(bmin, AT(v.gRes, e)), b);
          }
        }
      }
    }
  }

  // P2: training gangs and LLM stage minima (step 8)
  static __device__ void phase2(Ctx& c, int32_t t, Tl& tl) {
    const LV& v = *c.vp;
  const int LANE = c.lane;
    const LParams& Pm = *c.P;
    if (!c.active) return;
    const int par = t & 1;
    const int32_t* rR = v.rR + ((size_t)par * Pm.G * RES << 5);
    int32_t* gang = v.fGang + ((size_t)par * Pm.F << 5);
    int32_t* bmin = v.iBmin + ((size_t)par * Pm.I << 5);
    const int32_t lo = Pm.F * c.k / P, hi = Pm.F * (c.k + 1) / P;
    for (int32_t f = lo; f < hi; ++f) {
      if (!AT(v.fReg, f)) continue;
      const int32_t kind = AT(v.fKind, f);
      if (kind == K_TRAIN) {
        const int32_t gm = AT(gang, f);
        if (gm == BIG) continue;
        AT(gang, f) = BIG;
        int32_t nlive = 0;
        bool all_warm = true;
        for (int32_t s = AT(v.fLh, f); s >= 0; s = AT(v.iNext, s)) {
          ++nlive;
          all_warm &= st_l(AT(v.iMeta, s)) == ST_PLACED && AT(v.iReady, s) <= t;
        }
        if (all_warm) {
          tl.tprg += (long long)AT(v.fNw, f) * gm;
          tl.etot += (long long)nlive * gm;
        }
      } else if (kind == K_LLM) {
        for (int32_t s = AT(v.fLh, f); s >= 0; s = AT(v.iNext, s)) {
          const int32_t b = AT(bmin, s);
          if (b == BIG) continue;
          AT(bmin, s) = BIG;
          const int32_t meta = AT(v.iMeta, s);
          const int32_t nst = nst_l(meta);
          const int32_t e = AT(v.iPos, s * MAXST);
          const int32_t ibs = AT(v.rIbs, e), cst = AT(v.rCst, e);
          const int32_t rr = AT(rR, e);
          const long long capb = (long long)b * ibs;
          const int32_t served = capb < rr ? (int32_t)capb : rr;
          tl.rsrv += served;
          tl.rvio += rr - served;
          const long long ex = (long long)nst * b * cst;
          tl.iexe += ex;
          tl.etot += ex;
        }
      }
    }
  }
};

template <int P>
__global__ void __launch_bounds__(32 * P) k_lanes(LParams Pin, int32_t* next_grp, int32_t t0,
                                                  int32_t n_slots, int32_t n_req,
                                                  const int32_t* req_scn, const int32_t* req_func,
                                                  int32_t* out_gpu, int32_t* out_iid) {
  __shared__ LParams Pm;
  __shared__ Shr<P> sh;
  __shared__ LV sv;
  const int lane = threadIdx.x & 31, k = threadIdx.x >> 5;
  if (threadIdx.x == 0) Pm = Pin;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) sh.grp = atomicAdd(next_grp, 1);
    __syncthreads();
    const int32_t grp = sh.grp;
    if (grp >= Pm.ngroups) break;
    if (threadIdx.x == 0) sv = make_lv(Pm.state + (size_t)grp * Pm.L.bytes, Pm.L);
    __syncthreads();
    Ctx c;
    c.P = &Pm;
    c.k = k;
    c.lane = lane;
    const int32_t scn = grp * LN + lane;
    c.active = scn < Pm.S;
    c.vp = &sv;
    c.frow = Pm.funcs + (size_t)(c.active ? scn : 0) * Pm.F * 16;
    c.scn_id = c.active ? Pm.scen[scn * 4 + 0] : 0;
    c.om = c.active ? Pm.scen[scn * 4 + 1] : 0;
    c.ga = c.active ? Pm.scen[scn * 4 + 2] : 0;
    c.mode = c.active ? Pm.scen[scn * 4 + 3] : 0;
    const LV& v = *c.vp;
    const int LANE = c.lane;
    if (c.active && AT(v.h, LH_ERR)) c.active = false;
    Tl tl = {};
    if (n_req >= 0) {
      if (k == 0 && c.active) {
        for (int32_t jr = 0; jr < n_req && !AT(v.h, LH_ERR); ++jr) {
          if (req_scn[jr] != scn) continue;
          const int32_t f = req_func[jr];
          l_register(c, f, t0);
          out_iid[jr] = l_enqueue(c, f, AT(v.fKind, f) == K_TRAIN ? AT(v.fNw, f) : 1);
        }
        if (AT(v.h, LH_ERR)) c.active = false;
      }
      __syncthreads();
      // the error flag is per scenario: all parts re-read it
      if (c.active && AT(v.h, LH_ERR)) c.active = false;
      Engine<P>::pass(c, sh, t0, tl);
      if (k == 0 && c.active)
        for (int32_t jr = 0; jr < n_req; ++jr) {
          if (req_scn[jr] != scn) continue;
          const int32_t id = out_iid[jr];
          int32_t g = -1;
          for (int32_t s = AT(v.fLh, req_func[jr]); s >= 0; s = AT(v.iNext, s))
            if (AT(v.iId, s) == id) {
              if (st_l(AT(v.iMeta, s)) == ST_PLACED) g = AT(v.iG, s * MAXST);
              break;
            }
          out_gpu[jr] = g;
        }
    } else {
      for (int32_t t = t0; t < t0 + n_slots; ++t) {
        if (t % Pm.SPS == 0) {
          Engine<P>::boundary(c, sh, t, tl);
          if (c.active && AT(v.h, LH_ERR)) c.active = false;
        }
        Engine<P>::phase0(c, t, tl);
        if (k == 0 && c.active) {
          const long long na = AT(v.h, LH_NACT);
          tl.act += na;
          tl.memu += na * Pm.M - AT(v.h, LH_SUMU);
          tl.rows += Pm.G;
          tl.maxa = na > tl.maxa ? na : tl.maxa;
          tl.st[S_SLOT] += 1;
        }
        __syncthreads();
        Engine<P>::phase1(c, t, tl);
        __syncthreads();
        Engine<P>::phase2(c, t, tl);
        __syncthreads();
      }
    }
    // reduce the P parts of each scenario
    long long vals[9] = {tl.rtot, tl.rsrv, tl.rvio, tl.iexe, tl.tprg, tl.etot,
                         (long long)tl.hash, tl.nres, tl.nfun};
#pragma unroll
    for (int q = 0; q < 9; ++q) sh.acc[q][k][lane] = vals[q];
    __syncthreads();
    if (k == 0 && scn < Pm.S) {
      long long s9[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
      for (int q = 0; q < 9; ++q)
        for (int x = 0; x < P; ++x)
          s9[q] = (long long)((unsigned long long)s9[q] + (unsigned long long)sh.acc[q][x][lane]);
      long long* T = reinterpret_cast<long long*>(Pm.tally) + (size_t)scn * NT;
      T[T_ACT] += tl.act;
      T[T_SMU] += tl.act * Pm.T_slot - s9[5];
      T[T_MEMU] += tl.memu;
      T[T_RTOT] += s9[0];
      T[T_RSRV] += s9[1];
      T[T_RVIO] += s9[2];
      T[T_IEXE] += s9[3];
      T[T_TPRG] += s9[4];
      T[T_POK] += tl.pok;
      T[T_PFAIL] += tl.pfail;
      T[T_COLD] += tl.cold;
      T[T_SOUT] += tl.sout;
      T[T_SIN] += tl.sin;
      T[T_SPLIT] += tl.split;
      T[T_HASH] = (long long)((unsigned long long)T[T_HASH] + (unsigned long long)s9[6]);
      T[T_ROWS] += tl.rows;
      if (tl.maxa > T[T_MAXA]) T[T_MAXA] = tl.maxa;
      tl.st[S_RES] += s9[7];
      tl.st[S_FUN] += s9[8];
      long long* ST = reinterpret_cast<long long*>(Pm.stats) + (size_t)scn * NSTAT;
      for (int x = 0; x < NSTAT; ++x) ST[x] += tl.st[x];
    }
  }
}

// Initialise groups at slot 0: one CTA of 32 threads per group (thread = scenario).
__global__ void k_lanes_init(LParams P) {
  const int32_t grp = blockIdx.x, lane = threadIdx.x;
  const int LANE = lane;
  const int32_t scn = grp * LN + lane;
  LV v = make_lv(P.state + (size_t)grp * P.L.bytes, P.L);
  for (int k = 0; k < LH_WORDS; ++k) AT(v.h, k) = 0;
  AT(v.h, LH_FSTOP) = P.I;
  for (int32_t g = 0; g < P.G; ++g) {
    AT(v.gR, g) = 0; AT(v.gL, g) = 0; AT(v.gU, g) = 0; AT(v.gN, g) = 0; AT(v.gExcl, g) = 0;
    AT(v.gRel, g) = 0;
  }
  for (int32_t s = 0; s < P.I; ++s) {
    AT(v.iId, s) = -1; AT(v.iFunc, s) = -1; AT(v.iMeta, s) = ST_FREE; AT(v.iReady, s) = 0;
    AT(v.iNext, s) = -1;
    for (int k = 0; k < MAXST; ++k) {
      AT(v.iG, s * MAXST + k) = -1; AT(v.iShare, s * MAXST + k) = 0; AT(v.iPos, s * MAXST + k) = -1;
    }
    AT(v.iBmin, s) = BIG; AT(v.iBmin, P.I + s) = BIG;
    AT(v.fstack, s) = P.I - 1 - s;
    AT(v.qFunc, s) = 0; AT(v.qFirst, s) = 0; AT(v.qN, s) = 0; AT(v.qFail, s) = -1;
  }
  for (int k = 0; k < RLOG; ++k) { AT(v.rlG, k) = 0; AT(v.rlE, k) = 0; }
  const bool active = scn < P.S;
  const int32_t* rows = P.funcs + (size_t)(active ? scn : 0) * P.F * 16;
  const int32_t mode = active ? P.scen[scn * 4 + 3] : 0;
  for (int32_t f = 0; f < P.F; ++f) {
    const int32_t* r = rows + (size_t)f * 16;
    const int32_t kind = active ? r[0] : K_UNUSED;
    const int32_t req = (mode == M_STATIC_LIMIT || mode == M_EAGER) ? r[4] : r[3];
    const int32_t limq = mode == M_STATIC_REQUEST ? r[3] : r[4];
    AT(v.fKind, f) = kind; AT(v.fPrio, f) = r[1]; AT(v.fIbs, f) = r[2] > 0 ? r[2] : 1;
    AT(v.fReq, f) = req; AT(v.fLim, f) = limq; AT(v.fMem, f) = r[5];
    AT(v.fCb, f) = r[6] > 0 ? r[6] : 1; AT(v.fNw, f) = r[7]; AT(v.fCold, f) = r[9];
    AT(v.fCls, f) = r[10]; AT(v.fArr, f) = r[11]; AT(v.fDep, f) = r[12]; AT(v.fPat, f) = r[13];
    AT(v.fScale, f) = r[14];
    // training demand d = lim * duty; Exclusive owns the whole GPU (lim = T_slot, D7)
    const long long lim_tok = (long long)(mode == M_EXCLUSIVE ? 1000 : limq) * P.slot_ms;
    AT(v.fDtr, f) = kind == K_TRAIN ? (int32_t)(lim_tok * r[8] / 1000) : 0;
    AT(v.fCap1, f) = inf_l(kind) ? (long long)P.SPS * (((long long)req * P.slot_ms) / (r[6] > 0 ? r[6] : 1)) * r[2] : 0;
    AT(v.fReg, f) = 0; AT(v.fNsamp, f) = 0; AT(v.fAcc, f) = 0; AT(v.fHead, f) = 0;
    AT(v.fUp, f) = 0; AT(v.fDown, f) = 0; AT(v.fThrn, f) = -1; AT(v.fNlive, f) = 0;
    AT(v.fLh, f) = -1; AT(v.fLt, f) = -1; AT(v.fGang, f) = BIG; AT(v.fGang, P.F + f) = BIG;
    AT(v.fFlag, f) = 0; AT(v.fK, f) = 0; AT(v.fPidx, f) = 0; AT(v.fEvl, f) = 0;
  }
  if (active) {
    for (int k = 0; k < NT; ++k) P.tally[(size_t)scn * NT + k] = 0;
    for (int k = 0; k < NSTAT; ++k) P.stats[(size_t)scn * NSTAT + k] = 0;
  }
}

__global__ void k_lanes_snapshot(LParams P, int32_t id_cap, int32_t* out_gpu, int32_t* out_inst) {
  const int32_t grp = blockIdx.x, lane = threadIdx.x;
  const int LANE = lane;
  const int32_t scn = grp * LN + lane;
  if (scn >= P.S) return;
  LV v = make_lv(P.state + (size_t)grp * P.L.bytes, P.L);
  if (out_gpu)
    for (int32_t g = 0; g < P.G; ++g) {
      int32_t* o = out_gpu + ((size_t)scn * P.G + g) * 4;
      o[0] = AT(v.gR, g); o[1] = AT(v.gL, g); o[2] = AT(v.gU, g); o[3] = AT(v.gN, g);
    }
  if (!out_inst) return;
  const int32_t issued = AT(v.h, LH_NEXT_IID);
  for (int32_t id = 0; id < id_cap; ++id) {
    int32_t* o = out_inst + ((size_t)scn * id_cap + id) * 12;
    if (id >= issued) { for (int k = 0; k < 12; ++k) o[k] = -1; continue; }
    o[0] = -1; o[1] = 2; o[2] = 0; o[3] = -1;
    for (int k = 0; k < MAXST; ++k) { o[4 + k] = -1; o[8 + k] = 0; }
  }
  for (int32_t s = 0; s < P.I; ++s) {
    const int32_t meta = AT(v.iMeta, s);
    if (st_l(meta) == ST_FREE) continue;
    const int32_t id = AT(v.iId, s);
    if (id >= id_cap) continue;
    int32_t* o = out_inst + ((size_t)scn * id_cap + id) * 12;
    const bool pl = st_l(meta) == ST_PLACED;
    o[0] = AT(v.iFunc, s);
    o[1] = pl ? 1 : 0;
    o[2] = pl ? nst_l(meta) : 0;
    o[3] = pl ? AT(v.iReady, s) : -1;
    for (int k = 0; k < MAXST; ++k) {
      const bool on = pl && k < nst_l(meta);
      o[4 + k] = on ? AT(v.iG, s * MAXST + k) : -1;
      o[8 + k] = on ? AT(v.iShare, s * MAXST + k) : 0;
    }
  }
}

__global__ void k_lanes_errs(LParams P, int64_t* out) {
  const int32_t t = threadIdx.x;
  int32_t e = 0;
  for (int32_t scn = t; scn < P.S; scn += blockDim.x) {
    const int32_t grp = scn / LN, lane = scn % LN;
    const int32_t* h = reinterpret_cast<const int32_t*>(P.state + (size_t)grp * P.L.bytes + P.L.hdr) + lane;
    const int32_t x = h[(size_t)LH_ERR << 5];
    e = x > e ? x : e;
  }
  for (int o = 16; o > 0; o >>= 1) e = max(e, __shfl_xor_sync(0xffffffffu, e, o));
  if (t == 0) out[0] = e;
}

#undef AT
}  // namespace lanes
}  // namespace dilu
