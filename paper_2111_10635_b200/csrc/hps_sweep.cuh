// hps_sweep.cuh — fast path (v1) of the warp-per-plan evaluator.
//
// Same outputs as the literal path in hps_eval.cuh (and therefore as the reference), with the
// per-(candidate, stage) divisions replaced by exact table lookups:
//
//  * count(tau) of a stage entry is a non-increasing step function of tau (every operation of
//    _floor_count/_iceil is monotone under IEEE rounding). theta(m) = min{tau : count <= m} is
//    tabulated per instance (TE table, exact by bisection over double bit patterns), so
//    count(tau) = min{m : theta(m) <= tau}: an FP32 estimate seeds a galloping search over the
//    table, which alone decides the (exact) answer.
//  * bisection (ls/provisioner.py:430-437): lanes own stages; counts are pinned between
//    count(b) and count(a). Once every unpinned stage is within one step, quota_ok on (a, b)
//    switches at one of the thresholds theta_r(count(b)); that switch point tau* is found
//    exactly and the remaining bisection steps are comparisons mid >= tau*.
//  * _best_candidate (ls/provisioner.py:262-314): candidates round-robin over lanes; exact counts
//    come from an FP32 seed verified against the threshold table; a warm start around the
//    minimiser of a convex lower bound gives an upper bound ub, the bound confines the certified
//    candidates that can reach ub + 1e-15 to an interval, and a rigorous per-candidate lower
//    bound (E >= tau at a certified breakpoint, every unpinned stage's count bounded below in FP32
//    with its error margin, floored by its count at the interval's end) skips the candidates that
//    cannot reach the minimum or its 1e-15 tie window; evaluated candidates use the reference's
//    exact sequential per_second sum and its two cost divisions.
#pragma once
#include "hps_eval.cuh"

namespace hps {

struct CandQueue {    // survivors of cand_main's lower-bound filter, evaluated 32 at a time
  double q[64];
  int32_t qg[64];      // their generator: (leader << 16) | m, or -1 (tau_lo / tau_hi)
};

template <int MAXS>
struct SweepSmem {   // per-warp, per-plan constants of the fast candidate phase (broadcast reads)
  double pr[MAXS];   // price per second of stage r's type
  double etp[MAXS];  // exact et at the pinned count (kmin == kmax), else unused
  float fpr[MAXS];   // pr as FP32 (bounds only)
  int32_t kmi[MAXS]; // count at tau_hi (= kmin)
  int32_t kma[MAXS]; // count at tau_lo (= kmax)
  int32_t alo[MAXS], an[MAXS], blo[MAXS];  // restricted candidate ranges (cand_tau2)
  int32_t pre2[MAXS + 1];

  int32_t dom[MAXS]; // side_dominance over [tau_lo, tau_hi]: 1 oct, 2 odt, 0 both
  float est[MAXS][6];  // count_est seed constants (est_setup)
  int8_t lead[MAXS]; // class leader of stage r (stages of one class have identical counts)
  int32_t gex[MAXS]; // leader r: count_r(et_r(m)) == m for m <= gex[r] (tb.gex), else 0
  struct CandQueue* cq;  // the candidate kernel's survivor queue (prep does not need one)
  double p0;         // sum over pinned stages of pr * count (the bound's linear part)
  int32_t nu;        // unpinned stages, in stage order:
  int8_t ulist[MAXS];
  int16_t kb[MAXS];  // count at tb (cand_prep): the candidate filter's floor for tau <= tb
  double tb;         // right end of the restricted interval (-inf: none)
  float p0f;         // pinned stages' sum of pr * count in FP32 (cand_main)
  __device__ __forceinline__ float est_at(int r, int i) const { return est[r][i]; }
};

// FP32 estimate of count(tau) of unpinned stage r, clamped to [kmin, kmax]. Only a seed: the
// threshold table confirms or corrects it (count_verify), so it never affects a result.
// per-stage FP32 seed constants {rb, 1 - frac, frac} of both sides; a side that cannot decide the
// count (work 0, frac 0, or dominated per side_dominance) is {0, -1, 0} and contributes q = 0
template <int MAXS, class W>
__device__ __forceinline__ void est_setup(const W& w, SweepSmem<MAXS>& sw, int r) {
  const StageEntry& s = w.stage(r);
  const int dom = sw.dom[r];
#pragma unroll
  for (int side = 0; side < 2; side++) {
    const float rb = side ? s.f_rbd : s.f_rbo;
    const float frac = side ? s.f_beta : s.f_alpha;
    const bool on = (dom != 2 - side) && rb != 0.0f && frac != 0.0f;
    sw.est[r][3 * side + 0] = on ? rb : 0.0f;
    sw.est[r][3 * side + 1] = on ? (side ? s.f_omb : s.f_oma) : -1.0f;
    sw.est[r][3 * side + 2] = on ? frac : 0.0f;
  }
}

// FP32 estimate of count(tau) of unpinned stage r, clamped to [kmin, kmax]. Only a seed: the
// threshold table confirms or corrects it (count_verify), so it never affects a result.
template <int MAXS, class W, class SW>
__device__ __forceinline__ int count_est(const W& w, const SW& sw, int r, float tf) {
  const float q0 = sw.est_at(r, 2) * rcp_approx_f32(tf * sw.est_at(r, 0) - sw.est_at(r, 1));
  const float q1 = sw.est_at(r, 5) * rcp_approx_f32(tf * sw.est_at(r, 3) - sw.est_at(r, 4));
  const float q = fmaxf(1.0f, fmaxf(q0, q1));   // (NaN operands are ignored)
  const int lo = sw.kmi[r], hi = sw.kma[r];
  const int k = (q < 2.0e9f) ? (int)ceilf(q) : hi;
  return min(max(k, lo), hi);
}

// read-only table loads: {et(k), theta(k - 1)} in one 16-byte load, theta(k) separately
__device__ __forceinline__ double2 te_pair(const TEPair* row, int k) {
  return __ldg(reinterpret_cast<const double2*>(&HPS_TE(row, k - 1)));
}
__device__ __forceinline__ double te_theta(const TEPair* row, int k) { return __ldg(&HPS_TE(row, k).th); }

// Exact count(tau) for tau in [tau_lo, tau_hi] (count in [kmin, kmax]) given the seed k and the
// loads pk = {et(k), theta(k - 1)}, thk = theta(k): k is the count iff theta(k) <= tau <
// theta(k - 1) (count(tau) = min{m : theta(m) <= tau}); otherwise the exact galloping table search
// from k decides. Returns the count and et at it.
template <int MAXS, class W, class SW>
__device__ __forceinline__ int count_verify(const W& w, const SW& sw, int r,
                                            double tau, int k, double2 pk, double thk, double& et) {
  if (thk <= tau && tau < pk.y) {
    et = pk.x;
    return k;
  }
  const TEPair* row = w.row[r];
  k = count_tab(row, tau, sw.kmi[r], sw.kma[r], k);
  et = __ldg(&HPS_TE(row, k - 1).et);
  return k;
}

struct CostScalars {  // the four job constants the cost needs (no parameter-struct copies)
  double bo, batch, work, limit;
};

// exact cost of candidate tau (numpy column of _best_candidate, ls/provisioner.py:286-308);
// one out-of-line copy shared by every call site.
// gen = (g << 16) | m when tau = et_g(m) and tb.gex certifies count_g(tau) == m: every stage of
// g's class then has count m and et == tau exactly (the breakpoint value itself).
template <int MAXS, class W, class SW>
__device__ __noinline__ double cost_exact(const CostScalars cs, const W& w,
                                          const SW& sw, int S, double tau, int gen) {
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  const int g = (gen >= 0) ? (gen >> 16) : -1, gm = gen & 0xffff;
  const float tf = (float)tau;
  double P = 0.0, E = 0.0;
  for (int r = 0; r < S; r++) {
    double et;
    int k;
    if (sw.kma[r] == sw.kmi[r]) {
      k = sw.kmi[r];
      et = sw.etp[r];
    } else if (sw.lead[r] == g) {
      k = gm;
      et = tau;
    } else {
      const int k0 = count_est<MAXS>(w, sw, r, tf);
      const TEPair* row = w.row[r];
      k = count_verify<MAXS>(w, sw, r, tau, k0, te_pair(row, k0), te_theta(row, k0), et);
    }
    E = (r == 0) ? et : fmax(E, et);
    const double term = sw.pr[r] * (double)k;
    P = (r == 0) ? term : P + term;
  }
  const double thr = (E > 0) ? cs.batch / E : inf;
  if (!(thr > cs.limit)) return inf;
  return cs.work / thr * P;
}

// exact cost of one candidate into the lane's tie buffer (one out-of-line copy for every site)
template <int MAXS, class W, class SW>
__device__ __noinline__ void eval_insert(const CostScalars cs, const W& w, const SW& sw,
                                         int S, double tau, int gen, TieBuf& buf) {
  buf.insert(cost_exact<MAXS>(cs, w, sw, S, tau, gen), tau);
}

// FP32 lower bound on count(tau) of an unpinned stage (pruning only). Every FP32 input and
// operation carries a relative error of a few 2^-24; with kappa = B/h the headroom's relative
// error is <= 3e-7 kappa + 6e-8, so q~ = frac/h~ is within q (1 +- e0), e0 = 4e-7 (kappa + 2).
// lo = q~ (1 - e0 - 1e-6) is then <= q - 1e-9 whenever lo >= 1 (q >= 1e-3), and iceil is
// monotone, so ceil(lo) <= ceil(q - 1e-9) = count. dom (side_dominance) restricts it to the
// deciding side; a side with too much cancellation is skipped (1 is always a lower bound).
__device__ __forceinline__ int count_lb32(const StageEntry& s, float tau, int dom) {
  float lo = 1.0f;
#pragma unroll
  for (int side = 0; side < 2; side++) {
    if (dom == 2 - side) continue;   // dom 1 skips side 1, dom 2 skips side 0
    const float rb = side ? s.f_rbd : s.f_rbo;
    const float frac = side ? s.f_beta : s.f_alpha;
    if (rb == 0.0f || frac == 0.0f) continue;
    const float omf = side ? s.f_omb : s.f_oma;
    const float B = tau * rb;
    const float h = B - omf;
    if (!(h > 1e-3f * B)) continue;
    const float rh = rcp_approx_f32(h);
    const float e = 4e-7f * (B * rh + 2.0f) + 1e-6f;
    lo = fmaxf(lo, (frac * rh) * (1.0f - e));
  }
  return (int)ceilf(lo);
}

// count_lb32 from the count_est seed constants (est_setup): they hold the same FP32 side constants,
// with the sides count_lb32 skips (dominated, rb == 0 or frac == 0) set to rb = 0
__device__ __forceinline__ int count_lb32_est(const float* e, float tau) {
  float lo = 1.0f;
#pragma unroll
  for (int side = 0; side < 2; side++) {
    const float rb = e[3 * side], omf = e[3 * side + 1], frac = e[3 * side + 2];
    if (rb == 0.0f) continue;
    const float B = tau * rb;
    const float h = B - omf;
    if (!(h > 1e-3f * B)) continue;
    const float rh = rcp_approx_f32(h);
    const float ee = 4e-7f * (B * rh + 2.0f) + 1e-6f;
    lo = fmaxf(lo, (frac * rh) * (1.0f - ee));
  }
  return (int)ceilf(lo);
}

// candidate i: tau_lo, tau_hi, then the breakpoints et_sp(m) of the class leaders; gen as in
// cost_exact (-1 unless the leader's breakpoints are certified)
template <int MAXS, class W>
__device__ __forceinline__ double cand_tau(const W& w, const SweepSmem<MAXS>& sw, int i,
                                           int& sp, double tau_lo, double tau_hi, int& gen) {
  gen = -1;
  if (i < 2) return (i == 0) ? tau_lo : tau_hi;
  const int j = i - 2;
  while (w.pre[sp + 1] <= j) sp++;
  const int m = (int)w.kmin[sp] + (j - w.pre[sp]);
  if (m <= sw.gex[sp]) gen = (sp << 16) | m;
  return __ldg(&HPS_TE(w.row[sp], m - 1).et);
}

// candidate i of the restricted list: tau_lo, tau_hi, then per class leader sp the certified
// breakpoints m in [alo, alo + an) (those inside the bound interval) and the uncertified ones
// m in [blo, kmax]
template <int MAXS, class W, class SW>
__device__ __forceinline__ double cand_tau2(const W& w, const SW& sw, int i,
                                            int& sp, double tau_lo, double tau_hi, int& gen) {
  gen = -1;
  if (i < 2) return (i == 0) ? tau_lo : tau_hi;
  const int j = i - 2;
  while (sw.pre2[sp + 1] <= j) sp++;
  const int o = j - sw.pre2[sp];
  int m;
  if (o < sw.an[sp]) {
    m = sw.alo[sp] + o;
    gen = (sp << 16) | m;
  } else {
    m = sw.blo[sp] + (o - sw.an[sp]);
  }
  return __ldg(&HPS_TE(w.row[sp], m - 1).et);
}

#ifndef HPS_GRID
#define HPS_GRID 16
#endif
constexpr int kGrid = HPS_GRID;   // grid points per level of the interval search (power of 2)
#ifndef HPS_GRID_LEVELS
#define HPS_GRID_LEVELS 2
#endif

// Continuous lower bound of the cost of every certified breakpoint candidate tau:
//   L(tau) = (work/batch) tau sum_r pr_r max(kmin_r, q_r(tau)(1 - 1e-8) - 1e-9),
// q_r = max over sides of frac / (tau bo/work - (1 - frac)): count_r(tau) = ceil(max(1, q) - 1e-9)
// >= both terms (the 1e-8 relative slack covers the rounding of q here and in the reference), and
// E >= tau (certified breakpoint). Each term tau max(kmin, q(1-d) - e) is a max of convex
// functions of tau (tau q(tau) = (frac/b)(1 + c/(b tau - c)) with c = 1 - frac), so L is convex.
// Returns L and a subgradient dL/dtau at tau.
template <int MAXS, class W>
__device__ __noinline__ void lb_cont(const W& w, const SweepSmem<MAXS>& sw, int S, double bo,
                                        double C, double tau, double& L, double& dL, bool half = false) {
  // kGrid points per level: lanes p, p + kGrid, ... share point p and split the unpinned stages,
  // combined by butterfly steps; pinned stages contribute tau * p0 (slope p0), counted once.
  // A stage whose count one side decides on [tau_lo, tau_hi] (side_dominance) uses that side.
  // half: one plan per 16 lanes (hps_half.cuh), each lane takes all stages of its point.
  const int grp = half ? 0 : (threadIdx.x & 31) / kGrid, step = half ? 1 : 32 / kGrid;
  double P = (grp == 0) ? tau * sw.p0 : 0.0, dP = (grp == 0) ? sw.p0 : 0.0;
  for (int j = grp; j < sw.nu; j += step) {
    const int r = sw.ulist[j];
    const int dom = sw.dom[r];
    const double km = (double)sw.kmi[r];
    double v = km * tau, dv = km;
    const StageEntry& s = w.stage(r);
#pragma unroll
    for (int side = 0; side < 2; side++) {
      if (dom == 2 - side) continue;
      const double work = side ? s.odt : s.oct;
      const double frac = side ? s.beta : s.alpha;
      if (work == 0.0 || frac == 0.0) continue;
      const double cc = side ? s.omb : s.oma;
      const double h = tau * (bo * (side ? s.rwd : s.rwo)) - cc;
      if (!(h > 0.0)) { v = __longlong_as_double(0x7ff0000000000000LL); dv = 0.0; continue; }
      const double rh = rcp_1nt(h);
      const double q = frac * rh;
      const double vq = tau * (q * (1.0 - 1e-8) - 1e-9);
      // d(tau q)/dtau = -q^2 c / frac = -q c / h
      if (vq > v) { v = vq; dv = (1.0 - 1e-8) * (-q * cc * rh) - 1e-9; }
    }
    P += sw.pr[r] * v;
    dP += sw.pr[r] * dv;
  }
  if (!half)
    for (int o = kGrid; o < 32; o <<= 1) {
      P += __shfl_xor_sync(0xffffffffu, P, o);
      dP += __shfl_xor_sync(0xffffffffu, dP, o);
    }
  L = C * P;
  dL = C * dP;
}

// One level of the interval search: lane j < 16 holds (t, L, dL) at grid point j of [ta, tb]
// (point 15 = tb). On each cell, convexity bounds L from below by max(tangent at the left end, tangent
// at the right end); [ta, tb] shrinks to the cells whose bound does not exceed thr (ta > tb when
// none does).
static __device__ __noinline__ void interval_cells(double t, double L, double d, double thr, double& ta, double& tb) {
  const int lane = threadIdx.x & 31;
  const double t1 = __shfl_down_sync(0xffffffffu, t, 1);
  const double L1 = __shfl_down_sync(0xffffffffu, L, 1);
  const double d1 = __shfl_down_sync(0xffffffffu, d, 1);
  double lb;
  if (d >= 0.0) lb = L;
  else if (d1 <= 0.0) lb = L1;
  else {
    // any x gives min(left tangent, right tangent) <= the minimum of their maximum, so an
    // approximate intersection is still a valid lower bound
    const double x = (L1 - L + d * t - d1 * t1) * rcp_1nt(d - d1);
    lb = fmin(fmin(L + d * (x - t), L1 + d1 * (x - t1)), fmin(L, L1));
  }
  const bool keep = (lane < kGrid - 1) && !(lb > thr);   // NaN keeps
  const unsigned mk = __ballot_sync(0xffffffffu, keep);
  if (!mk) { ta = 1.0; tb = 0.0; return; }
  const int f = __ffs(mk) - 1, l = 31 - __clz(mk);
  const double nta = __shfl_sync(0xffffffffu, t, f);
  tb = __shfl_sync(0xffffffffu, t, l + 1);
  ta = nta;
}

template <int MAXS>
__device__ __forceinline__ double grid_point(double ta, double tb) {
  const int p = threadIdx.x & (kGrid - 1);   // lanes p, p + kGrid, ... hold the same point
  return (p == kGrid - 1) ? tb : ta + (tb - ta) * (double)p * (1.0 / (kGrid - 1));
}

// tie buffer overflow (rare): the largest tau of the restricted list whose exact cost is <= lim
template <int MAXS, class W>
__device__ __noinline__ double overflow_pass(const CostScalars cs, const W& w, const SweepSmem<MAXS>& sw,
                                             int S, double tau_lo, double tau_hi, int n2, double lim) {
  double bt = -__longlong_as_double(0x7ff0000000000000LL);
  int sp = 0;
  for (int i = (threadIdx.x & 31); i < n2; i += 32) {
    int gen;
    const double tau = cand_tau2<MAXS>(w, sw, i, sp, tau_lo, tau_hi, gen);
    if (!(tau >= tau_lo && tau <= tau_hi) || !(tau > bt)) continue;
    if (cost_exact<MAXS>(cs, w, sw, S, tau, gen) <= lim) bt = tau;
  }
  return bt;
}

// _best_candidate: round-robin candidates over lanes. A warm-start round evaluates 32 candidates
// (16 in the half-warp prep) around the grid minimiser of the convex bound L exactly (upper bound
// ub on the minimum). L
// (lb_cont) then confines every certified breakpoint that could reach ub + 1e-15 to an
// interval [ta, tb] (two grid levels, interval_cells); for each class leader those are the m in
// [count(tb), count(ta)] (certified: count(et(m)) == m, counts non-increasing). Only these,
// tau_lo, tau_hi and the uncertified breakpoints remain; each gets a per-candidate bound
// (E >= tau, the generator's class at count m, every other unpinned stage at the larger of its
// FP32 count lower bound and its count at tb (tau <= tb) or tau_hi; FP32 slack 1e-5) and is
// evaluated exactly only when the bound does not exceed the best cost so far + 1e-15. A skipped candidate costs more than the final minimum + 1e-15: it is
// neither the minimum nor a tie.
// Part 1 (cand_prep): per-plan constants, warm start, interval and restricted ranges (alo, an,
// blo); returns ub. Part 2 (cand_main): the filter and exact evaluation over the restricted list.
// The split path runs them in separate kernels (instruction-cache footprint): part 2 then starts
// with an empty tie buffer, which loses nothing, because every warm-start candidate that can be
// the minimum or a tie (cost <= ub + 1e-15) lies in the restricted list and passes the filter.
template <int MAXS, class W>
__device__ double cand_prep(const InstanceConsts& c, const DeviceTables& tb, const W& w,
                            SweepSmem<MAXS>& sw, int S, double tau_lo, double tau_hi, int n_cand, TieBuf& buf) {
  const int lane = threadIdx.x & 31;
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  int fl[2];   // first stage of each stage's class
  first_same2(S, (lane < S) ? w.cls[lane] : 0, (lane + 32 < S) ? w.cls[lane + 32] : 0, fl[0], fl[1]);
#pragma unroll 1
  for (int r = lane; r < S; r += 32) {
    const bool pinned = (w.kmax[r] == w.kmin[r]);
    sw.pr[r] = c.price_s[w.stage(r).type];
    sw.fpr[r] = (float)sw.pr[r];
    sw.kmi[r] = (int)w.kmin[r];
    sw.kma[r] = (int)w.kmax[r];
    sw.etp[r] = pinned ? w.row[r][(int)w.kmin[r] - 1].et : 0.0;
    sw.dom[r] = pinned ? 0 : side_dominance(w.stage(r), tau_lo, tau_hi, c.bo);
    est_setup<MAXS>(w, sw, r);
    const int ld = fl[r >> 5];
    sw.lead[r] = (int8_t)ld;
    sw.gex[r] = (ld == r && !pinned) ? __ldg(tb.gex + w.ent[r]) : 0;
  }
  {  // unpinned stages in order, and the pinned stages' part of the bound
    double p0 = 0.0;
    int base = 0;
#pragma unroll
    for (int slot = 0; slot < 2; slot++) {
      const int r = lane + 32 * slot;
      const bool unp = r < S && w.kmax[r] != w.kmin[r];
      if (r < S && !unp) p0 += c.price_s[w.stage(r).type] * w.kmin[r];
      const unsigned m = __ballot_sync(0xffffffffu, unp);
      if (unp) sw.ulist[base + __popc(m & ((1u << lane) - 1u))] = (int8_t)r;
      base += __popc(m);
    }
    for (int o = 16; o; o >>= 1) p0 += __shfl_xor_sync(0xffffffffu, p0, o);
    if (lane == 0) { sw.nu = base; sw.p0 = p0; }
  }
  __syncwarp();
  if (lane == 0) {
    HPS_STAT(ST_NCAND, n_cand);
    HPS_STAT(ST_PLANS_FAST, 1);
    HPS_STAT(ST_STAGES, S);
  }
  __syncwarp();
  const CostScalars cs{c.bo, c.batch, c.work, c.limit};
  int sp = 0;
  const double C = c.work / c.batch;
  // level-0 grid of the convex bound L over [tau_lo, tau_hi]
  const bool grid = tau_hi > tau_lo;
  double g_t = tau_lo, g_L = 0.0, g_d = 0.0;
  if (grid) {
    g_t = grid_point<MAXS>(tau_lo, tau_hi);
    lb_cont<MAXS>(w, sw, S, c.bo, C, g_t, g_L, g_d);
  }
  {  // warm start: 32 certified breakpoints around the grid minimiser of L (the optimum is
     // usually there), else spread over the whole candidate range
    double lmin = grid ? g_L : 0.0;
    lmin = warp_min(lmin);
    const unsigned at = __ballot_sync(0xffffffffu, grid && g_L == lmin);
    const double tstar = __shfl_sync(0xffffffffu, g_t, at ? __ffs(at) - 1 : 0);
    // leaders with certified breakpoints, their count at tstar
    int cstar = 0;
    bool ok = false;
    if (lane < S) {
      const int lo = sw.kmi[lane], chi = min(sw.kma[lane], sw.gex[lane]);
      ok = grid && w.pre[lane + 1] > w.pre[lane] && chi >= lo;
      if (ok) cstar = min(max(count_seeded(w.stage(lane), w.row[lane], tstar, lo, sw.kma[lane]), lo), chi);
    }
    const unsigned lm = __ballot_sync(0xffffffffu, ok);
    const int nl = __popc(lm);
    double tau = -inf;
    int gen = -1;
    if (nl > 0) {
      const int li = lane % nl, k = lane / nl;   // leader #li, offset 0, +1, -1, +2, -2, ...
      const int r = __fns(lm, 0, li + 1);
      const int cr = __shfl_sync(0xffffffffu, cstar, r);
      const int off = (k & 1) ? (k + 1) >> 1 : -(k >> 1);
      const int m = cr + off;
      if (r < S && m >= sw.kmi[r] && m <= min(sw.kma[r], sw.gex[r])) {
        gen = (r << 16) | m;
        tau = __ldg(&HPS_TE(w.row[r], m - 1).et);
      }
    } else {
      const int i = (int)(((long long)lane * n_cand) >> 5);
      tau = cand_tau<MAXS>(w, sw, i, sp, tau_lo, tau_hi, gen);
    }
    if (tau >= tau_lo && tau <= tau_hi) {
      HPS_STAT(ST_CANDS, 1);
      eval_insert<MAXS>(cs, w, sw, S, tau, gen, buf);
    }
  }
  double ub = warp_min(buf.mn);
  // ---- interval of the certified breakpoints that can still reach ub + 1e-15 ----
  double ta = tau_lo, tbh = tau_hi;
  if (grid && ub < inf) {
    const double thr = (ub + 1e-15) * (1.0 + 1e-7);
    interval_cells(g_t, g_L, g_d, thr, ta, tbh);
#pragma unroll 1
    for (int lvl = 1; lvl < HPS_GRID_LEVELS && ta <= tbh; lvl++) {
      const double t1 = grid_point<MAXS>(ta, tbh);
      double L1, d1;
      lb_cont<MAXS>(w, sw, S, c.bo, C, t1, L1, d1);
      interval_cells(t1, L1, d1, thr, ta, tbh);
    }
  }
  {
    if (lane == 0) sw.tb = (ta <= tbh) ? tbh : -inf;
#pragma unroll
    for (int slot = 0; slot < 2; slot++) {
      const int r = lane + 32 * slot;
      // count at tau_b of every stage: a candidate tau <= tau_b has count_r(tau) >= it
      int kbv = 0;
      SeedConsts scr;   // stage r's seed constants for both searches
      if (r < S) {
        scr.load(w.stage(r));
        kbv = sw.kmi[r];
        if (sw.kma[r] != sw.kmi[r] && ta <= tbh) kbv = count_seeded_r(scr, w.row[r], tbh, sw.kmi[r], sw.kma[r]);
        sw.kb[r] = (int16_t)kbv;
      }
      if (r < S && w.pre[r + 1] > w.pre[r]) {  // class leader with breakpoints
        const int lo = sw.kmi[r], hi = sw.kma[r];
        int alo = 0, an = 0;
        const int chi = min(hi, sw.gex[r]);   // certified part [lo, chi]
        if (ta <= tbh && chi >= lo) {
          const int ma = kbv;  // smallest certified m
          const int mb = count_seeded_r(scr, w.row[r], ta, lo, hi);   // largest certified m
          alo = max(ma, lo);
          an = max(0, min(mb, chi) - alo + 1);
        }
        const int blo = max(lo, sw.gex[r] + 1);
        sw.alo[r] = alo;
        sw.an[r] = an;
        sw.blo[r] = blo;
      } else if (r < S) {
        sw.alo[r] = 0;
        sw.an[r] = 0;
        sw.blo[r] = sw.kma[r] + 1;   // no breakpoints
      }
    }
  }
  __syncwarp();
  return ub;
}

// exclusive prefix of the restricted per-stage candidate counts an + (kmax - blo + 1)
template <int MAXS>
__device__ __forceinline__ void restricted_prefix(SweepSmem<MAXS>& sw, int S) {
  const int lane = threadIdx.x & 31;
  int cnt[2] = {0, 0};
#pragma unroll
  for (int slot = 0; slot < 2; slot++) {
    const int r = lane + 32 * slot;
    if (r < S) cnt[slot] = sw.an[r] + max(0, sw.kma[r] - sw.blo[r] + 1);
  }
  int inc0 = cnt[0];
  for (int o = 1; o < 32; o <<= 1) { const int v = __shfl_up_sync(0xffffffffu, inc0, o); if (lane >= o) inc0 += v; }
  const int tot0 = __shfl_sync(0xffffffffu, inc0, 31);
  int inc1 = cnt[1];
  for (int o = 1; o < 32; o <<= 1) { const int v = __shfl_up_sync(0xffffffffu, inc1, o); if (lane >= o) inc1 += v; }
  const int tot1 = __shfl_sync(0xffffffffu, inc1, 31);
  if (lane < S) sw.pre2[lane] = inc0 - cnt[0];
  if (lane + 32 < S) sw.pre2[lane + 32] = tot0 + inc1 - cnt[1];
  if (lane == 0) sw.pre2[S] = tot0 + tot1;
  __syncwarp();
}

template <int MAXS, class W>
__device__ double cand_main(const InstanceConsts& c, const W& w, SweepSmem<MAXS>& sw, int S,
                            double tau_lo, double tau_hi, double ub, TieBuf& buf) {
  const int lane = threadIdx.x & 31;
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  const CostScalars cs{c.bo, c.batch, c.work, c.limit};
  restricted_prefix<MAXS>(sw, S);
  const double C = c.work / c.batch;
  const int n2 = 2 + sw.pre2[S];
#ifdef HPS_STATS
  if (lane == 0) {
    HPS_STAT(ST_N2, n2);
    int unc = 0;
    for (int r = 0; r < S; r++) unc += max(0, sw.kma[r] - sw.blo[r] + 1);
    HPS_STAT(ST_UNCERT, unc);
  }
#endif
  const float fC = (float)C;
  {  // unpinned stages in order, and the pinned stages' part of the filter bound
    float p0f = 0.0f;
    int base = 0;
#pragma unroll
    for (int slot = 0; slot < 2; slot++) {
      const int r = lane + 32 * slot;
      const bool unp = r < S && sw.kma[r] != sw.kmi[r];
      if (r < S && !unp) p0f += sw.fpr[r] * (float)sw.kmi[r];
      const unsigned m = __ballot_sync(0xffffffffu, unp);
      if (unp) sw.ulist[base + __popc(m & ((1u << lane) - 1u))] = (int8_t)r;
      base += __popc(m);
    }
    for (int o = 16; o; o >>= 1) p0f += __shfl_xor_sync(0xffffffffu, p0f, o);
    if (lane == 0) { sw.nu = base; sw.p0f = p0f; }
    __syncwarp();
  }
  int sp = 0;
  // per-candidate filter; survivors are compacted into sw.q and evaluated densely (a warp only
  // saves work when all 32 lanes skip, so skipping must be compacted). A warm-start candidate
  // may pass again; re-inserting it is harmless (same cost and tau).
  sp = 0;
  int qn = 0;
  const unsigned lt = (1u << lane) - 1u;
  const int rounds = (n2 + 31) >> 5;
  for (int jr = 0; jr < rounds; jr++) {
    const int i = jr * 32 + lane;
    double tau = 0.0;
    int gen = -1;
    bool keep = false;
    if (i < n2) {
      tau = cand_tau2<MAXS>(w, sw, i, sp, tau_lo, tau_hi, gen);
      keep = tau >= tau_lo && tau <= tau_hi;
      if (keep && gen >= 0) {   // cost >= C tau P(tau) (E >= tau at a certified breakpoint)
        const int g = gen >> 16, m = gen & 0xffff;
        const float tf = (float)tau;
        // g's class has count m; every other unpinned stage's count is >= its count at tau_hi
        // (at tau_b when tau <= tau_b) and >= the FP32 lower bound; pinned stages are exact
        const bool inb = tau <= sw.tb;
        float P = sw.p0f;
        for (int j = 0; j < sw.nu; j++) {
          const int r = sw.ulist[j];
          const int k = (sw.lead[r] == g) ? m
                        : max(inb ? (int)sw.kb[r] : sw.kmi[r], count_lb32_est(sw.est[r], tf));
          P += sw.fpr[r] * (float)k;
        }
        keep = !((double)(fC * tf * P) * (1.0 - 1e-5) > ub + 1e-15);
      }
    }
    const unsigned mk = __ballot_sync(0xffffffffu, keep);
    if (keep) { sw.cq->q[qn + __popc(mk & lt)] = tau; sw.cq->qg[qn + __popc(mk & lt)] = gen; }
    qn += __popc(mk);
    __syncwarp();
    if (qn >= 32) {
      const double t = sw.cq->q[qn - 32 + lane];
      const int tg = sw.cq->qg[qn - 32 + lane];
      HPS_STAT(ST_CANDS, 1);
      eval_insert<MAXS>(cs, w, sw, S, t, tg, buf);
      qn -= 32;
      ub = fmin(ub, warp_min(buf.mn));
      __syncwarp();
    }
  }
  if (qn > 0) {
    if (lane < qn) {
      const double t = sw.cq->q[lane];
      HPS_STAT(ST_CANDS, 1);
      eval_insert<MAXS>(cs, w, sw, S, t, sw.cq->qg[lane], buf);
    }
  }
  const double mf = warp_min(buf.mn);
  if (!(mf < inf)) return __longlong_as_double(0x7ff8000000000000LL);
  const double lim = mf + 1e-15;
  double bt;
  if (__any_sync(0xffffffffu, buf.overflow)) {  // rare: exact second pass with the final limit
    bt = overflow_pass<MAXS>(cs, w, sw, S, tau_lo, tau_hi, n2, lim);
  } else {
    bt = buf.best_tau(lim);
  }
  return warp_max(bt);
}

template <int MAXS, class W>
__device__ double phase_candidates_fast(const InstanceConsts& c, const DeviceTables& tb,
                                        const W& w, SweepSmem<MAXS>& sw, int S,
                                        double tau_lo, double tau_hi, int n_cand) {
  TieBuf buf;
  buf.init();
  __shared__ CandQueue fused_queue[32];   // (fused eval_kernel path only; <= 32 warps per block)
  if ((threadIdx.x & 31) == 0) sw.cq = &fused_queue[threadIdx.x >> 5];
  __syncwarp();
  const double ub = cand_prep<MAXS>(c, tb, w, sw, S, tau_lo, tau_hi, n_cand, buf);
  return cand_main<MAXS>(c, w, sw, S, tau_lo, tau_hi, ub, buf);
}

// Whole plan, fast path. Falls back to the literal path's pending marker for >4096 candidates.
template <int MAXS, class W>
__device__ void eval_plan_fast(const InstanceConsts& c, const DeviceTables& tb, W& w,
                               SweepSmem<MAXS>& sw, int d0, int d1, PlanOut& out) {
  out.ps = 0;
  out.gap = 0.0;
  double tau_lo, tau_hi;
  int n_cand;
#ifdef HPS_STATS
  const long long t0 = clock64();
#endif
  if (!phase_stages_bisect<MAXS, true>(c, tb, w, d0, d1, out, tau_lo, tau_hi, n_cand)) return;
  if (n_cand > kBpLimit) { out.status = kStPending; return; }
#ifdef HPS_STATS
  const long long t1 = clock64();
#endif
  const double tau = phase_candidates_fast<MAXS>(c, tb, w, sw, out.S, tau_lo, tau_hi, n_cand);
#ifdef HPS_STATS
  const long long t2 = clock64();
  if ((threadIdx.x & 31) == 0) { HPS_STAT(ST_CYC_A, t1 - t0); HPS_STAT(ST_CYC_B, t2 - t1); }
#endif
  if (tau != tau) {
    out.status = HPS_ST_NO_CANDIDATE; out.gap = 1.0;
    out.cost = c.penalty_scale * (1.0 + 1.0);
    return;
  }
#ifdef HPS_STATS
  const long long t3 = clock64();
#endif
  phase_final_fast<MAXS>(c, w, out.S, tau, out);
#ifdef HPS_STATS
  if ((threadIdx.x & 31) == 0) HPS_STAT(ST_CYC_C, clock64() - t3);
#endif
}

}  // namespace hps
