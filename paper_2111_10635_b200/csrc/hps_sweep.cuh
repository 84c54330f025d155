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
//  * _best_candidate (ls/provisioner.py:262-314): candidates round-robin over lanes; counts are
//    CERTIFIED arithmetic counts (reciprocal + rigorous error bound, count_cert) with the exact
//    table search as fallback; a warm start plus a rigorous lower bound (E >= tau at a certified
//    breakpoint, per-round exact counts at the round's largest tau, FP32 bounds of the top
//    stage) skips the candidates that cannot reach the minimum or its 1e-15 tie window;
//    evaluated candidates use the reference's exact sequential per_second sum and its two cost
//    divisions.
#pragma once
#include "hps_eval.cuh"

namespace hps {

#ifndef HPS_TOP
#define HPS_TOP 1
#endif
#ifndef HPS_ROUNDB
#define HPS_ROUNDB 0   // 1: per-round exact counts at the round's largest candidate in the bound (measured slower)
#endif
constexpr int kTop = HPS_TOP;   // unpinned stages bounded per candidate (count_lb32)

template <int MAXS>
struct SweepSmem {   // per-warp, per-plan constants of the fast candidate phase (broadcast reads)
  double pr[MAXS];   // price per second of stage r's type
  double etp[MAXS];  // exact et at the pinned count (kmin == kmax), else unused
  float fpr[MAXS];   // pr as FP32 (bounds only)
  int32_t kmi[MAXS]; // count at tau_hi (= kmin)
  int32_t kma[MAXS]; // count at tau_lo (= kmax)
  int32_t kr[MAXS];  // exact counts at the current round's largest candidate (bounds only)

  int32_t top[kTop > 0 ? kTop : 1]; // unpinned stages with the largest price-weighted count span (-1: none)
  int32_t dom[MAXS]; // side_dominance over [tau_lo, tau_hi]: 1 oct, 2 odt, 0 both
  int8_t lead[MAXS]; // class leader of stage r (stages of one class have identical counts)
  int32_t gex[MAXS]; // leader r: count_r(et_r(m)) == m for m <= gex[r] (tb.gex), else 0
  double q[64];      // survivors of the lower-bound filter, evaluated 32 at a time
  int32_t qg[64];    // their generator: (leader << 16) | m, or -1 (tau_lo / tau_hi)
};

// FP32 estimate of count(tau) of unpinned stage r, clamped to [kmin, kmax]. Only a seed: the
// threshold table confirms or corrects it (count_verify), so it never affects a result.
template <int MAXS>
__device__ __forceinline__ int count_est(const WarpSmem<MAXS>& w, const SweepSmem<MAXS>& sw, int r, float tf) {
  const StageEntry& s = w.st[r];
  const int dom = sw.dom[r];
  float q = 1.0f;
#pragma unroll
  for (int side = 0; side < 2; side++) {
    if (dom == 2 - side) continue;
    const float rb = side ? s.f_rbd : s.f_rbo;
    const float frac = side ? s.f_beta : s.f_alpha;
    if (rb == 0.0f || frac == 0.0f) continue;
    const float h = tf * rb - (side ? s.f_omb : s.f_oma);
    q = (h > 0.0f) ? fmaxf(q, frac * rcp_approx_f32(h)) : 3.0e38f;
  }
  const int lo = sw.kmi[r], hi = sw.kma[r];
  const int k = (q < 2.0e9f) ? (int)ceilf(q) : hi;
  return min(max(k, lo), hi);
}

// read-only table loads: {et(k), theta(k - 1)} in one 16-byte load, theta(k) separately
__device__ __forceinline__ double2 te_pair(const TEPair* row, int k) {
  return __ldg(reinterpret_cast<const double2*>(row + (k - 1)));
}
__device__ __forceinline__ double te_theta(const TEPair* row, int k) { return __ldg(&row[k].th); }

// Exact count(tau) for tau in [tau_lo, tau_hi] (count in [kmin, kmax]) given the seed k and the
// loads pk = {et(k), theta(k - 1)}, thk = theta(k): k is the count iff theta(k) <= tau <
// theta(k - 1) (count(tau) = min{m : theta(m) <= tau}); otherwise the exact galloping table search
// from k decides. Returns the count and et at it.
template <int MAXS>
__device__ __forceinline__ int count_verify(const WarpSmem<MAXS>& w, const SweepSmem<MAXS>& sw, int r,
                                            double tau, int k, double2 pk, double thk, double& et) {
  if (thk <= tau && tau < pk.y) {
    et = pk.x;
    return k;
  }
  const TEPair* row = w.row[r];
  k = count_tab(row, tau, sw.kmi[r], sw.kma[r], k);
  et = __ldg(&row[k - 1].et);
  return k;
}

struct CostScalars {  // the four job constants the cost needs (no parameter-struct copies)
  double bo, batch, work, limit;
};

// exact cost of candidate tau (numpy column of _best_candidate, ls/provisioner.py:286-308);
// one out-of-line copy shared by every call site.
// gen = (g << 16) | m when tau = et_g(m) and tb.gex certifies count_g(tau) == m: every stage of
// g's class then has count m and et == tau exactly (the breakpoint value itself).
template <int MAXS>
__device__ __noinline__ double cost_exact(const CostScalars cs, const WarpSmem<MAXS>& w,
                                          const SweepSmem<MAXS>& sw, int S, double tau, int gen) {
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

// candidate i: tau_lo, tau_hi, then the breakpoints et_sp(m) of the class leaders; gen as in
// cost_exact (-1 unless the leader's breakpoints are certified)
template <int MAXS>
__device__ __forceinline__ double cand_tau(const WarpSmem<MAXS>& w, const SweepSmem<MAXS>& sw, int i,
                                           int& sp, double tau_lo, double tau_hi, int& gen) {
  gen = -1;
  if (i < 2) return (i == 0) ? tau_lo : tau_hi;
  const int j = i - 2;
  while (w.pre[sp + 1] <= j) sp++;
  const int m = (int)w.kmin[sp] + (j - w.pre[sp]);
  if (m <= sw.gex[sp]) gen = (sp << 16) | m;
  return __ldg(&w.row[sp][m - 1].et);
}

// _best_candidate: round-robin candidates over lanes. A warm-start round evaluates 32 candidates
// spread over the candidate range exactly; every other candidate is evaluated exactly only when a
// rigorous lower bound on its cost does not exceed the best cost so far + 1e-15. A skipped
// candidate therefore costs more than the final minimum + 1e-15: neither the minimum nor a tie.
//
// The bound of a certified breakpoint tau = et_g(m) (count_g(tau) == m, tb.gex): cost =
// (work/batch) E P with E >= et_g(m) = tau and P = sum_r pr_r count_r(tau), where
//   * count_g(tau) = m;
//   * count_r(tau) >= count_r(tau_max) for every r, tau_max = the round's largest candidate
//     (counts are non-increasing in tau): exact counts at tau_max are computed once per round,
//     one stage per lane, and the warp sums them;
//   * the top stage(s) also get a per-candidate FP32 lower bound (count_lb32).
// All FP32 arithmetic of the bound is covered by a 1e-5 relative slack. tau_lo, tau_hi and
// uncertified breakpoints are always evaluated.
template <int MAXS>
__device__ double phase_candidates_fast(const InstanceConsts& c, const DeviceTables& tb,
                                        const WarpSmem<MAXS>& w, SweepSmem<MAXS>& sw, int S,
                                        double tau_lo, double tau_hi, int n_cand) {
  const int lane = threadIdx.x & 31;
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  for (int r = lane; r < S; r += 32) {
    const bool pinned = (w.kmax[r] == w.kmin[r]);
    sw.pr[r] = c.price_s[w.st[r].type];
    sw.fpr[r] = (float)sw.pr[r];
    sw.kmi[r] = (int)w.kmin[r];
    sw.kma[r] = (int)w.kmax[r];
    sw.etp[r] = pinned ? w.row[r][(int)w.kmin[r] - 1].et : 0.0;
    sw.dom[r] = pinned ? 0 : side_dominance(w.st[r], tau_lo, tau_hi, c.bo);
    int ld = 0;  // first stage of r's class
    while (w.cls[ld] != w.cls[r]) ld++;
    sw.lead[r] = (int8_t)ld;
    sw.gex[r] = (ld == r && !pinned) ? __ldg(tb.gex + w.ent[r]) : 0;
  }
  __syncwarp();
  if (lane == 0) {
    int t[kTop > 0 ? kTop : 1];
    double v[kTop > 0 ? kTop : 1];
#pragma unroll
    for (int q = 0; q < kTop; q++) { t[q] = -1; v[q] = -1.0; }
    for (int r = 0; r < S; r++) {
      if (w.kmax[r] == w.kmin[r]) continue;
      double vv = sw.pr[r] * (w.kmax[r] - w.kmin[r]);
      int tt = r;
#pragma unroll
      for (int q = 0; q < kTop; q++) {   // insertion into the descending top list
        if (vv > v[q]) {
          const double v2 = v[q]; const int t2 = t[q];
          v[q] = vv; t[q] = tt; vv = v2; tt = t2;
        }
      }
    }
#pragma unroll
    for (int q = 0; q < kTop; q++) sw.top[q] = t[q];

    HPS_STAT(ST_NCAND, n_cand);
    HPS_STAT(ST_PLANS_FAST, 1);
    HPS_STAT(ST_STAGES, S);
  }
  __syncwarp();
  const CostScalars cs{c.bo, c.batch, c.work, c.limit};
  TieBuf buf;
  buf.init();
  const int rounds = (n_cand + 31) >> 5;
  int sp = 0;
  {  // warm start: one round of 32 candidates spread evenly over the candidate range
    const int i = (int)(((long long)lane * n_cand) >> 5);
    int gen;
    const double tau = cand_tau<MAXS>(w, sw, i, sp, tau_lo, tau_hi, gen);
    if (tau >= tau_lo && tau <= tau_hi) {
      HPS_STAT(ST_CANDS, 1);
      buf.insert(cost_exact<MAXS>(cs, w, sw, S, tau, gen), tau);
    }
  }
  double ub = warp_min(buf.mn);
  const float fC = (float)(c.work / c.batch);
#if !HPS_ROUNDB
  float pl0 = 0.0f;  // counts at tau_hi
  for (int r = lane; r < S; r += 32) {
    sw.kr[r] = sw.kmi[r];
    pl0 += sw.fpr[r] * (float)sw.kmi[r];
  }
  for (int o = 16; o; o >>= 1) pl0 += __shfl_xor_sync(0xffffffffu, pl0, o);
  __syncwarp();
#endif
  int top[kTop > 0 ? kTop : 1];
#pragma unroll
  for (int q = 0; q < kTop; q++) top[q] = sw.top[q];
  // every candidate: lower-bound filter; survivors are compacted into sw.q and evaluated
  // densely (a warp only saves work when all 32 lanes skip, so skipping must be compacted).
  // A warm-start candidate may pass again; re-inserting it is harmless (same cost and tau).
  sp = 0;
  int qn = 0;
  const unsigned lt = (1u << lane) - 1u;
  for (int jr = 0; jr < rounds; jr++) {
    const int i = jr * 32 + lane;
    double tau = 0.0;
    int gen = -1;
    bool inr = false;
    if (i < n_cand) {
      tau = cand_tau<MAXS>(w, sw, i, sp, tau_lo, tau_hi, gen);
      inr = tau >= tau_lo && tau <= tau_hi;
    }
    const double tmax = warp_max(inr ? tau : -inf);
    if (!(tmax > -inf)) continue;  // warp-uniform
#if HPS_ROUNDB
    float pl = 0.0f;
    for (int r = lane; r < S; r += 32) {
      int k = sw.kmi[r];
      double et_unused;
      if (sw.kma[r] != k) {
        const int k0 = count_est<MAXS>(w, sw, r, (float)tmax);
        k = count_verify<MAXS>(w, sw, r, tmax, k0, te_pair(w.row[r], k0), te_theta(w.row[r], k0), et_unused);
      }
      sw.kr[r] = k;
      pl += sw.fpr[r] * (float)k;
    }
    for (int o = 16; o; o >>= 1) pl += __shfl_xor_sync(0xffffffffu, pl, o);
    __syncwarp();
#else
    const float pl = pl0;
#endif
    bool keep = inr;
    if (inr && gen >= 0) {
      const int g = gen >> 16, m = gen & 0xffff;
      const float tf = (float)tau;
      float P = pl + sw.fpr[g] * (float)(m - sw.kr[g]);
#pragma unroll
      for (int q = 0; q < kTop; q++) {
        const int r = top[q];
        if (r < 0 || r == g) continue;
        const int d = count_lb32(w.st[r], tf, sw.dom[r]) - sw.kr[r];
        if (d > 0) P += sw.fpr[r] * (float)d;
      }
      keep = !((double)(fC * tf * P) * (1.0 - 1e-5) > ub + 1e-15);
    }
    const unsigned mk = __ballot_sync(0xffffffffu, keep);
    if (keep) { sw.q[qn + __popc(mk & lt)] = tau; sw.qg[qn + __popc(mk & lt)] = gen; }
    qn += __popc(mk);
    __syncwarp();
    if (qn >= 32) {
      const double t = sw.q[qn - 32 + lane];
      const int tg = sw.qg[qn - 32 + lane];
      HPS_STAT(ST_CANDS, 1);
      buf.insert(cost_exact<MAXS>(cs, w, sw, S, t, tg), t);
      qn -= 32;
      ub = fmin(ub, warp_min(buf.mn));
      __syncwarp();
    }
  }
  if (qn > 0) {
    if (lane < qn) {
      const double t = sw.q[lane];
      HPS_STAT(ST_CANDS, 1);
      buf.insert(cost_exact<MAXS>(cs, w, sw, S, t, sw.qg[lane]), t);
    }
  }
  const double mf = warp_min(buf.mn);
  if (!(mf < inf)) return __longlong_as_double(0x7ff8000000000000LL);
  const double lim = mf + 1e-15;
  double bt;
  if (__any_sync(0xffffffffu, buf.overflow)) {  // rare: exact second pass with the final limit
    bt = -inf;
    sp = 0;
    for (int i = lane; i < n_cand; i += 32) {
      int gen;
      const double tau = cand_tau<MAXS>(w, sw, i, sp, tau_lo, tau_hi, gen);
      if (!(tau >= tau_lo && tau <= tau_hi) || !(tau > bt)) continue;
      if (cost_exact<MAXS>(cs, w, sw, S, tau, gen) <= lim) bt = tau;
    }
  } else {
    bt = buf.best_tau(lim);
  }
  return warp_max(bt);
}

// Whole plan, fast path. Falls back to the literal path's pending marker for >4096 candidates.
template <int MAXS>
__device__ void eval_plan_fast(const InstanceConsts& c, const DeviceTables& tb, WarpSmem<MAXS>& w,
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
  phase_final<MAXS, true>(c, tb, w, out.S, tau, out);
#ifdef HPS_STATS
  if ((threadIdx.x & 31) == 0) HPS_STAT(ST_CYC_C, clock64() - t3);
#endif
}

}  // namespace hps
