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
//  * _best_candidate (ls/provisioner.py:262-314): candidates are spread round-robin over the
//    lanes; each unpinned stage's count at a candidate is a CERTIFIED arithmetic count
//    (reciprocal + rigorous error bound, count_cert) with the exact table search as fallback;
//    pinned stages (count(tau_hi) == count(tau_lo)) cost nothing; per_second is the reference's
//    exact sequential sum and the cost the reference's two divisions.
#pragma once
#include "hps_eval.cuh"

namespace hps {

constexpr int kTopK = 3;

template <int MAXS>
struct SweepSmem {   // per-warp, per-plan constants of the fast candidate phase (broadcast reads)
  double pr[MAXS];   // price per second of stage r's type
  double etp[MAXS];  // exact et at the pinned count (kmin == kmax), else unused
  double pmin_rest;  // sum of price*kmin over the stages outside the top-K set
  double ep_max;     // max over pinned stages of their exact et
  int32_t top[kTopK];  // unpinned stages with the largest price*(kmax-kmin) (-1: none)
  int32_t ntop;
};

// exact count of stage r at tau in [tau_lo, tau_hi]: certified arithmetic, exact table fallback
template <int MAXS>
__device__ __noinline__ int count_in_range(const InstanceConsts& c, const DeviceTables& tb,
                                              const WarpSmem<MAXS>& w, int r, double tau) {
  const StageEntry& st = w.st[r];
  const int k = count_cert(st, tau, c.bo);
  if (k > 0) return k;
  const TEPair* row = te_row(c, tb, st.type, w.ent[r]);
  return count_tab(row, tau, (int)w.kmin[r], (int)w.kmax[r], est_count(st, tau));
}

// Rigorous lower bound on the cost of candidate tau from stage s (count m): exact counts for s
// and the top-K stages, count(tau_hi) for the rest; E >= their et, P >= their price sum.
template <int MAXS>
__device__ __noinline__ double cost_lower_bound(const InstanceConsts& c, const DeviceTables& tb,
                                                   const WarpSmem<MAXS>& w, const SweepSmem<MAXS>& sw,
                                                   int s, double tau) {
  double E = sw.ep_max, P = sw.pmin_rest;
  bool s_in_top = false;
  for (int q = 0; q < sw.ntop; q++) {
    const int r = sw.top[q];
    s_in_top |= (r == s);
    const int k = count_in_range<MAXS>(c, tb, w, r, tau);
    P += sw.pr[r] * (double)k;
    E = fmax(E, et_approx(w.st[r], (double)k));
  }
  if (s >= 0 && !s_in_top && w.kmax[s] != w.kmin[s]) {
    const int k = count_in_range<MAXS>(c, tb, w, s, tau);
    P += sw.pr[s] * ((double)k - w.kmin[s]);
    E = fmax(E, et_approx(w.st[s], (double)k));
  }
  // cost_ref = fl(fl(work / fl(batch / E)) * P_seq) >= (work/batch) E P (1 - (2S + 16) u)
  return c.work / c.batch * E * P * (1.0 - 1e-13);
}

// cost of candidate tau (numpy column of _best_candidate, ls/provisioner.py:286-308): exact
// counts, exact sequential per_second, exact E = max_r et_r(k_r) (approximate et values pick the
// maximiser; every stage within the approximation band is resolved exactly from the TE table).
template <int MAXS>
__device__ __noinline__ double cost_fast(const InstanceConsts& c, const DeviceTables& tb,
                                            const WarpSmem<MAXS>& w, const SweepSmem<MAXS>& sw,
                                            int S, double tau) {
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  double P = 0.0, best = -1.0, second = -1.0;
  int kb = 0, rb = -1;
  for (int r = 0; r < S; r++) {
    const double kmin = w.kmin[r];
    double k, ea;
    if (w.kmax[r] == kmin) {
      k = kmin;
      ea = sw.etp[r];
    } else {
      k = (double)count_in_range<MAXS>(c, tb, w, r, tau);
      ea = et_approx(w.st[r], k);
    }
    if (ea > best) { second = best; best = ea; rb = r; kb = (int)k; }
    else if (ea > second) second = ea;
    const double term = sw.pr[r] * k;
    P = (r == 0) ? term : P + term;
  }
  double E;
  if (second >= best * (1.0 - 1e-14)) {  // near-tie between stages: resolve all candidates
    E = 0.0;
    for (int r = 0; r < S; r++) {
      double k = w.kmin[r];
      if (w.kmax[r] != k) k = (double)count_in_range<MAXS>(c, tb, w, r, tau);
      E = fmax(E, te_row(c, tb, w.st[r].type, w.ent[r])[(int)k - 1].et);
    }
  } else {
    E = (w.kmax[rb] == w.kmin[rb]) ? sw.etp[rb] : te_row(c, tb, w.st[rb].type, w.ent[rb])[kb - 1].et;
  }
  const double thr = (E > 0) ? c.batch / E : inf;
  if (!(thr > c.limit)) return inf;
  return c.work / thr * P;
}

template <int MAXS>
__device__ __forceinline__ double cand_tau(const InstanceConsts& c, const DeviceTables& tb,
                                           const WarpSmem<MAXS>& w, int i, double tau_lo,
                                           double tau_hi, int& sp, int& s_out) {
  if (i < 2) { s_out = -1; return (i == 0) ? tau_lo : tau_hi; }
  const int j = i - 2;
  while (w.pre[sp + 1] <= j) sp++;
  s_out = sp;
  const int m = (int)w.kmin[sp] + (j - w.pre[sp]);
  return te_row(c, tb, w.st[sp].type, w.ent[sp])[m - 1].et;
}

template <int MAXS>
__device__ double phase_candidates_fast(const InstanceConsts& c, const DeviceTables& tb,
                                        const WarpSmem<MAXS>& w, SweepSmem<MAXS>& sw, int S,
                                        double tau_lo, double tau_hi, int n_cand) {
  const int lane = threadIdx.x & 31;
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  for (int r = lane; r < S; r += 32) {
    sw.pr[r] = c.price_s[w.st[r].type];
    sw.etp[r] = (w.kmax[r] == w.kmin[r])
                    ? te_row(c, tb, w.st[r].type, w.ent[r])[(int)w.kmin[r] - 1].et : 0.0;
  }
  __syncwarp();
  if (lane == 0) {  // top-K unpinned stages by price-weighted count span, and the rest's floor
    int top[kTopK];
    double wt[kTopK];
    int nt = 0;
    double ep = 0.0;
    for (int r = 0; r < S; r++) {
      if (w.kmax[r] == w.kmin[r]) { ep = fmax(ep, sw.etp[r]); continue; }
      const double v = sw.pr[r] * (w.kmax[r] - w.kmin[r]);
      int pos = nt < kTopK ? nt : kTopK;
      while (pos > 0 && wt[pos - 1] < v) { if (pos < kTopK) { wt[pos] = wt[pos - 1]; top[pos] = top[pos - 1]; } pos--; }
      if (pos < kTopK) { wt[pos] = v; top[pos] = r; if (nt < kTopK) nt++; }
    }
    double pm = 0.0;
    for (int r = 0; r < S; r++) {
      bool in = false;
      for (int q = 0; q < nt; q++) in |= (top[q] == r);
      if (!in) pm += sw.pr[r] * w.kmin[r];
    }
    for (int q = 0; q < kTopK; q++) sw.top[q] = q < nt ? top[q] : -1;
    sw.ntop = nt;
    sw.pmin_rest = pm * (1.0 - 1e-13);
    sw.ep_max = ep;
  }
  __syncwarp();
  TieBuf buf;
  buf.init();
  const int rounds = (n_cand + 31) >> 5;
  // warm start: every 8th round of candidates, exactly
  int sp = 0, s_of;
  for (int jr = 0; jr < rounds; jr += 8) {
    const int i = jr * 32 + lane;
    if (i >= n_cand) continue;
    const double tau = cand_tau<MAXS>(c, tb, w, i, tau_lo, tau_hi, sp, s_of);
    if (!(tau >= tau_lo && tau <= tau_hi)) continue;
    buf.insert(cost_fast<MAXS>(c, tb, w, sw, S, tau), tau);
  }
  double ub = warp_min(buf.mn);
  // remaining candidates: full evaluation only when the lower bound can reach ub + 1e-15
  sp = 0;
  for (int jr = 0; jr < rounds; jr++) {
    if ((jr & 7) == 0) continue;
    const int i = jr * 32 + lane;
    if (i < n_cand) {
      const double tau = cand_tau<MAXS>(c, tb, w, i, tau_lo, tau_hi, sp, s_of);
      if (tau >= tau_lo && tau <= tau_hi) {
        const double lim = ub + 1e-15;
        if (!(cost_lower_bound<MAXS>(c, tb, w, sw, s_of, tau) > lim))
          buf.insert(cost_fast<MAXS>(c, tb, w, sw, S, tau), tau);
      }
    }
    ub = fmin(ub, warp_min(buf.mn));
  }
  const double mf = warp_min(buf.mn);
  if (!(mf < inf)) return __longlong_as_double(0x7ff8000000000000LL);
  const double lim = mf + 1e-15;
  double bt;
  if (__any_sync(0xffffffffu, buf.overflow)) {  // rare: exact second pass with the final limit
    bt = -inf;
    sp = 0;
    for (int i = lane; i < n_cand; i += 32) {
      const double tau = cand_tau<MAXS>(c, tb, w, i, tau_lo, tau_hi, sp, s_of);
      if (!(tau >= tau_lo && tau <= tau_hi)) continue;
      if (tau > bt && !(cost_lower_bound<MAXS>(c, tb, w, sw, s_of, tau) > lim) &&
          cost_fast<MAXS>(c, tb, w, sw, S, tau) <= lim)
        bt = tau;
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
  if (!phase_stages_bisect<MAXS, true>(c, tb, w, d0, d1, out, tau_lo, tau_hi, n_cand)) return;
  if (n_cand > kBpLimit) { out.status = kStPending; return; }
  const double tau = phase_candidates_fast<MAXS>(c, tb, w, sw, out.S, tau_lo, tau_hi, n_cand);
  if (tau != tau) {
    out.status = HPS_ST_NO_CANDIDATE; out.gap = 1.0;
    out.cost = c.penalty_scale * (1.0 + 1.0);
    return;
  }
  phase_final<MAXS, true>(c, tb, w, out.S, tau, out);
}

}  // namespace hps
