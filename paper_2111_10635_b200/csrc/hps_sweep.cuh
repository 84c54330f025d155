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
//    table search as fallback; a warm start plus a rigorous two-stage lower bound skips the
//    candidates that cannot reach the minimum or its 1e-15 tie window; evaluated candidates use
//    the reference's exact sequential per_second sum and its two cost divisions.
#pragma once
#include "hps_eval.cuh"

namespace hps {

#ifndef HPS_TOP
#define HPS_TOP 2
#endif
constexpr int kTop = HPS_TOP;   // unpinned stages bounded individually by cost_bound

template <int MAXS>
struct SweepSmem {   // per-warp, per-plan constants of the fast candidate phase (broadcast reads)
  double pr[MAXS];   // price per second of stage r's type
  double etp[MAXS];  // exact et at the pinned count (kmin == kmax), else unused
  double pmin_rest;  // sum over non-top stages of price * kmin, rounded down by 1e-13
  double ep_max;     // max over pinned stages of their exact et
  int32_t top[kTop]; // unpinned stages with the largest price-weighted count span (-1: none)
  int32_t dom[MAXS]; // side_dominance over [tau_lo, tau_hi]: 1 oct, 2 odt, 0 both
  double q[64];      // survivors of the lower-bound filter, evaluated 32 at a time
};

// exact count at tau in [tau_lo, tau_hi] (count in [kmin, kmax]): certified (one side when it
// provably dominates), table fallback
template <int MAXS>
__device__ __forceinline__ int count_fast(double bo, const WarpSmem<MAXS>& w, int r, double tau,
                                          int dom) {
  const StageEntry& s = w.st[r];
  const int k = (dom == 1)   ? count_cert1(s.alpha, s.oma, s.rwo, tau, bo)
                : (dom == 2) ? count_cert1(s.beta, s.omb, s.rwd, tau, bo)
                             : count_cert(s, tau, bo);
  if (k > 0) return k;
  return count_tab(w.row[r], tau, (int)w.kmin[r], (int)w.kmax[r], est_count(w.st[r], tau));
}

struct CostScalars {  // the four job constants the cost needs (no parameter-struct copies)
  double bo, batch, work, limit;
};

// exact cost of candidate tau (numpy column of _best_candidate, ls/provisioner.py:286-308);
// one out-of-line copy shared by every call site
template <int MAXS>
__device__ __noinline__ double cost_exact(const CostScalars cs, const WarpSmem<MAXS>& w,
                                          const SweepSmem<MAXS>& sw, int S, double tau) {
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  double P = 0.0, E = 0.0;
  for (int r = 0; r < S; r++) {
    double et;
    int k;
    if (w.kmax[r] == w.kmin[r]) {
      k = (int)w.kmin[r];
      et = sw.etp[r];
    } else {
      k = count_fast<MAXS>(cs.bo, w, r, tau, sw.dom[r]);
      et = w.row[r][k - 1].et;
    }
    E = (r == 0) ? et : fmax(E, et);
    const double term = sw.pr[r] * (double)k;
    P = (r == 0) ? term : P + term;
  }
  const double thr = (E > 0) ? cs.batch / E : inf;
  if (!(thr > cs.limit)) return inf;
  return cs.work / thr * P;
}

// rigorous lower bound from FP32 one-sided count bounds of the two top stages and count(tau_hi)
// for the others: P >= sum price k_lo, E >= max(pinned et, et(k_hi) of the top stages).
// Everything FP32 carries a 1e-5 relative slack, so the bound never exceeds the exact cost.
template <int MAXS>
__device__ __forceinline__ double cost_bound(const CostScalars cs, const WarpSmem<MAXS>& w,
                                             const SweepSmem<MAXS>& sw, double tau) {
  const float tf = (float)tau;
  float P = (float)sw.pmin_rest, E = (float)sw.ep_max;
#pragma unroll
  for (int q = 0; q < kTop; q++) {
    const int r = sw.top[q];
    if (r < 0) continue;
    int kl, ku;
    count_bounds32(w.st[r], tf, sw.dom[r], kl, ku);
    const int lo = (int)w.kmin[r], hi = (int)w.kmax[r];
    kl = max(kl, lo);
    P += (float)sw.pr[r] * (float)kl;
    if (ku > 0) {
      const StageEntry& st = w.st[r];
      const float k = (float)min(ku, hi);
      const float rk = rcp_approx_f32(k);
      E = fmaxf(E, fmaxf(st.f_coct * (st.f_oma + st.f_alpha * rk), st.f_codt * (st.f_omb + st.f_beta * rk)));
    }
  }
  return (double)((float)(cs.work / cs.batch) * E * P) * (1.0 - 1e-5);
}

template <int MAXS>
__device__ __forceinline__ double cand_tau(const WarpSmem<MAXS>& w, int i, int& sp, double tau_lo,
                                           double tau_hi) {
  if (i < 2) return (i == 0) ? tau_lo : tau_hi;
  const int j = i - 2;
  while (w.pre[sp + 1] <= j) sp++;
  const int m = (int)w.kmin[sp] + (j - w.pre[sp]);
  return w.row[sp][m - 1].et;
}

// _best_candidate: round-robin candidates over lanes. A warm-start pass evaluates every 8th
// round exactly; the remaining candidates are evaluated exactly only when a rigorous lower bound
// (two top stages exact) does not exceed the best cost so far + 1e-15. A skipped candidate
// therefore costs more than the final minimum + 1e-15: it is neither the minimum nor a tie.
template <int MAXS>
__device__ double phase_candidates_fast(const InstanceConsts& c, const DeviceTables& tb,
                                        const WarpSmem<MAXS>& w, SweepSmem<MAXS>& sw, int S,
                                        double tau_lo, double tau_hi, int n_cand) {
  const int lane = threadIdx.x & 31;
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  for (int r = lane; r < S; r += 32) {
    sw.pr[r] = c.price_s[w.st[r].type];
    sw.etp[r] = (w.kmax[r] == w.kmin[r]) ? w.row[r][(int)w.kmin[r] - 1].et : 0.0;
    sw.dom[r] = (w.kmax[r] == w.kmin[r]) ? 0 : side_dominance(w.st[r], tau_lo, tau_hi, c.bo);
  }
  __syncwarp();
  if (lane == 0) {
    int t[kTop];
    double v[kTop];
#pragma unroll
    for (int q = 0; q < kTop; q++) { t[q] = -1; v[q] = -1.0; }
    double ep = 0.0;
    for (int r = 0; r < S; r++) {
      if (w.kmax[r] == w.kmin[r]) { ep = fmax(ep, sw.etp[r]); continue; }
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
    double pm = 0.0;
    for (int r = 0; r < S; r++) {
      bool in_top = false;
#pragma unroll
      for (int q = 0; q < kTop; q++) in_top |= (t[q] == r);
      if (!in_top) pm += sw.pr[r] * w.kmin[r];
    }
#pragma unroll
    for (int q = 0; q < kTop; q++) sw.top[q] = t[q];
    sw.pmin_rest = pm * (1.0 - 1e-13);
    sw.ep_max = ep;
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
    const double tau = cand_tau<MAXS>(w, i, sp, tau_lo, tau_hi);
    if (tau >= tau_lo && tau <= tau_hi) {
      HPS_STAT(ST_CANDS, 1);
      buf.insert(cost_exact<MAXS>(cs, w, sw, S, tau), tau);
    }
  }
  double ub = warp_min(buf.mn);
  // every candidate: lower-bound filter; survivors are compacted into sw.q and evaluated
  // densely (a warp only saves work when all 32 lanes skip, so skipping must be compacted).
  // A warm-start candidate may pass again; re-inserting it is harmless (same cost and tau).
  sp = 0;
  int qn = 0;
  const unsigned lt = (1u << lane) - 1u;
  for (int jr = 0; jr < rounds; jr++) {
    const int i = jr * 32 + lane;
    bool keep = false;
    double tau = 0.0;
    if (i < n_cand) {
      tau = cand_tau<MAXS>(w, i, sp, tau_lo, tau_hi);
      keep = tau >= tau_lo && tau <= tau_hi && !(cost_bound<MAXS>(cs, w, sw, tau) > ub + 1e-15);
    }
    const unsigned mk = __ballot_sync(0xffffffffu, keep);
    if (keep) sw.q[qn + __popc(mk & lt)] = tau;
    qn += __popc(mk);
    __syncwarp();
    if (qn >= 32) {
      const double t = sw.q[qn - 32 + lane];
      HPS_STAT(ST_CANDS, 1);
      buf.insert(cost_exact<MAXS>(cs, w, sw, S, t), t);
      qn -= 32;
      ub = fmin(ub, warp_min(buf.mn));
      __syncwarp();
    }
  }
  if (qn > 0) {
    if (lane < qn) {
      const double t = sw.q[lane];
      HPS_STAT(ST_CANDS, 1);
      buf.insert(cost_exact<MAXS>(cs, w, sw, S, t), t);
    }
  }
  const double mf = warp_min(buf.mn);
  if (!(mf < inf)) return __longlong_as_double(0x7ff8000000000000LL);
  const double lim = mf + 1e-15;
#ifdef HPS_STATS
  {  // diagnostics: survivors the filter would keep with the final minimum as its bound
    int sp2 = 0, ideal = 0, unp = 0;
    for (int i = lane; i < n_cand; i += 32) {
      const double tau = cand_tau<MAXS>(w, i, sp2, tau_lo, tau_hi);
      if (tau >= tau_lo && tau <= tau_hi && !(cost_bound<MAXS>(cs, w, sw, tau) > lim)) ideal++;
    }
    for (int r = lane; r < S; r += 32) unp += (w.kmax[r] != w.kmin[r]);
    HPS_STAT(ST_CHUNKS, ideal);
    HPS_STAT(ST_UNPINNED, unp);
  }
#endif
  double bt;
  if (__any_sync(0xffffffffu, buf.overflow)) {  // rare: exact second pass with the final limit
    bt = -inf;
    sp = 0;
    for (int i = lane; i < n_cand; i += 32) {
      const double tau = cand_tau<MAXS>(w, i, sp, tau_lo, tau_hi);
      if (!(tau >= tau_lo && tau <= tau_hi) || !(tau > bt)) continue;
      if (!(cost_bound<MAXS>(cs, w, sw, tau) > lim) && cost_exact<MAXS>(cs, w, sw, S, tau) <= lim) bt = tau;
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
