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
//  * _best_candidate (ls/provisioner.py:262-314): lanes own tau-intervals (quantiles of a
//    warp-sorted sample of 32 candidates); each lane merges every leader stage's breakpoint
//    stream inside its interval in increasing tau, so each threshold is crossed once, keeps
//    every stage's exact count and next threshold, and per candidate does the reference's
//    exact sequential per_second sum and cost division.
#pragma once
#include "hps_eval.cuh"

namespace hps {

template <int MAXS>
struct SweepSmem {   // per-warp state of the fast path, next to WarpSmem
  double pr[MAXS];               // price per second of stage r's type
  double nt[MAXS][kWarp];        // per lane: tau at which stage r's count drops next
  double hd[MAXS][kWarp];        // per lane: tau of stage r's next breakpoint candidate (+inf: none)
  uint16_t kk[MAXS][kWarp];      // per lane: stage r's count at the lane's current tau
  uint16_t mp[MAXS][kWarp];      // per lane: count m whose breakpoint is hd[r]
  // counts fit 16 bits: the fast path is only enabled when every quota <= 16384
};

// tau of candidate index i of the implicit list {tau_lo, tau_hi, leaders' breakpoints}
template <int MAXS>
__device__ __forceinline__ double candidate_tau(const InstanceConsts& c, const DeviceTables& tb,
                                                const WarpSmem<MAXS>& w, int S, int i,
                                                double tau_lo, double tau_hi) {
  if (i == 0) return tau_lo;
  if (i == 1) return tau_hi;
  const int j = i - 2;
  int s = 0;
  while (w.pre[s + 1] <= j) s++;
  const double m = w.kmin[s] + (double)(j - w.pre[s]);
  return te_row(c, tb, w.st[s].type, w.ent[s])[(int)m - 1].et;
}

// Visit the candidates with tau in this lane's interval [b_lo, b_hi), in increasing tau (a merge
// of every leader stage's breakpoint stream), maintaining every stage's exact count.
// MODE 0: feed the tie buffer. MODE 1: return the largest tau with cost <= lim.
template <int MAXS, int MODE>
__device__ double sweep_lane(const InstanceConsts& c, const DeviceTables& tb, const WarpSmem<MAXS>& w,
                             SweepSmem<MAXS>& sw, int S, double tau_lo, double tau_hi,
                             double b_lo, double b_hi, TieBuf& buf, double lim) {
  const int lane = threadIdx.x & 31;
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  double best_tau = -inf;
  // heads: for each leader stage, the largest m in [kmin, kmax] with et(m) >= b_lo
  double first = inf;
  int fs = -1;
  for (int r = 0; r < S; r++) {
    double h = inf;
    int mm = 0;
    const int lo = (int)w.kmin[r], hi = (int)w.kmax[r];
    if (w.pre[r + 1] > w.pre[r]) {  // a class leader whose breakpoints are candidates
      const TEPair* row = te_row(c, tb, w.st[r].type, w.ent[r]);
      const double x = fmax(b_lo, tau_lo);
      if (row[lo - 1].et >= x) {  // some m has et(m) >= x; find the largest (et non-increasing in m)
        int a = lo, b = hi + 1;   // et(a) >= x, et(b) < x or b out of range
        while (b - a > 1) { const int md = (a + b) >> 1; if (row[md - 1].et >= x) a = md; else b = md; }
        const double e = row[a - 1].et;
        if (e < b_hi && e <= tau_hi) { h = e; mm = a; }
      }
    }
    sw.hd[r][lane] = h;
    sw.mp[r][lane] = (uint16_t)mm;
    if (h < first) { first = h; fs = r; }
  }
  const bool has_lo = (tau_lo >= b_lo && tau_lo < b_hi);
  const bool has_hi = (tau_hi >= b_lo && tau_hi < b_hi);
  double tau = has_lo ? tau_lo : first;
  if (!(tau < inf) && !has_hi) return best_tau;
  if (!(tau < inf)) tau = tau_hi;
  if (!has_lo && fs >= 0) {  // the first candidate is stage fs's head: consume it
    const TEPair* row = te_row(c, tb, w.st[fs].type, w.ent[fs]);
    const int m = sw.mp[fs][lane] - 1;
    double h = inf;
    if (m >= (int)w.kmin[fs]) {
      const double e = row[m - 1].et;
      if (e < b_hi && e <= tau_hi) h = e;
    }
    sw.hd[fs][lane] = h;
    sw.mp[fs][lane] = (uint16_t)m;
  }
  // state at the first candidate
  double E = 0.0;
  for (int r = 0; r < S; r++) {
    const StageEntry& st = w.st[r];
    const TEPair* row = te_row(c, tb, st.type, w.ent[r]);
    const int lo = (int)w.kmin[r], hi = (int)w.kmax[r];
    const int k = count_tab(row, tau, lo, hi, est_count(st, tau));
    const TEPair p = row[k - 1];
    sw.kk[r][lane] = (uint16_t)k;
    sw.nt[r][lane] = (k > lo) ? p.th : inf;
    E = (r == 0) ? p.et : fmax(E, p.et);
  }
  bool did_hi = false;
  for (;;) {
    // evaluate the current tau: advance crossed stages, exact sequential per_second
    double P = 0.0, nxt = inf;
    int ns = -1;
    for (int r = 0; r < S; r++) {
      int k = sw.kk[r][lane];
      if (tau >= sw.nt[r][lane]) {
        const StageEntry& st = w.st[r];
        const TEPair* row = te_row(c, tb, st.type, w.ent[r]);
        const int lo = (int)w.kmin[r];
        // one step down is the common case: count == k-1 iff tau < theta(k-2)
        TEPair p = row[k - 2];  // {et(k-1), theta(k-2)}
        if (k - 1 > lo && tau >= p.th) {
          k = count_tab(row, tau, lo, k - 2, est_count(st, tau));
          p = row[k - 1];
        } else {
          k = k - 1;
        }
        sw.kk[r][lane] = (uint16_t)k;
        sw.nt[r][lane] = (k > lo) ? p.th : inf;
        E = fmax(E, p.et);
      }
      const double term = sw.pr[r] * (double)k;
      P = (r == 0) ? term : P + term;
      const double h = sw.hd[r][lane];
      if (h < nxt) { nxt = h; ns = r; }
    }
    const double thr = (E > 0) ? c.batch / E : inf;
    const double cost = (thr > c.limit) ? c.work / thr * P : inf;
    if (MODE == 0) buf.insert(cost, tau); else if (cost <= lim && tau > best_tau) best_tau = tau;
    if (tau == tau_hi && has_hi) did_hi = true;
    // next candidate: pop the smallest head (a tau equal to the current one is re-evaluated
    // harmlessly: same state, same cost)
    if (ns >= 0 && nxt < inf) {
      const TEPair* row = te_row(c, tb, w.st[ns].type, w.ent[ns]);
      const int m = sw.mp[ns][lane] - 1;
      double h = inf;
      if (m >= (int)w.kmin[ns]) {
        const double e = row[m - 1].et;
        if (e < b_hi && e <= tau_hi) h = e;
      }
      sw.hd[ns][lane] = h;
      sw.mp[ns][lane] = (uint16_t)m;
      tau = fmax(tau, nxt);
    } else if (has_hi && !did_hi) {
      tau = tau_hi;
    } else {
      break;
    }
  }
  return best_tau;
}

template <int MAXS>
__device__ double phase_candidates_fast(const InstanceConsts& c, const DeviceTables& tb,
                                        const WarpSmem<MAXS>& w, SweepSmem<MAXS>& sw, int S,
                                        double tau_lo, double tau_hi, int n_cand) {
  const int lane = threadIdx.x & 31;
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  for (int r = lane; r < S; r += 32) sw.pr[r] = c.price_s[w.st[r].type];
  // lane intervals: 128 evenly spaced candidate indices (4 per lane), sorted across the warp
  // (bitonic over element index e = 4*lane + q), boundaries at every 4th sorted sample
  double v[4];
#pragma unroll
  for (int q = 0; q < 4; q++) {
    const int e = lane * 4 + q;
    v[q] = candidate_tau<MAXS>(c, tb, w, S, (int)(((long long)e * n_cand) >> 7), tau_lo, tau_hi);
    v[q] = fmin(fmax(v[q], tau_lo), tau_hi);
  }
#pragma unroll
  for (int k = 2; k <= 128; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j >= 4) {  // partner in lane ^ (j/4), same q
#pragma unroll
        for (int q = 0; q < 4; q++) {
          const int e = lane * 4 + q;
          const double o = __shfl_xor_sync(0xffffffffu, v[q], j >> 2);
          const bool up = (e & k) == 0, lower = (e & j) == 0;
          v[q] = (lower == up) ? fmin(v[q], o) : fmax(v[q], o);
        }
      } else {  // partner inside the lane
#pragma unroll
        for (int q = 0; q < 4; q++) {
          if ((q & j) == 0) {
            const int e = lane * 4 + q;
            const bool up = (e & k) == 0;
            const double a = v[q], b = v[q | j];
            v[q] = up ? fmin(a, b) : fmax(a, b);
            v[q | j] = up ? fmax(a, b) : fmin(a, b);
          }
        }
      }
    }
  }
  const double nb = __shfl_down_sync(0xffffffffu, v[0], 1);
  const double b_lo = (lane == 0) ? -inf : v[0];
  const double b_hi = (lane == 31) ? inf : nb;
  __syncwarp();
  TieBuf buf;
  buf.init();
  sweep_lane<MAXS, 0>(c, tb, w, sw, S, tau_lo, tau_hi, b_lo, b_hi, buf, 0.0);
  const double mf = warp_min(buf.mn);
  if (!(mf < inf)) return __longlong_as_double(0x7ff8000000000000LL);
  const double lim = mf + 1e-15;
  double bt;
  if (__any_sync(0xffffffffu, buf.overflow))
    bt = sweep_lane<MAXS, 1>(c, tb, w, sw, S, tau_lo, tau_hi, b_lo, b_hi, buf, lim);
  else
    bt = buf.best_tau(lim);
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
