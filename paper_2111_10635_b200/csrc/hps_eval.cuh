// hps_eval.cuh — warp-per-plan evaluation of one scheduling plan (the body of
// PlanScorer.__call__, ls/scoring.py:79-101), shared by the scoring, enumeration and
// random-sweep kernels.
//
// Work split inside a warp (32 lanes, one plan):
//   * stage construction: lane s owns stage s (and s+32): runs from a ballot over layer
//     boundaries, aggregates from the instance stage table (exact Neumaier sums done once);
//   * optimize_k1 exits + 60-step quota bisection (ls/provisioner.py:394-437): lanes evaluate
//     their stages' counts in parallel; a stage whose count is pinned by monotonicity
//     (count(b) == count(a)) is not re-evaluated;
//   * _best_candidate (ls/provisioner.py:262-314): the breakpoint candidates are spread over
//     lanes; each lane keeps a Pareto buffer of near-minimal (cost, tau) pairs and the warp
//     merges them. Candidates are never sorted: the reference's choice (minimum cost, then the
//     lexicographically smallest count vector among costs <= best + 1e-15) is a function of
//     the candidate SET, and counts are non-increasing in tau, so "lexicographically smallest"
//     == "largest tau among the ties".
//   * quota feasibility of candidates needs no work: every candidate lies in [tau_lo, tau_hi]
//     where counts are <= count(tau_lo), which passed quota_ok.
#pragma once
#include "hps_device.cuh"

namespace hps {

#ifndef HPS_BISECT_PROBES
#define HPS_BISECT_PROBES 0   // 1: the probing bisection (bisect_fast) instead of bisect_direct
#endif

constexpr int kTieBuf = 4;
constexpr uint8_t kStPending = 0xFE;  // internal: needs the block-per-plan slow path

template <int MAXS>
struct WarpSmem {
  StageEntry st[MAXS];
  double kmin[MAXS];   // count at tau_hi  (m_min, ls/provisioner.py:444)
  double kmax[MAXS];   // count at tau_lo  (m_max, ls/provisioner.py:445)
  double kres[MAXS];   // final counts
  int32_t ent[MAXS];   // stage-table entry
  int32_t cls[MAXS];   // ET-equivalence class of the entry
  int32_t pre[MAXS + 1];  // exclusive prefix of candidate counts over class leaders
  unsigned long long tsum[kMaxT];
  const TEPair* row[MAXS];  // TE row of stage r's entry (fast path)
  __device__ __forceinline__ const StageEntry& stage(int r) const { return st[r]; }
  __device__ __forceinline__ void bind(int r, const StageEntry* e) { st[r] = *e; }
};

// Lean per-warp view of the split path's candidate kernels: the stage entries stay in the
// (L1-cached, read-only) stage table instead of a 128-byte copy per stage and warp, which leaves
// the SM's unified L1/shared memory to the threshold-table loads of the exact evaluations.
template <int MAXS>
struct WarpSmemL {
  const StageEntry* sp[MAXS];  // stage-table entry of stage r
  int32_t kmin[MAXS];   // count at tau_hi
  int32_t kmax[MAXS];   // count at tau_lo
  double kres[MAXS];    // final counts (Python ints: the quota-gap path can see huge ones)
  int32_t ent[MAXS];
  int32_t cls[MAXS];
  int32_t pre[MAXS + 1];
  unsigned long long tsum[kMaxT];
  const TEPair* row[MAXS];
  __device__ __forceinline__ const StageEntry& stage(int r) const { return *sp[r]; }
  __device__ __forceinline__ void bind(int r, const StageEntry* e) { sp[r] = e; }
};

struct PlanOut {
  double cost, gap;
  int status;  // HPS_ST_* | overflow flag, or kStPending
  int S;
  int ps;
};

// `steps` of the reference's quota bisection (ls/provisioner.py:430-436) once quota_ok(mid) is known to
// be (mid >= tstar); returns the final b (the caller's tau_lo; the final a is not used).
//  * A step whose midpoint equals a or b is the last that can change b (the next midpoints repeat
//    it, or a == b), so the loop stops there.
//  * Once a and b are positive normals of one binade [2^e, 2^(e+1)) with ulp u, a = A u and b = B u,
//    and every step is exact integer arithmetic: fl(a + b) = 2u round_half_even((A + B) / 2), so
//    mid = M u with M = round_half_even((A + B) / 2) and the gap d = B - A becomes at most
//    ceil(d / 2). After ceil(log2 d) + 1 steps the outcome is fixed: b stays when tstar > b (or is
//    NaN; a alone moves); b = tstar when a < tstar <= b (tstar is then a multiple of u, and the
//    gap closes onto it); when tstar <= a only b moves, reaches a + u and then takes
//    M = round_half_even(A + 1/2): b = a for even A, a + u for odd A. With that many steps left
//    the loop jumps to this end state (bit-identical to running them).
__device__ __forceinline__ double halvings(double a, double b, double tstar, int steps) {
  for (int it = 0; it < steps; it++) {
    const long long ia = __double_as_longlong(a), ib = __double_as_longlong(b);
    const int ea = (int)(ia >> 52);
    if (ea == (int)(ib >> 52) && ea > 52 && ea < 2047 && ia > 0) {   // one binade, positive normals
      if (ia == ib) return b;
      const double u = __longlong_as_double((long long)(ea - 52) << 52);
      const double d = (b - a) / u;   // exact: Sterbenz, then a power-of-two scale
      const long long id = __double_as_longlong(d);
      const int need = (int)(id >> 52) - 1023 + ((id & 0xfffffffffffffLL) != 0) + 1;
      if (steps - it >= need) {
        if (!(tstar <= b)) return b;
        if (tstar <= a) return (ia & 1) ? a + u : a;
        return tstar;
      }
    }
    const double mid = (a + b) / 2.0;
    const bool last = (mid == a) || (mid == b);
    if (mid >= tstar) b = mid; else a = mid;
    if (last) break;
  }
  return b;
}

// For stages r = lane (slot 0) and lane + 32 (slot 1) of an S-stage plan (S <= 64): the first
// stage with the same key (k0 / k1, keys >= 0). One MATCH per slot; a slot-1 stage whose key also
// occurs in slot 0 takes the first such slot-0 stage (a 32-shuffle scan, only when S > 32).
__device__ __forceinline__ void first_same2(int S, int k0, int k1, int& f0, int& f1) {
  const int lane = threadIdx.x & 31;
  const int a = (lane < S) ? k0 : -1 - lane;        // absent stages get distinct negative keys
  const int b = (lane + 32 < S) ? k1 : -33 - lane;
  f0 = __ffs(__match_any_sync(0xffffffffu, a)) - 1;
  f1 = 32 + __ffs(__match_any_sync(0xffffffffu, b)) - 1;
  if (S > 32) {
    int g = 64;
#pragma unroll 4
    for (int q = 0; q < 32; q++) {
      const int kq = __shfl_sync(0xffffffffu, a, q);
      if (kq == b && q < g) g = q;
    }
    if (g < 64) f1 = g;
  }
}

struct TieBuf {  // Pareto set: costs ascending, taus ascending, all <= lane_min + 1e-15
  double c[kTieBuf], t[kTieBuf];
  int n;
  bool overflow;
  double mn;
  __device__ __forceinline__ void init() { n = 0; overflow = false; mn = __longlong_as_double(0x7ff0000000000000LL); }
  __device__ __noinline__ void insert(double cost, double tau) {
    if (!(cost <= mn + 1e-15) && n > 0) return;  // cannot be within 1e-15 of the minimum
    if (cost < mn) {
      mn = cost;
      const double lim = mn + 1e-15;
      int m = 0;
      for (int i = 0; i < n; i++)
        if (c[i] <= lim) { c[m] = c[i]; t[m] = t[i]; m++; }
      n = m;
    }
    // dominated by an existing entry (cheaper-or-equal and later-or-equal)?
    for (int i = 0; i < n; i++)
      if (c[i] <= cost && t[i] >= tau) return;
    int m = 0;
    for (int i = 0; i < n; i++)
      if (!(cost <= c[i] && tau >= t[i])) { c[m] = c[i]; t[m] = t[i]; m++; }
    n = m;
    if (n == kTieBuf) { overflow = true; return; }
    c[n] = cost; t[n] = tau; n++;
  }
  // largest tau whose cost is <= lim (the lexicographically smallest vector among ties)
  __device__ __forceinline__ double best_tau(double lim) const {
    double bt = -__longlong_as_double(0x7ff0000000000000LL);
    for (int i = 0; i < n; i++)
      if (c[i] <= lim && t[i] > bt) bt = t[i];
    return bt;
  }
};

// (operands are never NaN: plain compares instead of fmax/fmin's NaN handling)
__device__ __forceinline__ double warp_max(double v) {
  for (int o = 16; o; o >>= 1) { const double u = __shfl_xor_sync(0xffffffffu, v, o); v = (u > v) ? u : v; }
  return v;
}
__device__ __forceinline__ double warp_min(double v) {
  for (int o = 16; o; o >>= 1) { const double u = __shfl_xor_sync(0xffffffffu, v, o); v = (u < v) ? u : v; }
  return v;
}
__device__ __forceinline__ int warp_sum_i(int v) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ long long warp_sum_ll(long long v) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

constexpr int kOver = 0x7fffffff;  // "count above quota (or _floor_count raised)"

// single-precision seed of count(tau); correctness never depends on it
__device__ __forceinline__ int est_count(const StageEntry& s, double tau) {
  const float t = (float)tau;
  float q = 1.0f;
  if (s.oct != 0) {
    const float h = t * s.f_rbo - s.f_oma;
    q = (h > 0.f) ? fmaxf(q, __fdividef(s.f_alpha, h)) : 3.0e38f;
  }
  if (s.odt != 0) {
    const float h = t * s.f_rbd - s.f_omb;
    q = (h > 0.f) ? fmaxf(q, __fdividef(s.f_beta, h)) : 3.0e38f;
  }
  const float cf = ceilf(q - 1e-9f);
  return (cf < 2.0e9f && cf == cf) ? (int)cf : 2000000000;
}

// Exact count(tau) given count(tau) in [lo, hi] (hi <= table cap). row[c].th = theta(c).
static __device__ HPS_NOINLINE_RARE int count_tab(const TEPair* row, double tau, int lo, int hi, int g) {
  if (lo >= hi) return lo;
  HPS_STAT(ST_TAB, 1);
  const int m = min(max(g, lo), hi);
  if (HPS_TE(row, m).th <= tau) {  // count <= m: gallop down
    int hb = m, lb, step = 1;
    for (;;) {
      const int cnd = hb - step;
      if (cnd < lo) { lb = lo - 1; break; }
      if (HPS_TE(row, cnd).th <= tau) { hb = cnd; step <<= 1; } else { lb = cnd; break; }
    }
    while (hb - lb > 1) { const int md = (lb + hb) >> 1; if (HPS_TE(row, md).th <= tau) hb = md; else lb = md; }
    return hb;
  }
  int lb = m, hb, step = 1;  // count > m: gallop up (count <= hi is guaranteed)
  for (;;) {
    const int cnd = lb + step;
    if (cnd >= hi) { hb = hi; break; }
    if (HPS_TE(row, cnd).th <= tau) { hb = cnd; break; }
    lb = cnd;
    step <<= 1;
  }
  while (hb - lb > 1) { const int md = (lb + hb) >> 1; if (HPS_TE(row, md).th <= tau) hb = md; else lb = md; }
  return hb;
}

// per-type sums of counts <= quota for all types (lanes own stages r and r+32)
__device__ __forceinline__ bool quota_sums_ok(const InstanceConsts& c, unsigned types_present,
                                              int t0, int k0, int t1, int k1) {
  bool ok = true;
  while (types_present) {
    const int t = __ffs(types_present) - 1;
    types_present &= types_present - 1;
    const unsigned v = (t0 == t ? (unsigned)k0 : 0u) + (t1 == t ? (unsigned)k1 : 0u);
    const unsigned sum = __reduce_add_sync(0xffffffffu, v);
    ok = ok && ((long long)sum <= c.quota[t]);
  }
  return ok;
}

// Bisection on quota_ok (ls/provisioner.py:430-437). Inputs: counts at tau_hi in kb[] (finite,
// quota-feasible). Output: tau_lo and the counts at tau_lo.
template <class W>
__device__ __forceinline__ double bisect_fast(const InstanceConsts& c, const DeviceTables& tb, const W& w,
                                              int S, double a, double b, const double kb_in[2], int kb_out[2]) {
  const int lane = threadIdx.x & 31;
  int lb[2], ub[2], ty[2] = {-1, -1}, Q[2] = {0, 0};
  const TEPair* row[2] = {nullptr, nullptr};
  double thq[2] = {0.0, 0.0};
  unsigned present = 0;
  for (int slot = 0; slot < 2; slot++) {
    const int s = lane + 32 * slot;
    lb[slot] = ub[slot] = 0;
    if (s < S) {
      ty[slot] = w.stage(s).type;
      Q[slot] = (int)c.quota[ty[slot]];
      row[slot] = te_row(c, tb, ty[slot], w.ent[s]);
      lb[slot] = (int)kb_in[slot];
      ub[slot] = kOver;
      thq[slot] = row[slot][Q[slot]].th;  // count <= Q  <=>  tau >= theta(Q)
    }
  }
  present = __reduce_or_sync(0xffffffffu, (ty[0] >= 0 ? 1u << ty[0] : 0u) | (ty[1] >= 0 ? 1u << ty[1] : 0u));
  int it = 0;
  {  // probes below L* = max_r theta_r(Q): some stage is over its quota, so quota_ok fails
    double lstar = -__longlong_as_double(0x7ff0000000000000LL);
    for (int slot = 0; slot < 2; slot++)
      if (ty[slot] >= 0) lstar = fmax(lstar, thq[slot]);
    lstar = warp_max(lstar);
    for (; it < 60; it++) {
      const double mid = (a + b) / 2.0;
      if (!(mid < lstar)) break;
      a = mid;
    }
  }
  bool closed = false;
  double tstar_single = 0.0;
  int n_unres = -1;   // unresolved stages when the closed-form test last ran
  for (; it < 60; it++) {
    // (1) each type has at most one unresolved stage r: on (a, b) its type's constraint is
    //     count_r(mid) <= K_r = Q_t - sum of the type's other (pinned) counts, i.e.
    //     mid >= theta_r(K_r); quota_ok switches at the max of those thresholds.
    //     The test can only change outcome when a stage got resolved since it last ran.
    const int n_now = __popc(__ballot_sync(0xffffffffu, ty[0] >= 0 && ub[0] != lb[0])) +
                      __popc(__ballot_sync(0xffffffffu, ty[1] >= 0 && ub[1] != lb[1]));
    if (n_now != n_unres) {
      n_unres = n_now;
      const bool u0 = ty[0] >= 0 && ub[0] != lb[0], u1 = ty[1] >= 0 && ub[1] != lb[1];
      const unsigned tm = (u0 ? 1u << ty[0] : 0u) | (u1 ? 1u << ty[1] : 0u);
      const unsigned types_u = __reduce_or_sync(0xffffffffu, tm);
      bool single = !(u0 && u1 && ty[0] == ty[1]);
      single = __all_sync(0xffffffffu, single);
      unsigned rem = types_u;
      while (single && rem) {
        const int t = __ffs(rem) - 1;
        rem &= rem - 1;
        single = __popc(__ballot_sync(0xffffffffu, (tm >> t) & 1u)) <= 1;
      }
      if (single && types_u) {
        double th = -__longlong_as_double(0x7ff0000000000000LL);
        unsigned rem2 = types_u;
        while (rem2) {
          const int t = __ffs(rem2) - 1;
          rem2 &= rem2 - 1;
          const unsigned v = (ty[0] == t ? (unsigned)lb[0] : 0u) + (ty[1] == t ? (unsigned)lb[1] : 0u);
          const long long sum_b = (long long)__reduce_add_sync(0xffffffffu, v);  // counts at b
          for (int slot = 0; slot < 2; slot++) {
            const bool mine = (slot ? u1 : u0) && ty[slot] == t;
            if (mine) {
              const long long K = c.quota[t] - (sum_b - lb[slot]);  // >= lb (quota_ok(b))
              th = fmax(th, HPS_TE(row[slot], (int)K).th);                  // count <= K <=> tau >= theta(K)
            }
          }
        }
        tstar_single = warp_max(th);
        closed = true;
        break;
      }
    }
    const bool wide = (ub[0] - lb[0] > 1 && ub[0] != kOver) || (ub[1] - lb[1] > 1 && ub[1] != kOver) ||
                      (ub[0] == kOver && lb[0] < Q[0]) || (ub[1] == kOver && lb[1] < Q[1]);
    if (!__any_sync(0xffffffffu, wide)) break;
    if (lane == 0) HPS_STAT(ST_PROBES_EXACT, 1);
    const double mid = (a + b) / 2.0;
    int km[2];
    // some stage certainly above its quota (mid < theta(Q)): quota_ok(mid) is false, no counts
    const bool over0 = (ub[0] == kOver && mid < thq[0]) || (ub[1] == kOver && mid < thq[1]);
    if (__any_sync(0xffffffffu, over0)) {
      a = mid;
      for (int slot = 0; slot < 2; slot++)
        if (ub[slot] == kOver && mid < thq[slot]) ub[slot] = kOver;  // (unchanged: still over)
      continue;
    }
    bool over = false;
    for (int slot = 0; slot < 2; slot++) {
      km[slot] = lb[slot];
      if (ub[slot] != lb[slot]) {
        if (ub[slot] == kOver && mid < thq[slot]) {
          km[slot] = kOver;
          over = true;
        } else {
          const int s = lane + 32 * slot;
          const int hi = (ub[slot] == kOver) ? Q[slot] : ub[slot];
          const int kc = count_cert(w.stage(s), mid, c.bo);  // mid >= theta(Q): no raise here
          km[slot] = (kc >= lb[slot] && kc <= hi) ? kc : count_tab(row[slot], mid, lb[slot], hi, est_count(w.stage(s), mid));
        }
      }
    }
    const bool any_over = __any_sync(0xffffffffu, over);
    // counts at b satisfy the quotas; only a count above its value at b can break them
    const bool rose = __any_sync(0xffffffffu, km[0] != lb[0] || km[1] != lb[1]);
    const bool ok = !any_over && (!rose || quota_sums_ok(c, present, ty[0], km[0], ty[1], km[1]));
    if (ok) { b = mid; lb[0] = km[0]; lb[1] = km[1]; }
    else { a = mid; ub[0] = km[0]; ub[1] = km[1]; }
  }
  if (closed) {
    if (lane == 0) HPS_STAT(ST_PROBES_CLOSED, 60 - it);
    for (; it < 60; it++) {
      const double mid = (a + b) / 2.0;
      if (mid >= tstar_single) b = mid; else a = mid;
    }
    // counts at the final b: unresolved stages resolve by their threshold
    for (int slot = 0; slot < 2; slot++)
      if (ty[slot] >= 0 && ub[slot] != lb[slot]) {
        const int hi = (ub[slot] == kOver) ? Q[slot] : ub[slot];
        const int kc = count_cert(w.stage(lane + 32 * slot), b, c.bo);
        lb[slot] = (kc >= lb[slot] && kc <= hi) ? kc
                                                 : count_tab(row[slot], b, lb[slot], hi, est_count(w.stage(lane + 32 * slot), b));
      }
  } else if (it < 60) {
    // every unpinned stage has count(a) == count(b) + 1 (or "over" with count(b) == Q):
    // on (a, b) its count is lb + [tau < theta(lb)], so quota_ok switches at one of those
    // thresholds (or stays true up to b). Find the switch point tau* exactly.
    double cand[2] = {__longlong_as_double(0x7ff0000000000000LL), __longlong_as_double(0x7ff0000000000000LL)};
    double thr_lb[2] = {0.0, 0.0};
    for (int slot = 0; slot < 2; slot++) {
      if (ub[slot] != lb[slot]) {
        thr_lb[slot] = row[slot][lb[slot]].th;  // count <= lb  <=>  tau >= theta(lb)
        if (thr_lb[slot] > a && thr_lb[slot] <= b) cand[slot] = thr_lb[slot];
      }
    }
    double tstar = b;
    // candidates in ascending order; the predicate is monotone, so the first true one wins
    double lo_bound = -__longlong_as_double(0x7ff0000000000000LL);
    for (;;) {
      // next smallest candidate above lo_bound
      double mine = fmin(cand[0] > lo_bound ? cand[0] : __longlong_as_double(0x7ff0000000000000LL),
                         cand[1] > lo_bound ? cand[1] : __longlong_as_double(0x7ff0000000000000LL));
      const double x = warp_min(mine);
      if (!(x < b)) break;  // b itself is feasible
      int kx[2];
      bool ov = false;
      for (int slot = 0; slot < 2; slot++) {
        kx[slot] = lb[slot];
        if (ub[slot] != lb[slot] && x < thr_lb[slot]) { kx[slot] = ub[slot]; ov |= (ub[slot] == kOver); }
      }
      const bool okx = !__any_sync(0xffffffffu, ov) && quota_sums_ok(c, present, ty[0], kx[0], ty[1], kx[1]);
      if (okx) { tstar = x; break; }
      lo_bound = x;
    }
    if (lane == 0) HPS_STAT(ST_PROBES_CLOSED, 60 - it);
    b = halvings(a, b, tstar, 60 - it);
    for (int slot = 0; slot < 2; slot++)
      if (ub[slot] != lb[slot] && b < thr_lb[slot]) lb[slot] = ub[slot];
  }
  kb_out[0] = lb[0];
  kb_out[1] = lb[1];
  return b;
}


// Exact count(tau) of a stage known to lie in [lo, hi] (hi <= table cap): FP32 seed, confirmed by
// theta(k) <= tau < theta(k - 1) or corrected by the galloping table search.
// the FP32 seed constants of a stage, held in registers across repeated count searches
struct SeedConsts {
  float rb[2], om[2], fr[2];
  __device__ __forceinline__ void load(const StageEntry& s) {
    rb[0] = s.f_rbo; rb[1] = s.f_rbd;
    om[0] = s.f_oma; om[1] = s.f_omb;
    fr[0] = s.f_alpha; fr[1] = s.f_beta;
  }
};

// count_seeded from register-held seed constants (same seed arithmetic, same exact table test)
static __device__ __noinline__ int count_seeded_r(const SeedConsts sc, const TEPair* row, double tau, int lo, int hi) {
  const float tf = (float)tau;
  float q = 1.0f;
#pragma unroll
  for (int side = 0; side < 2; side++) {
    const float rb = sc.rb[side], frac = sc.fr[side];
    if (rb == 0.0f || frac == 0.0f) continue;
    const float h = tf * rb - sc.om[side];
    q = (h > 0.0f) ? fmaxf(q, frac * rcp_approx_f32(h)) : 3.0e38f;
  }
  int k = (q < 2.0e9f) ? (int)ceilf(q) : hi;
  k = min(max(k, lo), hi);
  const double2 pk = __ldg(reinterpret_cast<const double2*>(&HPS_TE(row, k - 1)));  // {et(k), theta(k-1)}
  const double thk = __ldg(&HPS_TE(row, k).th);
  if (thk <= tau && tau < pk.y) return k;
  return count_tab(row, tau, lo, hi, k);
}

static __device__ __noinline__ int count_seeded(const StageEntry& s, const TEPair* row, double tau, int lo, int hi) {
  const float tf = (float)tau;
  float q = 1.0f;
#pragma unroll
  for (int side = 0; side < 2; side++) {
    const float rb = side ? s.f_rbd : s.f_rbo;
    const float frac = side ? s.f_beta : s.f_alpha;
    if (rb == 0.0f || frac == 0.0f) continue;
    const float h = tf * rb - (side ? s.f_omb : s.f_oma);
    q = (h > 0.0f) ? fmaxf(q, frac * rcp_approx_f32(h)) : 3.0e38f;
  }
  int k = (q < 2.0e9f) ? (int)ceilf(q) : hi;
  k = min(max(k, lo), hi);
  const double2 pk = __ldg(reinterpret_cast<const double2*>(&HPS_TE(row, k - 1)));  // {et(k), theta(k-1)}
  const double thk = __ldg(&HPS_TE(row, k).th);
  if (thk <= tau && tau < pk.y) return k;
  return count_tab(row, tau, lo, hi, k);
}

// q_cont from register-held seed constants (same arithmetic)
__device__ __forceinline__ float q_cont_r(const SeedConsts& s, float tau, float& dq) {
  float q = 1.0f;
  dq = 0.0f;
#pragma unroll
  for (int side = 0; side < 2; side++) {
    const float rb = s.rb[side], frac = s.fr[side];
    if (rb == 0.0f || frac == 0.0f) continue;
    const float h = tau * rb - s.om[side];
    const float rh = rcp_approx_f32(h);
    const float v = (h > 0.0f) ? frac * rh : 3.0e38f;
    if (v > q) { q = v; dq = (h > 0.0f) ? -v * rb * rh : -3.0e38f; }
  }
  return q;
}

// FP32 continuous count q(tau) = max(1, frac / (tau rb - (1 - frac))) of both sides and dq/dtau
// (seed arithmetic only)
__device__ __forceinline__ float q_cont(const StageEntry& s, float tau, float& dq) {
  float q = 1.0f;
  dq = 0.0f;
#pragma unroll
  for (int side = 0; side < 2; side++) {
    const float rb = side ? s.f_rbd : s.f_rbo;
    const float frac = side ? s.f_beta : s.f_alpha;
    if (rb == 0.0f || frac == 0.0f) continue;
    const float h = tau * rb - (side ? s.f_omb : s.f_oma);
    const float rh = rcp_approx_f32(h);            // seed arithmetic: MUFU reciprocal
    const float v = (h > 0.0f) ? frac * rh : 3.0e38f;
    if (v > q) { q = v; dq = (h > 0.0f) ? -v * rb * rh : -3.0e38f; }
  }
  return q;
}

// Quota bisection (ls/provisioner.py:430-437) by its switch point. quota_ok(tau) holds iff for
// every type t the sum of its stages' counts is <= Q_t, and counts are non-increasing
// right-continuous step functions (count(tau) <= k <=> tau >= theta(k)), so quota_ok(tau) <=>
// tau >= tau* = max_t tau*_t. Per type: tau*_t >= L_t = max_r theta_r(Q_t) (below it one stage
// alone exceeds the quota); an FP32 Newton solve of sum_r q_r(tau) = Q_t - n/2 seeds tau_e in
// [L_t, tau_hi]; the exact counts at tau_e (sum S_e) then select tau*_t exactly from the
// thresholds next to tau_e: if S_e <= Q_t it is the (Q_t - S_e + 1)-th largest threshold below
// (count increments), else the (S_e - Q_t)-th smallest above (decrements), never below L_t.
// With tau* exact, the reference's 60 halvings are replayed as comparisons mid >= tau*, and the
// counts at the final b (= tau_lo) are read from the tables. Mids in (serial, tau_hi) never
// raise in _floor_count except where counts exceed every quota (mid < L_t), where quota_ok is
// false either way.
template <class W>
__device__ __forceinline__ double bisect_direct(const InstanceConsts& c, const W& w, int S, double a, double b,
                                                const double kb_in[2], int kb_out[2]) {
  const TEPair* const* rows = w.row;
  const int lane = threadIdx.x & 31;
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  int ty[2], kb[2];
  const TEPair* row[2];
  SeedConsts sc[2];   // the stages' seed constants, read once for every search below
#pragma unroll
  for (int slot = 0; slot < 2; slot++) {
    const int s = lane + 32 * slot;
    ty[slot] = (s < S) ? w.stage(s).type : -1;
    kb[slot] = (s < S) ? (int)kb_in[slot] : 0;
    row[slot] = (s < S) ? rows[s] : nullptr;
    if (s < S) sc[slot].load(w.stage(s));
  }
  const unsigned present =
      __reduce_or_sync(0xffffffffu, (ty[0] >= 0 ? 1u << ty[0] : 0u) | (ty[1] >= 0 ? 1u << ty[1] : 0u));
  double tstar = -inf;
  unsigned rem = present;
  while (rem) {
    const int t = __ffs(rem) - 1;
    rem &= rem - 1;
    const int Q = (int)c.quota[t];
    const bool mb[2] = {ty[0] == t, ty[1] == t};
    double lt = -inf;
#pragma unroll
    for (int slot = 0; slot < 2; slot++)
      if (mb[slot]) lt = fmax(lt, __ldg(&HPS_TE(row[slot], Q).th));
    lt = warp_max(lt);
    // exact counts at L_t (each <= Q there): when their sum is within the quota, tau*_t = L_t
    int cnt[2] = {0, 0};
#pragma unroll
    for (int slot = 0; slot < 2; slot++)
      if (mb[slot]) cnt[slot] = count_seeded_r(sc[slot], row[slot], lt, kb[slot], Q);
    const int sl = (int)__reduce_add_sync(0xffffffffu, (unsigned)(cnt[0] + cnt[1]));
    if (sl <= Q) {
      tstar = fmax(tstar, lt);
      continue;
    }
    // ---- FP32 seed of the root of sum_r q_r(tau) = Q_t - n/2 in (L_t, tau_hi]: Newton on
    // 1/F - 1/target from L_t (exact in one step for a single hyperbola c/(tau - p)) ----
    const int n = (int)__reduce_add_sync(0xffffffffu, (unsigned)mb[0] + (unsigned)mb[1]);
    const float target = (float)Q - 0.5f * (float)n;
    const float flo = (float)lt, fhi = (float)b;
    float x = flo;
    for (int itn = 0; itn < 12; itn++) {
      if (lane == 0) HPS_STAT(ST_CERT, 1);
      float F = 0.0f, dF = 0.0f;
#pragma unroll
      for (int slot = 0; slot < 2; slot++)
        if (mb[slot]) {
          float d;
          F += q_cont_r(sc[slot], x, d);
          dF += d;
        }
      for (int o = 16; o; o >>= 1) {
        F += __shfl_xor_sync(0xffffffffu, F, o);
        dF += __shfl_xor_sync(0xffffffffu, dF, o);
      }
      if (fabsf(F - target) <= 0.25f || !(dF < 0.0f) || !(F < 3.0e37f)) break;
      float nx = x + F * (1.0f - __fdividef(F, target)) * rcp_approx_f32(dF);
      nx = fminf(fmaxf(nx, flo), fhi);
      const bool done = fabsf(nx - x) <= 1e-7f * x;
      x = nx;
      if (done) break;
    }
    double te = fmin(fmax((double)x, lt), b);
    // ---- exact counts at te and exact selection of tau*_t ----
#pragma unroll
    for (int slot = 0; slot < 2; slot++)
      if (mb[slot]) cnt[slot] = count_seeded_r(sc[slot], row[slot], te, kb[slot], Q);
    const int se = (int)__reduce_add_sync(0xffffffffu, (unsigned)(cnt[0] + cnt[1]));
    double tt;
    if (se <= Q) {
      // descending thresholds below te: theta_r(cnt) (count cnt -> cnt + 1 below it); only
      // values >= L_t matter (below L_t the type is over its quota regardless)
      double nx[2];
#pragma unroll
      for (int slot = 0; slot < 2; slot++) {
        nx[slot] = -inf;
        if (mb[slot] && cnt[slot] < Q) {
          const double v = __ldg(&row[slot][cnt[slot]].th);
          if (v >= lt) nx[slot] = v;
        }
      }
      int d = Q - se + 1;
      if (d > 48) return __longlong_as_double(0x7ff8000000000000LL);  // poor seed: caller falls back
      tt = lt;
      for (;;) {
        const double mine = fmax(nx[0], nx[1]);
        const double e = warp_max(mine);
        if (lane == 0) HPS_STAT(ST_PROBES_EXACT, 1);
        if (!(e > -inf)) { tt = lt; break; }
        if (--d == 0) { tt = fmax(e, lt); break; }
        const unsigned own = __ballot_sync(0xffffffffu, mine == e);
        if (lane == __ffs(own) - 1) {
          const int sl = (nx[0] == e) ? 0 : 1;
          const int k = ++cnt[sl];
          double v = -inf;
          if (k < Q) {
            v = __ldg(&HPS_TE(row[sl], k).th);
            if (!(v >= lt)) v = -inf;
          }
          nx[sl] = v;
        }
      }
    } else {
      // ascending thresholds above te: theta_r(cnt - 1) (count cnt -> cnt - 1 from it on), down to
      // the count at tau_hi
      double nx[2];
#pragma unroll
      for (int slot = 0; slot < 2; slot++)
        nx[slot] = (mb[slot] && cnt[slot] > kb[slot]) ? __ldg(&row[slot][cnt[slot] - 1].th) : inf;
      int d = se - Q;
      if (d > 48) return __longlong_as_double(0x7ff8000000000000LL);
      tt = b;
      for (;;) {
        const double mine = fmin(nx[0], nx[1]);
        const double e = warp_min(mine);
        if (lane == 0) HPS_STAT(ST_CERT_FAIL, 1);
        if (!(e < inf)) { tt = b; break; }  // (cannot happen: quota_ok(tau_hi) holds)
        if (--d == 0) { tt = e; break; }
        const unsigned own = __ballot_sync(0xffffffffu, mine == e);
        if (lane == __ffs(own) - 1) {
          const int sl = (nx[0] == e) ? 0 : 1;
          const int k = --cnt[sl];
          nx[sl] = (k > kb[sl]) ? __ldg(&HPS_TE(row[sl], k - 1).th) : inf;
        }
      }
    }
    tstar = fmax(tstar, tt);
  }
  if (lane == 0) HPS_STAT(ST_PROBES_CLOSED, 60);
  b = halvings(a, b, tstar, 60);
#pragma unroll
  for (int slot = 0; slot < 2; slot++)
    kb_out[slot] = (ty[slot] >= 0) ? count_seeded_r(sc[slot], row[slot], b, kb[slot], (int)c.quota[ty[slot]])
                                   : kb[slot];
  return b;
}

// Evaluate one candidate tau: numpy _best_candidate column (ls/provisioner.py:286-308).
// Returns +inf when the column is not ok (throughput <= limit).
template <int MAXS, bool CERT = false>
__device__ __forceinline__ double candidate_cost(const InstanceConsts& c, const DeviceTables& tb,
                                                 const WarpSmem<MAXS>& w, int S, double tau) {
  double E = 0.0, P = 0.0;
  for (int r = 0; r < S; r++) {
    const StageEntry& s = w.stage(r);
    double k = w.kmin[r];
    if (w.kmax[r] != k) {
      const int kc = CERT ? count_cert(s, tau, c.bo) : -1;
      k = (kc > 0) ? (double)kc : count_at(s, tau, c.bo);
    }
    double et = et_lookup(c, tb, s, w.ent[r], k);
    double term = c.price_s[s.type] * k;
    if (r == 0) { E = et; P = term; } else { E = fmax(E, et); P = P + term; }
  }
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  double thr = (E > 0) ? c.batch / E : inf;
  if (!(thr > c.limit)) return inf;
  return c.work / thr * P;
}

// m_min / m_max and class leaders (ls/provisioner.py:442-455): counts at tau_lo in kb (lane
// slots), then the candidate count over class leaders (identical (oct, odt, alpha, beta) =>
// identical counts and breakpoints, so only the first stage of a class contributes distinct
// values) and its exclusive prefix in w.pre; n_cand includes tau_lo and tau_hi.
template <int MAXS, class W>
__device__ __forceinline__ void cands_prefix(const DeviceTables& tb, W& w, int S, const double kb[2],
                                             int& n_cand) {
  const int lane = threadIdx.x & 31;
  for (int slot = 0; slot < 2; slot++) {
    const int s = lane + 32 * slot;
    if (s < S) {
      w.kmax[s] = kb[slot];
      w.cls[s] = tb_class(tb, w.ent[s]);
    }
  }
  __syncwarp();
  int f[2];
  first_same2(S, (lane < S) ? w.cls[lane] : 0, (lane + 32 < S) ? w.cls[lane + 32] : 0, f[0], f[1]);
  int cnt[2] = {0, 0};
  for (int slot = 0; slot < 2; slot++) {
    const int s = lane + 32 * slot;
    if (s < S) {
      const bool leader = f[slot] == s;   // first stage of its class
      double span = w.kmax[s] - w.kmin[s];
      if (leader && span <= (double)kBpLimit) cnt[slot] = (int)span + 1;
    }
  }
  // exclusive prefix over s = 0..S-1 (slot 0 then slot 1)
  int inc0 = cnt[0];
  for (int o = 1; o < 32; o <<= 1) { int v = __shfl_up_sync(0xffffffffu, inc0, o); if (lane >= o) inc0 += v; }
  int tot0 = __shfl_sync(0xffffffffu, inc0, 31);
  int inc1 = cnt[1];
  for (int o = 1; o < 32; o <<= 1) { int v = __shfl_up_sync(0xffffffffu, inc1, o); if (lane >= o) inc1 += v; }
  int tot1 = __shfl_sync(0xffffffffu, inc1, 31);
  if (lane < S) w.pre[lane] = inc0 - cnt[0];
  if (lane + 32 < S) w.pre[lane + 32] = tot0 + inc1 - cnt[1];
  if (lane == 0) w.pre[S] = tot0 + tot1;
  __syncwarp();
  n_cand = tot0 + tot1 + 2;
}

// Fast-path bisection from the counts at tau_hi (w.kmin) on (serial, tau_hi), then the candidate
// prefix. Needs w.st, w.ent, w.row, w.kmin.
template <int MAXS, class W>
__device__ __forceinline__ void phase_bisect_cands(const InstanceConsts& c, const DeviceTables& tb, W& w,
                                                   int S, double a, double b, double& tau_lo_out, int& n_cand) {
  const int lane = threadIdx.x & 31;
  double kb[2] = {0.0, 0.0};
  for (int slot = 0; slot < 2; slot++) {
    const int s = lane + 32 * slot;
    if (s < S) kb[slot] = w.kmin[s];
  }
  int kl[2];
#if HPS_BISECT_PROBES
  b = bisect_fast(c, tb, w, S, a, b, kb, kl);
#else
  const double bd = bisect_direct(c, w, S, a, b, kb, kl);
  if (bd == bd) b = bd;
  else {  // (rare) seed too far off
    if (lane == 0) HPS_STAT(ST_UNPINNED, 1);
    b = bisect_fast(c, tb, w, S, a, b, kb, kl);
  }
#endif
  kb[0] = (double)kl[0];
  kb[1] = (double)kl[1];
  tau_lo_out = b;
  cands_prefix<MAXS>(tb, w, S, kb, n_cand);
}

// Phase A: stages, optimize_k1 exits and the bisection. Returns false when the plan is
// finished (infeasible / invalid); otherwise fills w.kmin/kmax and tau_lo/tau_hi.
// Lane l holds digits d0 (layer l) and d1 (layer l+32).
template <int MAXS, bool FAST = false, bool HI_ONLY = false, class W>
__device__ bool phase_stages_bisect(const InstanceConsts& c, const DeviceTables& tb,
                                    W& w, int d0, int d1, PlanOut& out,
                                    double& tau_lo_out, double& tau_hi_out, int& n_cand) {
  const int lane = threadIdx.x & 31;
  const int L = c.L;
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  // --- runs (ls/domain.py:293-296): stage starts where the type changes ---
  int prev0 = __shfl_up_sync(0xffffffffu, d0, 1);
  int last_lo = __shfl_sync(0xffffffffu, d0, 31);
  int prev1 = __shfl_up_sync(0xffffffffu, d1, 1);
  if (lane == 0) prev1 = last_lo;
  bool start0 = (lane < L) && (lane == 0 || d0 != prev0);
  bool start1 = (lane + 32 < L) && (d1 != prev1);
  unsigned m0 = __ballot_sync(0xffffffffu, start0), m1 = __ballot_sync(0xffffffffu, start1);
  bool bad_digit = (lane < L && (d0 < 0 || d0 >= c.T)) || (lane + 32 < L && (d1 < 0 || d1 >= c.T));
  if (__any_sync(0xffffffffu, bad_digit)) {
    out.status = HPS_ST_INVALID; out.cost = __longlong_as_double(0x7ff8000000000000LL); out.gap = 0; out.S = 0;
    return false;
  }
  const int c0 = __popc(m0);
  const int S = c0 + __popc(m1);
  out.S = S;
  HPS_CHECK(S <= MAXS, "more stages than the warp view holds");
  // lane s builds stage s and s+32
  bool invalid = false;
  for (int slot = 0; slot < 2; slot++) {
    const int s = lane + 32 * slot;
    int first = -1, last = -1;
    if (s < S) {
      first = (s < c0) ? (int)__fns(m0, 0, s + 1) : 32 + (int)__fns(m1, 0, s - c0 + 1);
      int nx = s + 1;
      if (nx < S) last = ((nx < c0) ? (int)__fns(m0, 0, nx + 1) : 32 + (int)__fns(m1, 0, nx - c0 + 1)) - 1;
      else last = L - 1;
    }
    int src = first & 31;
    int t0 = __shfl_sync(0xffffffffu, d0, src), t1 = __shfl_sync(0xffffffffu, d1, src);
    if (s < S) {
      const int type = (first < 32) ? t0 : t1;
      const int e = entry_index(c.P, type, first, last);
      w.bind(s, tb.stages + e);
      w.ent[s] = e;
      w.row[s] = tb.te + c.te_off[type] + (int64_t)(e - type * c.P) * (int64_t)(c.et_cap[type] + 1);
      invalid |= (w.stage(s).valid == 0);
    }
  }
  __syncwarp();
  if (__any_sync(0xffffffffu, invalid)) {
    out.status = HPS_ST_INVALID; out.cost = __longlong_as_double(0x7ff8000000000000LL); out.gap = 0;
    return false;
  }
  // --- stage-0 bound and tau_hi (ls/provisioner.py:394-397) ---
  const int type0 = w.stage(0).type;
  const int last0 = (S > 1) ? ((1 < c0) ? (int)__fns(m0, 0, 2) : 32 + (int)__fns(m1, 0, 1)) - 1 : L - 1;
  const Stage0Info s0 = tb.stage0[type0 * L + last0];
  if (s0.status != HPS_ST_OK) {
    out.status = s0.status; out.gap = s0.gap; out.cost = c.penalty_scale * (1.0 + pmax(0.0, s0.gap));
    return false;
  }
  const double tau_hi = s0.tau_hi;
  // --- serial floor (ls/provisioner.py:399-412) ---
  double ser = 0.0;
  for (int s = lane; s < S; s += 32) ser = fmax(ser, w.stage(s).serial);
  ser = warp_max(ser);
  if (ser >= tau_hi) {
    out.status = HPS_ST_SERIAL; out.gap = clamp_gap((ser - tau_hi) / tau_hi);
    out.cost = c.penalty_scale * (1.0 + pmax(0.0, out.gap));
    return false;
  }
  // --- counts at tau_hi + quota (ls/provisioner.py:413-427) ---
  if (lane < kMaxT) w.tsum[lane] = 0ull;
  __syncwarp();
  double kb[2] = {inf, inf}, ka[2] = {inf, inf}, gapv[2] = {0.0, 0.0};
  bool raised[2] = {false, false};
  for (int slot = 0; slot < 2; slot++) {
    const int s = lane + 32 * slot;
    if (s < S) {
      double r;
      if (floor_count(w.stage(s), tau_hi, c.bo, r, gapv[slot])) {
        kb[slot] = iceil(r);
        atomicAdd(&w.tsum[w.stage(s).type], sat_count(kb[slot]));
      } else {
        raised[slot] = true;
      }
    }
  }
  __syncwarp();
  bool over = (lane < c.T) && (w.tsum[lane] > (unsigned long long)c.quota[lane]);
  unsigned over_mask = __ballot_sync(0xffffffffu, over);
  unsigned r0 = __ballot_sync(0xffffffffu, raised[0]), r1 = __ballot_sync(0xffffffffu, raised[1]);
  if (r0 | r1 | over_mask) {
    if (r0 | r1) {  // _counts_at(tau_hi) raises from the first raising stage (:414)
      int src = r0 ? (__ffs(r0) - 1) : (__ffs(r1) - 1);
      double g = __shfl_sync(0xffffffffu, r0 ? gapv[0] : gapv[1], src);
      out.status = HPS_ST_FLOOR_TAU_HI; out.gap = g;
    } else {  // first offending type in ascending id (:418-420), exact Python-int totals
      for (int slot = 0; slot < 2; slot++) {
        const int s = lane + 32 * slot;
        if (s < S) w.kres[s] = kb[slot];
      }
      __syncwarp();
      const int off = __ffs(over_mask) - 1;
      double g = 0.0;
      if (lane == 0) {
        u128 tot = 0;
        for (int s = 0; s < S; s++)
          if (w.stage(s).type == off) tot += dbl_to_u128(w.kres[s]);
        g = clamp_gap(int_true_div(tot - (u128)c.quota[off], c.quota[off]));
      }
      out.status = HPS_ST_QUOTA_TAU_HI; out.gap = __shfl_sync(0xffffffffu, g, 0);
    }
    out.cost = c.penalty_scale * (1.0 + pmax(0.0, out.gap));
    return false;
  }
  for (int slot = 0; slot < 2; slot++) {
    const int s = lane + 32 * slot;
    if (s < S) w.kmin[s] = kb[slot];
  }
  tau_hi_out = tau_hi;
  if (HI_ONLY) {  // split path: the bisection runs in its own kernel (bisect_kernel)
    tau_lo_out = ser;
    n_cand = 0;
    return true;
  }
  // --- bisection (ls/provisioner.py:430-437); counts monotone in tau => pinning ---
  if (FAST) {
    phase_bisect_cands<MAXS>(c, tb, w, S, ser, tau_hi, tau_lo_out, n_cand);
    return true;
  }
  double a = ser, b = tau_hi;
  {
    for (int it = 0; it < 60; it++) {
      const double mid = (a + b) / 2.0;
      double km[2] = {inf, inf};
      bool rz = false;
      if (lane < kMaxT) w.tsum[lane] = 0ull;
      __syncwarp();
      for (int slot = 0; slot < 2; slot++) {
        const int s = lane + 32 * slot;
        if (s < S) {
          km[slot] = (ka[slot] == kb[slot]) ? kb[slot] : count_at(w.stage(s), mid, c.bo);
          if (km[slot] == inf) rz = true; else atomicAdd(&w.tsum[w.stage(s).type], sat_count(km[slot]));
        }
      }
      __syncwarp();
      bool bad = rz || ((lane < c.T) && (w.tsum[lane] > (unsigned long long)c.quota[lane]));
      const bool ok = !__any_sync(0xffffffffu, bad);
      if (ok) { b = mid; kb[0] = km[0]; kb[1] = km[1]; }
      else { a = mid; ka[0] = km[0]; ka[1] = km[1]; }
    }
  }
  tau_lo_out = b;
  cands_prefix<MAXS>(tb, w, S, kb, n_cand);
  return true;
}

}  // namespace hps

namespace hps {

// Phase B: _best_candidate over the implicit candidate set {tau_lo, tau_hi} U breakpoints of
// class leaders (ls/provisioner.py:442-455, 262-314). Returns the chosen tau, or NaN when no
// candidate is feasible (InfeasibleError(gap=1.0), ls/provisioner.py:473-477).
template <int MAXS, bool CERT = false>
__device__ double phase_candidates(const InstanceConsts& c, const DeviceTables& tb,
                                   const WarpSmem<MAXS>& w, int S, double tau_lo, double tau_hi,
                                   int n_cand) {
  const int lane = threadIdx.x & 31;
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  TieBuf buf;
  buf.init();
  int sp = 0;
  for (int i = lane; i < n_cand; i += 32) {
    double tau;
    if (i < 2) {
      tau = (i == 0) ? tau_lo : tau_hi;
    } else {
      const int j = i - 2;
      while (w.pre[sp + 1] <= j) sp++;
      const double m = w.kmin[sp] + (double)(j - w.pre[sp]);
      tau = et_lookup(c, tb, w.st[sp], w.ent[sp], m);
      if (!(tau >= tau_lo && tau <= tau_hi)) continue;
    }
    buf.insert(candidate_cost<MAXS, CERT>(c, tb, w, S, tau), tau);
  }
  const double mf = warp_min(buf.mn);
  if (!(mf < inf)) return __longlong_as_double(0x7ff8000000000000LL);
  const double lim = mf + 1e-15;
  double bt;
  if (__any_sync(0xffffffffu, buf.overflow)) {  // rare: exact second pass with the final limit
    bt = -inf;
    sp = 0;
    for (int i = lane; i < n_cand; i += 32) {
      double tau;
      if (i < 2) {
        tau = (i == 0) ? tau_lo : tau_hi;
      } else {
        const int j = i - 2;
        while (w.pre[sp + 1] <= j) sp++;
        tau = et_lookup(c, tb, w.st[sp], w.ent[sp], w.kmin[sp] + (double)(j - w.pre[sp]));
        if (!(tau >= tau_lo && tau <= tau_hi)) continue;
      }
      if (tau > bt && candidate_cost<MAXS, CERT>(c, tb, w, S, tau) <= lim) bt = tau;
    }
  } else {
    bt = buf.best_tau(lim);
  }
  return warp_max(bt);
}

// Phase C: counts at the chosen tau, add_ps_cores (ls/provisioner.py:486-513) and the final
// evaluate() whose monetary_cost is the score (ls/scoring.py:96-97, ls/costmodel.py:102-167).
template <int MAXS, bool FAST = false>
__device__ __noinline__ void phase_final(const InstanceConsts& c, const DeviceTables& tb, WarpSmem<MAXS>& w,
                            int S, double tau, PlanOut& out) {
  const int lane = threadIdx.x & 31;
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  long long accel = 0, on_ps = 0;
  double emax = 0.0;
  for (int s = lane; s < S; s += 32) {
    double k = w.kmin[s];
    if (w.kmax[s] != k) {
      if (FAST) {
        const TEPair* row = te_row(c, tb, w.st[s].type, w.ent[s]);
        k = (double)count_tab(row, tau, (int)w.kmin[s], (int)w.kmax[s], est_count(w.st[s], tau));
      } else {
        k = count_at(w.st[s], tau, c.bo);
      }
    }
    w.kres[s] = k;
    const int t = w.st[s].type;
    if (!c.is_cpu[t]) accel += (long long)k;
    if (t == c.ps_type) on_ps += (long long)k;
    emax = fmax(emax, et_lookup(c, tb, w.st[s], w.ent[s], k));
  }
  accel = warp_sum_ll(accel);
  on_ps = warp_sum_ll(on_ps);
  emax = warp_max(emax);
  __syncwarp();
  int ps = 0;
  if (c.with_ps && accel != 0) {
    if (c.ps_type < 0) { out.status = HPS_ST_NO_CPU_TYPE; out.cost = __longlong_as_double(0x7ff8000000000000LL); out.gap = 0; return; }
    ps = (int)ceil(c.ps_cores_per_gpu * (double)accel - 1e-9);
    const long long would = on_ps + ps;
    if (would > c.quota[c.ps_type]) {
      out.status = HPS_ST_PS_QUOTA;
      out.gap = clamp_gap((double)(would - c.quota[c.ps_type]) / (double)c.quota[c.ps_type]);
      out.cost = c.penalty_scale * (1.0 + pmax(0.0, out.gap));
      return;
    }
  }
  // evaluate(): overall = min_s B/et_s = B/max_s et_s (division is monotone); zero-time
  // stages give inf (ls/costmodel.py:127-128)
  const double overall = (emax > 0) ? c.batch / emax : inf;
  const double exec_time = (overall > 0 && overall != inf) ? c.work / overall : 0.0;
  double cost = 0.0;
  if (lane == 0) {  // per_type_totals in insertion order (ls/domain.py:342-348)
    int order[kMaxT];
    long long tot[kMaxT];
    int n = 0;
    unsigned seen = 0;
    for (int s = 0; s < S; s++) {
      const int t = w.st[s].type;
      if (!(seen >> t & 1u)) { seen |= 1u << t; order[n] = t; tot[n] = 0; n++; }
      for (int j = 0; j < n; j++)
        if (order[j] == t) { tot[j] += (long long)w.kres[s]; break; }
    }
    if (ps > 0) {
      const int t = c.ps_type;
      if (!(seen >> t & 1u)) { order[n] = t; tot[n] = 0; n++; }
      for (int j = 0; j < n; j++)
        if (order[j] == t) { tot[j] += ps; break; }
    }
    double per_second = 0.0;
    for (int j = 0; j < n; j++) per_second += c.price_s[order[j]] * (double)tot[j];  // price / 3600.0
    cost = exec_time * per_second;
  }
  out.cost = __shfl_sync(0xffffffffu, cost, 0);
  out.status = HPS_ST_OK;
  out.gap = 0.0;
  out.ps = ps;
}

// Phase C on the fast path (quotas <= the table cap, so every count and per-type total fits 32
// bits): counts at the chosen tau from the tables, add_ps_cores (ls/provisioner.py:486-513) and
// evaluate()'s monetary cost (ls/costmodel.py:102-167) with per_type_totals in insertion order
// (ls/domain.py:342-348). One compact out-of-line copy (runs once per plan).
template <int MAXS, class W>
__device__ __forceinline__ void phase_final_fast(const InstanceConsts& c, W& w, int S, double tau,
                                                 PlanOut& out) {
  const int lane = threadIdx.x & 31;
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  int accel = 0, on_ps = 0;
  double emax = 0.0;
  int ks[2] = {0, 0}, ts[2] = {-1, -1};   // count and type of stages lane and lane + 32
#pragma unroll
  for (int slot = 0; slot < 2; slot++) {
    const int s = lane + 32 * slot;
    if (s >= S) continue;
    const int lo = (int)w.kmin[s], hi = (int)w.kmax[s];
    const int k = (lo == hi) ? lo : count_seeded(w.stage(s), w.row[s], tau, lo, hi);
    w.kres[s] = (double)k;
    const int t = w.stage(s).type;
    ks[slot] = k;
    ts[slot] = t;
    if (!c.is_cpu[t]) accel += k;
    if (t == c.ps_type) on_ps += k;
    const double et = __ldg(&HPS_TE(w.row[s], k - 1).et);
    emax = (et > emax) ? et : emax;
  }
  accel = (int)__reduce_add_sync(0xffffffffu, (unsigned)accel);
  on_ps = (int)__reduce_add_sync(0xffffffffu, (unsigned)on_ps);
  emax = warp_max(emax);
  int ps = 0;
  if (c.with_ps && accel != 0) {
    if (c.ps_type < 0) { out.status = HPS_ST_NO_CPU_TYPE; out.cost = __longlong_as_double(0x7ff8000000000000LL); out.gap = 0; return; }
    ps = (int)ceil(c.ps_cores_per_gpu * (double)accel - 1e-9);
    const long long would = (long long)on_ps + ps;
    if (would > c.quota[c.ps_type]) {
      out.status = HPS_ST_PS_QUOTA;
      out.gap = clamp_gap((double)(would - c.quota[c.ps_type]) / (double)c.quota[c.ps_type]);
      out.cost = c.penalty_scale * (1.0 + pmax(0.0, out.gap));
      return;
    }
  }
  // evaluate(): overall = min_s B/et_s = B/max_s et_s (division is monotone); zero-time stages
  // give inf (ls/costmodel.py:127-128)
  const double overall = (emax > 0) ? c.batch / emax : inf;
  const double exec_time = (overall > 0 && overall != inf) ? c.work / overall : 0.0;
  // per-type totals; the sum runs over types in order of first occurrence (the stages that lead
  // their type's MATCH group, visited in stage order), then the PS type
  int f0, f1;
  first_same2(S, ts[0], ts[1], f0, f1);
  unsigned fo0 = __ballot_sync(0xffffffffu, lane < S && f0 == lane);
  unsigned fo1 = __ballot_sync(0xffffffffu, lane + 32 < S && f1 == lane + 32);
  double per_second = 0.0;
  bool first = true, seen_ps = false;
  while (fo0 | fo1) {
    int t;
    if (fo0) { const int j = __ffs(fo0) - 1; fo0 &= fo0 - 1; t = __shfl_sync(0xffffffffu, ts[0], j); }
    else { const int j = __ffs(fo1) - 1; fo1 &= fo1 - 1; t = __shfl_sync(0xffffffffu, ts[1], j); }
    const unsigned tot = __reduce_add_sync(0xffffffffu, (ts[0] == t ? (unsigned)ks[0] : 0u) +
                                                            (ts[1] == t ? (unsigned)ks[1] : 0u));
    const double term = c.price_s[t] * (double)((unsigned long long)tot + (t == c.ps_type ? (unsigned long long)ps : 0ull));
    per_second = first ? term : per_second + term;
    first = false;
    seen_ps |= (t == c.ps_type);
  }
  if (ps > 0 && !seen_ps) {
    const double term = c.price_s[c.ps_type] * (double)ps;
    per_second = first ? term : per_second + term;
  }
  const double cost = exec_time * per_second;
  out.cost = cost;
  out.status = HPS_ST_OK;
  out.gap = 0.0;
  out.ps = ps;
}

// Whole plan on one warp. Returns with out.status == kStPending when the breakpoint count
// may exceed 4096 (the block-per-plan slow path then finishes the plan).
template <int MAXS, bool HYBRID = false>
__device__ void eval_plan_warp(const InstanceConsts& c, const DeviceTables& tb, WarpSmem<MAXS>& w,
                               int d0, int d1, PlanOut& out) {
  out.ps = 0;
  out.gap = 0.0;
  double tau_lo, tau_hi;
  int n_cand;
  if (!phase_stages_bisect<MAXS, HYBRID>(c, tb, w, d0, d1, out, tau_lo, tau_hi, n_cand)) return;
  if (n_cand > kBpLimit) { out.status = kStPending; return; }
  const double tau = phase_candidates<MAXS, HYBRID>(c, tb, w, out.S, tau_lo, tau_hi, n_cand);
  if (tau != tau) {
    out.status = HPS_ST_NO_CANDIDATE; out.gap = 1.0;
    out.cost = c.penalty_scale * (1.0 + 1.0);
    return;
  }
  phase_final<MAXS, HYBRID>(c, tb, w, out.S, tau, out);
}

}  // namespace hps
