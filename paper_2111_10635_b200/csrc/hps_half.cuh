// hps_half.cuh — the quota bisection with TWO plans per warp (models of at most 16 layers).
//
// bisect_kernel gives each plan a warp whose lanes own its stages; with S <= 16 half the lanes
// idle, and the warp-uniform parts (the per-type threshold search and the reference's 60
// replayed halvings) run once per plan. Here each 16-lane half of a warp owns one plan: every
// warp-wide step becomes a 16-lane segment step (xor / up shuffles by 8, 4, 2, 1 stay inside a
// half; each collective names its own half, so the halves may take different paths), and whatever
// the two plans do alike issues once for both. Same arithmetic as bisect_direct /
// cands_prefix (hps_eval.cuh), so the same bits.
#pragma once

namespace hps {

// the 16 lanes of this thread's half: every collective below names exactly its segment (the two
// halves may be at different points of their plans; each half's lanes all reach each call)
__device__ __forceinline__ unsigned seg_mask() { return 0xffffu << (threadIdx.x & 16); }

__device__ __forceinline__ double seg_max(double v) {
  const unsigned am = seg_mask();
#pragma unroll
  for (int o = 8; o; o >>= 1) { const double u = __shfl_xor_sync(am, v, o); v = (u > v) ? u : v; }
  return v;
}
__device__ __forceinline__ double seg_min(double v) {
  const unsigned am = seg_mask();
#pragma unroll
  for (int o = 8; o; o >>= 1) { const double u = __shfl_xor_sync(am, v, o); v = (u < v) ? u : v; }
  return v;
}
__device__ __forceinline__ int seg_sum(int v) {
  const unsigned am = seg_mask();
#pragma unroll
  for (int o = 8; o; o >>= 1) v += __shfl_xor_sync(am, v, o);
  return v;
}
__device__ __forceinline__ float seg_sumf(float v) {
  const unsigned am = seg_mask();
#pragma unroll
  for (int o = 8; o; o >>= 1) v += __shfl_xor_sync(am, v, o);
  return v;
}
__device__ __forceinline__ unsigned seg_or(unsigned v) {
  const unsigned am = seg_mask();
#pragma unroll
  for (int o = 8; o; o >>= 1) v |= __shfl_xor_sync(am, v, o);
  return v;
}
// this half's 16 ballot bits (bit i = segment lane i)
__device__ __forceinline__ unsigned seg_ballot(bool p) {
  const unsigned m = __ballot_sync(seg_mask(), p);
  return (m >> (threadIdx.x & 16)) & 0xffffu;
}

// bisect_direct (hps_eval.cuh) for the plan of this half: segment lane sl owns stage sl
template <class W>
__device__ double bisect_half(const InstanceConsts& c, const W& w, int S, double a, double b, int kb_in,
                              int& kb_out) {
  const int sl = threadIdx.x & 15;
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  const int ty = (sl < S) ? w.stage(sl).type : -1;
  const int kb = (sl < S) ? kb_in : 0;
  const TEPair* row = (sl < S) ? w.row[sl] : nullptr;
  const unsigned present = seg_or(ty >= 0 ? 1u << ty : 0u);
  double tstar = -inf;
  unsigned rem = present;
  while (rem) {
    const int t = __ffs(rem) - 1;
    rem &= rem - 1;
    const int Q = (int)c.quota[t];
    const bool mb = ty == t;
    const double lt = seg_max(mb ? __ldg(&HPS_TE(row, Q).th) : -inf);
    int cnt = mb ? count_seeded(w.stage(sl), row, lt, kb, Q) : 0;
    if (seg_sum(cnt) <= Q) {
      tstar = fmax(tstar, lt);
      continue;
    }
    const int nst = seg_sum(mb ? 1 : 0);
    const float target = (float)Q - 0.5f * (float)nst;
    const float flo = (float)lt, fhi = (float)b;
    float x = flo;
    for (int itn = 0; itn < 12; itn++) {
      float F = 0.0f, dF = 0.0f;
      if (mb) F = q_cont(w.stage(sl), x, dF);
      F = seg_sumf(F);
      dF = seg_sumf(dF);
      if (fabsf(F - target) <= 0.25f || !(dF < 0.0f) || !(F < 3.0e37f)) break;
      float nx = x + F * (1.0f - __fdividef(F, target)) * rcp_approx_f32(dF);
      nx = fminf(fmaxf(nx, flo), fhi);
      const bool done = fabsf(nx - x) <= 1e-7f * x;
      x = nx;
      if (done) break;
    }
    const double te = fmin(fmax((double)x, lt), b);
    cnt = mb ? count_seeded(w.stage(sl), row, te, kb, Q) : 0;
    const int se = seg_sum(cnt);
    double tt;
    if (se <= Q) {   // descending thresholds below te (count increments)
      double nx = -inf;
      if (mb && cnt < Q) {
        const double v = __ldg(&HPS_TE(row, cnt).th);
        if (v >= lt) nx = v;
      }
      int d = Q - se + 1;
      if (d > 48) return __longlong_as_double(0x7ff8000000000000LL);  // poor seed: caller falls back
      tt = lt;
      for (;;) {
        const double e = seg_max(nx);
        if (!(e > -inf)) { tt = lt; break; }
        if (--d == 0) { tt = fmax(e, lt); break; }
        const unsigned own = seg_ballot(nx == e);
        if (sl == __ffs(own) - 1) {
          const int k = ++cnt;
          double v = -inf;
          if (k < Q) {
            v = __ldg(&HPS_TE(row, k).th);
            if (!(v >= lt)) v = -inf;
          }
          nx = v;
        }
      }
    } else {   // ascending thresholds above te (count decrements), down to the count at tau_hi
      double nx = (mb && cnt > kb) ? __ldg(&HPS_TE(row, cnt - 1).th) : inf;
      int d = se - Q;
      if (d > 48) return __longlong_as_double(0x7ff8000000000000LL);
      tt = b;
      for (;;) {
        const double e = seg_min(nx);
        if (!(e < inf)) { tt = b; break; }
        if (--d == 0) { tt = e; break; }
        const unsigned own = seg_ballot(nx == e);
        if (sl == __ffs(own) - 1) {
          const int k = --cnt;
          nx = (k > kb) ? __ldg(&HPS_TE(row, k - 1).th) : inf;
        }
      }
    }
    tstar = fmax(tstar, tt);
  }
  for (int it = 0; it < 60; it++) {   // the reference's halvings (ls/provisioner.py:430-436)
    const double mid = (a + b) / 2.0;
    if (mid >= tstar) b = mid; else a = mid;
  }
  kb_out = (ty >= 0) ? count_seeded(w.stage(sl), row, b, kb, (int)c.quota[ty]) : kb;
  return b;
}

// cands_prefix (hps_eval.cuh) for the plan of this half: kmax, class ids, candidate prefix
template <class W>
__device__ void cands_prefix_half(const DeviceTables& tb, W& w, int S, int kb, int& n_cand) {
  const int sl = threadIdx.x & 15, base = threadIdx.x & 16;
  if (sl < S) {
    w.kmax[sl] = kb;
    w.cls[sl] = tb_class(tb, w.ent[sl]);
  }
  __syncwarp(seg_mask());
  int cnt = 0;
  if (sl < S) {
    bool leader = true;
    for (int q = 0; q < sl; q++)
      if (w.cls[q] == w.cls[sl]) { leader = false; break; }
    const int span = w.kmax[sl] - w.kmin[sl];
    if (leader && span <= kBpLimit) cnt = span + 1;
  }
  const unsigned am = seg_mask();
  int inc = cnt;
#pragma unroll
  for (int o = 1; o < 16; o <<= 1) {
    const int v = __shfl_up_sync(am, inc, o);
    if (sl >= o) inc += v;
  }
  const int tot = __shfl_sync(am, inc, base + 15);
  if (sl < S) w.pre[sl] = inc - cnt;
  if (sl == 0) w.pre[S] = tot;
  __syncwarp(am);
  n_cand = tot + 2;
}

// two plans per warp; falls back to the slow path for the (rare) plan whose bisection seed is
// too far off (the slow kernel re-evaluates it from scratch with the probing bisection)
template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32, HPS_STAGE_MINB / WARPS)
bisect_kernel_h(const InstanceConsts c, const DeviceTables tb, Cont cont, Pending pend) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, half = lane >> 4, sl = lane & 15;
  WarpSmemL<16>& w = reinterpret_cast<WarpSmemL<16>*>(smem_raw)[warp * 2 + half];
  StageBuf<16, false>& sb =
      reinterpret_cast<StageBuf<16, false>*>(smem_raw + (sizeof(WarpSmemL<16>) * WARPS * 2 + 15) / 16 * 16)[warp * 2 + half];
  PlanState<16>* states = reinterpret_cast<PlanState<16>*>(cont.states);
  const unsigned int n = *cont.count;
  const uint64_t gh = ((uint64_t)blockIdx.x * WARPS + warp) * 2 + half, nh = (uint64_t)gridDim.x * WARPS * 2;
  if (sl == 0) {
    mbar_init(&sb.bar[0], 1);
    mbar_init(&sb.bar[1], 1);
    mbar_init_fence();
  }
  __syncwarp();
  auto issue = [&](int slot, uint64_t q) {
    if (sl == 0) {
      fence_proxy_async_smem();
      mbar_arrive_expect_tx(&sb.bar[slot], sizeof(PlanState<16>));
      bulk_g2s(&sb.ps[slot], states + q, sizeof(PlanState<16>), &sb.bar[slot]);
    }
  };
  if (gh < n) issue(0, gh);
  uint32_t it = 0;
  for (uint64_t q = gh; q < n; q += nh, it++) {
    const int slot = it & 1;
    if (q + nh < n) issue(slot ^ 1, q + nh);
    mbar_wait(&sb.bar[slot], (it >> 1) & 1);
    const PlanState<16>& ps = sb.ps[slot];
    PlanState<16>& out = states[q];
    const int S = ps.S;
    if (sl < S) {
      const int e = ps.ent[sl];
      const int type = __ldg(&tb.stages[e].type);
      w.sp[sl] = tb.stages + e;
      w.ent[sl] = e;
      w.row[sl] = tb.te + c.te_off[type] + (int64_t)(e - type * c.P) * (int64_t)(c.et_cap[type] + 1);
      w.kmin[sl] = ps.kmin[sl];
    }
    __syncwarp(seg_mask());
    int klo = 0;
    const double tau_lo = bisect_half(c, w, S, ps.tau_lo, ps.tau_hi, (sl < S) ? ps.kmin[sl] : 0, klo);
    int n_cand = kBpLimit + 1;   // NaN tau_lo (poor seed): the slow path finishes the plan
    if (tau_lo == tau_lo) cands_prefix_half(tb, w, S, klo, n_cand);
    if (n_cand > kBpLimit) {
      if (sl == 0) {
        HPS_STAT(ST_PENDING, 1);
        const unsigned int at = atomicAdd(pend.count, 1u);
        HPS_CHECK(at < pend.cap, "pending list overflow");
        if (at < pend.cap) pend.list[at] = ps.p;
        out.n_cand = -1;
      }
    } else {
      if (sl < S) {
        out.kmax[sl] = w.kmax[sl];
        out.pre[sl] = w.pre[sl];
      }
      if (sl == 0) {
        out.pre[S] = w.pre[S];
        out.tau_lo = tau_lo;
        out.n_cand = n_cand;
      }
    }
    __syncwarp(seg_mask());
  }
}

}  // namespace hps

namespace hps {

__device__ __forceinline__ unsigned long long seg_sum_u64(unsigned long long v) {
  const unsigned am = seg_mask();
#pragma unroll
  for (int o = 8; o; o >>= 1) v += __shfl_xor_sync(am, v, o);
  return v;
}
__device__ __forceinline__ unsigned long long seg_or_u64(unsigned long long v) {
  const unsigned am = seg_mask();
#pragma unroll
  for (int o = 8; o; o >>= 1) v |= __shfl_xor_sync(am, v, o);
  return v;
}

// phase_stages_bisect<16, true, true> (hps_eval.cuh) for the plan of this half: runs, stages,
// min_k1 / tau_hi, serial floor, counts at tau_hi and the quota check (ls/provisioner.py:
// 394-427). Segment lane sl holds the digit of layer sl and builds stage sl.
template <class W>
__device__ bool stage_phase_half(const InstanceConsts& c, const DeviceTables& tb, W& w, int d, PlanOut& out,
                                 double& tau_lo_out, double& tau_hi_out) {
  const int sl = threadIdx.x & 15, base = threadIdx.x & 16;
  const int L = c.L;
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  const unsigned am = seg_mask();
  const int prev = __shfl_up_sync(am, d, 1);   // (segment lane 0 ignores it)
  const bool start = (sl < L) && (sl == 0 || d != prev);
  const unsigned m = seg_ballot(start);
  if (seg_ballot(sl < L && (d < 0 || d >= c.T))) {
    out.status = HPS_ST_INVALID; out.cost = __longlong_as_double(0x7ff8000000000000LL); out.gap = 0; out.S = 0;
    return false;
  }
  const int S = __popc(m);
  out.S = S;
  int first = 0, last = 0;
  if (sl < S) {
    first = (int)__fns(m, 0, sl + 1);
    last = (sl + 1 < S) ? (int)__fns(m, 0, sl + 2) - 1 : L - 1;
  }
  const int type = __shfl_sync(am, d, base + (first & 15));
  bool invalid = false;
  if (sl < S) {
    const int e = entry_index(c.P, type, first, last);
    w.bind(sl, tb.stages + e);
    w.ent[sl] = e;
    w.row[sl] = tb.te + c.te_off[type] + (int64_t)(e - type * c.P) * (int64_t)(c.et_cap[type] + 1);
    invalid = (w.stage(sl).valid == 0);
  }
  __syncwarp(am);
  if (seg_ballot(invalid)) {
    out.status = HPS_ST_INVALID; out.cost = __longlong_as_double(0x7ff8000000000000LL); out.gap = 0;
    return false;
  }
  // stage-0 bound and tau_hi (ls/provisioner.py:394-397)
  const int type0 = w.stage(0).type;
  const int last0 = (S > 1) ? (int)__fns(m, 0, 2) - 1 : L - 1;
  const Stage0Info s0 = tb.stage0[type0 * L + last0];
  if (s0.status != HPS_ST_OK) {
    out.status = s0.status; out.gap = s0.gap; out.cost = c.penalty_scale * (1.0 + pmax(0.0, s0.gap));
    return false;
  }
  const double tau_hi = s0.tau_hi;
  // serial floor (ls/provisioner.py:399-412)
  const double ser = seg_max((sl < S) ? fmax(0.0, w.stage(sl).serial) : 0.0);
  if (ser >= tau_hi) {
    out.status = HPS_ST_SERIAL; out.gap = clamp_gap((ser - tau_hi) / tau_hi);
    out.cost = c.penalty_scale * (1.0 + pmax(0.0, out.gap));
    return false;
  }
  // counts at tau_hi and the quotas (ls/provisioner.py:413-427)
  double kb = inf, gapv = 0.0;
  bool raised = false;
  const int ty = (sl < S) ? w.stage(sl).type : -1;
  if (sl < S) {
    double r;
    if (floor_count(w.stage(sl), tau_hi, c.bo, r, gapv)) kb = iceil(r); else raised = true;
  }
  const unsigned rm = seg_ballot(raised);
  unsigned over = 0;
  if (!rm) {
    unsigned present = seg_or(ty >= 0 ? 1u << ty : 0u);
    while (present) {
      const int t = __ffs(present) - 1;
      present &= present - 1;
      const unsigned long long sum = seg_sum_u64(ty == t ? sat_count(kb) : 0ull);
      if (sum > (unsigned long long)c.quota[t]) over |= 1u << t;
    }
  }
  if (rm | over) {
    if (rm) {   // _counts_at(tau_hi) raises from the first raising stage (:414)
      out.status = HPS_ST_FLOOR_TAU_HI;
      out.gap = __shfl_sync(am, gapv, base + __ffs(rm) - 1);
    } else {    // first offending type in ascending id (:418-420), exact Python-int totals
      if (sl < S) w.kres[sl] = kb;
      __syncwarp(am);
      const int off = __ffs(over) - 1;
      double g = 0.0;
      if (sl == 0) {
        u128 tot = 0;
        for (int s = 0; s < S; s++)
          if (w.stage(s).type == off) tot += dbl_to_u128(w.kres[s]);
        g = clamp_gap(int_true_div(tot - (u128)c.quota[off], c.quota[off]));
      }
      out.status = HPS_ST_QUOTA_TAU_HI;
      out.gap = __shfl_sync(am, g, base);
    }
    out.cost = c.penalty_scale * (1.0 + pmax(0.0, out.gap));
    return false;
  }
  if (sl < S) w.kmin[sl] = (int)kb;
  tau_hi_out = tau_hi;
  tau_lo_out = ser;
  return true;
}

}  // namespace hps
