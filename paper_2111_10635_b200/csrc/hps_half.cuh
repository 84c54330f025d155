// hps_half.cuh — the quota bisection with TWO plans per warp (models of at most 16 layers).
//
// bisect_kernel gives each plan a warp whose lanes own its stages; with S <= 16 half the lanes
// idle, and the warp-uniform parts (the per-type threshold search and the reference's 60
// replayed halvings) run once per plan. Here each 16-lane half of a warp owns one plan: every
// warp-wide step becomes a 16-lane segment step (xor / up shuffles by 8, 4, 2, 1 stay inside a
// half; masks come from __activemask, so the halves may take different paths), and whatever
// the two plans do alike issues once for both. Same arithmetic as bisect_direct /
// cands_prefix (hps_eval.cuh), so the same bits.
#pragma once

namespace hps {

__device__ __forceinline__ double seg_max(double v) {
  const unsigned am = __activemask();
#pragma unroll
  for (int o = 8; o; o >>= 1) { const double u = __shfl_xor_sync(am, v, o); v = (u > v) ? u : v; }
  return v;
}
__device__ __forceinline__ double seg_min(double v) {
  const unsigned am = __activemask();
#pragma unroll
  for (int o = 8; o; o >>= 1) { const double u = __shfl_xor_sync(am, v, o); v = (u < v) ? u : v; }
  return v;
}
__device__ __forceinline__ int seg_sum(int v) {
  const unsigned am = __activemask();
#pragma unroll
  for (int o = 8; o; o >>= 1) v += __shfl_xor_sync(am, v, o);
  return v;
}
__device__ __forceinline__ float seg_sumf(float v) {
  const unsigned am = __activemask();
#pragma unroll
  for (int o = 8; o; o >>= 1) v += __shfl_xor_sync(am, v, o);
  return v;
}
__device__ __forceinline__ unsigned seg_or(unsigned v) {
  const unsigned am = __activemask();
#pragma unroll
  for (int o = 8; o; o >>= 1) v |= __shfl_xor_sync(am, v, o);
  return v;
}
// this half's 16 ballot bits (bit i = segment lane i)
__device__ __forceinline__ unsigned seg_ballot(bool p) {
  const unsigned m = __ballot_sync(__activemask(), p);
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
  __syncwarp(__activemask());
  int cnt = 0;
  if (sl < S) {
    bool leader = true;
    for (int q = 0; q < sl; q++)
      if (w.cls[q] == w.cls[sl]) { leader = false; break; }
    const int span = w.kmax[sl] - w.kmin[sl];
    if (leader && span <= kBpLimit) cnt = span + 1;
  }
  const unsigned am = __activemask();
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
    __syncwarp(__activemask());
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
    __syncwarp(__activemask());
  }
}

}  // namespace hps
