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

#ifndef HPS_END_REFINE
#define HPS_END_REFINE 1   // second grid level refines the end cells of the first (not uniform)
#endif
#ifndef HPS_WARM_ROUNDS
#define HPS_WARM_ROUNDS 1          // warm-start rounds of 16 exact evaluations in cand_prep_half (2: -1.7%)
#endif
#ifndef HPS_HALF_BISECT_STAGED
#define HPS_HALF_BISECT_STAGED 1   // bulk-copy staging of the plan states in bisect_kernel_h
#endif

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
  SeedConsts sc;   // this lane's stage seed constants, read once for every search below
  if (sl < S) sc.load(w.stage(sl));
  const unsigned present = seg_or(ty >= 0 ? 1u << ty : 0u);
  double tstar = -inf;
  unsigned rem = present;
  while (rem) {
    const int t = __ffs(rem) - 1;
    rem &= rem - 1;
    const int Q = (int)c.quota[t];
    const bool mb = ty == t;
    const double lt = seg_max(mb ? __ldg(&HPS_TE(row, Q).th) : -inf);
    int cnt = mb ? count_seeded_r(sc, row, lt, kb, Q) : 0;
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
      if (mb) F = q_cont_r(sc, x, dF);
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
    cnt = mb ? count_seeded_r(sc, row, te, kb, Q) : 0;
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
  b = halvings(a, b, tstar, 60);   // the reference's halvings (ls/provisioner.py:430-436)
  kb_out = (ty >= 0) ? count_seeded_r(sc, row, b, kb, (int)c.quota[ty]) : kb;
  return b;
}

// cands_prefix (hps_eval.cuh) for the plan of this half: kmax, class ids, candidate prefix
template <class W>
__device__ void cands_prefix_half(const DeviceTables& tb, W& w, int S, int kb, int& n_cand) {
  const int sl = threadIdx.x & 15, base = threadIdx.x & 16;
  const unsigned am = seg_mask();
  const int cl = (sl < S) ? tb_class(tb, w.ent[sl]) : -1 - sl;
  if (sl < S) {
    w.kmax[sl] = kb;
    w.cls[sl] = cl;
  }
  // class leader = the first stage of its class (one MATCH over the half)
  const bool leader = (__ffs(__match_any_sync(am, cl)) - 1 - base) == sl;
  __syncwarp(am);
  int cnt = 0;
  if (sl < S) {
    const int span = kb - w.kmin[sl];
    if (leader && span <= kBpLimit) cnt = span + 1;
  }
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
  PlanState<16>* states = reinterpret_cast<PlanState<16>*>(cont.states);
  const unsigned int n = *cont.count;
  const uint64_t gh = ((uint64_t)blockIdx.x * WARPS + warp) * 2 + half, nh = (uint64_t)gridDim.x * WARPS * 2;
#if HPS_HALF_BISECT_STAGED
  StageBuf<16, false>& sb =
      reinterpret_cast<StageBuf<16, false>*>(smem_raw + (sizeof(WarpSmemL<16>) * WARPS * 2 + 15) / 16 * 16)[warp * 2 + half];
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
#endif
  uint32_t it = 0;
  for (uint64_t q = gh; q < n; q += nh, it++) {
#if HPS_HALF_BISECT_STAGED
    const int slot = it & 1;
    if (q + nh < n) issue(slot ^ 1, q + nh);
    mbar_wait(&sb.bar[slot], (it >> 1) & 1);
    const PlanState<16>& ps = sb.ps[slot];
#else
    const PlanState<16>& ps = states[q];   // (copied to registers/shared below before `out` is written)
#endif
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

namespace hps {

__device__ __forceinline__ double seg_sumd(double v) {
  const unsigned am = seg_mask();
#pragma unroll
  for (int o = 8; o; o >>= 1) v += __shfl_xor_sync(am, v, o);
  return v;
}

// WarpSmemL (hps_eval.cuh) without the final-phase fields (kres, tsum): the plan view of
// prep_kernel_h, small enough that eight blocks of four warps (16 plans with their SweepSmem) fit
// the 132 KB shared-memory configuration and leave the rest of the SM's 256 KB to the L1
struct WarpSmemP {
  const StageEntry* sp[16];
  int32_t kmin[16];
  int32_t kmax[16];
  int32_t ent[16];
  int32_t cls[16];
  int32_t pre[17];
  const TEPair* row[16];
  __device__ __forceinline__ const StageEntry& stage(int r) const { return *sp[r]; }
};

// interval_cells (hps_sweep.cuh) for the plan of this half: segment lane j holds grid point j
__device__ __noinline__ void interval_cells_half(double t, double L, double d, double thr, double& ta, double& tb,
                                                 double& ta_in, double& tb_in) {
  const int sl = threadIdx.x & 15, base = threadIdx.x & 16;
  const unsigned am = seg_mask();
  const double t1 = __shfl_down_sync(am, t, 1, 16);
  const double L1 = __shfl_down_sync(am, L, 1, 16);
  const double d1 = __shfl_down_sync(am, d, 1, 16);
  double lb;
  if (d >= 0.0) lb = L;
  else if (d1 <= 0.0) lb = L1;
  else {
    const double x = (L1 - L + d * t - d1 * t1) * rcp_1nt(d - d1);
    lb = fmin(fmin(L + d * (x - t), L1 + d1 * (x - t1)), fmin(L, L1));
  }
  const bool keep = (sl < kGrid - 1) && !(lb > thr);   // NaN keeps
  const unsigned mk = seg_ballot(keep);
  if (!mk) { ta = 1.0; tb = 0.0; return; }
  const int f = __ffs(mk) - 1, l = 31 - __clz(mk);
  const double nta = __shfl_sync(am, t, base + f);
  tb = __shfl_sync(am, t, base + l + 1);
  // inner ends of the first and last kept cells (equal to tb / ta when one cell is kept)
  ta_in = __shfl_sync(am, t, base + f + 1);
  tb_in = __shfl_sync(am, t, base + l);
  ta = nta;
}

// cand_prep (hps_sweep.cuh) for the plan of this half (S <= 16): segment lane sl owns stage sl
// and grid point sl; the warm start evaluates the same 32 candidates in two rounds of 16.
template <int MAXS, class W>
__device__ double cand_prep_half(const InstanceConsts& c, const DeviceTables& tb, const W& w, SweepSmem<MAXS>& sw,
                                 int S, double tau_lo, double tau_hi, int n_cand, TieBuf& buf,
                                 int& kbv, double& tb_out) {
  const int sl = threadIdx.x & 15, base = threadIdx.x & 16;
  const unsigned am = seg_mask();
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  const int r = sl;
  const bool mine = r < S;
  const bool pinned = mine && (w.kmax[r] == w.kmin[r]);
  SeedConsts scr;   // stage r's seed constants for the count searches below
  if (mine) scr.load(w.stage(r));
  // class leader: the first stage of r's class (one MATCH over the half instead of a scan)
  const unsigned same = __match_any_sync(am, mine ? w.cls[r] : -1 - sl);
  const int ld = __ffs(same) - 1 - base;
  double prr = 0.0;
  if (mine) {
    prr = c.price_s[w.stage(r).type];
    sw.pr[r] = prr;
    sw.fpr[r] = (float)prr;
    sw.kmi[r] = (int)w.kmin[r];
    sw.kma[r] = (int)w.kmax[r];
    sw.etp[r] = pinned ? __ldg(&HPS_TE(w.row[r], (int)w.kmin[r] - 1).et) : 0.0;
    const int dom = pinned ? 0 : side_dominance(w.stage(r), tau_lo, tau_hi, c.bo);
    sw.dom[r] = dom;
#pragma unroll
    for (int side = 0; side < 2; side++) {   // est_setup (hps_sweep.cuh) from the register copy
      const bool on = (dom != 2 - side) && scr.rb[side] != 0.0f && scr.fr[side] != 0.0f;
      sw.est[r][3 * side + 0] = on ? scr.rb[side] : 0.0f;
      sw.est[r][3 * side + 1] = on ? scr.om[side] : -1.0f;
      sw.est[r][3 * side + 2] = on ? scr.fr[side] : 0.0f;
    }
    sw.lead[r] = (int8_t)ld;
    sw.gex[r] = (ld == r && !pinned) ? __ldg(tb.gex + w.ent[r]) : 0;
  }
  {  // unpinned stages in order, and the pinned stages' part of the bound
    const bool unp = mine && !pinned;
    const double p0 = seg_sumd((mine && pinned) ? prr * w.kmin[r] : 0.0);
    const unsigned m = seg_ballot(unp);
    if (unp) sw.ulist[__popc(m & ((1u << sl) - 1u))] = (int8_t)r;
    if (sl == 0) { sw.nu = __popc(m); sw.p0 = p0; }
  }
  __syncwarp(am);
  const CostScalars cs{c.bo, c.batch, c.work, c.limit};
  const double C = c.work / c.batch;
  const bool grid = tau_hi > tau_lo;
  double g_t = tau_lo, g_L = 0.0, g_d = 0.0;
  if (grid) {
    g_t = grid_point<MAXS>(tau_lo, tau_hi);
    lb_cont<MAXS>(w, sw, S, c.bo, C, g_t, g_L, g_d, true);
  }
  {  // warm start: the 32 candidates of cand_prep, 16 per round
    const double lmin = seg_min(grid ? g_L : 0.0);
    const unsigned at = seg_ballot(grid && g_L == lmin);
    const double tstar = __shfl_sync(am, g_t, base + (at ? __ffs(at) - 1 : 0));
    int cstar = 0;
    bool ok = false;
    if (mine) {
      const int lo = sw.kmi[r], chi = min(sw.kma[r], sw.gex[r]);
      ok = grid && w.pre[r + 1] > w.pre[r] && chi >= lo;
      if (ok) cstar = min(max(count_seeded_r(scr, w.row[r], tstar, lo, sw.kma[r]), lo), chi);
    }
    const unsigned lm = seg_ballot(ok);
    const int nl = __popc(lm);
    int sp = 0;
#pragma unroll 1
    for (int round = 0; round < HPS_WARM_ROUNDS; round++) {
      const int vl = sl + 16 * round;   // the lane of cand_prep's 32-lane warm start
      double tau = -inf;
      int gen = -1;
      if (nl > 0) {
        const int li = vl % nl, k = vl / nl;
        const int rr = __fns(lm, 0, li + 1);
        const int cr = __shfl_sync(am, cstar, base + (rr & 15));
        const int off = (k & 1) ? (k + 1) >> 1 : -(k >> 1);
        const int mm = cr + off;
        if (rr < S && mm >= sw.kmi[rr] && mm <= min(sw.kma[rr], sw.gex[rr])) {
          gen = (rr << 16) | mm;
          tau = __ldg(&HPS_TE(w.row[rr], mm - 1).et);
        }
      } else {
        const int i = (int)(((long long)vl * n_cand) / (16 * HPS_WARM_ROUNDS));
        tau = cand_tau<MAXS>(w, sw, i, sp, tau_lo, tau_hi, gen);
      }
      if (tau >= tau_lo && tau <= tau_hi) eval_insert<MAXS>(cs, w, sw, S, tau, gen, buf);
    }
  }
  const double ub = seg_min(buf.mn);
  double ta = tau_lo, tbh = tau_hi;
  if (grid && ub < inf) {
    const double thr = (ub + 1e-15) * (1.0 + 1e-7);
    double ta_in, tb_in;
    interval_cells_half(g_t, g_L, g_d, thr, ta, tbh, ta_in, tb_in);
#pragma unroll 1
    for (int lvl = 1; lvl < HPS_GRID_LEVELS && ta <= tbh; lvl++) {
#if HPS_END_REFINE
      // L is convex, so {L <= thr} is one interval whose ends lie in the first and last kept
      // cells: with more than one kept cell, 8 points refine each end cell (the interior cell
      // between them keeps its valid tangent bound); one kept cell is refined uniformly
      double t1;
      if (ta_in < tbh && tb_in > ta && ta_in <= tb_in) {
        t1 = (sl < 8) ? ((sl == 7) ? ta_in : ta + (ta_in - ta) * (double)sl * (1.0 / 7))
                      : ((sl == 15) ? tbh : tb_in + (tbh - tb_in) * (double)(sl - 8) * (1.0 / 7));
      } else {
        t1 = grid_point<MAXS>(ta, tbh);
      }
#else
      const double t1 = grid_point<MAXS>(ta, tbh);
#endif
      double L1, d1;
      lb_cont<MAXS>(w, sw, S, c.bo, C, t1, L1, d1, true);
      interval_cells_half(t1, L1, d1, thr, ta, tbh, ta_in, tb_in);
    }
  }
  // count of every stage at tau_b: a candidate tau <= tau_b has count_r(tau) >= count_r(tau_b)
  // for every r (counts are non-increasing), the candidate filter's base (cand_main_half)
  kbv = mine ? sw.kmi[r] : 0;
  if (mine && !pinned && ta <= tbh) kbv = count_seeded_r(scr, w.row[r], tbh, sw.kmi[r], sw.kma[r]);
  tb_out = (ta <= tbh) ? tbh : -inf;
  if (mine) {
    if (w.pre[r + 1] > w.pre[r]) {  // class leader with breakpoints
      const int lo = sw.kmi[r], hi = sw.kma[r];
      int alo = 0, an = 0;
      const int chi = min(hi, sw.gex[r]);
      if (ta <= tbh && chi >= lo) {
        const int ma = kbv;
        const int mb = count_seeded_r(scr, w.row[r], ta, lo, hi);
        alo = max(ma, lo);
        an = max(0, min(mb, chi) - alo + 1);
      }
      sw.alo[r] = alo;
      sw.an[r] = an;
      sw.blo[r] = max(lo, sw.gex[r] + 1);
    } else {
      sw.alo[r] = 0;
      sw.an[r] = 0;
      sw.blo[r] = sw.kma[r] + 1;
    }
  }
  __syncwarp(am);
  return ub;
}

}  // namespace hps

namespace hps {

// per-plan view of candidate_kernel_h (S <= 16): exactly what cost_exact, cand_tau2, the filter and
// the final counts read, packed so that eight blocks of four warps (16 plans) fit the 132 KB
// shared-memory configuration and leave the rest of the SM's 256 KB to the L1 (table loads).
// It serves as both the plan view (row) and the sweep constants of the shared helpers.
struct __align__(16) CandView {
  const TEPair* row[16];
  double pr[16];       // price per second of stage r's type
  double etp[16];      // et at the pinned count (kmin == kmax)
  // per stage, two 16-byte records read by one LDS.128 each: {rb, 1 - frac, frac} of side 0 (oct)
  // and side 1 (odt) = the count_est seeds (a side off per side_dominance is {0, -1, 0}), then
  // pr as FP32 and the counts at tau_hi (low 16 bits) and tau_b (high 16 bits)
  float4 fe[16][2];
  int32_t kmi[16], kma[16];
  int32_t pre2[17];
  int16_t alo[16], an[16], blo[16];
  int8_t lead[16], type[16];
  uint32_t tsum[kMaxT];
  double tb;           // tau_b: right end of the restricted interval (-inf: none)
  float p0f;           // FP32 sum of pr * count over the pinned stages
  uint32_t umask;      // unpinned stages (bit r)
  __device__ __forceinline__ float est_at(int r, int i) const {
    const float4& q = fe[r][i / 3];
    const int j = i % 3;
    return j == 0 ? q.x : (j == 1 ? q.y : q.z);
  }
  __device__ __forceinline__ float fpr(int r) const { return fe[r][0].w; }
};

// FP32 lower bound of P(tau) = sum_r pr_r count_r(tau) at a certified breakpoint tau = et_g(m) in
// [tau_lo, tau_hi]: g's class has count m; every other unpinned stage's count is >= its count at
// tau_hi (at tau_b when tau <= tau_b) and >= count_lb32_est; pinned stages are exact (p0f).
__device__ __forceinline__ float filter_P(const CandView& v, int g, int m, double tau, float tf) {
  const int sh = (tau <= v.tb) ? 16 : 0;   // floor: count at tau_b, else at tau_hi
  float P = v.p0f;
  for (unsigned um = v.umask; um; um &= um - 1) {
    const int r = __ffs(um) - 1;
    const float4 a = v.fe[r][0], b = v.fe[r][1];
    float lo = 1.0f;   // count_lb32_est over the two sides
#pragma unroll
    for (int side = 0; side < 2; side++) {
      const float rb = side ? b.x : a.x, omf = side ? b.y : a.y, frac = side ? b.z : a.z;
      const float B = tf * rb;
      const float h = B - omf;
      if (rb != 0.0f && h > 1e-3f * B) {
        // count_lb32's bound with fused steps (each rounds once, so the same margins cover it):
        // ee = 4e-7 (kappa + 2) + 1e-6, lo = q (1 - ee)
        const float rh = rcp_approx_f32(h);
        const float ee = __fmaf_rn(4e-7f, B * rh, 1.8e-6f);
        const float q = frac * rh;
        lo = fmaxf(lo, __fmaf_rn(-q, ee, q));
      }
    }
    const int fl = (int)((__float_as_uint(b.w) >> sh) & 0xffffu);
    const int k = (v.lead[r] == g) ? m : max(fl, (int)ceilf(lo));
    P = __fmaf_rn(a.w, (float)k, P);
  }
  return P;
}

// overflow_pass (hps_sweep.cuh) for the plan of this half: candidates strided over 16 lanes
__device__ __noinline__ double overflow_pass_half(const CostScalars cs, const CandView& v, int S, double tau_lo,
                                                  double tau_hi, int n2, double lim) {
  double bt = -__longlong_as_double(0x7ff0000000000000LL);
  int sp = 0;
  for (int i = (threadIdx.x & 15); i < n2; i += 16) {
    int gen;
    const double tau = cand_tau2<16>(v, v, i, sp, tau_lo, tau_hi, gen);
    if (!(tau >= tau_lo && tau <= tau_hi) || !(tau > bt)) continue;
    if (cost_exact<16>(cs, v, v, S, tau, gen) <= lim) bt = tau;
  }
  return bt;
}

// cand_main (hps_sweep.cuh) for the plan of this half (S <= 16): filter rounds of 16 candidates,
// survivors compacted into this half's 32 slots of the warp's queue and evaluated 16 at a time.
// The FP32 bound sums in another order than the 32-lane version; the filter's 1e-5 slack covers
// that (a skipped candidate still costs more than the minimum + 1e-15), so the result is the same.
__device__ double cand_main_half(const InstanceConsts& c, CandView& v, CandQueue& cq, int S, double tau_lo,
                                 double tau_hi, double ub, TieBuf& buf) {
  const int sl = threadIdx.x & 15, base = threadIdx.x & 16;
  const unsigned am = seg_mask();
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  const CostScalars cs{c.bo, c.batch, c.work, c.limit};
  // restricted_prefix over the segment
  const int cnt = (sl < S) ? v.an[sl] + max(0, v.kma[sl] - v.blo[sl] + 1) : 0;
  int inc = cnt;
#pragma unroll
  for (int o = 1; o < 16; o <<= 1) {
    const int u = __shfl_up_sync(am, inc, o);
    if (sl >= o) inc += u;
  }
  const int tot = __shfl_sync(am, inc, base + 15);
  if (sl < S) v.pre2[sl] = inc - cnt;
  if (sl == 0) v.pre2[S] = tot;
  __syncwarp(am);
  const int n2 = 2 + tot;
#ifdef HPS_STATS
  if (sl == 0) {
    HPS_STAT(ST_N2, n2);
    int unc = 0;
    for (int r = 0; r < S; r++) unc += max(0, v.kma[r] - v.blo[r] + 1);
    HPS_STAT(ST_UNCERT, unc);
  }
#endif
  const float fC = (float)(c.work / c.batch);
  {  // unpinned stages in order, and the pinned stages' part of filter_P
    const bool unp = sl < S && v.kma[sl] != v.kmi[sl];
    const unsigned um = seg_ballot(unp);
    const float p0f = seg_sumf((sl < S && !unp) ? v.fpr(sl) * (float)v.kmi[sl] : 0.0f);
    if (sl == 0) { v.umask = um; v.p0f = p0f; }
    __syncwarp(am);
  }
  double* qt = cq.q + 2 * base;      // this half's 32 queue slots
  int32_t* qg = cq.qg + 2 * base;
  int sp = 0, qn = 0;
  const unsigned lt = (1u << sl) - 1u;
  const int rounds = (n2 + 15) >> 4;
  for (int jr = 0; jr < rounds; jr++) {
    const int i = jr * 16 + sl;
    double tau = 0.0;
    int gen = -1;
    bool keep = false;
    if (i < n2) {
      tau = cand_tau2<16>(v, v, i, sp, tau_lo, tau_hi, gen);
      keep = tau >= tau_lo && tau <= tau_hi;
      if (keep && gen >= 0) {   // cost >= C tau P(tau) (E >= tau at a certified breakpoint)
        const float tf = (float)tau;
        const float P = filter_P(v, gen >> 16, gen & 0xffff, tau, tf);
        keep = !((double)(fC * tf * P) * (1.0 - 1e-5) > ub + 1e-15);
      }
    }
    const unsigned mk = seg_ballot(keep);
    if (keep) { qt[qn + __popc(mk & lt)] = tau; qg[qn + __popc(mk & lt)] = gen; }
    qn += __popc(mk);
    __syncwarp(am);
    if (qn >= 16) {
      const double t = qt[qn - 16 + sl];
      const int tg = qg[qn - 16 + sl];
      HPS_STAT(ST_CANDS, 1);
      eval_insert<16>(cs, v, v, S, t, tg, buf);
      qn -= 16;
      ub = fmin(ub, seg_min(buf.mn));
      __syncwarp(am);
    }
  }
  if (sl < qn) {
    HPS_STAT(ST_CANDS, 1);
    eval_insert<16>(cs, v, v, S, qt[sl], qg[sl], buf);
  }
  const double mf = seg_min(buf.mn);
#ifdef HPS_STATS
  {  // analysis only: survivors of the same filter with the final minimum as ub (IDEAL), and with
     // exact counts of every stage except E >= tau (IDEAL2: the best any count bound can do)
    int spx = 0;
    for (int jr = 0; jr < rounds; jr++) {
      const int i = jr * 16 + sl;
      if (i >= n2) continue;
      int gen;
      const double tau = cand_tau2<16>(v, v, i, spx, tau_lo, tau_hi, gen);
      if (!(tau >= tau_lo && tau <= tau_hi)) continue;
      bool keep = true, keep2 = true;
      if (gen >= 0) {
        const float tf = (float)tau;
        const float P = filter_P(v, gen >> 16, gen & 0xffff, tau, tf);
        keep = !((double)(fC * tf * P) * (1.0 - 1e-5) > mf + 1e-15);
        // exact P at tau
        double Px = 0.0;
        for (int r = 0; r < S; r++) {
          int k;
          if (v.kma[r] == v.kmi[r]) k = v.kmi[r];
          else { double et; const int k0 = count_est<16>(v, v, r, tf); k = count_verify<16>(v, v, r, tau, k0, te_pair(v.row[r], k0), te_theta(v.row[r], k0), et); }
          Px += v.pr[r] * (double)k;
        }
        keep2 = !((c.work / c.batch) * tau * Px * (1.0 - 1e-12) > mf + 1e-15);
      }
      if (keep) HPS_STAT(ST_IDEAL, 1);
      if (keep2) HPS_STAT(ST_IDEAL2, 1);
      if (cost_exact<16>(cs, v, v, S, tau, gen) <= mf * (1.0 + 1e-3)) HPS_STAT(ST_NEAR, 1);
    }
  }
#endif
  if (!(mf < inf)) return __longlong_as_double(0x7ff8000000000000LL);
  const double lim = mf + 1e-15;
  double bt;
  if (seg_ballot(buf.overflow)) {  // rare: exact second pass with the final limit
    bt = overflow_pass_half(cs, v, S, tau_lo, tau_hi, n2, lim);
  } else {
    bt = buf.best_tau(lim);
  }
  return seg_max(bt);
}

// phase_final_fast (hps_eval.cuh) for the plan of this half: counts at tau (segment lane sl keeps
// stage sl's in k), add_ps_cores, cost
__device__ void final_half(const InstanceConsts& c, CandView& v, const StageEntry* st, int S, double tau,
                           PlanOut& out, int& k) {
  const int sl = threadIdx.x & 15, base = threadIdx.x & 16;
  const unsigned am = seg_mask();
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  int accel = 0, on_ps = 0, t = -1;
  double emax = 0.0;
  k = 0;
  if (sl < S) {
    const int lo = v.kmi[sl], hi = v.kma[sl];
    if (lo == hi) {
      k = lo;
    } else {   // seed constants from the view (a dominated side is off: still a valid seed)
      SeedConsts sc;
      const float4 a = v.fe[sl][0], b = v.fe[sl][1];
      sc.rb[0] = a.x; sc.om[0] = a.y; sc.fr[0] = a.z;
      sc.rb[1] = b.x; sc.om[1] = b.y; sc.fr[1] = b.z;
      k = count_seeded_r(sc, v.row[sl], tau, lo, hi);
    }
    t = v.type[sl];
    if (!c.is_cpu[t]) accel = k;
    if (t == c.ps_type) on_ps = k;
    emax = __ldg(&HPS_TE(v.row[sl], k - 1).et);
  }
  accel = seg_sum(accel);
  on_ps = seg_sum(on_ps);
  emax = seg_max(emax);
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
  // evaluate(): overall = B / max_s et_s; zero-time stages give inf (ls/costmodel.py:127-128)
  const double overall = (emax > 0) ? c.batch / emax : inf;
  const double exec_time = (overall > 0 && overall != inf) ? c.work / overall : 0.0;
  // per-type totals, summed over types in order of first occurrence, then the PS type: the
  // first-occurrence stages are the lanes that lead their type's MATCH group, visited in order
  const unsigned same = __match_any_sync(am, t >= 0 ? t : 64 + sl);
  unsigned fo = seg_ballot(t >= 0 && (__ffs(same) - 1 - base) == sl);
  double per_second = 0.0;
  bool first = true, seen_ps = false;
  while (fo) {
    const int j = __ffs(fo) - 1;
    fo &= fo - 1;
    const int ty = __shfl_sync(am, t, base + j);
    const int tot = seg_sum(t == ty ? k : 0);
    const double term = c.price_s[ty] * (double)((unsigned long long)(unsigned)tot +
                                                  (ty == c.ps_type ? (unsigned long long)ps : 0ull));
    per_second = first ? term : per_second + term;
    first = false;
    seen_ps |= (ty == c.ps_type);
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

}  // namespace hps

