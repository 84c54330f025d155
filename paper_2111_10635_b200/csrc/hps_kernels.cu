// hps_kernels.cu — sm_100a kernels of the plan evaluator and the extern "C" ABI (include/hps.h).
//
// Kernels (SURVEY.md §2 numbering):
//   setup      stage table (Neumaier aggregates of every (type, first, last) run), stage-0
//              exits (min_k1 / tau_hi) and the ET table et(e, m) for m <= quota
//   K1         score_kernel       PlanScorer.__call__ over a plan batch, one warp per plan
//   K2         argmin_kernel      brute_force / random_search loop with a fused (cost, rank)
//                                 argmin; plans decoded (enumeration index) or generated
//                                 (numpy PCG64 + Lemire) in-kernel
//   K7         slow_kernel        block per plan for the >4096-breakpoint path: sort, dedup,
//                                 Newton/golden + subsample (ls/provisioner.py:456-470)
//   reduce     finish_argmin      deterministic merge of per-block keys
#include "hps_launch.h"
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "hps_sweep.cuh"
#include "hps_tma.cuh"

using namespace hps;

namespace {

thread_local std::string g_last_error;

int set_err(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

#define CUDA_TRY(expr)                                                                  \
  do {                                                                                  \
    cudaError_t _e = (expr);                                                            \
    if (_e != cudaSuccess)                                                              \
      return set_err(HPS_E_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));   \
  } while (0)

constexpr int kEtCapMax = 16384;
#ifndef HPS_SLOW_THREADS
#define HPS_SLOW_THREADS 256
#endif
constexpr int kSlowThreads = HPS_SLOW_THREADS;
#ifndef HPS_SLOW_SORT
#define HPS_SLOW_SORT 2048  // 2048/4096 (3 blocks per SM) measured 0.8-1.2% faster per sweep than 8192 (2)
#endif
constexpr int kSlowSmemSort = HPS_SLOW_SORT;  // doubles of dynamic shared memory for the slow path's sort

// ------------------------------------------------------------------ plan sources

struct PlanSource {
  int32_t mode;          // 0 plans array, 1 enumeration index, 2 numpy PCG64 integers(),
                         // 3 subtrees of surviving prefixes (enumeration index
                         //   prefixes[q / stride] * stride + q % stride, q = begin + p)
  int32_t tbits;         // mode 2: log2(T)
  const uint8_t* plans;  // mode 0
  uint64_t begin;        // mode 1/2: first enumeration index / first random plan
  uint64_t stride;       // mode 1: plan p is enumeration index begin + p * stride; mode 3: subtree size
  const uint32_t* prefixes;  // mode 3: surviving prefix ids
  uint64_t tpow[kMaxL];  // mode 1: T^(L-1-l)
  // mode 2: state after (first*L/2 + 1) steps is computed per warp; A_j/C_j advance it by j
  uint64_t s0_hi, s0_lo, inc_hi, inc_lo;
  uint64_t jA_hi[33], jA_lo[33], jC_hi[33], jC_lo[33];
};

__host__ __device__ __forceinline__ u128 mk(uint64_t hi, uint64_t lo) { return ((u128)hi << 64) | lo; }

// digits of plan number p (relative to src.begin) for this lane: d0 = layer lane, d1 = lane+32
template <int MODE>
__device__ __forceinline__ void load_digits(const InstanceConsts& c, const PlanSource& src,
                                            uint64_t p, int& d0, int& d1, u128& rank) {
  const int lane = threadIdx.x & 31;
  const int L = c.L;
  d0 = 0;
  d1 = 0;
  if (MODE == 0) {
    const uint8_t* row = src.plans + p * (uint64_t)L;
    if (lane < L) d0 = row[lane];
    if (lane + 32 < L) d1 = row[lane + 32];
    rank = 0;
    if (src.tbits > 0) {  // argmin over an explicit batch: packed lexicographic rank
      u128 part = 0;
      for (int slot = 0; slot < 2; slot++) {
        const int l = lane + 32 * slot;
        if (l < L) part |= (u128)((slot ? d1 : d0) & ((1 << src.tbits) - 1)) << ((L - 1 - l) * src.tbits);
      }
      uint64_t hi = (uint64_t)(part >> 64), lo = (uint64_t)part;
      for (int o = 16; o; o >>= 1) {
        hi |= __shfl_xor_sync(0xffffffffu, hi, o);
        lo |= __shfl_xor_sync(0xffffffffu, lo, o);
      }
      rank = mk(hi, lo);
    }
  } else if (MODE == 1 || MODE == 3) {
    uint64_t idx;
    if (MODE == 1) {
      idx = src.begin + p * src.stride;
    } else {
      const uint64_t q = src.begin + p;
      const uint64_t r = q / src.stride;
      idx = (uint64_t)__ldg(src.prefixes + r) * src.stride + (q - r * src.stride);
    }
    if (idx < 0xffffffffull && src.tpow[0] < 0xffffffffull) {  // 32-bit division is much cheaper
      const uint32_t i32 = (uint32_t)idx, t32 = (uint32_t)c.T;
      if (lane < L) d0 = (int)((i32 / (uint32_t)src.tpow[lane]) % t32);
      if (lane + 32 < L) d1 = (int)((i32 / (uint32_t)src.tpow[lane + 32]) % t32);
    } else {
      if (lane < L) d0 = (int)((idx / src.tpow[lane]) % (uint64_t)c.T);
      if (lane + 32 < L) d1 = (int)((idx / src.tpow[lane + 32]) % (uint64_t)c.T);
    }
    rank = idx;
  } else {
    const uint64_t g = src.begin + p;
    if (c.T > 1) {
      // 32-bit half h = g*L + l of the PCG64 stream: draw h>>1, low half first
      const u128 h0 = (u128)g * (u128)L;
      const u128 base = h0 >> 1;
      u128 sb = 0;
      if (lane == 0) sb = pcg_advance(mk(src.s0_hi, src.s0_lo), mk(src.inc_hi, src.inc_lo), base + 1);
      uint64_t sb_hi = __shfl_sync(0xffffffffu, (uint64_t)(sb >> 64), 0);
      uint64_t sb_lo = __shfl_sync(0xffffffffu, (uint64_t)sb, 0);
      sb = mk(sb_hi, sb_lo);
      for (int slot = 0; slot < 2; slot++) {
        const int l = lane + 32 * slot;
        if (l < L) {
          const u128 h = h0 + (u128)l;
          const int j = (int)((h >> 1) - base);
          const u128 st = mk(src.jA_hi[j], src.jA_lo[j]) * sb + mk(src.jC_hi[j], src.jC_lo[j]);
          const uint64_t v = pcg_output(st);
          const uint32_t u = (h & 1) ? (uint32_t)(v >> 32) : (uint32_t)v;
          const int dg = (int)(u >> (32 - src.tbits));
          if (slot == 0) d0 = dg; else d1 = dg;
        }
      }
    }
    // lexicographic rank: base-T digits, layer 0 most significant (T = 2^tbits)
    u128 part = 0;
    for (int slot = 0; slot < 2; slot++) {
      const int l = lane + 32 * slot;
      if (l < L) part |= (u128)(slot ? d1 : d0) << ((L - 1 - l) * src.tbits);
    }
    uint64_t hi = (uint64_t)(part >> 64), lo = (uint64_t)part;
    for (int o = 16; o; o >>= 1) {
      hi |= __shfl_xor_sync(0xffffffffu, hi, o);
      lo |= __shfl_xor_sync(0xffffffffu, lo, o);
    }
    rank = mk(hi, lo);
  }
}

// ------------------------------------------------------------------ argmin keys

struct Key {
  double cost;  // +inf = nothing
  uint64_t hi, lo;
  uint32_t status;
};

__device__ __forceinline__ bool key_less(const Key& a, const Key& b) {
  if (a.cost != b.cost) return a.cost < b.cost;
  if (a.hi != b.hi) return a.hi < b.hi;
  return a.lo < b.lo;
}

struct KeyPart {  // per-block partial of an argmin launch
  Key best;
  unsigned long long evaluated, feasible;
  uint32_t flags;  // bit0: a plan needed NO_CPU_TYPE, bit1: INVALID
};

struct Outputs {  // mode 0 per-plan outputs (HpsPlanResults)
  double* cost;
  uint8_t* status;
  double* gap;
  int32_t* ps;
  int32_t* num_stages;
  int32_t* k;
};

struct Pending {
  unsigned long long* list;  // plan numbers that need the slow path
  unsigned int* count;
  unsigned int cap;          // == the plans of the launch it serves: every plan is pushed at most
                             // once per super-chunk, so the list cannot overflow (run_super)
};

template <int MAXS, class W>
__device__ __forceinline__ void write_plan(const InstanceConsts& c, const W& w,
                                           const Outputs& o, uint64_t p, const PlanOut& r) {
  const int lane = threadIdx.x & 31;
  const bool ok = (r.status & 0x7f) == HPS_ST_OK;
  const bool counts = ok || (r.status & 0x7f) == HPS_ST_PS_QUOTA;  // final counts exist
  if (lane == 0) {
    o.cost[p] = r.cost;
    o.status[p] = (uint8_t)r.status;
    if (o.gap) o.gap[p] = r.gap;
    if (o.ps) o.ps[p] = ok ? r.ps : 0;
    if (o.num_stages) o.num_stages[p] = r.S;
  }
  if (o.k) {
    for (int s = lane; s < c.L; s += 32)
      o.k[p * (uint64_t)c.L + s] = (counts && s < r.S) ? (int32_t)w.kres[s] : 0;
  }
}

// ------------------------------------------------------------------ K1 / K2

template <int MAXS, int WARPS, bool ARGMIN, bool FAST, int SRC>
#ifndef HPS_MINB
#define HPS_MINB 24
#endif
__global__ void __launch_bounds__(WARPS * 32, HPS_MINB / WARPS)
eval_kernel(const InstanceConsts c, const DeviceTables tb, const PlanSource src, uint64_t n,
            Outputs o, Pending pend, int feasible_only, KeyPart* parts) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  WarpSmem<MAXS>* sm = reinterpret_cast<WarpSmem<MAXS>*>(smem_raw);
  SweepSmem<MAXS>* ss = reinterpret_cast<SweepSmem<MAXS>*>(smem_raw + sizeof(WarpSmem<MAXS>) * WARPS);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  WarpSmem<MAXS>& w = sm[warp];
  const uint64_t gw = (uint64_t)blockIdx.x * WARPS + warp, nw = (uint64_t)gridDim.x * WARPS;
  Key best;
  best.cost = __longlong_as_double(0x7ff0000000000000LL);
  best.hi = best.lo = ~0ull;
  best.status = 0;
  unsigned long long feas = 0;
  uint32_t flags = 0;
  for (uint64_t p = gw; p < n; p += nw) {
    int d0, d1;
    u128 rank;
    load_digits<SRC>(c, src, p, d0, d1, rank);
    PlanOut r;
#ifdef HPS_HYBRID
    if (FAST) eval_plan_warp<MAXS, true>(c, tb, w, d0, d1, r);
#else
    if (FAST) eval_plan_fast<MAXS>(c, tb, w, ss[warp], d0, d1, r);
#endif
    else eval_plan_warp<MAXS>(c, tb, w, d0, d1, r);
    if (lane == 0) HPS_STAT(ST_PLANS, 1);
    if (r.status == kStPending) {
      if (lane == 0) {
        HPS_STAT(ST_PENDING, 1);
        unsigned int at = atomicAdd(pend.count, 1u);
        HPS_CHECK(at < pend.cap, "pending list overflow");
        if (at < pend.cap) pend.list[at] = p;
      }
    } else if (!ARGMIN) {
      write_plan<MAXS>(c, w, o, p, r);
    } else {
      const int code = r.status & 0x7f;
      if (code == HPS_ST_OK) feas++;
      if (code == HPS_ST_NO_CPU_TYPE) flags |= 1u;
      if (code == HPS_ST_INVALID) flags |= 2u;
      const bool take = feasible_only ? (code == HPS_ST_OK) : (code != HPS_ST_NO_CPU_TYPE && code != HPS_ST_INVALID);
      if (take) {
        Key k{r.cost, (uint64_t)(rank >> 64), (uint64_t)rank, (uint32_t)r.status};
        if (key_less(k, best)) best = k;
      }
    }
    __syncwarp();
  }
  if (ARGMIN && lane == 0) parts[gw] = KeyPart{best, 0ull, feas, flags};  // one partial per warp
}

// ------------------------------------------------------------------ K7 slow path

// _CostModel.real_cost (ls/provisioner.py:230-249), evaluated by one warp: lanes compute the
// stages' real counts and times; the per_second sum stays CPython's sequential Neumaier sum in
// stage order (lane 0), so the value is bit-identical to the reference's. Each warp of the slow
// block has its own term row, so the block evaluates up to 8 points at once.
__device__ double real_cost_dev(const InstanceConsts& c, const WarpSmem<64>& w, int S, double tau) {
  const int lane = threadIdx.x & 31;
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  __shared__ double terms_all[kSlowThreads / 32][64];
  double* terms = terms_all[threadIdx.x >> 5];
  bool raised = false;
  double et = 0.0;
  for (int s = lane; s < S; s += 32) {
    double r, g;
    if (!floor_count(w.st[s], tau, c.bo, r, g)) { raised = true; continue; }
    const double k = pmax(1.0, r);
    et = fmax(et, stage_et(w.st[s], k));  // max over stages: order-free
    terms[s] = c.price_s[w.st[s].type] * k;
  }
  if (__any_sync(0xffffffffu, raised)) return inf;
  et = warp_max(et);
  __syncwarp();
  double out = 0.0;
  if (lane == 0) {
    if (et <= 0) {
      out = 0.0;
    } else {
      const double thr = c.batch / et;
      if (!(thr > c.limit)) {
        out = inf;
      } else {
        PySum ps;
        for (int s = 0; s < S; s++) ps.add(terms[s]);
        out = c.work / thr * ps.result();
      }
    }
  }
  return __shfl_sync(0xffffffffu, out, 0);
}

// Block-parallel continuous search of the >4096-breakpoint path. The reference's sequence of
// points and comparisons is kept exactly; only independent real_cost evaluations run on
// different warps at the same time.
struct SlowSearch {
  double x[kSlowThreads / 32];   // points evaluated this round (one per warp)
  double f[kSlowThreads / 32];
};

// every warp w < n evaluates x[w] into f[w]
__device__ __forceinline__ void eval_points(const InstanceConsts& c, const WarpSmem<64>& w, int S, SlowSearch& ss,
                                            int n) {
  const int warp = threadIdx.x >> 5;
  __syncthreads();
  if (warp < n) {
    const double v = real_cost_dev(c, w, S, ss.x[warp]);
    if ((threadIdx.x & 31) == 0) ss.f[warp] = v;
  }
  __syncthreads();
}

// _newton_minimize (ls/provisioner.py:317-345): the three finite-difference points of an
// iteration are evaluated by three warps; the convergence check's point follows.
__device__ bool newton_block(const InstanceConsts& c, const WarpSmem<64>& w, int S, double lo, double hi,
                             SlowSearch& ss, double& xo) {
  const double h = pmax(c.fd_step * (hi - lo), 1e-12);
  double x = pmin(hi - h, lo + pmax(h, (hi - lo) * 0.25));
  if (x <= lo + h) return false;
  for (int it = 0; it < c.newton_max_iters; it++) {
    if (threadIdx.x == 0) { ss.x[0] = x - h; ss.x[1] = x; ss.x[2] = x + h; }
    eval_points(c, w, S, ss, 3);
    const double fm = ss.f[0], f0 = ss.f[1], fp = ss.f[2];
    if (!(isfinite(fm) && isfinite(f0) && isfinite(fp))) return false;
    const double d1 = (fp - fm) / (2.0 * h);
    const double d2 = (fp - 2.0 * f0 + fm) / (h * h);
    if (fabs(d2) < 1e-18) return false;
    const double step = d1 / d2;
    const double xn = x - step;
    if (!isfinite(xn) || xn < lo || xn > hi) return false;
    if (fabs(xn - x) < c.newton_tol * pmax(1.0, fabs(x))) {
      if (threadIdx.x == 0) ss.x[0] = xn;
      eval_points(c, w, S, ss, 1);
      if (ss.f[0] <= f0 + 1e-12) { xo = xn; return true; }
      return false;
    }
    x = xn;
  }
  return false;
}

// _golden_minimize (ls/provisioner.py:348-371). The 17-point scan is evaluated 8 points at a
// time. Each golden iteration evaluates one new point whose position depends on the earlier
// comparisons; the block evaluates the 7 candidate points of the next 3 iterations (the binary
// tree of outcomes of iterations 2 and 3; iteration 1's outcome is already known) and then
// replays the 3 iterations exactly, so 60 iterations take 20 rounds of evaluation.
__device__ double golden_block(const InstanceConsts& c, const WarpSmem<64>& w, int S, double lo, double hi,
                               SlowSearch& ss) {
  if (hi <= lo) return lo;
  constexpr int n = 17, kW = kSlowThreads / 32;
  double vals[n];
  for (int i0 = 0; i0 < n; i0 += kW) {
    if (threadIdx.x == 0)
      for (int q = 0; q < kW && i0 + q < n; q++) ss.x[q] = lo + (hi - lo) * (double)(i0 + q) / (double)(n - 1);
    eval_points(c, w, S, ss, min(kW, n - i0));
    for (int q = 0; q < kW && i0 + q < n; q++) vals[i0 + q] = ss.f[q];
  }
  int best = 0;
  for (int i = 1; i < n; i++)
    if (vals[i] < vals[best]) best = i;
  auto xs = [&](int i) { return lo + (hi - lo) * (double)i / (double)(n - 1); };   // xs[i] as the scan
  double a = xs(best > 0 ? best - 1 : 0), b = xs(best + 1 < n ? best + 1 : n - 1);
  const double inv_phi = (sqrt(5.0) - 1.0) / 2.0;
  double cc = b - inv_phi * (b - a), dd = a + inv_phi * (b - a);
  if (threadIdx.x == 0) { ss.x[0] = cc; ss.x[1] = dd; }
  eval_points(c, w, S, ss, 2);
  double fc = ss.f[0], fd = ss.f[1];
  // one iteration of the reference's loop; `take_c` = (fc <= fd); returns the new point
  struct St { double a, b, cc, dd; };
  auto step = [&](St& t, bool take_c) {
    if (take_c) { t.b = t.dd; t.dd = t.cc; t.cc = t.b - inv_phi * (t.b - t.a); return t.cc; }
    t.a = t.cc; t.cc = t.dd; t.dd = t.a + inv_phi * (t.b - t.a); return t.dd;
  };
  for (int it = 0; it < 60;) {
    const int depth = min(3, 60 - it);
    // tree nodes: node 0 = iteration it (outcome known); nodes 1-2 = iteration it+1 after
    // outcome bit b1 of its comparison; nodes 3-6 = iteration it+2 after bits (b1, b2)
    if (threadIdx.x == 0) {
      const bool t0 = fc <= fd;
      for (int node = 0; node < (1 << depth) - 1; node++) {
        const int d = (node == 0) ? 0 : (node < 3 ? 1 : 2);
        const int bits = node - ((1 << d) - 1);   // outcome bits of iterations it+1 .. it+d
        St t{a, b, cc, dd};
        double xn = step(t, t0);
        for (int q = 0; q < d; q++) xn = step(t, (bits >> (d - 1 - q)) & 1);
        ss.x[node] = xn;
      }
    }
    eval_points(c, w, S, ss, (1 << depth) - 1);
    // replay the iterations with the evaluated values
    int bits = 0;
    for (int q = 0; q < depth; q++) {
      const bool take_c = fc <= fd;
      if (q > 0) bits = (bits << 1) | (take_c ? 1 : 0);
      const int node = (q == 0) ? 0 : ((1 << q) - 1) + bits;
      St t{a, b, cc, dd};
      step(t, take_c);
      a = t.a; b = t.b; cc = t.cc; dd = t.dd;
      if (take_c) { fd = fc; fc = ss.f[node]; } else { fc = fd; fd = ss.f[node]; }
    }
    it += depth;
  }
  return (a + b) / 2.0;
}

// block-wide exclusive scan helper over per-thread counts (kSlowThreads threads): warp shuffles,
// then the warp totals (tmp[0..nwarps) scratch, tmp[kSlowThreads] = total)
__device__ unsigned block_excl_scan(unsigned v, unsigned* tmp, unsigned& total) {
  constexpr int kW = kSlowThreads / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned inc = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const unsigned y = __shfl_up_sync(0xffffffffu, inc, d);
    if (lane >= d) inc += y;
  }
  if (lane == 31) tmp[warp] = inc;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned acc = 0;
    for (int i = 0; i < kW; i++) { unsigned t = tmp[i]; tmp[i] = acc; acc += t; }
    tmp[kSlowThreads] = acc;
  }
  __syncthreads();
  const unsigned r = tmp[warp] + inc - v;
  total = tmp[kSlowThreads];
  __syncthreads();
  return r;
}

// block-wide fmin / fmax of one double per thread (order-independent); red[0..nwarps) scratch
template <bool MAX>
__device__ double block_minmax(double v, double* red) {
  constexpr int kW = kSlowThreads / 32;
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    const double y = __shfl_xor_sync(0xffffffffu, v, d);
    v = MAX ? fmax(v, y) : fmin(v, y);
  }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double r = red[0];
#pragma unroll
  for (int i = 1; i < kW; i++) r = MAX ? fmax(r, red[i]) : fmin(r, red[i]);
  __syncthreads();
  return r;
}

// FAST: quotas within the threshold tables (HpsInstance::fast): the exact table-driven bisection
// and final phase; otherwise the literal arithmetic of both.
template <bool FAST>
#ifndef HPS_SLOW_MINB
#define HPS_SLOW_MINB 6  // 40 registers, 6 resident blocks per SM: 653 -> 629 ms per cfg3 sweep (4: 633 ms)
#endif
__global__ void __launch_bounds__(kSlowThreads, HPS_SLOW_MINB)
slow_kernel(const InstanceConsts c, const DeviceTables tb, const PlanSource src, Outputs o,
            Pending pend, int argmin_mode, int feasible_only, KeyPart* slow_parts,
            double* scratch, size_t per_block) {
  __shared__ WarpSmem<64> w;
  __shared__ unsigned scan_tmp[kSlowThreads + 1];
  __shared__ double red_d[kSlowThreads];
  __shared__ unsigned long long red_i[kSlowThreads];
  __shared__ double s_tau_lo, s_tau_hi, s_tau_star;
  __shared__ int s_ncand, s_S, s_done;
  __shared__ PlanOut s_out;
  __shared__ u128 s_rank;
  __shared__ int s_bnd[kMaxL + 2];
  __shared__ int s_nseg, s_levels;
  __shared__ SlowSearch s_search;
  extern __shared__ double s_sort[];  // kSlowSmemSort doubles: the sort runs here when it fits
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* raw = scratch + (size_t)blockIdx.x * per_block;  // [per_block/2] sort buffer
  double* cand = raw + per_block / 2;                       // distinct / kept candidates
  const unsigned total = min(*pend.count, pend.cap);  // (count <= cap by construction)
  Key acc;  // per-block argmin partial (thread 0), written once at the end
  acc.cost = __longlong_as_double(0x7ff0000000000000LL);
  acc.hi = acc.lo = ~0ull;
  acc.status = 0;
  unsigned long long acc_feas = 0;
  uint32_t acc_flags = 0;
  for (unsigned item = blockIdx.x; item < total; item += gridDim.x) {
    const uint64_t p = pend.list[item];
    if (warp == 0) {
      int d0, d1;
      u128 rank;
      if (src.mode == 0) load_digits<0>(c, src, p, d0, d1, rank);
      else if (src.mode == 1) load_digits<1>(c, src, p, d0, d1, rank);
      else if (src.mode == 3) load_digits<3>(c, src, p, d0, d1, rank);
      else load_digits<2>(c, src, p, d0, d1, rank);
      PlanOut r;
      r.ps = 0; r.gap = 0.0;
      double tlo = 0, thi = 0;
      int ncand = 0;
      const bool go = phase_stages_bisect<64, FAST>(c, tb, w, d0, d1, r, tlo, thi, ncand);
      if (lane == 0) {
        s_out = r; s_tau_lo = tlo; s_tau_hi = thi; s_ncand = ncand; s_S = r.S; s_done = go ? 0 : 1;
        s_rank = rank;
      }
    }
    __syncthreads();
    if (!s_done) {
      const int S = s_S;
      const double tau_lo = s_tau_lo, tau_hi = s_tau_hi;
      const int nraw = s_ncand;
      int npow = 1;
      while (npow < nraw) npow <<= 1;
      HPS_CHECK((size_t)npow <= per_block / 2, "slow-path sort buffer too small");
      const double inf = __longlong_as_double(0x7ff0000000000000LL);
      // raw candidates: tau_lo, tau_hi, then each class leader's breakpoints et(m) for m from
      // kmax down to kmin (ascending: et is non-increasing in m); values below tau_lo become
      // -inf and above tau_hi +inf, which keeps every segment sorted
      double* srt;
      if (npow <= kSlowSmemSort) {
        srt = s_sort;
      } else {   // merge path: the segments are already sorted, so log2(#segments) merge passes
        if (tid == 0) {   // segment boundaries: {tau_lo, tau_hi}, then every non-empty leader
          int ns = 0;
          s_bnd[ns++] = 0;
          s_bnd[ns] = 2;
          for (int r2 = 0; r2 < S; r2++)
            if (w.pre[r2 + 1] > w.pre[r2]) s_bnd[++ns] = 2 + w.pre[r2 + 1];
          s_nseg = ns;
          int lv = 0;
          while ((1 << lv) < ns) lv++;
          s_levels = lv;
        }
        __syncthreads();
        srt = (s_levels & 1) ? cand : raw;   // the last merge pass writes into raw
      }
      for (int i = tid; i < (srt == s_sort ? npow : nraw); i += kSlowThreads) {
        double v = inf;
        if (i == 0) v = tau_lo;
        else if (i == 1) v = tau_hi;
        else if (i < nraw) {
          const int j = i - 2;
          int lo = 0, hi = S;  // find stage: pre[lo] <= j < pre[lo+1]
          while (hi - lo > 1) { int mid = (lo + hi) / 2; if (w.pre[mid] <= j) lo = mid; else hi = mid; }
          while (w.pre[lo + 1] <= j) lo++;
          v = et_lookup(c, tb, w.st[lo], w.ent[lo], w.kmax[lo] - (double)(j - w.pre[lo]));
          if (v < tau_lo) v = -inf;
          else if (!(v <= tau_hi)) v = inf;
        }
        srt[i] = v;
      }
      __syncthreads();
      bool bitonic = srt == s_sort;
      if (!bitonic) {   // every segment sorted? (et monotone in m needs alpha, beta, profiles >= 0)
        bool bad = false;
        int sg = 0;
        for (int i = tid; i < nraw; i += kSlowThreads) {
          while (s_bnd[sg + 1] <= i) sg++;
          if (i > s_bnd[sg] && srt[i - 1] > srt[i]) bad = true;
        }
        if (__syncthreads_or(bad)) {   // rare: general sort in raw
          for (int i = tid; i < npow; i += kSlowThreads) raw[i] = (i < nraw) ? srt[i] : inf;
          __syncthreads();
          srt = raw;
          bitonic = true;
        }
      }
      if (bitonic) {
        for (int k = 2; k <= npow; k <<= 1)  // bitonic sort ascending (one thread per pair)
          for (int j = k >> 1; j > 0; j >>= 1) {
            for (int t = tid; t < (npow >> 1); t += kSlowThreads) {
              const int i = 2 * t - (t & (j - 1));   // lower index of pair t at distance j
              const int l = i + j;
              const double a = srt[i], b = srt[l];
              const bool up = (i & k) == 0;
              if (up ? (a > b) : (a < b)) { srt[i] = b; srt[l] = a; }
            }
            __syncthreads();
          }
      } else {
        // pairwise merges of adjacent segments (stable merge path per thread's output slice)
        double* src = srt;
        double* dst = (srt == raw) ? cand : raw;
        while (s_nseg > 1) {
          const int ns = s_nseg, n = s_bnd[ns];
          const int per = (n + kSlowThreads - 1) / kSlowThreads;
          int o = min(n, tid * per);
          const int o1 = min(n, o + per);
          int p = 0;
          while (o < o1) {
            while (s_bnd[min(2 * p + 2, ns)] <= o) p++;
            const int b0 = s_bnd[2 * p], bm = s_bnd[min(2 * p + 1, ns)], b1 = s_bnd[min(2 * p + 2, ns)];
            const double* A = src + b0;
            const double* B = src + bm;
            const int nA = bm - b0, nB = b1 - bm;
            const int k = o - b0, end = min(o1, b1) - b0;
            int lo = max(0, k - nB), hi = min(k, nA);
            while (lo < hi) {   // merge path: A elements among the first k outputs (A first on ties)
              const int m = (lo + hi) >> 1;
              if (A[m] <= B[k - 1 - m]) lo = m + 1; else hi = m;
            }
            int ia = lo, ib = k - lo;
            for (int q = k; q < end; q++)
              dst[b0 + q] = (ia < nA && (ib >= nB || A[ia] <= B[ib])) ? A[ia++] : B[ib++];
            o = b0 + end;
          }
          __syncthreads();
          if (tid == 0) {
            const int nn = (ns + 1) / 2;
            for (int q = 1; q <= nn; q++) s_bnd[q] = s_bnd[min(2 * q, ns)];
            s_nseg = nn;
          }
          __syncthreads();
          double* t2 = src; src = dst; dst = t2;
        }
        srt = src;   // == raw (level parity chosen above)
      }
      // distinct finite values -> cand, in sorted order: rounds of kSlowThreads consecutive
      // entries (bank-conflict free), ballot + warp counts; stops at the first +inf (sorted)
      unsigned nc = 0;
      const int nsorted = bitonic ? npow : nraw;   // merged data is unpadded
      for (int r0 = 0; r0 < nsorted; r0 += kSlowThreads) {
        if (!(srt[r0] < inf)) break;  // block-uniform (sorted: +inf only at the end)
        const int i = r0 + tid;
        const bool f = i < nsorted && srt[i] < inf && srt[i] > -inf && (i == 0 || srt[i] != srt[i - 1]);
        const unsigned m = __ballot_sync(0xffffffffu, f);
        if (lane == 0) scan_tmp[warp] = __popc(m);
        __syncthreads();
        unsigned off = nc, tot = 0;
#pragma unroll
        for (int w2 = 0; w2 < kSlowThreads / 32; w2++) {
          const unsigned cw = scan_tmp[w2];
          if (w2 < warp) off += cw;
          tot += cw;
        }
        if (f) cand[off + __popc(m & ((1u << lane) - 1u))] = srt[i];
        nc += tot;
        __syncthreads();
      }
      bool ovf = false;
      if (nc > (unsigned)kBpLimit) {  // ls/provisioner.py:456-470
        ovf = true;
        {  // the reference's search, real_cost evaluations spread over the block's warps
          double ts;
          if (!newton_block(c, w, S, tau_lo, tau_hi, s_search, ts)) ts = golden_block(c, w, S, tau_lo, tau_hi, s_search);
          if (tid == 0) s_tau_star = ts;
        }
        __syncthreads();
        const double ts = s_tau_star;
        // centre = first index of the minimum |cand[i] - tau_star|
        double bd = __longlong_as_double(0x7ff0000000000000LL);
        unsigned long long bi = ~0ull;
        for (unsigned i = tid; i < nc; i += kSlowThreads) {
          double dd = fabs(cand[i] - ts);
          if (dd < bd || (dd == bd && i < bi)) { bd = dd; bi = i; }
        }
        red_d[tid] = bd; red_i[tid] = bi;
        __syncthreads();
        if (tid == 0) {
          for (int i = 1; i < kSlowThreads; i++)
            if (red_d[i] < red_d[0] || (red_d[i] == red_d[0] && red_i[i] < red_i[0])) { red_d[0] = red_d[i]; red_i[0] = red_i[i]; }
        }
        __syncthreads();
        const unsigned long long centre = red_i[0];
        const double step = (double)nc / (double)(kBpLimit / 2);
        // kept indices: {0, nc-1} U {int(i*step)} U [centre-256, centre+256)
        uint8_t* keep = reinterpret_cast<uint8_t*>(raw);  // raw is free now
        for (unsigned i = tid; i < nc; i += kSlowThreads) keep[i] = 0;
        __syncthreads();
        if (tid == 0) { keep[0] = 1; keep[nc - 1] = 1; }
        for (int i = tid; i < kBpLimit / 2; i += kSlowThreads) keep[(unsigned long long)((double)i * step)] = 1;
        const long long lo_i = (long long)centre >= 256 ? (long long)centre - 256 : 0;
        const long long hi_i = (long long)centre + 256 < (long long)nc ? (long long)centre + 256 : (long long)nc;
        for (long long i = lo_i + tid; i < hi_i; i += kSlowThreads) keep[i] = 1;
        __syncthreads();
        const int ch2 = (nc + kSlowThreads - 1) / kSlowThreads;
        const unsigned e0 = min(nc, (unsigned)(tid * ch2)), e1 = min(nc, e0 + ch2);
        unsigned kc = 0;
        for (unsigned i = e0; i < e1; i++) kc += keep[i];
        unsigned nk;
        unsigned pos = block_excl_scan(kc, scan_tmp, nk);
        double* kept = reinterpret_cast<double*>(raw) + (per_block / 4);  // upper half of raw
        for (unsigned i = e0; i < e1; i++)
          if (keep[i]) kept[pos++] = cand[i];
        __syncthreads();
        for (unsigned i = tid; i < nk; i += kSlowThreads) cand[i] = kept[i];
        __syncthreads();
        nc = nk;
      }
      // _best_candidate over the explicit list, all threads
      TieBuf buf;
      buf.init();
      for (unsigned i = tid; i < nc; i += kSlowThreads) buf.insert(candidate_cost<64, true>(c, tb, w, S, cand[i]), cand[i]);
      const double mf = block_minmax<false>(buf.mn, red_d);
      const bool any_ovf = __syncthreads_or(buf.overflow);
      double bt = -__longlong_as_double(0x7ff0000000000000LL);
      if (mf < __longlong_as_double(0x7ff0000000000000LL)) {
        const double lim = mf + 1e-15;
        if (any_ovf) {
          for (unsigned i = tid; i < nc; i += kSlowThreads)
            if (cand[i] > bt && candidate_cost<64, true>(c, tb, w, S, cand[i]) <= lim) bt = cand[i];
        } else {
          bt = buf.best_tau(lim);
        }
      }
      const double tau = block_minmax<true>(bt, red_d);
      if (warp == 0) {
        PlanOut r = s_out;
        if (!(mf < __longlong_as_double(0x7ff0000000000000LL))) {
          r.status = HPS_ST_NO_CANDIDATE; r.gap = 1.0; r.cost = c.penalty_scale * 2.0;
        } else {
          if (FAST) phase_final_fast<64>(c, w, S, tau, r);
          else phase_final<64>(c, tb, w, S, tau, r);
        }
        if (ovf) r.status |= HPS_ST_OVERFLOW_FLAG;
        if (lane == 0) s_out = r;
      }
      __syncthreads();
    }
    // emit
    if (warp == 0) {
      PlanOut r = s_out;
      if (!argmin_mode) {
        write_plan<64>(c, w, o, p, r);
      } else if (lane == 0) {
        const int code = r.status & 0x7f;
        acc_feas += (code == HPS_ST_OK);
        acc_flags |= (code == HPS_ST_NO_CPU_TYPE ? 1u : 0u) | (code == HPS_ST_INVALID ? 2u : 0u);
        const bool take = feasible_only ? (code == HPS_ST_OK) : (code != HPS_ST_NO_CPU_TYPE && code != HPS_ST_INVALID);
        const Key k{r.cost, (uint64_t)(s_rank >> 64), (uint64_t)s_rank, (uint32_t)r.status};
        if (take && key_less(k, acc)) acc = k;
      }
    }
    __syncthreads();
  }
  if (argmin_mode && tid == 0) slow_parts[blockIdx.x] = KeyPart{acc, 0ull, acc_feas, acc_flags};
}

__global__ void finish_argmin(const KeyPart* parts, int nparts, const KeyPart* slow_parts, int nslow,
                              uint64_t evaluated, HpsArgmin* out) {
  __shared__ KeyPart red[256];
  KeyPart acc;
  acc.best.cost = __longlong_as_double(0x7ff0000000000000LL);
  acc.best.hi = acc.best.lo = ~0ull;
  acc.best.status = 0;
  acc.feasible = 0;
  acc.flags = 0;
  for (int i = threadIdx.x; i < nparts + nslow; i += blockDim.x) {
    const KeyPart& k = (i < nparts) ? parts[i] : slow_parts[i - nparts];
    if (key_less(k.best, acc.best)) acc.best = k.best;
    acc.feasible += k.feasible;
    acc.flags |= k.flags;
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < (int)blockDim.x; i++) {
      if (key_less(red[i].best, acc.best)) acc.best = red[i].best;
      acc.feasible += red[i].feasible;
      acc.flags |= red[i].flags;
    }
    out->cost = acc.best.cost;
    out->rank_hi = acc.best.hi;
    out->rank_lo = acc.best.lo;
    out->evaluated = evaluated;
    out->feasible = acc.feasible;
    out->status = acc.best.status;
    out->flags = acc.flags;
  }
}

// merge of per-super-chunk results (argmin_common): same total order, counts summed
__global__ void merge_argmin(const HpsArgmin* keys, int n, uint64_t evaluated, HpsArgmin* out) {
  if (threadIdx.x != 0) return;
  HpsArgmin acc = keys[0];
  for (int i = 1; i < n; i++) {
    const HpsArgmin& k = keys[i];
    const bool less = (k.cost != acc.cost) ? (k.cost < acc.cost)
                      : (k.rank_hi != acc.rank_hi) ? (k.rank_hi < acc.rank_hi) : (k.rank_lo < acc.rank_lo);
    const unsigned long long feas = acc.feasible + k.feasible;
    const uint32_t flags = acc.flags | k.flags;
    if (less) acc = k;
    acc.feasible = feas;
    acc.flags = flags;
  }
  acc.evaluated = evaluated;
  *out = acc;
}

// ------------------------------------------------------------------ setup kernels

struct RawTables {
  const double *oct, *odt, *alpha, *beta;  // [T][L]
};

__global__ void stage_table_kernel(const InstanceConsts c, RawTables raw, StageEntry* out) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= c.T * c.P) return;
  const int t = idx / c.P, pe = idx % c.P;
  int last = 0;
  while ((last + 1) * (last + 2) / 2 <= pe) last++;
  const int first = pe - last * (last + 1) / 2;
  const int L = c.L;
  // build_stages aggregates (ls/domain.py:298-325)
  PySum so, sw, sa, sd, sv, sb;
  bool valid = true;
  for (int l = first; l <= last; l++) {
    const double o = raw.oct[t * L + l], d = raw.odt[t * L + l], a = raw.alpha[t * L + l], b = raw.beta[t * L + l];
    if (o != o || d != d || a != a || b != b) valid = false;
    so.add(o);
    sw.add(o * a);
    sa.add(a);
    sd.add(d);
    sv.add(d * b);
    sb.add(b);
  }
  const int n = last - first + 1;
  StageEntry e;
  e.oct = so.result();
  e.alpha = (e.oct > 0) ? sw.result() / e.oct : sa.result() / (double)n;
  const double odt_sum = sd.result();
  e.beta = (odt_sum > 0) ? sv.result() / odt_sum : sb.result() / (double)n;
  e.odt = raw.odt[t * L + last];
  e.c_oct = e.oct / c.bo;
  e.c_odt = e.odt / c.bo;
  e.oma = 1.0 - e.alpha;
  e.omb = 1.0 - e.beta;
  e.serial = pmax(e.c_oct * e.oma, e.c_odt * e.omb);
  e.valid = valid ? 1 : 0;
  e.type = t;
  e.f_rbo = (e.oct != 0) ? (float)(c.bo / e.oct) : 0.f;
  e.f_rbd = (e.odt != 0) ? (float)(c.bo / e.odt) : 0.f;
  e.f_oma = (float)e.oma;
  e.f_omb = (float)e.omb;
  e.f_alpha = (float)e.alpha;
  e.f_beta = (float)e.beta;
  e.f_coct = (float)e.c_oct;
  e.f_codt = (float)e.c_odt;
  e.rwo = (e.oct != 0) ? 1.0 / e.oct : 0.0;
  e.rwd = (e.odt != 0) ? 1.0 / e.odt : 0.0;
  out[idx] = e;
}

__global__ void stage0_kernel(const InstanceConsts c, const StageEntry* st, Stage0Info* out) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= c.T * c.L) return;
  const int t = idx / c.L, last = idx % c.L;
  const StageEntry& s = st[entry_index(c.P, t, 0, last)];
  Stage0Info r;
  r.status = HPS_ST_OK;
  r.gap = 0.0;
  r.pad = 0;
  // min_k1 (ls/provisioner.py:80-104)
  const double budget = c.limit * c.bo;
  double b[2] = {0.0, 0.0};
  const double works[2] = {s.oct, s.odt}, fr[2] = {s.alpha, s.beta};
  for (int i = 0; i < 2 && r.status == HPS_ST_OK; i++) {
    if (works[i] == 0) continue;
    const double denom = budget - (1.0 - fr[i]) * works[i];
    if (denom <= 0) {
      r.status = HPS_ST_MIN_K1;
      r.gap = clamp_gap(((1.0 - fr[i]) * works[i] - budget) / budget);
    } else {
      b[i] = fr[i] * works[i] / denom;
    }
  }
  double tau_hi = c.tau_limit;
  if (r.status == HPS_ST_OK) {
    const double k1 = pmax(b[0], b[1]);
    if (k1 > 1.0) tau_hi = pmin(tau_hi, stage_et(s, k1));
  }
  r.tau_hi = tau_hi;
  out[idx] = r;
}

// TE[e][m-1] = {et(m), theta(m-1)}; theta(j) = min{tau >= 0 : count(tau) <= j}, found by
// bisection over the bit patterns of non-negative doubles with the exact count function
// (count is monotone in tau, so the predicate is monotone in the bit pattern).
__device__ double theta_exact(const StageEntry& s, double bo, double j) {
  if (count_at(s, 0.0, bo) <= j) return 0.0;
  unsigned long long lo = 0ull, hi = 0x7ff0000000000000ull;  // pred(lo) false, pred(hi) true
  while (hi - lo > 1ull) {
    const unsigned long long mid = lo + ((hi - lo) >> 1);
    if (count_at(s, __longlong_as_double((long long)mid), bo) <= j) hi = mid; else lo = mid;
  }
  return __longlong_as_double((long long)hi);
}

__global__ void te_table_kernel(const InstanceConsts c, const StageEntry* st, TEPair* te, int t,
                                int64_t count, int64_t off) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= count) return;
  const int rows = c.et_cap[t] + 1;
  const int64_t pe = idx / rows;
  const int m = (int)(idx % rows) + 1;
  const StageEntry& s = st[t * c.P + pe];
  TEPair p;
  p.et = stage_et(s, (double)m);
  p.th = (m == 1) ? __longlong_as_double(0x7ff0000000000000LL) : theta_exact(s, c.bo, (double)(m - 1));
  te[off + idx] = p;
}

// Per entry: the largest M such that every breakpoint et(m), m in [1, M], has count exactly m
// (theta(m) <= et(m) gives count <= m, et(m) < theta(m - 1) gives count >= m). A candidate
// tau = et_r(m) with m <= M then pins stage r's count to m and E(tau) >= et_r(m) = tau, which the
// candidate phase's bound uses. (Rounding can break it for large m: the prefix stops there.)
__global__ void gen_exact_init_kernel(const InstanceConsts c, int32_t* gex, int t) {
  const int pe = blockIdx.x * blockDim.x + threadIdx.x;
  if (pe < c.P) gex[t * c.P + pe] = c.et_cap[t];
}
__global__ void gen_exact_kernel(const InstanceConsts c, const TEPair* te, int32_t* gex, int t,
                                 int64_t count) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= count) return;
  const int cap = c.et_cap[t];
  const int64_t pe = idx / cap;
  const int m = (int)(idx % cap) + 1;
  const TEPair* row = te + c.te_off[t] + pe * (cap + 1);
  const double et = HPS_TE(row, m - 1).et;  // et(m); row[m - 1].th = theta(m - 1), row[m].th = theta(m)
  if (!((HPS_TE(row, m).th <= et) && (et < HPS_TE(row, m - 1).th))) atomicMin(gex + t * c.P + pe, m - 1);
}

}  // namespace

// ===================================================================== C ABI

struct HpsInstance {
  InstanceConsts c;
  DeviceTables tb;
  StageEntry* d_stages = nullptr;
  Stage0Info* d_stage0 = nullptr;
  TEPair* d_te = nullptr;
  int32_t* d_cls = nullptr;
  int32_t* d_gex = nullptr;
  bool fast = false;
  std::vector<StageEntry> h_stages;
  int sm_count = 148;
  int grid_per_sm = 32;   // blocks per SM of the split kernels' grid (HPS_GRID_PER_SM; 16: +2%)
  int carveout = -1;      // shared-memory carveout % for the split kernels (HPS_CARVEOUT)
  size_t te_bytes = 0;    // threshold-table size (bounds of the checked build)
  uint64_t chunk = 0;     // plans per split-kernel chunk (HPS_CHUNK; 0: by MAXS)
  bool half_bisect = true;  // L <= 16: two plans per warp in the bisection (HPS_HALF_BISECT=0: one)
  bool half_stage = true;   // L <= 16: two plans per warp in the stage kernel (HPS_HALF_STAGE=0: one)
  bool half_prep = true;    // L <= 16: two plans per warp in the prep kernel (HPS_HALF_PREP=0: one)
  bool half_cand = true;    // L <= 16: two plans per warp in the candidate kernel (HPS_HALF_CAND=0: one)
  int slow_per_sm = -1;   // resident slow_kernel blocks per SM (occupancy API, first use)
  uint64_t super_chunk = 1ull << 26;  // plans per pending-list pass (HPS_SUPERCHUNK; tests shrink it)
  int dev = 0;               // device the tables live on
  size_t sz_stages = 0, sz_stage0 = 0, sz_cls = 0, sz_gex = 0;   // table sizes (allocation cache)
  int pipe = 2;              // split-kernel chunk pipeline streams (HPS_PIPE=1: one stream)
  uint64_t pipe_chunk = 1ull << 20;    // L <= 16 chunk size when pipelined (HPS_CHUNK overrides)
  cudaStream_t aux = nullptr;          // the pipeline's second stream
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
};

namespace {

// checked build: the threshold-table range the kernels of this stream may touch
int chk_bind(const HpsInstance* in, cudaStream_t st) {
#ifdef HPS_CHECKS
  // (a captured copy would read this host stack at replay: graph captures keep the binding of
  // the eager call that precedes them)
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  CUDA_TRY(cudaStreamIsCapturing(st, &cap));
  if (cap != cudaStreamCaptureStatusNone) return HPS_OK;
  const char* lo = reinterpret_cast<const char*>(in->d_te);
  const char* hi = lo + in->te_bytes;
  CUDA_TRY(cudaMemcpyToSymbolAsync(g_chk_te_lo, &lo, sizeof(lo), 0, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyToSymbolAsync(g_chk_te_hi, &hi, sizeof(hi), 0, cudaMemcpyHostToDevice, st));
#else
  (void)in; (void)st;
#endif
  return HPS_OK;
}

// ------------------------------------------------------------------ split fast path
// K1a: runs, exits and the quota bisection; finished (infeasible) plans are emitted here, the
// rest leave a compact state for K1b (candidate phase + final). Two small kernels keep each
// hot loop inside the instruction cache (one fused kernel stalled on instruction fetch).

template <int MAXS>
struct __align__(16) PlanState {   // 16-byte multiple: staged by 1-D bulk copies
  uint64_t p, rank_hi, rank_lo;
  double tau_lo, tau_hi;
  int32_t S, n_cand;
  int32_t ent[MAXS];
  int32_t kmin[MAXS], kmax[MAXS];
  int32_t pre[MAXS + 1];
};

struct Cont {
  void* states;
  unsigned int* count;
  unsigned int cap;   // PlanState slots (the chunk size)
};

// Per-plan result of cand_prep carried from prep_kernel to candidate_kernel.
template <int MAXS>
struct __align__(16) PrepState {
  double ub;
  double tb;      // right end of the restricted interval (-inf: none)
  int8_t dom[MAXS], lead[MAXS];
  int16_t alo[MAXS], an[MAXS], blo[MAXS];
  int16_t kb[MAXS];   // count at tb (half-warp kernels)
};

// double-buffered per-warp staging of the next plan's state records (bulk copies, hps_tma.cuh)
template <int MAXS, bool PREP>
struct StageBuf {
  PlanState<MAXS> ps[2];
  PrepState<MAXS> pp[PREP ? 2 : 1];
  uint64_t bar[2];
};

// shared-memory offset of the staging buffers: after the warp views and the sweep constants
template <int MAXS, int WARPS>
__host__ __device__ constexpr size_t stage_offset() {
  return ((sizeof(WarpSmemL<MAXS>) + sizeof(SweepSmem<MAXS>)) * WARPS + 15) / 16 * 16;
}

// staged only for MAXS <= 16: the 64-stage records (1 KB + 0.5 KB, double-buffered) would cost
// more occupancy (shared memory) than the staging saves
template <int MAXS>
__host__ __device__ constexpr bool staged() { return MAXS <= 16; }
template <int MAXS, bool PREP>
__host__ __device__ constexpr size_t stage_bytes() { return staged<MAXS>() ? sizeof(StageBuf<MAXS, PREP>) : 0; }

template <int MAXS, bool PREP>
__device__ __forceinline__ void stage_init(StageBuf<MAXS, PREP>& sb) {
  if (!staged<MAXS>()) return;
  if ((threadIdx.x & 31) == 0) {
    mbar_init(&sb.bar[0], 1);
    mbar_init(&sb.bar[1], 1);
    mbar_init_fence();
  }
  __syncwarp();
}

// lane 0: stage plan q's PlanState (and PrepState) into slot `slot`; the slot's previous
// contents were read by the whole warp before the __syncwarp that ended that iteration
template <int MAXS, bool PREP>
__device__ __forceinline__ void stage_issue(StageBuf<MAXS, PREP>& sb, int slot, const PlanState<MAXS>* states,
                                            const PrepState<MAXS>* prep, uint64_t q) {
  if (staged<MAXS>() && (threadIdx.x & 31) == 0) {
    fence_proxy_async_smem();
    const uint32_t bytes = sizeof(PlanState<MAXS>) + (PREP ? sizeof(PrepState<MAXS>) : 0);
    mbar_arrive_expect_tx(&sb.bar[slot], bytes);
    bulk_g2s(&sb.ps[slot], states + q, sizeof(PlanState<MAXS>), &sb.bar[slot]);
    if (PREP) bulk_g2s(&sb.pp[slot & (PREP ? 1 : 0)], prep + q, sizeof(PrepState<MAXS>), &sb.bar[slot]);
  }
}


__device__ __forceinline__ void merge_part(KeyPart* parts, uint64_t slot, int first, const Key& best,
                                           unsigned long long feas, uint32_t flags) {
  KeyPart kp{best, 0ull, feas, flags};
  if (!first) {
    const KeyPart o = parts[slot];
    if (key_less(o.best, kp.best)) kp.best = o.best;
    kp.feasible += o.feasible;
    kp.flags |= o.flags;
  }
  parts[slot] = kp;
}

#ifndef HPS_STAGE_MINB
#define HPS_STAGE_MINB 32
#endif
template <int MAXS, int WARPS, bool ARGMIN, int SRC>
__global__ void __launch_bounds__(WARPS * 32, HPS_STAGE_MINB / WARPS)
stage_kernel(const InstanceConsts c, const DeviceTables tb, const PlanSource src, uint64_t p0,
             uint64_t p1, Outputs o, Pending pend, Cont cont, int feasible_only, KeyPart* parts,
             int first) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  WarpSmemL<MAXS>* sm = reinterpret_cast<WarpSmemL<MAXS>*>(smem_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  WarpSmemL<MAXS>& w = sm[warp];
  const uint64_t gw = (uint64_t)blockIdx.x * WARPS + warp, nw = (uint64_t)gridDim.x * WARPS;
  PlanState<MAXS>* states = reinterpret_cast<PlanState<MAXS>*>(cont.states);
  Key best;
  best.cost = __longlong_as_double(0x7ff0000000000000LL);
  best.hi = best.lo = ~0ull;
  best.status = 0;
  uint32_t flags = 0;
  for (uint64_t p = p0 + gw; p < p1; p += nw) {
    int d0, d1;
    u128 rank;
    load_digits<SRC>(c, src, p, d0, d1, rank);
    PlanOut r;
    r.ps = 0;
    r.gap = 0.0;
    double tau_lo, tau_hi;
    int n_cand;
    if (lane == 0) HPS_STAT(ST_PLANS, 1);
    // up to the counts at tau_hi; the bisection runs in bisect_kernel (tau_lo holds the serial
    // floor, the bisection's lower end, until then)
    if (phase_stages_bisect<MAXS, true, true>(c, tb, w, d0, d1, r, tau_lo, tau_hi, n_cand)) {
      unsigned int at = 0;
      if (lane == 0) at = atomicAdd(cont.count, 1u);
      at = __shfl_sync(0xffffffffu, at, 0);
      HPS_CHECK(at < cont.cap, "plan-state chunk overflow");
      PlanState<MAXS>& ps = states[at];
      for (int s = lane; s < r.S; s += 32) {
        ps.ent[s] = w.ent[s];
        ps.kmin[s] = (int32_t)w.kmin[s];
      }
      if (lane == 0) {
        ps.p = p;
        ps.rank_hi = (uint64_t)(rank >> 64);
        ps.rank_lo = (uint64_t)rank;
        ps.tau_lo = tau_lo;
        ps.tau_hi = tau_hi;
        ps.S = r.S;
        ps.n_cand = 0;
      }
    } else if (!ARGMIN) {
      write_plan<MAXS>(c, w, o, p, r);
    } else {
      const int code = r.status & 0x7f;
      if (code == HPS_ST_NO_CPU_TYPE) flags |= 1u;
      if (code == HPS_ST_INVALID) flags |= 2u;
      const bool take = feasible_only ? false : (code != HPS_ST_NO_CPU_TYPE && code != HPS_ST_INVALID);
      if (take) {
        Key k{r.cost, (uint64_t)(rank >> 64), (uint64_t)rank, (uint32_t)r.status};
        if (key_less(k, best)) best = k;
      }
    }
    __syncwarp();
  }
  if (ARGMIN && lane == 0) merge_part(parts, gw, first, best, 0ull, flags);
}

#ifndef HPS_CAND_MINB
#define HPS_CAND_MINB 32
#endif

// K1a': the quota bisection (bisect_direct) and the candidate prefix of each surviving plan,
// in place on its PlanState; plans with more than 4096 breakpoints go to the slow path and
// are marked (n_cand = -1) for the kernels that follow.
template <int MAXS, int WARPS>
__global__ void __launch_bounds__(WARPS * 32, HPS_STAGE_MINB / WARPS)
bisect_kernel(const InstanceConsts c, const DeviceTables tb, Cont cont, Pending pend) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  WarpSmemL<MAXS>* sm = reinterpret_cast<WarpSmemL<MAXS>*>(smem_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  WarpSmemL<MAXS>& w = sm[warp];
  const uint64_t gw = (uint64_t)blockIdx.x * WARPS + warp, nw = (uint64_t)gridDim.x * WARPS;
  PlanState<MAXS>* states = reinterpret_cast<PlanState<MAXS>*>(cont.states);
  StageBuf<MAXS, false>& sb = reinterpret_cast<StageBuf<MAXS, false>*>(
      smem_raw + (sizeof(WarpSmemL<MAXS>) * WARPS + 15) / 16 * 16)[warp];
  const unsigned int n = *cont.count;
  stage_init(sb);
  if (gw < n) stage_issue(sb, 0, states, (const PrepState<MAXS>*)nullptr, gw);
  uint32_t it = 0;
  for (uint64_t q = gw; q < n; q += nw, it++) {
    const int slot = it & 1;
    if (q + nw < n) stage_issue(sb, slot ^ 1, states, (const PrepState<MAXS>*)nullptr, q + nw);
    if (staged<MAXS>()) mbar_wait(&sb.bar[slot], (it >> 1) & 1);
    const PlanState<MAXS>& ps = staged<MAXS>() ? sb.ps[slot] : states[q];   // results go to states[q]
    PlanState<MAXS>& out = states[q];
    const int S = ps.S;
#pragma unroll 1
    for (int s = lane; s < S; s += 32) {
      const int e = ps.ent[s];
      const int type = __ldg(&tb.stages[e].type);
      w.sp[s] = tb.stages + e;
      w.ent[s] = e;
      w.row[s] = tb.te + c.te_off[type] + (int64_t)(e - type * c.P) * (int64_t)(c.et_cap[type] + 1);
      w.kmin[s] = ps.kmin[s];
    }
    __syncwarp();
    double tau_lo;
    int n_cand;
    phase_bisect_cands<MAXS>(c, tb, w, S, ps.tau_lo, ps.tau_hi, tau_lo, n_cand);
    if (n_cand > kBpLimit) {
      if (lane == 0) {
        HPS_STAT(ST_PENDING, 1);
        const unsigned int at = atomicAdd(pend.count, 1u);
        HPS_CHECK(at < pend.cap, "pending list overflow");
        if (at < pend.cap) pend.list[at] = ps.p;
        out.n_cand = -1;
      }
    } else {
      for (int s = lane; s < S; s += 32) out.kmax[s] = (int32_t)w.kmax[s];
      for (int s = lane; s <= S; s += 32) out.pre[s] = w.pre[s];
      if (lane == 0) {
        out.tau_lo = tau_lo;
        out.n_cand = n_cand;
      }
    }
    __syncwarp();
  }
}

}  // namespace
#include "hps_half.cuh"
namespace {

// load_digits for a plan per 16-lane half: segment lane sl gets the digit of layer sl (L <= 16)
template <int MODE>
__device__ __forceinline__ void load_digits_half(const InstanceConsts& c, const PlanSource& src, uint64_t p,
                                                 int& d, u128& rank) {
  const int sl = threadIdx.x & 15, base = threadIdx.x & 16;
  const int L = c.L;
  d = 0;
  rank = 0;
  if (MODE == 1 || MODE == 3) {
    uint64_t idx;
    if (MODE == 1) {
      idx = src.begin + p * src.stride;
    } else {
      const uint64_t q = src.begin + p;
      const uint64_t r = q / src.stride;
      idx = (uint64_t)__ldg(src.prefixes + r) * src.stride + (q - r * src.stride);
    }
    if (sl < L) {
      if (idx < 0xffffffffull && src.tpow[0] < 0xffffffffull)
        d = (int)(((uint32_t)idx / (uint32_t)src.tpow[sl]) % (uint32_t)c.T);
      else
        d = (int)((idx / src.tpow[sl]) % (uint64_t)c.T);
    }
    rank = idx;
    return;
  }
  if (MODE == 0) {
    if (sl < L) d = src.plans[p * (uint64_t)L + sl];
  } else {   // numpy PCG64 integers(): 32-bit half h = g*L + l of the stream, low half first
    const uint64_t g = src.begin + p;
    if (c.T > 1) {
      const u128 h0 = (u128)g * (u128)L;
      const u128 hb = h0 >> 1;
      u128 sb = 0;
      if (sl == 0) sb = pcg_advance(mk(src.s0_hi, src.s0_lo), mk(src.inc_hi, src.inc_lo), hb + 1);
      const unsigned am = seg_mask();
      sb = mk(__shfl_sync(am, (uint64_t)(sb >> 64), base), __shfl_sync(am, (uint64_t)sb, base));
      if (sl < L) {
        const u128 h = h0 + (u128)sl;
        const int j = (int)((h >> 1) - hb);
        const u128 st = mk(src.jA_hi[j], src.jA_lo[j]) * sb + mk(src.jC_hi[j], src.jC_lo[j]);
        const uint64_t v = pcg_output(st);
        const uint32_t u = (h & 1) ? (uint32_t)(v >> 32) : (uint32_t)v;
        d = (int)(u >> (32 - src.tbits));
      }
    }
  }
  if (MODE == 2 || src.tbits > 0) {   // packed lexicographic rank, layer 0 most significant
    u128 part = 0;
    if (sl < L) part = (u128)(d & ((1 << src.tbits) - 1)) << ((L - 1 - sl) * src.tbits);
    rank = mk(seg_or_u64((uint64_t)(part >> 64)), seg_or_u64((uint64_t)part));
  }
}

// prep_kernel with two plans per warp (L <= 16, hps_half.cuh)
template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32, HPS_CAND_MINB / WARPS)
prep_kernel_h(const InstanceConsts c, const DeviceTables tb, Cont cont, PrepState<16>* prep) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, half = lane >> 4, sl = lane & 15;
  const int v = warp * 2 + half;
  WarpSmemP& w = reinterpret_cast<WarpSmemP*>(smem_raw)[v];
  SweepSmem<16>& sw = reinterpret_cast<SweepSmem<16>*>(smem_raw + sizeof(WarpSmemP) * WARPS * 2)[v];
  const PlanState<16>* states = reinterpret_cast<const PlanState<16>*>(cont.states);
  const unsigned int n = *cont.count;
  const uint64_t gh = ((uint64_t)blockIdx.x * WARPS + warp) * 2 + half, nh = (uint64_t)gridDim.x * WARPS * 2;
  // (no shared-memory staging of the plan states here: two plan views per warp already take
  // the shared memory, and the L1 is worth more to this kernel's table loads)
  for (uint64_t q = gh; q < n; q += nh) {
    const PlanState<16>& ps = states[q];
    if (ps.n_cand >= 0) {   // (slow-path plans are finished elsewhere)
      const int S = ps.S;
      if (sl < S) {
        const int e = ps.ent[sl];
        const int type = __ldg(&tb.stages[e].type);
        w.sp[sl] = tb.stages + e;
        w.ent[sl] = e;
        w.row[sl] = tb.te + c.te_off[type] + (int64_t)(e - type * c.P) * (int64_t)(c.et_cap[type] + 1);
        w.kmin[sl] = ps.kmin[sl];
        w.kmax[sl] = ps.kmax[sl];
        w.cls[sl] = tb_class(tb, e);
        w.pre[sl] = ps.pre[sl];
      }
      if (sl == 0) w.pre[S] = ps.pre[S];
      __syncwarp(seg_mask());
      TieBuf buf;
      buf.init();
      int kbv;
      double tbv;
      const double ub = cand_prep_half<16>(c, tb, w, sw, S, ps.tau_lo, ps.tau_hi, ps.n_cand, buf, kbv, tbv);
      PrepState<16>& out = prep[q];
      if (sl < S) {
        out.kb[sl] = (int16_t)kbv;
        out.dom[sl] = (int8_t)sw.dom[sl];
        out.lead[sl] = sw.lead[sl];
        out.alo[sl] = (int16_t)sw.alo[sl];
        out.an[sl] = (int16_t)sw.an[sl];
        out.blo[sl] = (int16_t)sw.blo[sl];
      }
      if (sl == 0) {
        out.ub = ub;
        out.tb = tbv;
      }
    }
    __syncwarp(seg_mask());
  }
}

// candidate_kernel with two plans per warp (L <= 16, hps_half.cuh): each half fills its CandView
// (segment lane sl: stage sl) and shares the warp's survivor queue (32 slots per half)
template <int WARPS, bool ARGMIN>
__global__ void __launch_bounds__(WARPS * 32, HPS_CAND_MINB / WARPS)
candidate_kernel_h(const InstanceConsts c, const DeviceTables tb, Cont cont, const PrepState<16>* prep, Outputs o,
                   int feasible_only, KeyPart* parts, int first) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, half = lane >> 4, sl = lane & 15;
  CandView& v = reinterpret_cast<CandView*>(smem_raw)[warp * 2 + half];
  CandQueue& cq = reinterpret_cast<CandQueue*>(smem_raw + sizeof(CandView) * WARPS * 2)[warp];
  const PlanState<16>* states = reinterpret_cast<const PlanState<16>*>(cont.states);
  const unsigned int n = *cont.count;
  const uint64_t gw = (uint64_t)blockIdx.x * WARPS + warp;
  const uint64_t gh = gw * 2 + half, nh = (uint64_t)gridDim.x * WARPS * 2;
  const unsigned am = seg_mask();
  Key best;
  best.cost = __longlong_as_double(0x7ff0000000000000LL);
  best.hi = best.lo = ~0ull;
  best.status = 0;
  unsigned long long feas = 0;
  uint32_t flags = 0;
  for (uint64_t q = gh; q < n; q += nh) {
    const PlanState<16>& ps = states[q];
    if (ps.n_cand < 0) { __syncwarp(am); continue; }  // slow path
    const int S = ps.S;
    const PrepState<16>& pp = prep[q];
    const StageEntry* st = nullptr;
    if (sl < S) {
      const int e = ps.ent[sl];
      st = tb.stages + e;
      const int type = __ldg(&st->type);
      const int lo = ps.kmin[sl], hi = ps.kmax[sl];
      const TEPair* row = tb.te + c.te_off[type] + (int64_t)(e - type * c.P) * (int64_t)(c.et_cap[type] + 1);
      v.row[sl] = row;
      v.type[sl] = (int8_t)type;
      v.pr[sl] = c.price_s[type];

      v.kmi[sl] = lo;
      v.kma[sl] = hi;
      v.etp[sl] = (lo == hi) ? __ldg(&HPS_TE(row, lo - 1).et) : 0.0;
      const int dom = pp.dom[sl];
      float4 fr[2];
#pragma unroll
      for (int side = 0; side < 2; side++) {   // est_setup (hps_sweep.cuh)
        const float rb = __ldg(side ? &st->f_rbd : &st->f_rbo);
        const float frac = __ldg(side ? &st->f_beta : &st->f_alpha);
        const bool on = (dom != 2 - side) && rb != 0.0f && frac != 0.0f;
        fr[side].x = on ? rb : 0.0f;
        fr[side].y = on ? __ldg(side ? &st->f_omb : &st->f_oma) : -1.0f;
        fr[side].z = on ? frac : 0.0f;
      }
      fr[0].w = (float)c.price_s[type];
      fr[1].w = __uint_as_float((uint32_t)(lo & 0xffff) | ((uint32_t)(pp.kb[sl] & 0xffff) << 16));
      v.fe[sl][0] = fr[0];
      v.fe[sl][1] = fr[1];
      v.lead[sl] = pp.lead[sl];
      v.alo[sl] = pp.alo[sl];
      v.an[sl] = pp.an[sl];
      v.blo[sl] = pp.blo[sl];
    }
    if (sl == 0) v.tb = pp.tb;
    __syncwarp(am);
    PlanOut r;
    r.ps = 0;
    r.gap = 0.0;
    r.S = S;
    TieBuf buf;
    buf.init();
    const double tau = cand_main_half(c, v, cq, S, ps.tau_lo, ps.tau_hi, pp.ub, buf);
    int k = 0;
    if (tau != tau) {
      r.status = HPS_ST_NO_CANDIDATE;
      r.gap = 1.0;
      r.cost = c.penalty_scale * (1.0 + 1.0);
    } else {
      final_half(c, v, st, S, tau, r, k);
    }
    if (!ARGMIN) {   // write_plan for this half's plan
      const bool ok = (r.status & 0x7f) == HPS_ST_OK;
      const bool counts = ok || (r.status & 0x7f) == HPS_ST_PS_QUOTA;
      const uint64_t p = ps.p;
      if (sl == 0) {
        o.cost[p] = r.cost;
        o.status[p] = (uint8_t)r.status;
        if (o.gap) o.gap[p] = r.gap;
        if (o.ps) o.ps[p] = ok ? r.ps : 0;
        if (o.num_stages) o.num_stages[p] = r.S;
      }
      if (o.k && sl < c.L) o.k[p * (uint64_t)c.L + sl] = (counts && sl < r.S) ? (int32_t)k : 0;
    } else {
      const int code = r.status & 0x7f;
      if (code == HPS_ST_OK) feas++;
      if (code == HPS_ST_NO_CPU_TYPE) flags |= 1u;
      const bool take = feasible_only ? (code == HPS_ST_OK) : (code != HPS_ST_NO_CPU_TYPE && code != HPS_ST_INVALID);
      if (take) {
        Key kk{r.cost, ps.rank_hi, ps.rank_lo, (uint32_t)r.status};
        if (key_less(kk, best)) best = kk;
      }
    }
    __syncwarp(am);
  }
  if (ARGMIN) {   // the two halves' partials meet, lane 0 writes the warp's
    __syncwarp();
    Key ob;
    ob.cost = __shfl_xor_sync(0xffffffffu, best.cost, 16);
    ob.hi = __shfl_xor_sync(0xffffffffu, best.hi, 16);
    ob.lo = __shfl_xor_sync(0xffffffffu, best.lo, 16);
    ob.status = __shfl_xor_sync(0xffffffffu, best.status, 16);
    flags |= __shfl_xor_sync(0xffffffffu, flags, 16);
    feas += __shfl_xor_sync(0xffffffffu, feas, 16);
    if (key_less(ob, best)) best = ob;
    if (lane == 0) merge_part(parts, gw, first, best, feas, flags);
  }
}

// stage_kernel with two plans per warp (L <= 16, hps_half.cuh)
template <int WARPS, bool ARGMIN, int SRC>
__global__ void __launch_bounds__(WARPS * 32, HPS_STAGE_MINB / WARPS)
stage_kernel_h(const InstanceConsts c, const DeviceTables tb, const PlanSource src, uint64_t p0,
               uint64_t p1, Outputs o, Pending pend, Cont cont, int feasible_only, KeyPart* parts,
               int first) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, half = lane >> 4, sl = lane & 15;
  WarpSmemL<16>& w = reinterpret_cast<WarpSmemL<16>*>(smem_raw)[warp * 2 + half];
  const uint64_t gw = (uint64_t)blockIdx.x * WARPS + warp, nw = (uint64_t)gridDim.x * WARPS;
  const uint64_t gh = gw * 2 + half, nh = nw * 2;
  PlanState<16>* states = reinterpret_cast<PlanState<16>*>(cont.states);
  Key best;
  best.cost = __longlong_as_double(0x7ff0000000000000LL);
  best.hi = best.lo = ~0ull;
  best.status = 0;
  uint32_t flags = 0;
  for (uint64_t p = p0 + gh; p < p1; p += nh) {
    int d;
    u128 rank;
    load_digits_half<SRC>(c, src, p, d, rank);
    PlanOut r;
    r.ps = 0;
    r.gap = 0.0;
    double tau_lo, tau_hi;
    if (stage_phase_half(c, tb, w, d, r, tau_lo, tau_hi)) {
      const unsigned am = seg_mask();
      unsigned int at = 0;
      if (sl == 0) at = atomicAdd(cont.count, 1u);
      at = __shfl_sync(am, at, lane & 16);
      HPS_CHECK(at < cont.cap, "plan-state chunk overflow");
      PlanState<16>& ps = states[at];
      if (sl < r.S) {
        ps.ent[sl] = w.ent[sl];
        ps.kmin[sl] = w.kmin[sl];
      }
      if (sl == 0) {
        ps.p = p;
        ps.rank_hi = (uint64_t)(rank >> 64);
        ps.rank_lo = (uint64_t)rank;
        ps.tau_lo = tau_lo;
        ps.tau_hi = tau_hi;
        ps.S = r.S;
        ps.n_cand = 0;
      }
    } else if (!ARGMIN) {   // write_plan for this half's plan
      const bool ok = (r.status & 0x7f) == HPS_ST_OK;
      if (sl == 0) {
        o.cost[p] = r.cost;
        o.status[p] = (uint8_t)r.status;
        if (o.gap) o.gap[p] = r.gap;
        if (o.ps) o.ps[p] = ok ? r.ps : 0;
        if (o.num_stages) o.num_stages[p] = r.S;
      }
      if (o.k)
        for (int s = sl; s < c.L; s += 16) o.k[p * (uint64_t)c.L + s] = 0;   // infeasible here
    } else {
      const int code = r.status & 0x7f;
      if (code == HPS_ST_NO_CPU_TYPE) flags |= 1u;
      if (code == HPS_ST_INVALID) flags |= 2u;
      const bool take = feasible_only ? false : (code != HPS_ST_NO_CPU_TYPE && code != HPS_ST_INVALID);
      if (take) {
        Key k{r.cost, (uint64_t)(rank >> 64), (uint64_t)rank, (uint32_t)r.status};
        if (key_less(k, best)) best = k;
      }
    }
    __syncwarp(seg_mask());
  }
  if (ARGMIN) {   // the two halves' partials meet, lane 0 writes the warp's
    __syncwarp();
    Key ob;
    ob.cost = __shfl_xor_sync(0xffffffffu, best.cost, 16);
    ob.hi = __shfl_xor_sync(0xffffffffu, best.hi, 16);
    ob.lo = __shfl_xor_sync(0xffffffffu, best.lo, 16);
    ob.status = __shfl_xor_sync(0xffffffffu, best.status, 16);
    flags |= __shfl_xor_sync(0xffffffffu, flags, 16);
    if (key_less(ob, best)) best = ob;
    if (lane == 0) merge_part(parts, gw, first, best, 0ull, flags);
  }
}

// load PlanState q into the warp's shared-memory view; per-stage constants of the sweep
template <int MAXS>
__device__ __forceinline__ void load_state(const InstanceConsts& c, const DeviceTables& tb, const PlanState<MAXS>& ps,
                                           WarpSmemL<MAXS>& w) {
  const int lane = threadIdx.x & 31;
  const int S = ps.S;
#pragma unroll 1
  for (int s = lane; s < S; s += 32) {
    const int e = ps.ent[s];
    const int type = __ldg(&tb.stages[e].type);
    w.sp[s] = tb.stages + e;
    w.ent[s] = e;
    w.row[s] = tb.te + c.te_off[type] + (int64_t)(e - type * c.P) * (int64_t)(c.et_cap[type] + 1);
    w.kmin[s] = ps.kmin[s];
    w.kmax[s] = ps.kmax[s];
    w.cls[s] = tb_class(tb, e);
  }
  for (int s = lane; s <= S; s += 32) w.pre[s] = ps.pre[s];
  __syncwarp();
}

// K1b: per-plan sweep constants, warm start, bound interval and restricted candidate ranges
template <int MAXS, int WARPS>
__global__ void __launch_bounds__(WARPS * 32, HPS_CAND_MINB / WARPS)
prep_kernel(const InstanceConsts c, const DeviceTables tb, Cont cont, PrepState<MAXS>* prep) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  WarpSmemL<MAXS>* sm = reinterpret_cast<WarpSmemL<MAXS>*>(smem_raw);
  SweepSmem<MAXS>* ss = reinterpret_cast<SweepSmem<MAXS>*>(smem_raw + sizeof(WarpSmemL<MAXS>) * WARPS);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  WarpSmemL<MAXS>& w = sm[warp];
  SweepSmem<MAXS>& sw = ss[warp];
  const uint64_t gw = (uint64_t)blockIdx.x * WARPS + warp, nw = (uint64_t)gridDim.x * WARPS;
  const PlanState<MAXS>* states = reinterpret_cast<const PlanState<MAXS>*>(cont.states);
  StageBuf<MAXS, false>& sb = reinterpret_cast<StageBuf<MAXS, false>*>(smem_raw + stage_offset<MAXS, WARPS>())[warp];
  const unsigned int n = *cont.count;
  stage_init(sb);
  if (gw < n) stage_issue(sb, 0, states, (const PrepState<MAXS>*)nullptr, gw);
  uint32_t it = 0;
  for (uint64_t q = gw; q < n; q += nw, it++) {
    const int slot = it & 1;
    if (q + nw < n) stage_issue(sb, slot ^ 1, states, (const PrepState<MAXS>*)nullptr, q + nw);
    if (staged<MAXS>()) mbar_wait(&sb.bar[slot], (it >> 1) & 1);
    const PlanState<MAXS>& ps = staged<MAXS>() ? sb.ps[slot] : states[q];
    if (ps.n_cand < 0) { __syncwarp(); continue; }  // slow path
    load_state<MAXS>(c, tb, ps, w);
    const int S = ps.S;
    TieBuf buf;
    buf.init();
    const double ub = cand_prep<MAXS>(c, tb, w, sw, S, ps.tau_lo, ps.tau_hi, ps.n_cand, buf);
    PrepState<MAXS>& out = prep[q];
    for (int s = lane; s < S; s += 32) {
      out.kb[s] = sw.kb[s];
      out.dom[s] = (int8_t)sw.dom[s];
      out.lead[s] = sw.lead[s];
      out.alo[s] = (int16_t)sw.alo[s];
      out.an[s] = (int16_t)sw.an[s];
      out.blo[s] = (int16_t)sw.blo[s];
    }
    if (lane == 0) {
      out.ub = ub;
      out.tb = sw.tb;
    }
    __syncwarp();
  }
}

// K1c: filter + exact evaluation over the restricted list, add_ps_cores, final cost, argmin
template <int MAXS, int WARPS, bool ARGMIN>
__global__ void __launch_bounds__(WARPS * 32, HPS_CAND_MINB / WARPS)
candidate_kernel(const InstanceConsts c, const DeviceTables tb, Cont cont, const PrepState<MAXS>* prep, Outputs o,
                 int feasible_only, KeyPart* parts, int first) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  WarpSmemL<MAXS>* sm = reinterpret_cast<WarpSmemL<MAXS>*>(smem_raw);
  SweepSmem<MAXS>* ss = reinterpret_cast<SweepSmem<MAXS>*>(smem_raw + sizeof(WarpSmemL<MAXS>) * WARPS);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  WarpSmemL<MAXS>& w = sm[warp];
  SweepSmem<MAXS>& sw = ss[warp];
  const uint64_t gw = (uint64_t)blockIdx.x * WARPS + warp, nw = (uint64_t)gridDim.x * WARPS;
  const PlanState<MAXS>* states = reinterpret_cast<const PlanState<MAXS>*>(cont.states);
  StageBuf<MAXS, true>& sb = reinterpret_cast<StageBuf<MAXS, true>*>(
      smem_raw + stage_offset<MAXS, WARPS>())[warp];
  CandQueue* queues = reinterpret_cast<CandQueue*>(smem_raw + stage_offset<MAXS, WARPS>() +
                                                   stage_bytes<MAXS, true>() * WARPS);
  if (lane == 0) sw.cq = &queues[warp];
  const unsigned int n = *cont.count;
  Key best;
  best.cost = __longlong_as_double(0x7ff0000000000000LL);
  best.hi = best.lo = ~0ull;
  best.status = 0;
  unsigned long long feas = 0;
  uint32_t flags = 0;
  stage_init(sb);
  if (gw < n) stage_issue(sb, 0, states, prep, gw);
  uint32_t it = 0;
  for (uint64_t q = gw; q < n; q += nw, it++) {
    const int slot = it & 1;
    if (q + nw < n) stage_issue(sb, slot ^ 1, states, prep, q + nw);
    if (staged<MAXS>()) mbar_wait(&sb.bar[slot], (it >> 1) & 1);
    const PlanState<MAXS>& ps = staged<MAXS>() ? sb.ps[slot] : states[q];
    if (ps.n_cand < 0) { __syncwarp(); continue; }  // slow path
    load_state<MAXS>(c, tb, ps, w);
    const int S = ps.S;
    const PrepState<MAXS>& pp = staged<MAXS>() ? sb.pp[slot] : prep[q];
#pragma unroll 1
    for (int r = lane; r < S; r += 32) {
      const int lo = ps.kmin[r], hi = ps.kmax[r];
      sw.pr[r] = c.price_s[w.stage(r).type];
      sw.fpr[r] = (float)sw.pr[r];
      sw.kmi[r] = lo;
      sw.kma[r] = hi;
      sw.etp[r] = (lo == hi) ? __ldg(&HPS_TE(w.row[r], lo - 1).et) : 0.0;
      sw.dom[r] = pp.dom[r];
      est_setup<MAXS>(w, sw, r);
      sw.lead[r] = pp.lead[r];
      sw.alo[r] = pp.alo[r];
      sw.an[r] = pp.an[r];
      sw.blo[r] = pp.blo[r];
      sw.kb[r] = pp.kb[r];
    }
    if (lane == 0) {
      sw.tb = pp.tb;
    }
    __syncwarp();
    PlanOut r;
    r.ps = 0;
    r.gap = 0.0;
    r.S = S;
    TieBuf buf;
    buf.init();
    const double tau = cand_main<MAXS>(c, w, sw, S, ps.tau_lo, ps.tau_hi, pp.ub, buf);
    if (tau != tau) {
      r.status = HPS_ST_NO_CANDIDATE;
      r.gap = 1.0;
      r.cost = c.penalty_scale * (1.0 + 1.0);
    } else {
      phase_final_fast<MAXS>(c, w, S, tau, r);
    }
    if (!ARGMIN) {
      write_plan<MAXS>(c, w, o, ps.p, r);
    } else {
      const int code = r.status & 0x7f;
      if (code == HPS_ST_OK) feas++;
      if (code == HPS_ST_NO_CPU_TYPE) flags |= 1u;
      const bool take = feasible_only ? (code == HPS_ST_OK) : (code != HPS_ST_NO_CPU_TYPE && code != HPS_ST_INVALID);
      if (take) {
        Key k{r.cost, ps.rank_hi, ps.rank_lo, (uint32_t)r.status};
        if (key_less(k, best)) best = k;
      }
    }
    __syncwarp();
  }
  if (ARGMIN && lane == 0) merge_part(parts, gw, first, best, feas, flags);
}

template <int MAXS, int WARPS, bool ARGMIN, bool FAST, int SRC>
int launch_eval(HpsInstance* in, const PlanSource& src, uint64_t n, const Outputs& o, Pending pend,
                int feasible_only, KeyPart* parts, int grid, cudaStream_t st) {
  const size_t smem = sizeof(WarpSmem<MAXS>) * WARPS + (FAST ? sizeof(SweepSmem<MAXS>) * WARPS : 0);
  auto kern = eval_kernel<MAXS, WARPS, ARGMIN, FAST, SRC>;
  CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  HPS_COUNT_LAUNCH();
  kern<<<grid, WARPS * 32, smem, st>>>(in->c, in->tb, src, n, o, pend, feasible_only, parts);
  CUDA_TRY(cudaGetLastError());
  return HPS_OK;
}

template <int MAXS, int WARPS, bool ARGMIN, bool FAST>
int launch_src(HpsInstance* in, const PlanSource& src, uint64_t n, const Outputs& o, Pending pend,
               int feasible_only, KeyPart* parts, int grid, cudaStream_t st) {
  if (src.mode == 0) return launch_eval<MAXS, WARPS, ARGMIN, FAST, 0>(in, src, n, o, pend, feasible_only, parts, grid, st);
  if (!ARGMIN) return set_err(HPS_E_INVALID_ARG, "per-plan outputs need an explicit plan batch");
  if (src.mode == 1) return launch_eval<MAXS, WARPS, ARGMIN, FAST, 1>(in, src, n, o, pend, feasible_only, parts, grid, st);
  if (src.mode == 3) return launch_eval<MAXS, WARPS, ARGMIN, FAST, 3>(in, src, n, o, pend, feasible_only, parts, grid, st);
  return launch_eval<MAXS, WARPS, ARGMIN, FAST, 2>(in, src, n, o, pend, feasible_only, parts, grid, st);
}

template <bool ARGMIN>
int dispatch_eval(HpsInstance* in, const PlanSource& src, uint64_t n, const Outputs& o, Pending pend,
                  int feasible_only, KeyPart* parts, int grid, cudaStream_t st) {
  if (in->c.L <= 16) return launch_src<16, 4, ARGMIN, false>(in, src, n, o, pend, feasible_only, parts, grid, st);
  if (in->c.L <= 32) return launch_src<32, 4, ARGMIN, false>(in, src, n, o, pend, feasible_only, parts, grid, st);
  return launch_src<64, 2, ARGMIN, false>(in, src, n, o, pend, feasible_only, parts, grid, st);
}

int warps_per_block(const HpsInstance* in) { return (in->c.L <= 32) ? 4 : 2; }

template <int MAXS, int WARPS, bool ARGMIN, int SRC>
int launch_stage(HpsInstance* in, const PlanSource& src, uint64_t p0, uint64_t p1, const Outputs& o,
                 Pending pend, Cont cont, int feasible_only, KeyPart* parts, int first, int grid,
                 cudaStream_t st) {
  if (MAXS == 16 && in->half_stage) {   // two plans per warp (hps_half.cuh)
    const size_t smem = sizeof(WarpSmemL<16>) * WARPS * 2;
    auto kern = stage_kernel_h<WARPS, ARGMIN, SRC>;
    CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    HPS_COUNT_LAUNCH();
    kern<<<grid, WARPS * 32, smem, st>>>(in->c, in->tb, src, p0, p1, o, pend, cont, feasible_only, parts, first);
    CUDA_TRY(cudaGetLastError());
    return HPS_OK;
  }
  const size_t smem = sizeof(WarpSmemL<MAXS>) * WARPS;
  auto kern = stage_kernel<MAXS, WARPS, ARGMIN, SRC>;
  CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (in->carveout >= 0) CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, in->carveout));
  HPS_COUNT_LAUNCH();
  kern<<<grid, WARPS * 32, smem, st>>>(in->c, in->tb, src, p0, p1, o, pend, cont, feasible_only, parts, first);
  CUDA_TRY(cudaGetLastError());
  return HPS_OK;
}

// identity partial keys (a pipeline stream that received no chunk)
__global__ void init_parts_kernel(KeyPart* parts, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    KeyPart kp;
    kp.best.cost = __longlong_as_double(0x7ff0000000000000LL);
    kp.best.hi = kp.best.lo = ~0ull;
    kp.best.status = 0;
    kp.evaluated = 0ull;
    kp.feasible = 0ull;
    kp.flags = 0u;
    parts[i] = kp;
  }
}

// streams of the chunk pipeline: 2 when the instance has its auxiliary stream (HPS_PIPE)
int pipe_streams(const HpsInstance* in) { return (in->pipe > 1 && in->aux) ? 2 : 1; }

// chunked K1a/K1b/K1c pipeline over plans [0, n); parts holds 2 * grid * WARPS partial keys per
// pipeline stream. With two streams, chunk j runs on stream j % 2 with its own plan-state buffer
// and partials, so one chunk's kernel tails overlap the other's kernels and a chunk's state
// records (written by one kernel, read by the next) stay in L2 at small chunk sizes.
template <int MAXS, int WARPS, bool ARGMIN>
int run_split(HpsInstance* in, const PlanSource& src, uint64_t n, const Outputs& o, Pending pend,
              int feasible_only, KeyPart* parts, int grid, cudaStream_t st) {
  int np = pipe_streams(in);
  const uint64_t def_chunk = (MAXS <= 16 ? (np > 1 ? in->pipe_chunk : (4ull << 20)) : (MAXS <= 32 ? (2ull << 20) : (1ull << 20)));
  const uint64_t base_chunk = in->chunk ? in->chunk : def_chunk;
  uint64_t chunk = std::min<uint64_t>(n, base_chunk);
  if (np > 1) chunk = std::min<uint64_t>(chunk, (n + 1) / 2);   // >= 2 chunks when n >= 2
  const uint64_t nchunks = (n + chunk - 1) / chunk;
  const int used = (int)std::min<uint64_t>((uint64_t)np, nchunks);
  char* buf = nullptr;
  const size_t state_bytes = (sizeof(PlanState<MAXS>) * chunk + 255) / 256 * 256;
  const size_t slot_bytes = 256 + state_bytes + (sizeof(PrepState<MAXS>) * chunk + 255) / 256 * 256;
  CUDA_TRY(cudaMallocAsync(&buf, slot_bytes * used, st));
  const size_t nkp = (size_t)grid * WARPS;   // partials per kernel
  if (ARGMIN && parts && used < np) {   // the second stream's partials are read by finish_argmin
    HPS_COUNT_LAUNCH();
    init_parts_kernel<<<8, 256, 0, st>>>(parts + 2 * nkp, (int)(2 * nkp));
    CUDA_TRY(cudaGetLastError());
  }
  const size_t smem3 = stage_offset<MAXS, WARPS>() + (stage_bytes<MAXS, true>() + sizeof(CandQueue)) * WARPS;
  const size_t smem1 = (sizeof(WarpSmemL<MAXS>) * WARPS + 15) / 16 * 16 + stage_bytes<MAXS, false>() * WARPS;
  auto kb = bisect_kernel<MAXS, WARPS>;
  CUDA_TRY(cudaFuncSetAttribute(kb, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem1));
  auto kbh = bisect_kernel_h<WARPS>;
  const size_t smemh = (sizeof(WarpSmemL<16>) * WARPS * 2 + 15) / 16 * 16 + sizeof(StageBuf<16, false>) * WARPS * 2;
  if (MAXS == 16) CUDA_TRY(cudaFuncSetAttribute(kbh, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smemh));
  auto kp = prep_kernel<MAXS, WARPS>;
  const size_t smemp = stage_offset<MAXS, WARPS>() + stage_bytes<MAXS, false>() * WARPS;
  CUDA_TRY(cudaFuncSetAttribute(kp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smemp));
  auto kph = prep_kernel_h<WARPS>;
  const size_t smemph = (sizeof(WarpSmemP) + sizeof(SweepSmem<16>)) * WARPS * 2;
  if (MAXS == 16) CUDA_TRY(cudaFuncSetAttribute(kph, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smemph));
  auto k2 = candidate_kernel<MAXS, WARPS, ARGMIN>;
  CUDA_TRY(cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem3));
  auto k2h = candidate_kernel_h<WARPS, ARGMIN>;
  const size_t smem2h = sizeof(CandView) * WARPS * 2 + sizeof(CandQueue) * WARPS;
  if (MAXS == 16) CUDA_TRY(cudaFuncSetAttribute(k2h, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2h));
  if (MAXS == 16 && in->carveout >= 0) CUDA_TRY(cudaFuncSetAttribute(k2h, cudaFuncAttributePreferredSharedMemoryCarveout, in->carveout));
  if (in->carveout >= 0) CUDA_TRY(cudaFuncSetAttribute(k2, cudaFuncAttributePreferredSharedMemoryCarveout, in->carveout));
  if (used > 1) {   // fork: the auxiliary stream starts after everything queued on st so far
    CUDA_TRY(cudaEventRecord(in->ev_fork, st));
    CUDA_TRY(cudaStreamWaitEvent(in->aux, in->ev_fork, 0));
  }
  for (uint64_t j = 0; j < nchunks; j++) {
    const int sl = (int)(j % (uint64_t)used);
    cudaStream_t s = sl ? in->aux : st;
    const uint64_t c0 = j * chunk, c1 = std::min(n, c0 + chunk);
    const int first = (j < (uint64_t)used);
    char* sb = buf + slot_bytes * sl;
    Cont cont{sb + 256, reinterpret_cast<unsigned int*>(sb), (unsigned int)chunk};
    PrepState<MAXS>* prep = reinterpret_cast<PrepState<MAXS>*>(sb + 256 + state_bytes);
    KeyPart* parts_a = parts ? parts + 2 * nkp * sl : nullptr;
    KeyPart* parts_b = parts ? parts_a + nkp : nullptr;
    CUDA_TRY(cudaMemsetAsync(cont.count, 0, sizeof(unsigned int), s));
    int rc;
    if (src.mode == 0) rc = launch_stage<MAXS, WARPS, ARGMIN, 0>(in, src, c0, c1, o, pend, cont, feasible_only, parts_a, first, grid, s);
    else if (src.mode == 1) rc = launch_stage<MAXS, WARPS, ARGMIN, 1>(in, src, c0, c1, o, pend, cont, feasible_only, parts_a, first, grid, s);
    else if (src.mode == 3) rc = launch_stage<MAXS, WARPS, ARGMIN, 3>(in, src, c0, c1, o, pend, cont, feasible_only, parts_a, first, grid, s);
    else rc = launch_stage<MAXS, WARPS, ARGMIN, 2>(in, src, c0, c1, o, pend, cont, feasible_only, parts_a, first, grid, s);
    if (rc) return rc;
    HPS_COUNT_LAUNCH();
    if (MAXS == 16 && in->half_bisect) {   // two plans per warp (hps_half.cuh)
      kbh<<<grid, WARPS * 32, smemh, s>>>(in->c, in->tb, cont, pend);
    } else {
      kb<<<grid, WARPS * 32, smem1, s>>>(in->c, in->tb, cont, pend);
    }
    CUDA_TRY(cudaGetLastError());
    HPS_COUNT_LAUNCH();
    if (MAXS == 16 && in->half_prep) {   // two plans per warp (hps_half.cuh)
      kph<<<grid, WARPS * 32, smemph, s>>>(in->c, in->tb, cont, reinterpret_cast<PrepState<16>*>(prep));
    } else {
      kp<<<grid, WARPS * 32, smemp, s>>>(in->c, in->tb, cont, prep);
    }
    CUDA_TRY(cudaGetLastError());
    HPS_COUNT_LAUNCH();
    if (MAXS == 16 && in->half_cand) {   // two plans per warp (hps_half.cuh)
      k2h<<<grid, WARPS * 32, smem2h, s>>>(in->c, in->tb, cont, reinterpret_cast<const PrepState<16>*>(prep), o,
                                           feasible_only, parts_b, first);
    } else {
      k2<<<grid, WARPS * 32, smem3, s>>>(in->c, in->tb, cont, prep, o, feasible_only, parts_b, first);
    }
    CUDA_TRY(cudaGetLastError());
  }
  if (used > 1) {   // join
    CUDA_TRY(cudaEventRecord(in->ev_join, in->aux));
    CUDA_TRY(cudaStreamWaitEvent(st, in->ev_join, 0));
  }
  CUDA_TRY(cudaFreeAsync(buf, st));
  return HPS_OK;
}

template <bool ARGMIN>
int dispatch_split(HpsInstance* in, const PlanSource& src, uint64_t n, const Outputs& o, Pending pend,
                   int feasible_only, KeyPart* parts, int grid, cudaStream_t st) {
  if (in->c.L <= 16) return run_split<16, 4, ARGMIN>(in, src, n, o, pend, feasible_only, parts, grid, st);
  if (in->c.L <= 32) return run_split<32, 4, ARGMIN>(in, src, n, o, pend, feasible_only, parts, grid, st);
  return run_split<64, 2, ARGMIN>(in, src, n, o, pend, feasible_only, parts, grid, st);
}

int grid_for(HpsInstance* in, uint64_t n_plans) {
  const int warps = warps_per_block(in);
  uint64_t blocks = (n_plans + warps - 1) / warps;
  uint64_t cap = (uint64_t)in->sm_count * in->grid_per_sm;
  return (int)std::max<uint64_t>(1, std::min(blocks, cap));
}

size_t slow_per_block(const HpsInstance* in) {
  size_t nraw = (size_t)in->c.L * (kBpLimit + 1) + 2;
  size_t npow = 1;
  while (npow < nraw) npow <<= 1;
  return 2 * npow;  // doubles: sort buffer + candidate buffer
}

// resident slow-path blocks (occupancy API, cached) and the grid: one launch per super-chunk
int slow_grid(HpsInstance* in, int& blocks) {
  auto ks = in->fast ? slow_kernel<true> : slow_kernel<false>;
  if (in->slow_per_sm < 0) {
    CUDA_TRY(cudaFuncSetAttribute(ks, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(kSlowSmemSort * sizeof(double))));
    int per_sm = 0;  // as many resident blocks as registers and shared memory allow
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ks, kSlowThreads, kSlowSmemSort * sizeof(double)));
    in->slow_per_sm = std::max(1, per_sm);
  }
  const size_t per_block = slow_per_block(in);
  const size_t cap_blocks = std::max<size_t>(8, ((size_t)4 << 30) / (per_block * sizeof(double)));
  blocks = (int)std::min<size_t>((size_t)in->sm_count * in->slow_per_sm, cap_blocks);
  return HPS_OK;
}

int run_slow(HpsInstance* in, const PlanSource& src, const Outputs& o, Pending pend, int argmin_mode,
             int feasible_only, KeyPart* slow_parts, cudaStream_t st) {
  int blocks = 0;
  if (int rc = slow_grid(in, blocks)) return rc;
  const size_t per_block = slow_per_block(in);
  double* scratch = nullptr;
  auto ks = in->fast ? slow_kernel<true> : slow_kernel<false>;
  CUDA_TRY(cudaMallocAsync(&scratch, per_block * blocks * sizeof(double), st));
  HPS_COUNT_LAUNCH();
  ks<<<blocks, kSlowThreads, kSlowSmemSort * sizeof(double), st>>>(in->c, in->tb, src, o, pend, argmin_mode, feasible_only,
                                                    slow_parts, scratch, per_block);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaFreeAsync(scratch, st));
  return HPS_OK;
}

// plan source advanced by `off` plans (a super-chunk of the caller's range)
PlanSource advance_source(const PlanSource& src, uint64_t off, int L) {
  PlanSource s = src;
  if (s.mode == 0) s.plans = src.plans + off * (uint64_t)L;
  else if (s.mode == 1) s.begin = src.begin + off * src.stride;
  else s.begin = src.begin + off;   // modes 2, 3: plan number offset
  return s;
}

void fill_random_source(HpsInstance* in, const HpsPcg64* g, uint64_t first, PlanSource& src) {
  src.mode = 2;
  src.begin = first;
  int b = 0;
  while ((1 << b) < in->c.T) b++;
  src.tbits = b;
  src.s0_hi = g->state_hi; src.s0_lo = g->state_lo;
  src.inc_hi = g->inc_hi; src.inc_lo = g->inc_lo;
  const u128 inc = mk(g->inc_hi, g->inc_lo), M = pcg_mult();
  u128 A = 1, Cc = 0;
  for (int j = 0; j <= 32; j++) {
    src.jA_hi[j] = (uint64_t)(A >> 64); src.jA_lo[j] = (uint64_t)A;
    src.jC_hi[j] = (uint64_t)(Cc >> 64); src.jC_lo[j] = (uint64_t)Cc;
    A = M * A;
    Cc = M * Cc + inc;
  }
}

// Argmin over plans [0, n) of src, in super-chunks of at most in->super_chunk plans: each runs the
// warp kernels, then the slow path over that chunk's pending list (sized to the chunk, so no plan
// is ever dropped), then the merge into one key per chunk; the chunk keys merge at the end.
int argmin_common(HpsInstance* in, PlanSource& src, uint64_t n, int feasible_only, HpsArgmin* d_best,
                  cudaStream_t st) {
  if (n == 0) {   // empty range: the identity key (cost +inf, nothing evaluated)
    HPS_COUNT_LAUNCH();
    finish_argmin<<<1, 256, 0, st>>>(nullptr, 0, nullptr, 0, 0, d_best);
    CUDA_TRY(cudaGetLastError());
    return HPS_OK;
  }
  if (int rc = chk_bind(in, st)) return rc;
  const uint64_t sc = in->super_chunk;
  const uint64_t nsc = (n + sc - 1) / sc;
  const uint64_t n0 = std::min(n, sc);
  const int grid = grid_for(in, n0);   // one grid for every chunk: every warp writes its partial
  const int nparts = grid * warps_per_block(in) * (in->fast ? 2 * pipe_streams(in) : 1);
  int nslow = 0;
  if (int rc = slow_grid(in, nslow)) return rc;
  const unsigned cap = (unsigned)n0;
  char* buf = nullptr;
  const size_t bytes = sizeof(KeyPart) * (nparts + nslow) + sizeof(HpsArgmin) * (nsc > 1 ? nsc : 0) +
                       sizeof(unsigned long long) * cap + 64;
  CUDA_TRY(cudaMallocAsync(&buf, bytes, st));
  KeyPart* parts = reinterpret_cast<KeyPart*>(buf);
  KeyPart* slow_parts = parts + nparts;
  HpsArgmin* chunk_keys = reinterpret_cast<HpsArgmin*>(slow_parts + nslow);
  unsigned long long* list = reinterpret_cast<unsigned long long*>(chunk_keys + (nsc > 1 ? nsc : 0));
  unsigned int* count = reinterpret_cast<unsigned int*>(list + cap);
  Outputs o{};
  for (uint64_t i = 0; i < nsc; i++) {
    const uint64_t s0 = i * sc, m = std::min(n, s0 + sc) - s0;
    const PlanSource sub = advance_source(src, s0, in->c.L);
    CUDA_TRY(cudaMemsetAsync(count, 0, sizeof(unsigned int), st));
    Pending pend{list, count, (unsigned)m};
    int rc = in->fast ? dispatch_split<true>(in, sub, m, o, pend, feasible_only, parts, grid, st)
                      : dispatch_eval<true>(in, sub, m, o, pend, feasible_only, parts, grid, st);
    if (rc) return rc;
    rc = run_slow(in, sub, o, pend, 1, feasible_only, slow_parts, st);
    if (rc) return rc;
    HPS_COUNT_LAUNCH();
    finish_argmin<<<1, 256, 0, st>>>(parts, nparts, slow_parts, nslow, m, nsc > 1 ? chunk_keys + i : d_best);
    CUDA_TRY(cudaGetLastError());
  }
  if (nsc > 1) {
    HPS_COUNT_LAUNCH();
    merge_argmin<<<1, 32, 0, st>>>(chunk_keys, (int)nsc, n, d_best);
    CUDA_TRY(cudaGetLastError());
  }
  CUDA_TRY(cudaFreeAsync(buf, st));
  return HPS_OK;
}

}  // namespace

#include "hps_prune.cuh"

extern "C" {

int hps_abi_version(void) { return HPS_ABI_VERSION; }

const char* hps_error_string(int code) {
  switch (code) {
    case HPS_OK: return "ok";
    case HPS_E_INVALID_ARG: return "invalid argument";
    case HPS_E_PLAN: return "plan does not fit the model graph or catalog";
    case HPS_E_CONFIG: return "configuration not supported";
    case HPS_E_CUDA: return "CUDA runtime failure";
    case HPS_E_NO_CPU_TYPE: return "catalog has no CPU-capable resource type";
    case HPS_E_NUMERIC: return "non-finite values";
    default: return "unknown error";
  }
}

const char* hps_last_error(void) { return g_last_error.c_str(); }

namespace {
int instance_build(const HpsInstanceDesc* d, HpsInstance* in, int dev, double*& d_raw);
}

int hps_instance_create(const HpsInstanceDesc* d, HpsInstance** out) {
  if (!d || !out) return set_err(HPS_E_INVALID_ARG, "null argument");
  *out = nullptr;
  const int L = d->num_layers, T = d->num_types;
  if (L < 1 || L > kMaxL || T < 1 || T > kMaxT) return set_err(HPS_E_CONFIG, "L or T out of range");
  if (!(d->throughput_limit > 0) || d->profile_batch_size < 1 || d->batch_size < 1)
    return set_err(HPS_E_INVALID_ARG, "bad job parameters");
  int dev = 0, ndev = 0;
  CUDA_TRY(cudaGetDeviceCount(&ndev));
  if (ndev < 1) return set_err(HPS_E_CUDA, "no CUDA device");
  CUDA_TRY(cudaGetDevice(&dev));
  auto* in = new HpsInstance();
  double* d_raw = nullptr;
  const int rc = instance_build(d, in, dev, d_raw);
  if (d_raw) cudaFree(d_raw);
  if (rc != HPS_OK) {   // every partially created table is released (destroy tolerates nulls)
    hps_instance_destroy(in);
    return rc;
  }
  *out = in;
  return HPS_OK;
}

}  // extern "C"

namespace {
// Device buffers of destroyed instances are kept (per device and size, up to 2 GB) and handed to
// the next instance of the same shape: re-staging an instance (the e2e path does it every call)
// then allocates nothing. Buffers enter the cache after a device synchronisation, so no queued
// kernel of the old instance can still read them.
std::mutex g_buf_mu;
std::multimap<std::pair<int, size_t>, void*> g_buf_cache;
size_t g_buf_bytes = 0;
constexpr size_t kBufCacheCap = 2ull << 30;

cudaError_t cached_alloc(void** p, size_t n, int dev) {
  {
    std::lock_guard<std::mutex> lock(g_buf_mu);
    auto it = g_buf_cache.find({dev, n});
    if (it != g_buf_cache.end()) {
      *p = it->second;
      g_buf_cache.erase(it);
      g_buf_bytes -= n;
      return cudaSuccess;
    }
  }
  return cudaMalloc(p, n);
}

void cached_release(void* p, size_t n, int dev) {
  if (!p) return;
  {
    std::lock_guard<std::mutex> lock(g_buf_mu);
    if (g_buf_bytes + n <= kBufCacheCap) {
      g_buf_cache.insert({{dev, n}, p});
      g_buf_bytes += n;
      return;
    }
  }
  cudaFree(p);
}

int instance_build(const HpsInstanceDesc* d, HpsInstance* in, int dev, double*& d_raw) {
  const int L = d->num_layers, T = d->num_types;
  cudaDeviceGetAttribute(&in->sm_count, cudaDevAttrMultiProcessorCount, dev);
  if (const char* e = getenv("HPS_GRID_PER_SM")) in->grid_per_sm = std::max(1, atoi(e));
  if (const char* e = getenv("HPS_CARVEOUT")) in->carveout = std::min(100, atoi(e));
  if (const char* e = getenv("HPS_HALF_BISECT")) in->half_bisect = atoi(e) != 0;
  if (const char* e = getenv("HPS_HALF_STAGE")) in->half_stage = atoi(e) != 0;
  if (const char* e = getenv("HPS_HALF_PREP")) in->half_prep = atoi(e) != 0;
  if (const char* e = getenv("HPS_HALF_CAND")) in->half_cand = atoi(e) != 0;
  if (const char* e = getenv("HPS_CHUNK")) in->chunk = (uint64_t)std::max(1024ll, atoll(e));
  if (const char* e = getenv("HPS_SUPERCHUNK")) in->super_chunk = (uint64_t)std::max(1ll, std::min(atoll(e), 1ll << 31));
  if (const char* e = getenv("HPS_PIPE")) in->pipe = std::max(1, std::min(2, atoi(e)));
  if (in->pipe > 1) {   // one auxiliary stream per device for the process (instances come and go;
                        // stream order plus the per-instance fork/join events keep each call ordered)
    static std::mutex mu;
    static cudaStream_t aux[256] = {};
    std::lock_guard<std::mutex> lock(mu);
    if (dev < 0 || dev >= 256) return set_err(HPS_E_CONFIG, "device index out of range");
    if (!aux[dev]) CUDA_TRY(cudaStreamCreateWithFlags(&aux[dev], cudaStreamNonBlocking));
    in->aux = aux[dev];
    CUDA_TRY(cudaEventCreateWithFlags(&in->ev_fork, cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&in->ev_join, cudaEventDisableTiming));
  }
  {  // keep stream-ordered scratch (slow-path buffers, argmin partials) mapped between calls
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = 8ull << 30;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  }
  InstanceConsts& c = in->c;
  memset(&c, 0, sizeof(c));
  c.L = L; c.T = T; c.P = L * (L + 1) / 2;
  c.with_ps = d->with_ps;
  c.newton_max_iters = d->newton_max_iters;
  c.bo = (double)d->profile_batch_size;
  c.batch = (double)d->batch_size;
  c.work = (double)(d->epochs * d->total_samples);
  c.limit = d->throughput_limit;
  c.ps_cores_per_gpu = d->ps_cores_per_gpu;
  c.newton_tol = d->newton_tol;
  c.fd_step = d->fd_step;
  c.tau_limit = c.batch / c.limit;
  double mx = d->price_per_hour[0];
  c.ps_type = -1;
  for (int t = 0; t < T; t++) {
    if (d->price_per_hour[t] > mx) mx = d->price_per_hour[t];
    c.price_h[t] = d->price_per_hour[t];
    c.price_s[t] = d->price_per_hour[t] / 3600.0;
    c.quota[t] = d->quota[t];
    c.is_cpu[t] = d->is_cpu[t] ? 1 : 0;
    if (c.is_cpu[t] && (c.ps_type < 0 || d->price_per_hour[t] < d->price_per_hour[c.ps_type])) c.ps_type = t;
  }
  c.penalty_scale = 1e6 * mx;
  int64_t off = 0;
  bool fast = true;
  for (int t = 0; t < T; t++) {
    c.et_cap[t] = (int32_t)std::max<int64_t>(1, std::min<int64_t>(d->quota[t], kEtCapMax));
    if (d->quota[t] > kEtCapMax) fast = false;  // counts could leave the threshold table
    c.te_off[t] = off;
    off += (int64_t)c.P * (c.et_cap[t] + 1);
  }
  c.redux_ok = fast ? 1 : 0;
  in->fast = fast && (getenv("HPS_FORCE_LITERAL") == nullptr);
  // raw tables -> device
  const size_t tl = (size_t)T * L * sizeof(double);
  in->dev = dev;
  CUDA_TRY(cudaMalloc(&d_raw, 4 * tl));
  CUDA_TRY(cudaMemcpy(d_raw, d->oct, tl, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy((char*)d_raw + tl, d->odt, tl, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy((char*)d_raw + 2 * tl, d->alpha, tl, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy((char*)d_raw + 3 * tl, d->beta, tl, cudaMemcpyHostToDevice));
  RawTables raw{d_raw, d_raw + T * L, d_raw + 2 * T * L, d_raw + 3 * T * L};
  const int ne = T * c.P;
  in->sz_stages = sizeof(StageEntry) * ne;
  in->sz_stage0 = sizeof(Stage0Info) * T * L;
  in->te_bytes = sizeof(TEPair) * off;
  in->sz_cls = in->sz_gex = sizeof(int32_t) * ne;
  CUDA_TRY(cached_alloc(reinterpret_cast<void**>(&in->d_stages), in->sz_stages, dev));
  CUDA_TRY(cached_alloc(reinterpret_cast<void**>(&in->d_stage0), in->sz_stage0, dev));
  CUDA_TRY(cached_alloc(reinterpret_cast<void**>(&in->d_te), in->te_bytes, dev));
  if (int rc = chk_bind(in, 0)) return rc;
  CUDA_TRY(cached_alloc(reinterpret_cast<void**>(&in->d_cls), in->sz_cls, dev));
  CUDA_TRY(cached_alloc(reinterpret_cast<void**>(&in->d_gex), in->sz_gex, dev));
  HPS_COUNT_LAUNCH();
  stage_table_kernel<<<(ne + 127) / 128, 128>>>(c, raw, in->d_stages);
  CUDA_TRY(cudaGetLastError());
  HPS_COUNT_LAUNCH();
  stage0_kernel<<<(T * L + 127) / 128, 128>>>(c, in->d_stages, in->d_stage0);
  CUDA_TRY(cudaGetLastError());
  for (int t = 0; t < T; t++) {
    const int64_t cnt = (int64_t)c.P * (c.et_cap[t] + 1);
    HPS_COUNT_LAUNCH();
    te_table_kernel<<<(unsigned)((cnt + 127) / 128), 128>>>(c, in->d_stages, in->d_te, t, cnt, c.te_off[t]);
    CUDA_TRY(cudaGetLastError());
  }
  for (int t = 0; t < T; t++) {
    HPS_COUNT_LAUNCH();
    gen_exact_init_kernel<<<(c.P + 127) / 128, 128>>>(c, in->d_gex, t);
    CUDA_TRY(cudaGetLastError());
    const int64_t cnt = (int64_t)c.P * c.et_cap[t];
    HPS_COUNT_LAUNCH();
    gen_exact_kernel<<<(unsigned)((cnt + 255) / 256), 256>>>(c, in->d_te, in->d_gex, t, cnt);
    CUDA_TRY(cudaGetLastError());
  }
  CUDA_TRY(cudaDeviceSynchronize());
  CUDA_TRY(cudaFree(d_raw));
  d_raw = nullptr;
  // ET-equivalence classes: group entries with bitwise-equal (oct, odt, alpha, beta)
  in->h_stages.resize(ne);
  CUDA_TRY(cudaMemcpy(in->h_stages.data(), in->d_stages, sizeof(StageEntry) * ne, cudaMemcpyDeviceToHost));
  std::map<std::tuple<uint64_t, uint64_t, uint64_t, uint64_t>, int> ids;
  std::vector<int32_t> cls(ne);
  for (int e = 0; e < ne; e++) {
    const StageEntry& s = in->h_stages[e];
    uint64_t k[4];
    memcpy(&k[0], &s.oct, 8); memcpy(&k[1], &s.odt, 8); memcpy(&k[2], &s.alpha, 8); memcpy(&k[3], &s.beta, 8);
    auto key = std::make_tuple(k[0], k[1], k[2], k[3]);
    auto it = ids.find(key);
    if (it == ids.end()) it = ids.emplace(key, (int)ids.size()).first;
    cls[e] = it->second;
  }
  CUDA_TRY(cudaMemcpy(in->d_cls, cls.data(), sizeof(int32_t) * ne, cudaMemcpyHostToDevice));
  in->tb = DeviceTables{in->d_stages, in->d_stage0, in->d_te, in->d_cls, in->d_gex};
  return HPS_OK;
}
}  // namespace

extern "C" {

int hps_instance_destroy(HpsInstance* in) {
  if (!in) return HPS_OK;
  int cur = 0;
  cudaGetDevice(&cur);
  cudaSetDevice(in->dev);
  cudaDeviceSynchronize();   // nothing queued may still read the tables once they are reused
  cached_release(in->d_stages, in->sz_stages, in->dev);
  cached_release(in->d_stage0, in->sz_stage0, in->dev);
  cached_release(in->d_te, in->te_bytes, in->dev);
  cached_release(in->d_cls, in->sz_cls, in->dev);
  cached_release(in->d_gex, in->sz_gex, in->dev);
  cudaSetDevice(cur);
  if (in->ev_fork) cudaEventDestroy(in->ev_fork);
  if (in->ev_join) cudaEventDestroy(in->ev_join);
  delete in;
  return HPS_OK;
}

int hps_stage_table(HpsInstance* in, int32_t t, int32_t first, int32_t last, double* out4) {
  if (!in || !out4) return set_err(HPS_E_INVALID_ARG, "null argument");
  if (t < 0 || t >= in->c.T || first < 0 || last < first || last >= in->c.L)
    return set_err(HPS_E_INVALID_ARG, "stage range out of bounds");
  const StageEntry& s = in->h_stages[entry_index(in->c.P, t, first, last)];
  if (!s.valid) return set_err(HPS_E_PLAN, "layer profiles do not cover the type");
  out4[0] = s.oct; out4[1] = s.odt; out4[2] = s.alpha; out4[3] = s.beta;
  return HPS_OK;
}

int hps_score_plans(HpsInstance* in, const uint8_t* d_plans, int64_t n, const HpsPlanResults* r,
                    void* stream) {
  if (!in || !r || !r->cost || !r->status || n < 0) return set_err(HPS_E_INVALID_ARG, "null argument");
  if (n == 0) return HPS_OK;
  cudaStream_t st = (cudaStream_t)stream;
  PlanSource src{};
  src.mode = 0;
  src.plans = d_plans;
  // super-chunks as in argmin_common: the pending list holds a whole chunk
  if (int rc = chk_bind(in, st)) return rc;
  const uint64_t sc = in->super_chunk;
  const uint64_t cap = std::min<uint64_t>((uint64_t)n, sc);
  char* buf = nullptr;
  CUDA_TRY(cudaMallocAsync(&buf, sizeof(unsigned long long) * cap + 64, st));
  unsigned long long* list = reinterpret_cast<unsigned long long*>(buf);
  unsigned int* count = reinterpret_cast<unsigned int*>(list + cap);
  const int L = in->c.L;
  for (uint64_t s0 = 0; s0 < (uint64_t)n; s0 += sc) {
    const uint64_t m = std::min<uint64_t>((uint64_t)n, s0 + sc) - s0;
    const PlanSource sub = advance_source(src, s0, L);
    Outputs o{r->cost + s0, r->status + s0, r->gap ? r->gap + s0 : nullptr, r->ps ? r->ps + s0 : nullptr,
              r->num_stages ? r->num_stages + s0 : nullptr, r->k ? r->k + s0 * (uint64_t)L : nullptr};
    CUDA_TRY(cudaMemsetAsync(count, 0, sizeof(unsigned int), st));
    Pending pend{list, count, (unsigned)m};
    int rc = in->fast ? dispatch_split<false>(in, sub, m, o, pend, 0, nullptr, grid_for(in, m), st)
                      : dispatch_eval<false>(in, sub, m, o, pend, 0, nullptr, grid_for(in, m), st);
    if (rc) return rc;
    rc = run_slow(in, sub, o, pend, 0, 0, nullptr, st);
    if (rc) return rc;
  }
  CUDA_TRY(cudaFreeAsync(buf, st));
  return HPS_OK;
}

int hps_enum_argmin(HpsInstance* in, uint64_t begin, uint64_t end, int32_t feasible_only,
                    HpsArgmin* d_best, void* stream) {
  if (!in || !d_best || end < begin) return set_err(HPS_E_INVALID_ARG, "bad range");
  // T^L must fit in 64 bits
  long double total = powl((long double)in->c.T, (long double)in->c.L);
  if (total > 1.8e19L) return set_err(HPS_E_CONFIG, "T^L does not fit a 64-bit enumeration index");
  uint64_t tot = 1;
  for (int l = 0; l < in->c.L; l++) tot *= (uint64_t)in->c.T;
  if (end > tot) return set_err(HPS_E_INVALID_ARG, "range beyond T^L");
  PlanSource src{};
  src.mode = 1;
  src.begin = begin;
  src.stride = 1;
  uint64_t pw = 1;
  for (int l = in->c.L - 1; l >= 0; l--) { src.tpow[l] = pw; pw *= (uint64_t)in->c.T; }
  return argmin_common(in, src, end - begin, feasible_only, d_best, (cudaStream_t)stream);
}

int hps_enum_argmin_strided(HpsInstance* in, uint64_t first, uint64_t stride, uint64_t count,
                            int32_t feasible_only, HpsArgmin* d_best, void* stream) {
  if (!in || !d_best || stride == 0) return set_err(HPS_E_INVALID_ARG, "bad stride");
  long double total = powl((long double)in->c.T, (long double)in->c.L);
  if (total > 1.8e19L) return set_err(HPS_E_CONFIG, "T^L does not fit a 64-bit enumeration index");
  uint64_t tot = 1;
  for (int l = 0; l < in->c.L; l++) tot *= (uint64_t)in->c.T;
  if (count > 0 && (first >= tot || (count - 1) > (tot - 1 - first) / stride))
    return set_err(HPS_E_INVALID_ARG, "strided range beyond T^L");
  PlanSource src{};
  src.mode = 1;
  src.begin = first;
  src.stride = stride;
  uint64_t pw = 1;
  for (int l = in->c.L - 1; l >= 0; l--) { src.tpow[l] = pw; pw *= (uint64_t)in->c.T; }
  return argmin_common(in, src, count, feasible_only, d_best, (cudaStream_t)stream);
}

int hps_enum_argmin_pruned(HpsInstance* in, int32_t depth, double incumbent, HpsArgmin* d_best,
                           HpsPruneStats* stats, void* stream) {
  if (!in || !d_best) return set_err(HPS_E_INVALID_ARG, "null argument");
  const int L = in->c.L, T = in->c.T;
  long double total = powl((long double)T, (long double)L);
  if (total > 1.8e19L) return set_err(HPS_E_CONFIG, "T^L does not fit a 64-bit enumeration index");
  if (depth < 1 || depth >= L) return set_err(HPS_E_INVALID_ARG, "prefix depth must be in [1, L)");
  uint64_t npref = 1, R = 1;
  for (int l = 0; l < depth; l++) npref *= (uint64_t)T;
  for (int l = depth; l < L; l++) R *= (uint64_t)T;
  if (npref > (1ull << 28)) return set_err(HPS_E_CONFIG, "too many prefixes (lower the depth)");
  // every plan the bound may skip must be one the reference scores without raising
  if (in->c.ps_type < 0) return set_err(HPS_E_CONFIG, "pruning needs a CPU type (PS cores)");
  for (const StageEntry& e : in->h_stages)
    if (!e.valid) return set_err(HPS_E_CONFIG, "pruning needs every layer profiled on every type");
  cudaStream_t st = (cudaStream_t)stream;
  // geometric E grid from the smallest serial floor of any stage to B / limit
  double emin = in->c.tau_limit;
  for (const StageEntry& e : in->h_stages)
    if (e.valid && e.serial > 0 && e.serial < emin) emin = e.serial;
  emin = std::max(emin, in->c.tau_limit * 1e-12);
  std::vector<double> grid(kPruneCells + 1);
  for (int k = 0; k <= kPruneCells; k++)
    grid[k] = emin * std::pow(in->c.tau_limit / emin, (double)k / kPruneCells);
  grid[kPruneCells] = in->c.tau_limit * (1.0 + 1e-12);
  const int ne = T * in->c.P;
  const size_t nF = (size_t)(kPruneCells + 1) * ne, nS = (size_t)(kPruneCells + 1) * (L + 1) * (T + 1);
  char* buf = nullptr;
  const size_t bytes = sizeof(double) * (grid.size() + nF + nS + npref + 1) + sizeof(uint32_t) * (npref + 4) +
                       sizeof(HpsArgmin) * 2 + 256;
  CUDA_TRY(cudaMallocAsync(&buf, bytes, st));
  double* dE = reinterpret_cast<double*>(buf);
  double* dF = dE + grid.size();
  double* dS = dF + nF;
  double* dLB = dS + nS;
  double* dminlb = dLB + npref;
  HpsArgmin* keys = reinterpret_cast<HpsArgmin*>(dminlb + 1);
  uint32_t* list = reinterpret_cast<uint32_t*>(keys + 2);
  uint32_t* misc = list + npref;   // [0] survivors, [1] best prefix
  CUDA_TRY(cudaMemcpyAsync(dE, grid.data(), sizeof(double) * grid.size(), cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemsetAsync(misc, 0, sizeof(uint32_t) * 4, st));
  HPS_COUNT_LAUNCH();
  prune_f_kernel<<<(unsigned)((nF + 255) / 256), 256, 0, st>>>(in->c, in->tb, dE, dF);
  CUDA_TRY(cudaGetLastError());
  HPS_COUNT_LAUNCH();
  prune_suffix_kernel<<<kPruneCells + 1, 32, 0, st>>>(in->c, dF, dS);
  CUDA_TRY(cudaGetLastError());
  HPS_COUNT_LAUNCH();
  prune_bound_kernel<<<(unsigned)((npref + 127) / 128), 128, 0, st>>>(in->c, in->tb, dE, dF, dS, depth, npref, dLB);
  CUDA_TRY(cudaGetLastError());
  HPS_COUNT_LAUNCH();
  prune_argmin_kernel<<<1, 256, 0, st>>>(dLB, npref, misc + 1, dminlb);
  CUDA_TRY(cudaGetLastError());
  uint32_t first = 0xffffffffu;
  double min_lb = 0.0;
  CUDA_TRY(cudaMemcpyAsync(&first, misc + 1, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(&min_lb, dminlb, sizeof(double), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  uint64_t evaluated = 0;
  const bool own_incumbent = !(incumbent < __builtin_inf());
  PlanSource src{};
  src.mode = 1;
  src.stride = 1;
  uint64_t pw = 1;
  for (int l = L - 1; l >= 0; l--) { src.tpow[l] = pw; pw *= (uint64_t)T; }
  if (own_incumbent && first != 0xffffffffu) {   // incumbent: the subtree with the smallest bound
    src.begin = (uint64_t)first * R;
    if (int rc = argmin_common(in, src, R, 1, keys, st)) return rc;
    evaluated += R;
  } else {
    first = 0xffffffffu;
    HPS_COUNT_LAUNCH();
    finish_argmin<<<1, 256, 0, st>>>(nullptr, 0, nullptr, 0, 0, keys);
    CUDA_TRY(cudaGetLastError());
  }
  HPS_COUNT_LAUNCH();
  prune_survivors_kernel<<<(unsigned)((npref + 255) / 256), 256, 0, st>>>(
      dLB, npref, own_incumbent ? keys : nullptr, incumbent, first, list, misc);
  CUDA_TRY(cudaGetLastError());
  uint32_t nsurv = 0;
  double inc_cost = incumbent;
  CUDA_TRY(cudaMemcpyAsync(&nsurv, misc, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
  if (own_incumbent) CUDA_TRY(cudaMemcpyAsync(&inc_cost, &keys->cost, sizeof(double), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  PlanSource sv{};
  sv.mode = 3;
  sv.stride = R;
  sv.prefixes = list;
  memcpy(sv.tpow, src.tpow, sizeof(src.tpow));
  if (int rc = argmin_common(in, sv, (uint64_t)nsurv * R, 1, keys + 1, st)) return rc;
  evaluated += (uint64_t)nsurv * R;
  HPS_COUNT_LAUNCH();
  merge_argmin<<<1, 32, 0, st>>>(keys, 2, evaluated, d_best);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaFreeAsync(buf, st));
  if (stats) {
    stats->prefixes = npref;
    stats->survivors = nsurv;
    stats->evaluated = evaluated;
    stats->incumbent_cost = inc_cost;
    stats->min_bound = min_lb;
    stats->depth = depth;
    stats->subtree = R;
  }
  return HPS_OK;
}

int hps_plans_argmin(HpsInstance* in, const uint8_t* d_plans, int64_t n, int32_t feasible_only,
                     HpsArgmin* d_best, void* stream) {
  if (!in || !d_best || n < 0) return set_err(HPS_E_INVALID_ARG, "null argument");
  PlanSource src{};
  src.mode = 0;
  src.plans = d_plans;
  int b = 0;
  while ((1 << b) < in->c.T) b++;
  src.tbits = b > 0 ? b : 1;
  if (src.tbits * in->c.L > 128) return set_err(HPS_E_CONFIG, "assignment rank exceeds 128 bits");
  return argmin_common(in, src, (uint64_t)n, feasible_only, d_best, (cudaStream_t)stream);
}

int hps_random_argmin(HpsInstance* in, const HpsPcg64* g, uint64_t first, uint64_t n,
                      HpsArgmin* d_best, void* stream) {
  if (!in || !g || !d_best) return set_err(HPS_E_INVALID_ARG, "null argument");
  if (in->c.T & (in->c.T - 1)) return set_err(HPS_E_CONFIG, "in-kernel plan generation needs a power-of-two T");
  PlanSource src{};
  fill_random_source(in, g, first, src);
  if (src.tbits * in->c.L > 128) return set_err(HPS_E_CONFIG, "assignment rank exceeds 128 bits");
  return argmin_common(in, src, n, 0, d_best, (cudaStream_t)stream);
}

}  // extern "C"

namespace {
__global__ void gen_plans_kernel(const InstanceConsts c, const PlanSource src, uint64_t n, uint8_t* out) {
  const int lane = threadIdx.x & 31;
  const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t p = gw; p < n; p += nw) {
    int d0, d1;
    u128 rank;
    load_digits<2>(c, src, p, d0, d1, rank);
    if (lane < c.L) out[p * c.L + lane] = (uint8_t)d0;
    if (lane + 32 < c.L) out[p * c.L + lane + 32] = (uint8_t)d1;
  }
}

__global__ void report_kernel(const InstanceConsts c, const DeviceTables tb, const uint8_t* plans,
                              const int32_t* k, const int32_t* ps, int64_t n, double* ct, double* dt,
                              double* et, double* tp, double* ptp, double* exec, double* cost,
                              uint8_t* feasible) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int L = c.L;
  const uint8_t* pl = plans + i * L;
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  int s = 0, start = 0;
  double overall = inf;
  int order[kMaxT];
  long long tot[kMaxT];
  int nt = 0;
  unsigned seen = 0;
  for (int pos = 1; pos <= L; pos++) {
    if (pos < L && pl[pos] == pl[start]) continue;
    const int t = pl[start];
    const StageEntry& e = tb.stages[entry_index(c.P, t, start, pos - 1)];
    const double kk = (double)k[i * L + s];
    const double a = e.c_oct * (e.oma + e.alpha / kk), b = e.c_odt * (e.omb + e.beta / kk);
    const double x = pmax(a, b);
    const double tpp = (x > 0) ? c.batch / x : inf;
    ct[i * L + s] = a; dt[i * L + s] = b; et[i * L + s] = x; tp[i * L + s] = tpp;
    overall = (s == 0) ? tpp : pmin(overall, tpp);
    if (!(seen >> t & 1u)) { seen |= 1u << t; order[nt] = t; tot[nt] = 0; nt++; }
    for (int j = 0; j < nt; j++) if (order[j] == t) { tot[j] += k[i * L + s]; break; }
    s++;
    start = pos;
  }
  const int pcount = ps ? ps[i] : 0;
  if (pcount > 0 && c.ps_type >= 0) {
    const int t = c.ps_type;
    if (!(seen >> t & 1u)) { seen |= 1u << t; order[nt] = t; tot[nt] = 0; nt++; }
    for (int j = 0; j < nt; j++) if (order[j] == t) { tot[j] += pcount; break; }
  }
  const double ex = (overall > 0 && overall != inf) ? c.work / overall : 0.0;
  double per_second = 0.0;
  bool quota_ok = true;
  for (int j = 0; j < nt; j++) {
    per_second += c.price_h[order[j]] / 3600.0 * (double)tot[j];
    if (tot[j] > c.quota[order[j]]) quota_ok = false;
  }
  ptp[i] = overall;
  exec[i] = ex;
  cost[i] = ex * per_second;
  feasible[i] = (overall > c.limit) && quota_ok;
}

// InfeasibleError details (ls/provisioner.py:98-101, 164-174, 407-411, 421-425, 508-511), one
// thread per plan: the fields the reference's message text names, recomputed from the stage
// table for the status the scorer returned.
__global__ void explain_kernel(const InstanceConsts c, const DeviceTables tb, const uint8_t* plans,
                               const uint8_t* status, const int32_t* k, int64_t n, HpsExplain* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int L = c.L;
  const uint8_t* pl = plans + i * L;
  HpsExplain e;
  memset(&e, 0, sizeof(e));
  e.status = status[i] & 0x7f;
  int ent[kMaxL];
  int S = 0, last0 = L - 1;
  for (int pos = 1, start = 0; pos <= L; pos++) {   // build_stages runs (ls/domain.py:293-296)
    if (pos < L && pl[pos] == pl[start]) continue;
    if (pl[start] >= c.T) { out[i] = e; return; }
    if (S == 0) last0 = pos - 1;
    ent[S++] = entry_index(c.P, pl[start], start, pos - 1);
    start = pos;
  }
  const StageEntry& s0 = tb.stages[ent[0]];
  const double tau_hi = tb.stage0[s0.type * L + last0].tau_hi;
  if (e.status == HPS_ST_MIN_K1) {   // min_k1: computation side first (ls/provisioner.py:89-101)
    const double budget = c.limit * c.bo;
    e.side = (s0.oct != 0 && budget - (1.0 - s0.alpha) * s0.oct <= 0) ? 0 : 1;
  } else if (e.status == HPS_ST_SERIAL) {   // max(stages, key=serial time): the first maximum
    double best = -1.0;
    for (int s = 0; s < S; s++) {
      const double v = tb.stages[ent[s]].serial;
      if (v > best) { best = v; e.stage = s; }
    }
    e.serial = 0.0;
    for (int s = 0; s < S; s++) {   // _serial_floor: max(floor, ct side, dt side) per stage
      const StageEntry& st = tb.stages[ent[s]];
      e.serial = pmax(pmax(e.serial, st.c_oct * st.oma), st.c_odt * st.omb);
    }
    e.tau_hi = tau_hi;
  } else if (e.status == HPS_ST_FLOOR_TAU_HI) {   // the first raising _floor_count at tau_hi
    for (int s = 0; s < S; s++) {
      const StageEntry& st = tb.stages[ent[s]];
      bool raised = false;
      for (int side = 0; side < 2 && !raised; side++) {
        const double work = side ? st.odt : st.oct, frac = side ? st.beta : st.alpha;
        if (work == 0) continue;
        const double h = tau_hi * c.bo / work - (side ? st.omb : st.oma);
        if (frac == 0.0 ? !(h >= 0) : (h <= 0)) {
          raised = true;
          e.stage = s; e.side = side; e.serial_side = (frac == 0.0);
        }
      }
      if (raised) break;
    }
  } else if (e.status == HPS_ST_QUOTA_TAU_HI) {   // first type (ascending id) over its quota
    u128 tot[kMaxT];
    for (int t = 0; t < c.T; t++) tot[t] = 0;
    for (int s = 0; s < S; s++) {
      const StageEntry& st = tb.stages[ent[s]];
      double r, g;
      if (floor_count(st, tau_hi, c.bo, r, g)) tot[st.type] += dbl_to_u128(iceil(r));
    }
    for (int t = 0; t < c.T; t++)
      if (tot[t] > (u128)c.quota[t]) {
        e.type = t;
        e.units_hi = (uint64_t)(tot[t] >> 64);
        e.units_lo = (uint64_t)tot[t];
        break;
      }
  } else if (e.status == HPS_ST_PS_QUOTA && k != nullptr && c.ps_type >= 0) {
    long long accel = 0, have = 0;
    for (int s = 0; s < S; s++) {
      const int t = tb.stages[ent[s]].type;
      const long long kk = k[i * L + s];
      if (!c.is_cpu[t]) accel += kk;
      if (t == c.ps_type) have += kk;
    }
    e.ps = (long long)ceil(c.ps_cores_per_gpu * (double)accel - 1e-9);
    e.type = c.ps_type;
    e.units_lo = (uint64_t)(have + e.ps);
  }
  out[i] = e;
}
}  // namespace

extern "C" int hps_explain(HpsInstance* in, const uint8_t* d_plans, const uint8_t* d_status,
                           const int32_t* d_k, int64_t n, HpsExplain* d_out, void* stream) {
  if (!in || !d_plans || !d_status || !d_out || n < 0) return set_err(HPS_E_INVALID_ARG, "null argument");
  if (n == 0) return HPS_OK;
  HPS_COUNT_LAUNCH();
  explain_kernel<<<(unsigned)((n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(in->c, in->tb, d_plans, d_status,
                                                                                d_k, n, d_out);
  CUDA_TRY(cudaGetLastError());
  return HPS_OK;
}

std::atomic<unsigned long long> hps::g_launches{0};

extern "C" uint64_t hps_launch_count(void) { return hps::g_launches.load(std::memory_order_relaxed); }

extern "C" int hps_stats_read(unsigned long long* out, int n, int reset) {
#ifdef HPS_STATS
  if (n > 24) n = 24;
  CUDA_TRY(cudaMemcpyFromSymbol(out, hps::g_stats, sizeof(unsigned long long) * n));
  if (reset) {
    unsigned long long z[24] = {0};
    CUDA_TRY(cudaMemcpyToSymbol(hps::g_stats, z, sizeof(z)));
  }
  return HPS_OK;
#else
  (void)out; (void)n; (void)reset;
  return set_err(HPS_E_CONFIG, "built without -DHPS_STATS");
#endif
}

extern "C" int hps_random_plans(HpsInstance* in, const HpsPcg64* g, uint64_t first, uint64_t n,
                                uint8_t* d_plans, void* stream) {
  if (!in || !g || !d_plans) return set_err(HPS_E_INVALID_ARG, "null argument");
  if (in->c.T & (in->c.T - 1)) return set_err(HPS_E_CONFIG, "in-kernel plan generation needs a power-of-two T");
  PlanSource src{};
  fill_random_source(in, g, first, src);
  if (n == 0) return HPS_OK;
  const uint64_t warps = std::min<uint64_t>(n, (uint64_t)in->sm_count * 64);
  HPS_COUNT_LAUNCH();
  gen_plans_kernel<<<(unsigned)((warps + 7) / 8), 256, 0, (cudaStream_t)stream>>>(in->c, src, n, d_plans);
  CUDA_TRY(cudaGetLastError());
  return HPS_OK;
}

extern "C" int hps_report(HpsInstance* in, const uint8_t* d_plans, const int32_t* d_k, const int32_t* d_ps,
                          int64_t n, double* d_ct, double* d_dt, double* d_et, double* d_tp,
                          double* d_pipeline_tp, double* d_exec_time, double* d_cost, uint8_t* d_feasible,
                          void* stream) {
  if (!in || n < 0) return set_err(HPS_E_INVALID_ARG, "bad argument");
  if (n == 0) return HPS_OK;
  HPS_COUNT_LAUNCH();
  report_kernel<<<(unsigned)((n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
      in->c, in->tb, d_plans, d_k, d_ps, n, d_ct, d_dt, d_et, d_tp, d_pipeline_tp, d_exec_time, d_cost, d_feasible);
  CUDA_TRY(cudaGetLastError());
  return HPS_OK;
}

// ---- static provisioning baselines (ls/provisioner.py:516-561) --------------------------------
namespace {
// One thread per plan. Counts are linear in the multiplier g (k_s = f_s * g, per-type totals
// m_t * g), so the quota break of the reference's scan is g_max = min_t floor(Q_t / m_t); the
// throughput test is monotone in g whenever every stage's ct/dt coefficients are >= 0 (et is
// then non-increasing in k under IEEE rounding), so the first feasible g is found by bisection
// over [1, g_max]. Otherwise the scan runs literally.
__device__ bool static_feasible(const InstanceConsts& c, const StageEntry* const* ent, const int* f,
                                int S, long long g, double& overall) {
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  overall = inf;
  for (int s = 0; s < S; s++) {
    const double kk = (double)((long long)f[s] * g);
    const double x = stage_et(*ent[s], kk);
    const double tp = (x > 0) ? c.batch / x : inf;
    overall = (s == 0) ? tp : pmin(overall, tp);
  }
  return overall > c.limit;
}

__global__ void static_kernel(const InstanceConsts c, const DeviceTables tb, const uint8_t* plans, int64_t n,
                              int mode, int cpu_per_gpu, Outputs o) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int L = c.L;
  const uint8_t* pl = plans + i * L;
  const double nan = __longlong_as_double(0x7ff8000000000000LL);
  int32_t* kout = o.k ? o.k + i * L : nullptr;
  if (kout) for (int s = 0; s < L; s++) kout[s] = 0;
  for (int l = 0; l < L; l++) {
    if (pl[l] >= c.T) {   // validate_plan (ls/provisioner.py:536)
      o.cost[i] = nan; o.status[i] = HPS_ST_INVALID;
      if (o.gap) o.gap[i] = 0.0;
      if (o.ps) o.ps[i] = 0;
      if (o.num_stages) o.num_stages[i] = 0;
      return;
    }
  }
  const StageEntry* ent[kMaxL];
  int f[kMaxL];
  int order[kMaxT + 1];
  long long m[kMaxT + 1];
  int nt = 0, S = 0, start = 0;
  long long n_acc = 0;
  bool mono = c.batch >= 0.0;
  for (int pos = 1; pos <= L; pos++) {   // build_stages (ls/domain.py:293-296)
    if (pos < L && pl[pos] == pl[start]) continue;
    const int t = pl[start];
    ent[S] = &tb.stages[entry_index(c.P, t, start, pos - 1)];
    f[S] = c.is_cpu[t] ? cpu_per_gpu : 1;
    if (!c.is_cpu[t]) n_acc++;
    mono = mono && ent[S]->c_oct >= 0.0 && ent[S]->alpha >= 0.0 && ent[S]->c_odt >= 0.0 &&
           ent[S]->beta >= 0.0;
    int j = 0;
    while (j < nt && order[j] != t) j++;
    if (j == nt) { order[nt] = t; m[nt] = 0; nt++; }
    m[j] += f[S];
    S++;
    start = pos;
  }
  if (o.num_stages) o.num_stages[i] = S;
  if (c.ps_type < 0) {   // catalog.cheapest_cpu_type() raises first (ls/provisioner.py:538)
    o.cost[i] = nan; o.status[i] = HPS_ST_NO_CPU_TYPE;
    if (o.gap) o.gap[i] = 0.0;
    if (o.ps) o.ps[i] = 0;
    return;
  }
  const long long ps_per_g = (mode == 2) ? (long long)cpu_per_gpu * n_acc : 0;
  if (ps_per_g > 0) {
    int j = 0;
    while (j < nt && order[j] != c.ps_type) j++;
    if (j == nt) { order[nt] = c.ps_type; m[nt] = 0; nt++; }
    m[j] += ps_per_g;
  }
  // over_quota(g) <=> some m_t * g > Q_t; max_quota bounds the scan (ls/provisioner.py:539-552)
  long long gmax = LLONG_MAX;
  long long maxq = 0;
  for (int t = 0; t < c.T; t++) maxq = (c.quota[t] > maxq) ? c.quota[t] : maxq;
  for (int j = 0; j < nt; j++) {
    if (m[j] <= 0) continue;
    const long long q = c.quota[order[j]];
    const long long gm = (q < 0) ? -1 : q / m[j];
    gmax = (gm < gmax) ? gm : gmax;
  }
  gmax = (maxq < gmax) ? maxq : gmax;
  long long g_found = 0;
  double overall = 0.0;
  if (gmax >= 1) {
    if (mono) {
      if (static_feasible(c, ent, f, S, gmax, overall)) {
        long long lo = 0, hi = gmax;   // feasible(hi), !feasible(lo) (lo = 0 is a sentinel)
        while (hi - lo > 1) {
          const long long mid = lo + (hi - lo) / 2;
          double ov;
          if (static_feasible(c, ent, f, S, mid, ov)) hi = mid; else lo = mid;
        }
        g_found = hi;
      }
    } else {
      for (long long g = 1; g <= gmax; g++) {
        double ov;
        if (static_feasible(c, ent, f, S, g, ov)) { g_found = g; break; }
      }
    }
  }
  if (g_found == 0) {   // InfeasibleError(gap=1.0) -> penalty_cost (ls/provisioner.py:557-561)
    o.cost[i] = c.penalty_scale * (1.0 + 1.0); o.status[i] = HPS_ST_STATIC_NONE;
    if (o.gap) o.gap[i] = 1.0;
    if (o.ps) o.ps[i] = 0;
    return;
  }
  static_feasible(c, ent, f, S, g_found, overall);
  // evaluate(): exec time and cost over per_type_totals in insertion order (ls/costmodel.py:90-99)
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  const double ex = (overall > 0 && overall != inf) ? c.work / overall : 0.0;
  double per_second = 0.0;
  for (int j = 0; j < nt; j++) per_second += c.price_h[order[j]] / 3600.0 * (double)(m[j] * g_found);
  o.cost[i] = ex * per_second;
  o.status[i] = HPS_ST_OK;
  if (o.gap) o.gap[i] = 0.0;
  if (o.ps) o.ps[i] = (int32_t)(ps_per_g * g_found);
  if (kout) for (int s = 0; s < S; s++) kout[s] = (int32_t)((long long)f[s] * g_found);
}
}  // namespace

extern "C" int hps_score_plans_static(HpsInstance* in, const uint8_t* d_plans, int64_t n, int32_t mode,
                                      int32_t cpu_per_gpu, const HpsPlanResults* r, void* stream) {
  if (!in || !r || !r->cost || !r->status || n < 0) return set_err(HPS_E_INVALID_ARG, "null argument");
  if (mode != HPS_MODE_STARATIO && mode != HPS_MODE_STAPSRATIO)
    return set_err(HPS_E_INVALID_ARG, "unknown static provisioning mode");
  if (cpu_per_gpu < 1) return set_err(HPS_E_INVALID_ARG, "cpu_per_gpu must be >= 1");
  if (n == 0) return HPS_OK;
  Outputs o{r->cost, r->status, r->gap, r->ps, r->num_stages, r->k};
  HPS_COUNT_LAUNCH();
  static_kernel<<<(unsigned)((n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(in->c, in->tb, d_plans, n, mode,
                                                                               cpu_per_gpu, o);
  CUDA_TRY(cudaGetLastError());
  return HPS_OK;
}
