// hps_prune.cuh — certified subtree pruning for the brute-force argmin (an exact accelerator of
// brute_force, ls/baselines.py:63-87: same winner, ties included; not a different search).
//
// Enumeration index order puts layer 0 most significant, so the plans sharing the assignment of
// layers 0..d-1 (a "prefix") are one contiguous index range of T^(L-d) plans. For every prefix a
// LOWER BOUND on the monetary cost of any plan in its range is computed; ranges whose bound
// exceeds an incumbent's cost are skipped, the rest are swept by the ordinary kernels.
//
// The bound. A plan's cost is exec_time * per_second = (work / B) * E * per_second with E the
// largest stage execution time (ls/costmodel.py:102-167), and per_second >= sum over stages of
// price_s * k_s (PS cores only add). Each stage's count satisfies et_s(k_s) <= E, i.e.
// k_s >= q_s(E) = max over sides of frac / (E * bo / work - (1 - frac)) (ls/provisioner.py:150-176)
// and k_s is an integer >= 1. q_s is non-increasing in E, so on a cell [Ea, Eb] of E:
//     cost >= (work / B) * Ea * sum_s price_s * max(1, ceil(q_s(Eb) (1 - 1e-12) - 1e-9)).
// The stages of a completion are the prefix's closed runs (known), the open last run extended
// to some layer e >= d-1, and any runs over layers e+1..L-1: the cheapest such suffix per cell is a
// small dynamic program over (layer, previous type) (prune_suffix_kernel). The plan's bound is
// the minimum over the cells E covers (from the prefix's largest serial floor up to B / limit,
// the largest E any feasible plan has, ls/provisioner.py:395). Quotas are ignored (relaxation).
// The 1e-12 / 1e-9 slacks and the enlarged headroom below cover every rounding of the reference's
// own arithmetic, and a range is skipped only when bound * (1 - 1e-9) > incumbent, so a skipped
// plan is strictly costlier than the winner (it can be neither the minimum nor a tie).
#pragma once

namespace hps {

constexpr int kPruneCells = 128;   // geometric cells of E between the smallest serial floor and B / limit

// price * max(1, ceil(q(E) - 1e-9)) lower bound for stage entry s at E (+inf: no count reaches E)
__device__ __forceinline__ double prune_stage_term(const InstanceConsts& c, const StageEntry& s, double E) {
  double q = 1.0;
  bool ambiguous = false;
#pragma unroll
  for (int side = 0; side < 2; side++) {
    const double work = side ? s.odt : s.oct;
    if (work == 0) continue;
    const double frac = side ? s.beta : s.alpha, omf = side ? s.omb : s.oma;
    const double hb = E * c.bo / work;
    const double h = hb - omf;
    const double err = (fabs(hb) + fabs(omf)) * 1e-15;   // >> the reference's rounding of h
    if (h + err < 0) return __longlong_as_double(0x7ff0000000000000LL);   // raises for every E' <= E
    if (frac == 0.0) continue;
    if (h - err <= 0) { ambiguous = true; continue; }
    q = fmax(q, frac / (h + err) * (1.0 - 1e-12));
  }
  const double k = ambiguous ? 1.0 : fmax(1.0, ceil(q - 1e-9));
  return c.price_s[s.type] * k;
}

// F[k][e] for grid point E[k] and stage entry e
__global__ void prune_f_kernel(const InstanceConsts c, const DeviceTables tb, const double* E, double* F) {
  const int ne = c.T * c.P;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (kPruneCells + 1) * ne) return;
  const int k = i / ne, e = i - k * ne;
  F[i] = tb.stages[e].valid ? prune_stage_term(c, tb.stages[e], E[k]) : __longlong_as_double(0x7ff0000000000000LL);
}

// SUF[k][j][tp]: cheapest sum of stage terms over layers j..L-1 whose first run's type differs
// from tp (tp == T: any type), at grid point k. One block per grid point.
__global__ void prune_suffix_kernel(const InstanceConsts c, const double* F, double* SUF) {
  const int k = blockIdx.x, tp = threadIdx.x, L = c.L, T = c.T, ne = T * c.P;
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  double* S = SUF + (size_t)k * (L + 1) * (T + 1);
  const double* Fk = F + (size_t)k * ne;
  if (tp <= T) S[L * (T + 1) + tp] = 0.0;
  __syncthreads();
  for (int j = L - 1; j >= 0; j--) {
    if (tp <= T) {
      double m = inf;
      for (int t = 0; t < T; t++) {
        if (t == tp) continue;
        for (int e = j; e < L; e++) {
          const double v = Fk[entry_index(c.P, t, j, e)] + S[(e + 1) * (T + 1) + t];
          m = v < m ? v : m;
        }
      }
      S[j * (T + 1) + tp] = m;
    }
    __syncthreads();
  }
}

// lower bound of every prefix id (layer 0 most significant digit of d digits)
__global__ void prune_bound_kernel(const InstanceConsts c, const DeviceTables tb, const double* E, const double* F,
                                   const double* SUF, int d, uint64_t npref, double* lb) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= npref) return;
  const int L = c.L, T = c.T, ne = T * c.P;
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  int dig[kMaxL];
  uint64_t x = i;
  for (int l = d - 1; l >= 0; l--) { dig[l] = (int)(x % (uint64_t)T); x /= (uint64_t)T; }
  // closed runs of the prefix and the open last run (tm, am)
  int closed[kMaxL];
  int nclosed = 0, start = 0;
  double emin = 0.0;
  for (int p = 1; p < d; p++)
    if (dig[p] != dig[start]) {
      const int e = entry_index(c.P, dig[start], start, p - 1);
      closed[nclosed++] = e;
      emin = fmax(emin, tb.stages[e].serial);
      start = p;
    }
  const int tm = dig[start], am = start;
  const double C = c.work / c.batch;
  double best = inf;
  // cells [E[k-1], E[k]] for k = 1..K, plus [emin, E[0]] evaluated at E[0]
  for (int k = 0; k <= kPruneCells; k++) {
    const double eb = E[k];
    if (eb < emin) continue;   // E >= the closed runs' serial floors
    const double ea = (k == 0) ? emin : fmax(E[k - 1], emin);
    const double* Fk = F + (size_t)k * ne;
    double fixed = 0.0;
    for (int q = 0; q < nclosed; q++) fixed += Fk[closed[q]];
    if (!(fixed < inf)) continue;
    const double* S = SUF + (size_t)k * (L + 1) * (T + 1);
    double m = inf;
    for (int e = d - 1; e < L; e++) {
      const double v = Fk[entry_index(c.P, tm, am, e)] + S[(e + 1) * (T + 1) + tm];
      m = v < m ? v : m;
    }
    const double b = C * ea * (fixed + m);
    best = b < best ? b : best;
  }
  lb[i] = best;
}

// index of the smallest bound (first on ties); one block
__global__ void prune_argmin_kernel(const double* lb, uint64_t n, uint32_t* out, double* out_lb) {
  __shared__ double sv[256];
  __shared__ uint32_t si[256];
  double bv = __longlong_as_double(0x7ff0000000000000LL);
  uint32_t bi = 0xffffffffu;
  for (uint64_t i = threadIdx.x; i < n; i += blockDim.x)
    if (lb[i] < bv) { bv = lb[i]; bi = (uint32_t)i; }
  sv[threadIdx.x] = bv;
  si[threadIdx.x] = bi;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int t = 1; t < (int)blockDim.x; t++)
      if (sv[t] < bv || (sv[t] == bv && si[t] < bi)) { bv = sv[t]; bi = si[t]; }
    *out = bi;
    *out_lb = bv;
  }
}

// prefixes that may hold a plan costing <= the incumbent (skip: already swept)
__global__ void prune_survivors_kernel(const double* lb, uint64_t n, const HpsArgmin* inc, double inc_cost,
                                       uint32_t skip, uint32_t* list, unsigned int* count) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || i == skip) return;
  const double best = inc ? inc->cost : inc_cost;
  if (lb[i] * (1.0 - 1e-9) > best) return;
  list[atomicAdd(count, 1u)] = (uint32_t)i;
}

}  // namespace hps
