// hps_policy.cu — the scheduling policy on the device: LSTM/Elman forward (K4), numpy-exact
// categorical sampling from the PCG64 stream (K3), REINFORCE round bookkeeping + BPTT + update
// (K5/K6). Reference: ls/policy/network.py:111-292, ls/policy/training.py:115-274.
//
// Exactness contract (SURVEY.md §7 hard part 4): everything elementwise (gates, c/h updates,
// softmax, outer-product gradient accumulation, winsorising, standardising, dlogits in trace
// order, the parameter update, numpy's pairwise mean/std) is restated operation for operation;
// the three dense contractions (xh @ W, h @ W_out, the BPTT mat-vecs) use FMA dot products whose
// summation order differs from OpenBLAS, so probabilities agree to ~1e-16 relative and sampled
// plans are identical unless a uniform draw lands within that distance of a CDF boundary.
// The hoisted input projection X @ W_x runs on the FP64 tensor cores (mma.sync m8n8k4 f64).
#include "hps_launch.h"
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "hps_device.cuh"

using namespace hps;

namespace {

thread_local std::string g_pol_err;
int perr(int code, const std::string& m) {
  g_pol_err = m;
  return code;
}
#define PCUDA(expr)                                                                      \
  do {                                                                                   \
    cudaError_t _e = (expr);                                                             \
    if (_e != cudaSuccess) return perr(HPS_E_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
  } while (0)

constexpr int kMaxH = 128;
constexpr int kMaxD = 160;

// numpy pairwise_sum (loops_utils.h.src): a block of n <= 128 elements is summed with eight
// accumulators (n < 8: sequentially from -0.0); longer arrays split at n2 = n/2 - (n/2) % 8 and
// return pw(left) + pw(right). No device recursion (it would need a runtime-sized stack): pw_tree
// walks the same tree with an explicit stack, taking leaf sums from a callback.
__device__ double pw_leaf(const double* a, long n, long stride) {
  if (n < 8) {
    double res = -0.0;
    for (long i = 0; i < n; i++) res += a[i * stride];
    return res;
  }
  double r[8];
  for (int j = 0; j < 8; j++) r[j] = a[j * stride];
  long i;
  for (i = 8; i < n - (n % 8); i += 8)
    for (int j = 0; j < 8; j++) r[j] += a[(i + j) * stride];
  double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
  for (; i < n; i++) res += a[i * stride];
  return res;
}

template <class Leaf>
__device__ double pw_tree(long n, Leaf leaf) {
  struct Fr { long off, n; double left; int state; };
  Fr fr[40];   // depth log2(n / 128) + 1
  int sp = 0;
  fr[sp++] = Fr{0, n, 0.0, 0};
  double ret = 0.0;
  while (sp) {
    Fr& f = fr[sp - 1];
    if (f.n <= 128) { ret = leaf(f.off, f.n); sp--; continue; }
    long m2 = f.n / 2;
    m2 -= m2 % 8;
    if (f.state == 0) { f.state = 1; fr[sp++] = Fr{f.off, m2, 0.0, 0}; continue; }
    if (f.state == 1) { f.left = ret; f.state = 2; fr[sp++] = Fr{f.off + m2, f.n - m2, 0.0, 0}; continue; }
    ret = f.left + ret;
    sp--;
  }
  return ret;
}

__device__ double np_pairwise(const double* a, long n, long stride) {
  return pw_tree(n, [&](long off, long m) { return pw_leaf(a + off * stride, m, stride); });
}

// np_pairwise of a[0..n) by a whole block: thread 0 lists the tree's leaves (leaf: >= 2 *
// (n / 64 + 2) ints), the block sums them in parallel (val), thread 0 combines them in the tree's
// order. Same bits as np_pairwise; called by every thread, result returned on all.
__device__ double block_pairwise(const double* a, long n, int* leaf, double* val, double* out) {
  __shared__ int s_nleaf;
  if (threadIdx.x == 0) {
    int nl = 0;
    pw_tree(n, [&](long off, long m) { leaf[2 * nl] = (int)off; leaf[2 * nl + 1] = (int)m; nl++; return 0.0; });
    s_nleaf = nl;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < s_nleaf; i += blockDim.x) val[i] = pw_leaf(a + leaf[2 * i], leaf[2 * i + 1], 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    int next = 0;
    *out = pw_tree(n, [&](long, long) { return val[next++]; });
  }
  __syncthreads();
  return *out;
}

__device__ __forceinline__ double sigmoid_np(double x) {  // ls/policy/network.py:132-138
  if (x >= 0) return 1.0 / (1.0 + exp(-x));
  const double ex = exp(x);
  return ex / (1.0 + ex);
}

struct PolicyDims {
  int L, D, H, T, G4;  // G4 = gates * H
  int lstm;            // 1 lstm, 0 elman
};

struct PolicyBufs {
  double *w_cell, *b_cell, *w_out, *b_out;          // params
  double *gw_cell, *gb_cell, *gw_out, *gb_out;      // grads
  double* feat;                                     // [L][D]
  double* xw;                                       // [L][G4] hoisted x_t @ W_x
  double *xh, *gi, *gf, *go, *gg, *cc, *cp, *tc, *hh;  // caches [L][...]
  double* probs;                                    // [L][T]
  double* cdf;                                      // [L][T] normalised cumulative
  double* dlogits;                                  // [L][T]
  double* scratch;                                  // [G] x 4 work arrays
  double* state;                                    // [16] baseline, best cost, entropy, ...
  int* flags;                                       // [4] non-finite flags
  double* dz;                                       // [L][G4] BPTT gate gradients
  unsigned long long* ctr;                          // [2] next round (1-based), draws consumed
  int* pw_leaf;                                     // block_pairwise leaf table
  double* pw_val;                                   // block_pairwise leaf sums
};

// ---------------------------------------------------------------- K4: forward

// x_t @ W_x for all t on the FP64 tensor cores: [L x D] @ [D x G4], mma.sync m8n8k4 f64.
// One warp per 8x8 output tile; K padded by zeros to a multiple of 4.
__global__ void xw_dmma_kernel(PolicyDims d, const double* feat, const double* w, double* xw) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int tiles_n = (d.G4 + 7) / 8, tiles_m = (d.L + 7) / 8;
  if (warp >= tiles_m * tiles_n) return;
  const int tm = warp / tiles_n, tn = warp % tiles_n;
  double acc[2] = {0.0, 0.0};
  // m8n8k4 f64 fragments: A (row) lane holds A[g][k] with g = lane>>2, k = lane&3;
  // B (col) lane holds B[k][n] with k = lane&3, n = lane>>2; C lane holds C[g][2*(lane&3)+{0,1}]
  const int g = lane >> 2, kq = lane & 3;
  for (int k0 = 0; k0 < d.D; k0 += 4) {
    const int row = tm * 8 + g, k = k0 + kq, col = tn * 8 + g;
    const double a = (row < d.L && k < d.D) ? feat[row * d.D + k] : 0.0;
    const double b = (k < d.D && col < d.G4) ? w[(long)k * d.G4 + col] : 0.0;
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
                 : "+d"(acc[0]), "+d"(acc[1])
                 : "d"(a), "d"(b));
  }
  const int row = tm * 8 + g;
  for (int q = 0; q < 2; q++) {
    const int col = tn * 8 + 2 * kq + q;
    if (row < d.L && col < d.G4) xw[row * d.G4 + col] = acc[q];
  }
}

// Recurrence over layers (ls/policy/network.py:147-200); one block of G4 (>= T) threads.
__global__ void forward_kernel(PolicyDims d, PolicyBufs b, double temperature) {
  extern __shared__ double sm[];
  double* h = sm;                 // [H]
  double* c = h + d.H;            // [H]
  double* z = c + d.H;            // [G4]
  double* lg = z + d.G4;          // [T]
  const int j = threadIdx.x;
  const int H = d.H, D = d.D, G4 = d.G4, T = d.T, DH = D + H;
  if (j < H) { h[j] = 0.0; c[j] = 0.0; }
  // this thread's column of the hidden-state weights W_h stays in registers for all L steps
  // (H <= 64; larger H reads it from global memory each step). Same FMA order either way.
  constexpr int kRegH = 64;
  double wh[kRegH];
  const bool reg = H <= kRegH;
#pragma unroll
  for (int i = 0; i < kRegH; i++) wh[i] = (reg && j < G4 && i < H) ? b.w_cell[(long)(D + i) * G4 + j] : 0.0;
  const double bj = (j < G4) ? b.b_cell[j] : 0.0;
  __syncthreads();
  for (int t = 0; t < d.L; t++) {
    // xh = concat(x_t, h)
    for (int k = j; k < DH; k += blockDim.x) b.xh[t * DH + k] = (k < D) ? b.feat[t * D + k] : h[k - D];
    if (j < G4) {  // z = xh @ W + b: hoisted x part (tensor cores) + h part
      double acc = b.xw[t * G4 + j];
      if (reg) {
#pragma unroll
        for (int i = 0; i < kRegH; i++)
          if (i < H) acc = fma(h[i], wh[i], acc);
      } else {
        for (int i = 0; i < H; i++) acc = fma(h[i], b.w_cell[(long)(D + i) * G4 + j], acc);
      }
      z[j] = acc + bj;
    }
    __syncthreads();
    if (j < H) {
      double hn;
      if (d.lstm) {
        const double gi = sigmoid_np(z[j]), gf = sigmoid_np(z[H + j]), go = sigmoid_np(z[2 * H + j]);
        const double gg = tanh(z[3 * H + j]);
        const double cprev = c[j];
        const double cn = gf * cprev + gi * gg;
        const double tcn = tanh(cn);
        hn = go * tcn;
        b.gi[t * H + j] = gi; b.gf[t * H + j] = gf; b.go[t * H + j] = go; b.gg[t * H + j] = gg;
        b.cc[t * H + j] = cn; b.cp[t * H + j] = cprev; b.tc[t * H + j] = tcn;
        c[j] = cn;
      } else {
        hn = tanh(z[j]);
      }
      b.hh[t * H + j] = hn;
    }
    __syncthreads();
    if (j < H) h[j] = b.hh[t * H + j];
    __syncthreads();
    if (j < T) {  // logits = h @ W_out + b_out
      double acc = 0.0;
      for (int i = 0; i < H; i++) acc = fma(h[i], b.w_out[i * T + j], acc);
      lg[j] = acc + b.b_out[j];
      if (!isfinite(lg[j])) atomicOr(&b.flags[0], 1);
    }
    __syncthreads();
    if (j == 0) {  // softmax(logits / temperature) (ls/policy/network.py:141-144,196-197)
      double sc[16], mx = 0.0;
      for (int a = 0; a < T; a++) { sc[a] = lg[a] / temperature; mx = (a == 0 || sc[a] > mx) ? sc[a] : mx; }
      double ex[16];
      for (int a = 0; a < T; a++) ex[a] = exp(sc[a] - mx);
      const double s = np_pairwise(ex, T, 1);
      double cum = 0.0;
      for (int a = 0; a < T; a++) {
        const double p = ex[a] / s;
        b.probs[t * T + a] = p;
        cum = (a == 0) ? p : cum + p;  // cdf = probs.cumsum() (Generator.choice)
        b.cdf[t * T + a] = cum;
      }
      for (int a = 0; a < T; a++) b.cdf[t * T + a] = b.cdf[t * T + a] / cum;  // cdf /= cdf[-1]
    }
    __syncthreads();
  }
  if (j == 0) {  // entropy_of: -(safe*log(safe)).sum(axis=1).mean()  (network.py:265-268)
    double rows[64];
    for (int t = 0; t < d.L; t++) {
      double e[16];
      for (int a = 0; a < T; a++) {
        double p = b.probs[t * T + a];
        p = p < 1e-300 ? 1e-300 : (p > 1.0 ? 1.0 : p);
        e[a] = -(p * log(p));
      }
      rows[t] = np_pairwise(e, T, 1);
    }
    b.state[2] = np_pairwise(rows, d.L, 1) / (double)d.L;
  }
}

// ---------------------------------------------------------------- K3: sampling

// plan g, layer t consumes draw (first_draw + g*L + t) of the PCG64 stream: one
// Generator.random() per Generator.choice(T, p) (ls/policy/network.py:258).
// first_draw == ~0: the policy's device counter (draws consumed by earlier rounds)
__global__ void sample_kernel(PolicyDims d, const double* cdf, const unsigned long long* ctr, u128 state0,
                              u128 inc, u128 first_draw, long n, uint8_t* plans) {
  const long g = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n) return;
  if (first_draw == (u128)~0ull) first_draw = ctr[1];
  u128 s = pcg_advance(state0, inc, first_draw + (u128)g * (u128)d.L);
  const u128 M = pcg_mult();
  for (int t = 0; t < d.L; t++) {
    s = s * M + inc;
    const uint64_t x = pcg_output(s);
    const double u = (double)(x >> 11) * (1.0 / 9007199254740992.0);
    int a = 0;
    for (int q = 0; q < d.T; q++) a += (cdf[t * d.T + q] <= u) ? 1 : 0;  // searchsorted right
    plans[g * d.L + t] = (uint8_t)a;
  }
}

// ---------------------------------------------------------------- K6: round bookkeeping

struct RoundIn {
  const double* cost;    // [G] ScoredPlan.cost
  const uint8_t* status; // [G]
  const uint8_t* plans;  // [G][L]
  long G;
  double temperature, lr, gamma;
  int round;             // 1-based
  double* history;       // [rounds][4]: mean_cost, best_cost, baseline, entropy
  uint8_t* best_plan;    // [L]
  long long* best_where; // [2]: round, index
};

// block-wide reductions (order-independent ops only: min / max / or)
template <bool MAX>
__device__ double block_minmax_d(double v, double* red) {
  for (int o = 16; o; o >>= 1) {
    const double u = __shfl_xor_sync(0xffffffffu, v, o);
    v = MAX ? (u > v ? u : v) : (u < v ? u : v);
  }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double r = red[0];
  for (int i = 1; i < (int)(blockDim.x >> 5); i++) r = MAX ? (red[i] > r ? red[i] : r) : (red[i] < r ? red[i] : r);
  __syncthreads();
  return r;
}

__device__ long block_min_l(long v, long* red) {
  for (int o = 16; o; o >>= 1) {
    const long u = __shfl_xor_sync(0xffffffffu, v, o);
    v = u < v ? u : v;
  }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  long r = red[0];
  for (int i = 1; i < (int)(blockDim.x >> 5); i++) r = red[i] < r ? red[i] : r;
  __syncthreads();
  return r;
}

// state[0] baseline, state[1] best cost (+inf before round 1), state[2] entropy of the round.
// One block of kRoundThreads threads. Every step is either elementwise (parallel), an
// order-independent min/max (block reductions), numpy's pairwise sum (block_pairwise: same
// recursion, leaves in parallel) or the trace-order dlogits accumulation (one thread per (t, a),
// sequential over g as numpy's `dlogits += ...` loop; its terms are precomputed in parallel).
constexpr int kRoundThreads = 1024;
__global__ void __launch_bounds__(kRoundThreads) round_update_kernel(PolicyDims d, PolicyBufs b, RoundIn in) {
  __shared__ double sh[8];
  __shared__ double red[32];
  __shared__ long redl[32];
  const int tid = threadIdx.x, nt = blockDim.x;
  const long G = in.G;
  double* R = b.scratch;           // rewards after winsorising
  double* X = b.scratch + G;       // R - baseline, then the gradient weights
  double* W = b.scratch + 2 * G;   // squared deviations
  const double base = b.state[0];
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  const int round = (in.round > 0) ? in.round : (int)b.ctr[0];
  // best-ever: the first plan (trace order) reaching the round's minimum, if it beats the best
  // so far (training.py:219-220: strict <, sequential = first index of the minimum)
  double mn = inf;
  for (long g = tid; g < G; g += nt) mn = in.cost[g] < mn ? in.cost[g] : mn;
  mn = block_minmax_d<false>(mn, red);
  const double bc = b.state[1];
  if (mn < bc) {
    long first = G;
    for (long g = tid; g < G; g += nt) if (in.cost[g] == mn && g < first) first = g;
    first = block_min_l(first, redl);
    for (int t = tid; t < d.L; t += nt) in.best_plan[t] = in.plans[first * d.L + t];
    if (tid == 0) {
      b.state[1] = mn;
      in.best_where[0] = round;
      in.best_where[1] = first;
    }
  }
  // rewards; any infeasible?
  int any_bad = 0;
  for (long g = tid; g < G; g += nt) {
    R[g] = -in.cost[g];
    if ((in.status[g] & 0x7f) != HPS_ST_OK) any_bad = 1;
  }
  any_bad = __syncthreads_or(any_bad);
  if (any_bad) {  // winsorise penalised rewards into [b-2u, b-u] (training.py:221-240)
    double spread = -inf, lo = inf, hi = -inf;
    int have = 0;
    for (long g = tid; g < G; g += nt) {
      if ((in.status[g] & 0x7f) == HPS_ST_OK) {
        const double v = fabs(R[g] - base);
        spread = v > spread ? v : spread;
        have = 1;
      } else {
        lo = R[g] < lo ? R[g] : lo;
        hi = R[g] > hi ? R[g] : hi;
      }
    }
    spread = block_minmax_d<true>(spread, red);
    lo = block_minmax_d<false>(lo, red);
    hi = block_minmax_d<true>(hi, red);
    have = __syncthreads_or(have);
    const double unit = 10.0 * (have ? spread : 1.0);
    for (long g = tid; g < G; g += nt)
      if ((in.status[g] & 0x7f) != HPS_ST_OK) {
        const double z = (hi == lo) ? 0.5 : (R[g] - lo) / (hi - lo);
        R[g] = base - unit * (2.0 - z);
      }
    __syncthreads();
  }
  for (long g = tid; g < G; g += nt) X[g] = R[g] - base;
  __syncthreads();
  // np.std(R - b) (pairwise mean, pairwise sum of squares) and np.mean(R)
  const double mean = block_pairwise(X, G, b.pw_leaf, b.pw_val, &sh[0]) / (double)G;
  for (long g = tid; g < G; g += nt) { const double v = X[g] - mean; W[g] = v * v; }
  __syncthreads();
  const double spread = sqrt(block_pairwise(W, G, b.pw_leaf, b.pw_val, &sh[1]) / (double)G);
  const double mean_r = block_pairwise(R, G, b.pw_leaf, b.pw_val, &sh[2]) / (double)G;
  const double scale = 1.0 / (double)G;
  for (long g = tid; g < G; g += nt) {  // gradient weights (training.py:245-252, 136-137)
    double r2 = R[g];
    if (spread > 1e-12) r2 = base + (R[g] - base) / spread;
    X[g] = (r2 - base) * scale;
  }
  __syncthreads();
  const double mean_cost = block_pairwise(in.cost, G, b.pw_leaf, b.pw_val, &sh[3]) / (double)G;
  if (tid == 0) {
    const double nb = (1.0 - in.gamma) * base + in.gamma * mean_r;
    b.state[0] = nb;
    double* hrow = in.history + (long)(round - 1) * 4;
    hrow[0] = mean_cost;
    hrow[1] = b.state[1];
    hrow[2] = nb;
    hrow[3] = b.state[2];
    b.ctr[0] = (unsigned long long)round + 1;   // device round counter (graph-replayed rounds)
    b.ctr[1] += (unsigned long long)G * d.L;
  }
}

// dlogits[t][a] = sum over traces g (in order) of (w_g * (onehot_g - p) / temperature)
// (training.py:134-143). One block per (t, a): the terms of a chunk of traces are formed in
// parallel in shared memory, then one thread adds them in trace order (the reference's
// `dlogits += ...` accumulation, starting from zeros).
constexpr int kDlChunk = 4096;
__global__ void dlogits_kernel(PolicyDims d, PolicyBufs b, const uint8_t* plans, long G, double temperature) {
  __shared__ double terms[kDlChunk];
  const int e = blockIdx.x, t = e / d.T, a = e - t * d.T;
  const double p = b.probs[e];
  const double* X = b.scratch + G;   // gradient weights (round_update_kernel)
  double acc = 0.0;
  for (long g0 = 0; g0 < G; g0 += kDlChunk) {
    const int n = (int)min((long)kDlChunk, G - g0);
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const long g = g0 + i;
      const double oh = (plans[g * d.L + t] == a) ? 1.0 : 0.0;
      terms[i] = X[g] * (oh - p) / temperature;
    }
    __syncthreads();
    if (threadIdx.x == 0)
      for (int i = 0; i < n; i++) acc = acc + terms[i];
    __syncthreads();
  }
  if (threadIdx.x == 0) b.dlogits[e] = acc;
}

__global__ void set_ctr_kernel(unsigned long long* ctr, unsigned long long round, unsigned long long draws) {
  ctr[0] = round;
  ctr[1] = draws;
}

// ---------------------------------------------------------------- K5: BPTT + update

// BPTT (network.py:203-248) split in two. bptt_kernel (one block) runs the sequential recurrence
// dh -> gates -> dz -> dh_next and stores dz for every step; grads_kernel (whole grid) then forms
// the weight gradients as the reference accumulates them: grads.w_cell[k][j] = sum over
// t = L-1 .. 0 of xh_t[k] * dz_t[j], product rounded, then added, in that order (np.outer then
// +=), so every element is the reference's bits given the same dz. (A DMMA tile would fuse
// product and sum into one rounding per k-step and lose that; the accumulation is 16 steps
// per element, memory-light, and parallel over 36 K elements, so CUDA cores are the right unit.)
__global__ void bptt_kernel(PolicyDims d, PolicyBufs b) {
  extern __shared__ double sm[];
  const int H = d.H, D = d.D, G4 = d.G4, T = d.T;
  double* dhn = sm;          // [H] dh_next
  double* dcn = dhn + H;     // [H] dc_next
  double* dz = dcn + H;      // [G4]
  double* dh = dz + G4;      // [H]
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  for (int i = tid; i < H; i += nt) { dhn[i] = 0.0; dcn[i] = 0.0; }
  __syncthreads();
  for (int t = d.L - 1; t >= 0; t--) {
    const double* dl = b.dlogits + t * T;
    for (int i = tid; i < H; i += nt) {  // dh = W_out @ dl + dh_next
      double acc = 0.0;
      for (int a = 0; a < T; a++) acc = fma(b.w_out[i * T + a], dl[a], acc);
      dh[i] = acc + dhn[i];
    }
    __syncthreads();
    for (int i = tid; i < H; i += nt) {
      if (d.lstm) {
        const double gi = b.gi[t * H + i], gf = b.gf[t * H + i], go = b.go[t * H + i], gg = b.gg[t * H + i];
        const double tc = b.tc[t * H + i], cp = b.cp[t * H + i];
        const double dov = dh[i] * tc;
        const double dc = dh[i] * go * (1.0 - tc * tc) + dcn[i];
        const double di = dc * gg, dg = dc * gi, df = dc * cp;
        dcn[i] = dc * gf;
        dz[i] = di * gi * (1.0 - gi);
        dz[H + i] = df * gf * (1.0 - gf);
        dz[2 * H + i] = dov * go * (1.0 - go);
        dz[3 * H + i] = dg * (1.0 - gg * gg);
      } else {
        const double h = b.hh[t * H + i];
        dz[i] = dh[i] * (1.0 - h * h);
      }
    }
    __syncthreads();
    for (int jj = tid; jj < G4; jj += nt) b.dz[t * G4 + jj] = dz[jj];
    // dh_next = (W_cell @ dz)[D:]: one warp per row, lanes over the G4 columns
    for (int i = warp; i < H; i += nw) {
      const double* wrow = b.w_cell + (long)(D + i) * G4;
      double acc = 0.0;
      for (int jj = lane; jj < G4; jj += 32) acc = fma(wrow[jj], dz[jj], acc);
      for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) dhn[i] = acc;
    }
    __syncthreads();
  }
}

// grads.w_cell += outer(xh_t, dz_t), grads.b_cell += dz_t, grads.w_out += outer(h_t, dl_t),
// grads.b_out += dl_t for t = L-1 .. 0, one thread per gradient element (grads start at zero)
__global__ void grads_kernel(PolicyDims d, PolicyBufs b) {
  const int G4 = d.G4, H = d.H, T = d.T, DH = d.D + d.H;
  const long n1 = (long)DH * G4, n2 = n1 + G4, n3 = n2 + (long)H * T, n4 = n3 + T;
  for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < n4; e += (long)gridDim.x * blockDim.x) {
    double acc = 0.0;
    if (e < n1) {
      const int k = (int)(e / G4), j = (int)(e - (long)k * G4);
      for (int t = d.L - 1; t >= 0; t--) acc = acc + b.xh[t * DH + k] * b.dz[t * G4 + j];
      b.gw_cell[e] = acc;
    } else if (e < n2) {
      const int j = (int)(e - n1);
      for (int t = d.L - 1; t >= 0; t--) acc = acc + b.dz[t * G4 + j];
      b.gb_cell[j] = acc;
    } else if (e < n3) {
      const int q = (int)(e - n2), i = q / T, a = q - i * T;
      for (int t = d.L - 1; t >= 0; t--) acc = acc + b.hh[t * H + i] * b.dlogits[t * T + a];
      b.gw_out[q] = acc;
    } else {
      const int a = (int)(e - n3);
      for (int t = d.L - 1; t >= 0; t--) acc = acc + b.dlogits[t * T + a];
      b.gb_out[a] = acc;
    }
  }
}

__global__ void update_kernel(PolicyDims d, PolicyBufs b, double lr) {  // training.py:255-262
  __shared__ double part[1024];
  const int tid = threadIdx.x, nt = blockDim.x;
  const long n1 = (long)(d.D + d.H) * d.G4, n2 = d.G4, n3 = (long)d.H * d.T, n4 = d.T;
  double acc = 0.0;  // ||grads.flat()||^2
  for (long e = tid; e < n1; e += nt) acc = fma(b.gw_cell[e], b.gw_cell[e], acc);
  for (long e = tid; e < n2; e += nt) acc = fma(b.gb_cell[e], b.gb_cell[e], acc);
  for (long e = tid; e < n3; e += nt) acc = fma(b.gw_out[e], b.gw_out[e], acc);
  for (long e = tid; e < n4; e += nt) acc = fma(b.gb_out[e], b.gb_out[e], acc);
  part[tid] = acc;
  __syncthreads();
  for (int s = nt / 2; s > 0; s >>= 1) {
    if (tid < s) part[tid] += part[tid + s];
    __syncthreads();
  }
  double scale = lr;
  const double update_norm = scale * sqrt(part[0]);
  if (update_norm > 50.0) scale *= 50.0 / update_norm;
  int bad = 0;
  for (long e = tid; e < n1; e += nt) { b.w_cell[e] = b.w_cell[e] + scale * b.gw_cell[e]; bad |= !isfinite(b.w_cell[e]); }
  for (long e = tid; e < n2; e += nt) { b.b_cell[e] = b.b_cell[e] + scale * b.gb_cell[e]; bad |= !isfinite(b.b_cell[e]); }
  for (long e = tid; e < n3; e += nt) { b.w_out[e] = b.w_out[e] + scale * b.gw_out[e]; bad |= !isfinite(b.w_out[e]); }
  for (long e = tid; e < n4; e += nt) { b.b_out[e] = b.b_out[e] + scale * b.gb_out[e]; bad |= !isfinite(b.b_out[e]); }
  if (bad) atomicOr(&b.flags[1], 1);
}

}  // namespace

// ===================================================================== C ABI

struct HpsPolicy {
  PolicyDims d;
  PolicyBufs b;
  std::vector<void*> allocs;
};

namespace {
template <typename T>
int palloc(HpsPolicy* p, T** ptr, size_t n) {
  void* q = nullptr;
  PCUDA(cudaMalloc(&q, sizeof(T) * (n ? n : 1)));
  PCUDA(cudaMemset(q, 0, sizeof(T) * (n ? n : 1)));
  p->allocs.push_back(q);
  *ptr = reinterpret_cast<T*>(q);
  return HPS_OK;
}
}  // namespace

extern "C" {

const char* hps_policy_last_error(void) { return g_pol_err.c_str(); }

int hps_policy_create(int32_t L, int32_t D, int32_t H, int32_t T, int32_t lstm, int64_t max_plans,
                      const double* features, HpsPolicy** out) {
  if (!out || !features || L < 1 || L > 64 || D < 1 || D > kMaxD || H < 1 || H > kMaxH || T < 1 ||
      T > 16 || max_plans < 1)
    return perr(HPS_E_INVALID_ARG, "policy dimensions out of range");
  auto* p = new HpsPolicy();
  p->d = PolicyDims{L, D, H, T, (lstm ? 4 : 1) * H, lstm ? 1 : 0};
  const int G4 = p->d.G4, DH = D + H;
  PolicyBufs& b = p->b;
  int rc = 0;
  rc |= palloc(p, &b.w_cell, (size_t)DH * G4); rc |= palloc(p, &b.b_cell, G4);
  rc |= palloc(p, &b.w_out, (size_t)H * T);    rc |= palloc(p, &b.b_out, T);
  rc |= palloc(p, &b.gw_cell, (size_t)DH * G4); rc |= palloc(p, &b.gb_cell, G4);
  rc |= palloc(p, &b.gw_out, (size_t)H * T);    rc |= palloc(p, &b.gb_out, T);
  rc |= palloc(p, &b.feat, (size_t)L * D);      rc |= palloc(p, &b.xw, (size_t)L * G4);
  rc |= palloc(p, &b.xh, (size_t)L * DH);
  for (double** q : {&b.gi, &b.gf, &b.go, &b.gg, &b.cc, &b.cp, &b.tc, &b.hh}) rc |= palloc(p, q, (size_t)L * H);
  rc |= palloc(p, &b.probs, (size_t)L * T);     rc |= palloc(p, &b.cdf, (size_t)L * T);
  rc |= palloc(p, &b.dlogits, (size_t)L * T);
  rc |= palloc(p, &b.scratch, (size_t)max_plans * 4);
  rc |= palloc(p, &b.state, 16);                rc |= palloc(p, &b.flags, 4);
  rc |= palloc(p, &b.dz, (size_t)L * G4);       rc |= palloc(p, &b.ctr, 2);
  rc |= palloc(p, &b.pw_leaf, (size_t)2 * (max_plans / 64 + 4));
  rc |= palloc(p, &b.pw_val, (size_t)(max_plans / 64 + 4));
  if (rc) { hps_policy_destroy(p); return HPS_E_CUDA; }
  const double init_state[3] = {0.0, __builtin_inf(), 0.0};
  const unsigned long long init_ctr[2] = {1ull, 0ull};
  if (cudaMemcpy(b.feat, features, sizeof(double) * L * D, cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(b.state, init_state, sizeof(init_state), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(b.ctr, init_ctr, sizeof(init_ctr), cudaMemcpyHostToDevice) != cudaSuccess) {
    hps_policy_destroy(p);
    return perr(HPS_E_CUDA, "policy upload failed");
  }
  *out = p;
  return HPS_OK;
}

int hps_policy_destroy(HpsPolicy* p) {
  if (!p) return HPS_OK;
  for (void* q : p->allocs) cudaFree(q);
  delete p;
  return HPS_OK;
}

// which: 0 w_cell, 1 b_cell, 2 w_out, 3 b_out; dir 0 host->device, 1 device->host
int hps_policy_params(HpsPolicy* p, int32_t which, int32_t dir, double* host, int64_t n) {
  if (!p || !host) return perr(HPS_E_INVALID_ARG, "null argument");
  double* dev[4] = {p->b.w_cell, p->b.b_cell, p->b.w_out, p->b.b_out};
  const int64_t sz[4] = {(int64_t)(p->d.D + p->d.H) * p->d.G4, p->d.G4, (int64_t)p->d.H * p->d.T, p->d.T};
  if (which < 0 || which > 3 || n != sz[which]) return perr(HPS_E_INVALID_ARG, "parameter size mismatch");
  if (dir == 0) PCUDA(cudaMemcpy(dev[which], host, sizeof(double) * n, cudaMemcpyHostToDevice));
  else PCUDA(cudaMemcpy(host, dev[which], sizeof(double) * n, cudaMemcpyDeviceToHost));
  return HPS_OK;
}

// K4: probs/cdf/cache for the current parameters. d_probs_out (optional) receives [L][T].
int hps_policy_forward(HpsPolicy* p, double temperature, double* d_probs_out, void* stream) {
  if (!p || !(temperature > 0)) return perr(HPS_E_INVALID_ARG, "temperature must be > 0");
  cudaStream_t st = (cudaStream_t)stream;
  const PolicyDims& d = p->d;
  const int tiles = ((d.L + 7) / 8) * ((d.G4 + 7) / 8);
  HPS_COUNT_LAUNCH();
  xw_dmma_kernel<<<(tiles * 32 + 127) / 128, 128, 0, st>>>(d, p->b.feat, p->b.w_cell, p->b.xw);
  PCUDA(cudaGetLastError());
  const int threads = ((d.G4 > d.T ? d.G4 : d.T) + 31) / 32 * 32;
  const size_t smem = sizeof(double) * (2 * d.H + d.G4 + d.T);
  HPS_COUNT_LAUNCH();
  forward_kernel<<<1, threads, smem, st>>>(d, p->b, temperature);
  PCUDA(cudaGetLastError());
  if (d_probs_out)
    PCUDA(cudaMemcpyAsync(d_probs_out, p->b.probs, sizeof(double) * d.L * d.T, cudaMemcpyDeviceToDevice, st));
  return HPS_OK;
}

// K3: n plans; plan g layer t uses draw (first_draw + g*L + t) of `gen`'s stream
int hps_policy_sample(HpsPolicy* p, const HpsPcg64* gen, uint64_t first_draw, int64_t n,
                      uint8_t* d_plans, void* stream) {
  if (!p || !gen || !d_plans || n < 0) return perr(HPS_E_INVALID_ARG, "null argument");
  if (n == 0) return HPS_OK;
  const u128 s0 = ((u128)gen->state_hi << 64) | gen->state_lo, inc = ((u128)gen->inc_hi << 64) | gen->inc_lo;
  HPS_COUNT_LAUNCH();
  const u128 fd = (first_draw == ~0ull) ? (u128)~0ull : (u128)first_draw;
  sample_kernel<<<(unsigned)((n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(p->d, p->b.cdf, p->b.ctr, s0, inc,
                                                                               fd, n, d_plans);
  PCUDA(cudaGetLastError());
  return HPS_OK;
}

// K6 + K5 + update: one REINFORCE round given the G scored plans (device arrays).
// history: device [rounds][4] (mean_cost, best_cost, baseline, entropy); best_plan: device [L];
// best_where: device [2] (round, index). Returns HPS_OK; non-finite logits/params are
// reported through hps_policy_flags.
int hps_policy_reinforce(HpsPolicy* p, const double* d_cost, const uint8_t* d_status,
                         const uint8_t* d_plans, int64_t G, int32_t round, double temperature,
                         double lr, double gamma, double* d_history, uint8_t* d_best_plan,
                         long long* d_best_where, void* stream) {
  if (!p || G < 1) return perr(HPS_E_INVALID_ARG, "bad argument");
  cudaStream_t st = (cudaStream_t)stream;
  RoundIn in{d_cost, d_status, d_plans, G, temperature, lr, gamma, round, d_history, d_best_plan, d_best_where};
  HPS_COUNT_LAUNCH();
  round_update_kernel<<<1, kRoundThreads, 0, st>>>(p->d, p->b, in);
  PCUDA(cudaGetLastError());
  HPS_COUNT_LAUNCH();
  dlogits_kernel<<<p->d.L * p->d.T, 256, 0, st>>>(p->d, p->b, d_plans, G, temperature);
  PCUDA(cudaGetLastError());
  const size_t smem = sizeof(double) * (3 * p->d.H + p->d.G4);
  HPS_COUNT_LAUNCH();
  bptt_kernel<<<1, 512, smem, st>>>(p->d, p->b);
  PCUDA(cudaGetLastError());
  const long ngrad = (long)(p->d.D + p->d.H) * p->d.G4 + p->d.G4 + (long)p->d.H * p->d.T + p->d.T;
  HPS_COUNT_LAUNCH();
  grads_kernel<<<(unsigned)((ngrad + 255) / 256), 256, 0, st>>>(p->d, p->b);
  PCUDA(cudaGetLastError());
  HPS_COUNT_LAUNCH();
  update_kernel<<<1, 1024, 0, st>>>(p->d, p->b, lr);
  PCUDA(cudaGetLastError());
  return HPS_OK;
}

// device round counter read by hps_policy_sample (first_draw = ~0) and hps_policy_reinforce
// (round = 0), advanced by every reinforce: lets a captured round be replayed unchanged
int hps_policy_counter(HpsPolicy* p, uint64_t round, uint64_t draws, void* stream) {
  if (!p || round < 1) return perr(HPS_E_INVALID_ARG, "bad counter");
  HPS_COUNT_LAUNCH();
  set_ctr_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(p->b.ctr, round, draws);
  PCUDA(cudaGetLastError());
  return HPS_OK;
}

// state: {baseline, best_cost, entropy}; flags: {nonfinite logits, nonfinite params}
int hps_policy_state(HpsPolicy* p, double* state3, int32_t* flags2) {
  if (!p) return perr(HPS_E_INVALID_ARG, "null argument");
  if (state3) PCUDA(cudaMemcpy(state3, p->b.state, sizeof(double) * 3, cudaMemcpyDeviceToHost));
  if (flags2) PCUDA(cudaMemcpy(flags2, p->b.flags, sizeof(int32_t) * 2, cudaMemcpyDeviceToHost));
  return HPS_OK;
}

}  // extern "C"
