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

// numpy pairwise_sum over a strided double array (loops_utils.h.src), n >= 0
__device__ double np_pairwise(const double* a, long n, long stride) {
  // iterative restatement of the recursion: split points as numpy's pw(a, n)
  if (n < 8) {
    double res = -0.0;
    for (long i = 0; i < n; i++) res += a[i * stride];
    return res;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; j++) r[j] = a[j * stride];
    long i;
    for (i = 8; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; j++) r[j] += a[(i + j) * stride];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; i++) res += a[i * stride];
    return res;
  }
  long n2 = n / 2;
  n2 -= n2 % 8;
  return np_pairwise(a, n2, stride) + np_pairwise(a + n2 * stride, n - n2, stride);
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
  __syncthreads();
  for (int t = 0; t < d.L; t++) {
    // xh = concat(x_t, h)
    for (int k = j; k < DH; k += blockDim.x) b.xh[t * DH + k] = (k < D) ? b.feat[t * D + k] : h[k - D];
    if (j < G4) {  // z = xh @ W + b: hoisted x part (tensor cores) + h part
      double acc = b.xw[t * G4 + j];
      for (int i = 0; i < H; i++) acc = fma(h[i], b.w_cell[(long)(D + i) * G4 + j], acc);
      z[j] = acc + b.b_cell[j];
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
__global__ void sample_kernel(PolicyDims d, const double* cdf, u128 state0, u128 inc, u128 first_draw,
                              long n, uint8_t* plans) {
  const long g = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n) return;
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

// state[0] baseline, state[1] best cost (+inf before round 1), state[2] entropy of the round
__global__ void round_update_kernel(PolicyDims d, PolicyBufs b, RoundIn in) {
  __shared__ double sh[64];
  const int tid = threadIdx.x, nt = blockDim.x;
  const long G = in.G;
  double* R = b.scratch;           // rewards after winsorising
  double* X = b.scratch + G;       // R - baseline, then standardised weights
  double* W = b.scratch + 2 * G;   // scratch
  const double base = b.state[0];
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  // best-ever: first plan (trace order) with cost < best so far (training.py:219-220)
  if (tid == 0) {
    double bc = b.state[1];
    long bi = -1;
    for (long g = 0; g < G; g++)
      if (in.cost[g] < bc) { bc = in.cost[g]; bi = g; }
    if (bi >= 0) {
      b.state[1] = bc;
      for (int t = 0; t < d.L; t++) in.best_plan[t] = in.plans[bi * d.L + t];
      in.best_where[0] = in.round;
      in.best_where[1] = bi;
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
    if (tid == 0) {
      double spread = -inf, lo = inf, hi = -inf;
      bool have = false;
      for (long g = 0; g < G; g++) {
        const bool ok = (in.status[g] & 0x7f) == HPS_ST_OK;
        if (ok) {
          const double v = fabs(R[g] - base);
          if (!have || v > spread) spread = v;
          have = true;
        } else {
          if (R[g] < lo) lo = R[g];
          if (R[g] > hi) hi = R[g];
        }
      }
      sh[0] = 10.0 * (have ? spread : 1.0);
      sh[1] = lo;
      sh[2] = hi;
    }
    __syncthreads();
    const double unit = sh[0], lo = sh[1], hi = sh[2];
    for (long g = tid; g < G; g += nt)
      if ((in.status[g] & 0x7f) != HPS_ST_OK) {
        const double z = (hi == lo) ? 0.5 : (R[g] - lo) / (hi - lo);
        R[g] = base - unit * (2.0 - z);
      }
    __syncthreads();
  }
  for (long g = tid; g < G; g += nt) X[g] = R[g] - base;
  __syncthreads();
  if (tid == 0) {  // np.std(R - b) and np.mean(R), np.mean(cost) (pairwise)
    const double mean = np_pairwise(X, G, 1) / (double)G;
    sh[3] = mean;
  }
  __syncthreads();
  for (long g = tid; g < G; g += nt) { const double v = X[g] - sh[3]; W[g] = v * v; }
  __syncthreads();
  if (tid == 0) {
    sh[4] = sqrt(np_pairwise(W, G, 1) / (double)G);
    sh[5] = np_pairwise(R, G, 1) / (double)G;  // mean reward
  }
  __syncthreads();
  const double spread = sh[4];
  const double scale = 1.0 / (double)G;
  for (long g = tid; g < G; g += nt) {  // gradient weights (training.py:245-252, 136-137)
    double r2 = R[g];
    if (spread > 1e-12) r2 = base + (R[g] - base) / spread;
    X[g] = (r2 - base) * scale;
  }
  __syncthreads();
  // dlogits accumulated in trace order (training.py:134-143); one thread per (t, a)
  for (int e = tid; e < d.L * d.T; e += nt) {
    const int t = e / d.T, a = e % d.T;
    const double p = b.probs[e];
    double acc = 0.0;
    for (long g = 0; g < G; g++) {
      const double oh = (in.plans[g * d.L + t] == a) ? 1.0 : 0.0;
      acc = acc + X[g] * (oh - p) / in.temperature;
    }
    b.dlogits[e] = acc;
  }
  if (tid == 0) {
    const double mean_cost = np_pairwise(in.cost, G, 1) / (double)G;
    const double nb = (1.0 - in.gamma) * base + in.gamma * sh[5];
    b.state[0] = nb;
    double* hrow = in.history + (long)(in.round - 1) * 4;
    hrow[0] = mean_cost;
    hrow[1] = b.state[1];
    hrow[2] = nb;
    hrow[3] = b.state[2];
  }
}

// ---------------------------------------------------------------- K5: BPTT + update

__global__ void backward_kernel(PolicyDims d, PolicyBufs b) {  // network.py:203-248
  extern __shared__ double sm[];
  const int H = d.H, D = d.D, G4 = d.G4, T = d.T, DH = D + H;
  double* dhn = sm;          // [H] dh_next
  double* dcn = dhn + H;     // [H] dc_next
  double* dz = dcn + H;      // [G4]
  double* dh = dz + G4;      // [H]
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int i = tid; i < H; i += nt) { dhn[i] = 0.0; dcn[i] = 0.0; }
  for (long e = tid; e < (long)DH * G4; e += nt) b.gw_cell[e] = 0.0;
  for (int e = tid; e < G4; e += nt) b.gb_cell[e] = 0.0;
  for (int e = tid; e < H * T; e += nt) b.gw_out[e] = 0.0;
  for (int e = tid; e < T; e += nt) b.gb_out[e] = 0.0;
  __syncthreads();
  for (int t = d.L - 1; t >= 0; t--) {
    const double* dl = b.dlogits + t * T;
    for (int e = tid; e < H * T; e += nt) {  // grads.w_out += outer(h, dl)
      const int i = e / T, a = e % T;
      b.gw_out[e] = b.gw_out[e] + b.hh[t * H + i] * dl[a];
    }
    for (int a = tid; a < T; a += nt) b.gb_out[a] = b.gb_out[a] + dl[a];
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
    const double* xh = b.xh + t * DH;
    for (long e = tid; e < (long)DH * G4; e += nt) {  // grads.w_cell += outer(xh, dz)
      const int k = (int)(e / G4), jj = (int)(e % G4);
      b.gw_cell[e] = b.gw_cell[e] + xh[k] * dz[jj];
    }
    for (int jj = tid; jj < G4; jj += nt) b.gb_cell[jj] = b.gb_cell[jj] + dz[jj];
    __syncthreads();
    for (int i = tid; i < H; i += nt) {  // dh_next = (W_cell @ dz)[D:]
      double acc = 0.0;
      for (int jj = 0; jj < G4; jj++) acc = fma(b.w_cell[(long)(D + i) * G4 + jj], dz[jj], acc);
      dhn[i] = acc;
    }
    __syncthreads();
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
  rc |= palloc(p, &b.dlogits, (size_t)L * T);   rc |= palloc(p, &b.scratch, (size_t)max_plans * 4);
  rc |= palloc(p, &b.state, 16);                rc |= palloc(p, &b.flags, 4);
  if (rc) return HPS_E_CUDA;
  PCUDA(cudaMemcpy(b.feat, features, sizeof(double) * L * D, cudaMemcpyHostToDevice));
  const double init_state[3] = {0.0, __builtin_inf(), 0.0};
  PCUDA(cudaMemcpy(b.state, init_state, sizeof(init_state), cudaMemcpyHostToDevice));
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
  sample_kernel<<<(unsigned)((n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(p->d, p->b.cdf, s0, inc,
                                                                               (u128)first_draw, n, d_plans);
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
  round_update_kernel<<<1, 256, 0, st>>>(p->d, p->b, in);
  PCUDA(cudaGetLastError());
  const size_t smem = sizeof(double) * (3 * p->d.H + p->d.G4);
  HPS_COUNT_LAUNCH();
  backward_kernel<<<1, 512, smem, st>>>(p->d, p->b);
  PCUDA(cudaGetLastError());
  HPS_COUNT_LAUNCH();
  update_kernel<<<1, 1024, 0, st>>>(p->d, p->b, lr);
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
