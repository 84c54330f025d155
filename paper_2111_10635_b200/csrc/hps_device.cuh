// hps_device.cuh — device-side data layout and exact arithmetic primitives of the plan
// evaluator. Compiled with --fmad=false and IEEE division/sqrt so every operation below
// rounds exactly like CPython/numpy binary64 (the bit-exact contract of SURVEY.md §7).
#pragma once
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "../../include/hps.h"

// HPS_NOINLINE: inlined helpers; HPS_NOINLINE_RARE: one out-of-line copy (rare paths, and hot
// helpers called from several sites, to keep the hot loops inside the instruction cache)
#define HPS_NOINLINE __forceinline__
#define HPS_NOINLINE_RARE __noinline__

namespace hps {

typedef unsigned __int128 u128;

// Optional device counters (build with -DHPS_STATS; see tools/sweep_stats.py)
enum {
  ST_PLANS, ST_CHUNKS, ST_CHUNKS_EVAL, ST_CANDS, ST_PROBES_EXACT, ST_PROBES_CLOSED, ST_CERT,
  ST_CERT_FAIL, ST_TAB, ST_PENDING, ST_STAGES, ST_UNPINNED, ST_NCAND, ST_PLANS_FAST,
  ST_CYC_A, ST_CYC_B, ST_CYC_C, ST_CYC_P1, ST_CYC_P2, ST_N2, ST_UNCERT, ST_IDEAL, ST_IDEAL2, ST_NEAR, ST_NSTAT
};
#ifdef HPS_STATS
__device__ unsigned long long g_stats[24];
#define HPS_STAT(i, v) atomicAdd(&hps::g_stats[i], (unsigned long long)(v))
#else
#define HPS_STAT(i, v) ((void)0)
#endif

// Bounds-checked build (-DHPS_CHECKS, `make checked`): every threshold-table access and the
// per-warp / pending-list indices below trap with a message when out of range. The tests run
// against that build on the GPU box in place of compute-sanitizer (closed on this pool).
#ifdef HPS_CHECKS
__device__ const char* g_chk_te_lo;   // [lo, hi) of the threshold table of the running launch
__device__ const char* g_chk_te_hi;
#define HPS_CHECK(cond, what)                                                                  \
  do {                                                                                         \
    if (!(cond)) {                                                                             \
      printf("HPS_CHECK failed: %s at %s:%d (block %d thread %d)\n", what, __FILE__, __LINE__,   \
             (int)blockIdx.x, (int)threadIdx.x);                                               \
      __trap();                                                                                \
    }                                                                                          \
  } while (0)
#else
#define HPS_CHECK(cond, what) ((void)0)
#endif

constexpr int kMaxL = HPS_MAX_LAYERS;
constexpr int kMaxT = HPS_MAX_TYPES;
constexpr int kBpLimit = HPS_BREAKPOINT_LIMIT;
constexpr int kWarp = 32;

// Aggregates of one stage = maximal run (type t, layers first..last), as build_stages makes
// them (ls/domain.py:275-328), plus the constants every formula of ls/provisioner.py needs.
struct __align__(16) StageEntry {
  double c_oct;   // oct / B_o
  double c_odt;   // odt / B_o
  double alpha;
  double beta;
  double oma;     // 1.0 - alpha
  double omb;     // 1.0 - beta
  double oct;     // Neumaier sum of member oct (ls/domain.py:306)
  double odt;     // last member's odt (ls/domain.py:324)
  double serial;  // max((oct/B_o)(1-alpha), (odt/B_o)(1-beta))  (ls/provisioner.py:184-193)
  int32_t valid;  // 0 when a member lacks a profile for the type (PlanValidationError)
  int32_t type;
  // single-precision constants for the count ESTIMATE that seeds the exact table search
  float f_rbo, f_rbd;    // B_o / oct, B_o / odt (0 when the work is 0)
  float f_oma, f_omb, f_alpha, f_beta;
  float f_coct, f_codt;  // oct / B_o, odt / B_o
  double rwo, rwd;       // fl(1/oct), fl(1/odt) (0 when the work is 0): certified counts
};

// Certified count: q = frac / (fl(fl(tau*bo)/work) - (1-frac)) evaluated with a reciprocal
// instead of the two IEEE divisions, together with a rigorous bound on its distance to the
// reference's value; when ceil(fl(v - 1e-9)) cannot change inside the bound the integer count
// is exact (monotone ops). Returns -1 when uncertain (caller falls back to the exact path).
// Valid only where the stage does not raise (tau inside [tau_lo, tau_hi] or above a point
// known not to raise), which is where callers use it.
__device__ __forceinline__ double rcp_refined(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);  // two Newton steps: error 2^-22 -> 2^-44 -> rounding level
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// one Newton step: relative error <= 2^-40 for any seed accurate to 2^-20 (counted in count_cert)
__device__ __forceinline__ double rcp_1nt(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

__device__ __forceinline__ double dmax_nn(double a, double b) { return a > b ? a : b; }  // no NaNs

__device__ __forceinline__ float rcp_approx_f32(float x) {  // MUFU.RCP, rel. error ~2^-23
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

static __device__ HPS_NOINLINE_RARE int count_cert(const StageEntry& s, double tau, double bo) {
  const double A = tau * bo;  // identical to the reference's first product
  double lo = 1.0, hi = 1.0;
#pragma unroll
  for (int side = 0; side < 2; side++) {
    const double work = side ? s.odt : s.oct;
    if (work == 0) continue;
    const double frac = side ? s.beta : s.alpha;
    const double omf = side ? s.omb : s.oma;
    const double B = A * (side ? s.rwd : s.rwo);
    const double h = B - omf;
    if (frac == 0.0) {
      // side is skipped when headroom >= 0; decide exactly only if clearly so
      if (h > 4e-16 * (B + 1.0)) continue;
      return -1;
    }
    const double eh = (4.0 * B + 3.0 * fabs(h)) * 1.1102230246251565e-16;  // |h - h_ref| bound
    if (!(h > 2.0 * eh)) return -1;
    const double rh = rcp_1nt(h);
    const double q = frac * rh;
    // |q - q_ref| <= q (eh/(h-eh) + 2^-40 + 4u) and eh/(h-eh) <= 2 eh/h since h > 2 eh
    const double dq = q * fma(2.02 * eh, rh, 1.0e-12);
    lo = dmax_nn(lo, q - dq);
    hi = dmax_nn(hi, q + dq);
  }
  const double c_lo = ceil(lo - 1e-9), c_hi = ceil(hi - 1e-9);
  HPS_STAT(ST_CERT, 1);
  if (c_lo != c_hi || !(c_hi < 2.0e9)) { HPS_STAT(ST_CERT_FAIL, 1); return -1; }
  return c_lo < 1.0 ? 1 : (int)c_lo;
}

// count_cert for a stage whose count is decided by ONE side (see side_dominance): the same
// certified arithmetic on that side only.
static __device__ HPS_NOINLINE_RARE int count_cert1(double frac, double omf, double rw, double tau,
                                                    double bo) {
  const double B = (tau * bo) * rw;
  const double h = B - omf;
  const double eh = (4.0 * B + 3.0 * fabs(h)) * 1.1102230246251565e-16;
  HPS_STAT(ST_CERT, 1);
  if (!(h > 2.0 * eh)) { HPS_STAT(ST_CERT_FAIL, 1); return -1; }
  const double rh = rcp_1nt(h);
  const double q = frac * rh;
  const double dq = q * fma(2.02 * eh, rh, 1.0e-12);
  const double c_lo = ceil(dmax_nn(1.0, q - dq) - 1e-9), c_hi = ceil(dmax_nn(1.0, q + dq) - 1e-9);
  if (c_lo != c_hi || !(c_hi < 2.0e9)) { HPS_STAT(ST_CERT_FAIL, 1); return -1; }
  return (int)c_lo;
}

// Which side of _floor_count (ls/provisioner.py:150-176) decides a stage's count for every tau
// in [tlo, thi]: 1 = computation, 2 = communication, 0 = undecided (use both). With both
// sides active, q_o - q_d = N / (h_o h_d) with N = alpha h_d - beta h_o LINEAR in tau, so a
// sign of N that holds with margin at both ends holds on the whole interval; the margin
// (relative 1e-9, far above the rounding of h and q) makes the reference's rounded q's obey
// the same order, and iceil is monotone, so max(iceil(q_o), iceil(q_d)) = iceil(q_dominant).
static __device__ __noinline__ int side_dominance(const StageEntry& s, double tlo, double thi, double bo) {
  if (s.odt == 0.0) return (s.oct != 0.0 && s.alpha > 0.0) ? 1 : 0;
  if (s.oct == 0.0) return (s.beta > 0.0) ? 2 : 0;
  if (!(s.alpha > 0.0) || !(s.beta > 0.0)) return 0;
  int sg[2];
#pragma unroll
  for (int e = 0; e < 2; e++) {
    const double A = (e ? thi : tlo) * bo;
    const double Bo = A * s.rwo, Bd = A * s.rwd;
    const double ho = Bo - s.oma, hd = Bd - s.omb;
    const double eo = (4.0 * Bo + 3.0 * fabs(ho)) * 1.1102230246251565e-16;
    const double ed = (4.0 * Bd + 3.0 * fabs(hd)) * 1.1102230246251565e-16;
    if (!(ho > 2.0 * eo) || !(hd > 2.0 * ed)) return 0;
    const double N = s.alpha * hd - s.beta * ho;
    const double M = 8.0 * (s.alpha * ed + s.beta * eo) + 1e-9 * (s.alpha * hd + s.beta * ho);
    sg[e] = (N > M) ? 1 : ((N < -M) ? 2 : 0);
  }
  return (sg[0] == sg[1]) ? sg[0] : 0;
}

// et(k) approximately (k >= 1 integer): within ~4 ulp of _stage_et(s, k)
__device__ __forceinline__ double et_approx(const StageEntry& s, double k) {
  const double rk = rcp_refined(k);
  const double ct = s.c_oct * fma(s.alpha, rk, s.oma);
  const double dt = s.c_odt * fma(s.beta, rk, s.omb);
  return fmax(ct, dt);
}

// Per (stage entry, count m) pair of the TE table: et(m) = _stage_et at integer count m, and
// th(m-1) = theta(m-1) = the smallest double tau with count(tau) <= m-1 (+inf for m == 1).
// count(tau) = min{m : theta(m) <= tau}; theta is exact: found by bisection over the bit
// patterns of tau with the exact _floor_count/_iceil (ls/provisioner.py:75-77,150-176).
struct __align__(16) TEPair {
  double et;
  double th;  // theta(m - 1)
};

// checked element access of a threshold-table row (plain indexing in the product build)
__device__ __forceinline__ const TEPair& te_checked(const TEPair* row, long i) {
#ifdef HPS_CHECKS
  const char* p = reinterpret_cast<const char*>(row + i);
  HPS_CHECK(p >= g_chk_te_lo && p + sizeof(TEPair) <= g_chk_te_hi, "threshold-table index out of range");
#endif
  return row[i];
}
#define HPS_TE(row, i) (::hps::te_checked((row), (i)))

// Stage-0 exits of optimize_k1 for an entry starting at layer 0 (ls/provisioner.py:394-397)
struct Stage0Info {
  double tau_hi;  // min(B/limit, et(stage0, k1_floor)) if k1_floor > 1
  double gap;     // InfeasibleError gap when status == HPS_ST_MIN_K1
  int32_t status; // HPS_ST_OK or HPS_ST_MIN_K1
  int32_t pad;
};

// Immutable per-instance constants, in __constant__-friendly form (passed by value).
struct InstanceConsts {
  int32_t L, T, P;        // P = L(L+1)/2 stage ranges per type
  int32_t with_ps;
  int32_t ps_type;        // cheapest CPU type (ls/domain.py:163-167), -1 if none
  int32_t newton_max_iters;
  double bo, batch, work, limit;
  double penalty_scale;   // 1e6 * max price (ls/scoring.py:47-50)
  double ps_cores_per_gpu, newton_tol, fd_step;
  double tau_limit;       // B / limit (ls/provisioner.py:395)
  double price_s[kMaxT];  // price_per_hour / 3600.0 (ls/provisioner.py:209)
  double price_h[kMaxT];  // price_per_hour
  int64_t quota[kMaxT];
  uint8_t is_cpu[kMaxT];
  int32_t et_cap[kMaxT];  // TE table holds m in [1, et_cap[t] + 1] for stages of type t
  int64_t te_off[kMaxT];  // TE table offset of type t's block (rows of et_cap[t] + 1)
  int32_t redux_ok;       // all quotas < 2^24: per-type sums fit 32-bit warp reductions
};

struct DeviceTables {
  const StageEntry* stages;   // [T * P]
  const Stage0Info* stage0;   // [T * L] indexed by (t, last)
  const TEPair* te;           // TE[e][m-1], m = 1 .. et_cap[t] + 1 (same offsets, stride cap+1)
  const int32_t* cls;         // [T * P] ET-equivalence class: entries with bitwise-equal
                              // (oct, odt, alpha, beta) share counts and breakpoints
  const int32_t* gex;         // [T * P] largest M with count(et(m)) == m for every m <= M:
                              // theta(m) <= et(m) < theta(m - 1) (exact generator counts)
};

__device__ __forceinline__ int tb_class(const DeviceTables& tb, int e) { return __ldg(tb.cls + e); }

__host__ __device__ __forceinline__ int pair_index(int first, int last) {
  return last * (last + 1) / 2 + first;
}
__host__ __device__ __forceinline__ int entry_index(int P, int t, int first, int last) {
  return t * P + pair_index(first, last);
}

// Python max(a, b) / min(a, b): the first argument unless the second is strictly better.
__device__ __forceinline__ double pmax(double a, double b) { return (b > a) ? b : a; }
__device__ __forceinline__ double pmin(double a, double b) { return (b < a) ? b : a; }
__device__ __forceinline__ double clamp_gap(double g) { return (g > 0.0) ? g : 0.0; }

// _stage_et (ls/provisioner.py:144-147) == compute_ct/compute_dt + max (ls/costmodel.py:50-66)
__device__ __forceinline__ double stage_et(const StageEntry& s, double k) {
  double ct = s.c_oct * (s.oma + s.alpha / k);
  double dt = s.c_odt * (s.omb + s.beta / k);
  return pmax(ct, dt);
}

// _floor_count (ls/provisioner.py:150-176): false on InfeasibleError (gap = -headroom).
__device__ __forceinline__ bool floor_count(const StageEntry& s, double tau, double bo,
                                            double& req, double& gap) {
  double required = 1.0;
  if (s.oct != 0) {
    double h = tau * bo / s.oct - s.oma;
    if (s.alpha == 0.0) {
      if (!(h >= 0)) { gap = clamp_gap(-h); return false; }
    } else {
      if (h <= 0) { gap = clamp_gap(-h); return false; }
      required = pmax(required, s.alpha / h);
    }
  }
  if (s.odt != 0) {
    double h = tau * bo / s.odt - s.omb;
    if (s.beta == 0.0) {
      if (!(h >= 0)) { gap = clamp_gap(-h); return false; }
    } else {
      if (h <= 0) { gap = clamp_gap(-h); return false; }
      required = pmax(required, s.beta / h);
    }
  }
  req = required;
  return true;
}

// _iceil (ls/provisioner.py:75-77) as an integer-valued double (Python int semantics)
__device__ __forceinline__ double iceil(double x) {
  double c = ceil(x - 1e-9);
  return c < 1.0 ? 1.0 : c;
}

// integer count at tau, +inf when _floor_count raises
__device__ __forceinline__ double count_at(const StageEntry& s, double tau, double bo) {
  double r, g;
  return floor_count(s, tau, bo, r, g) ? iceil(r) : __longlong_as_double(0x7ff0000000000000LL);
}

__device__ __forceinline__ const TEPair* te_row(const InstanceConsts& c, const DeviceTables& tb,
                                                int t, int e);

__device__ __forceinline__ double et_lookup(const InstanceConsts& c, const DeviceTables& tb,
                                            const StageEntry& s, int e, double k) {
  const int t = s.type;
  if (k <= (double)c.et_cap[t] + 1.0) return te_row(c, tb, t, e)[(int64_t)k - 1].et;
  return stage_et(s, k);
}

__device__ __forceinline__ const TEPair* te_row(const InstanceConsts& c, const DeviceTables& tb,
                                                int t, int e) {
  return tb.te + c.te_off[t] + (int64_t)(e - t * c.P) * (int64_t)(c.et_cap[t] + 1);
}

__device__ __forceinline__ uint64_t sat_count(double k) {  // saturating u64 of a count
  return (k < 1.125899906842624e15) ? (uint64_t)k : (uint64_t)1125899906842624ULL;  // 2^50
}

// Exact u128 of an integer-valued double in [1, 2^127) (Python int(count)).
__device__ __forceinline__ u128 dbl_to_u128(double x) {
  if (!(x < 1.7014118346046923e38)) return ~(u128)0 >> 1;
  int e;
  double m = frexp(x, &e);
  uint64_t mi = (uint64_t)ldexp(m, 53);
  return (e >= 53) ? ((u128)mi << (e - 53)) : ((u128)mi >> (53 - e));
}

// Python int/int true division (correctly rounded), 0 <= n < 2^127, d > 0.
static __device__ HPS_NOINLINE_RARE double int_true_div(u128 n, int64_t d) {
  if (n < ((u128)1 << 53)) return (double)(uint64_t)n / (double)d;
  u128 q = n / (u128)d, r = n % (u128)d;
  int e = 0;
  u128 mant = q;
  while ((mant >> 54) == 0) {
    r <<= 1;
    mant = (mant << 1) | (r >= (u128)d ? 1u : 0u);
    if (r >= (u128)d) r -= (u128)d;
    e--;
  }
  bool sticky = (r != 0);
  int nb = 0;
  for (u128 t = mant; t; t >>= 1) nb++;
  int drop = nb - 53;
  u128 low = mant & ((((u128)1) << drop) - 1);
  u128 half = ((u128)1) << (drop - 1);
  mant >>= drop;
  e += drop;
  if (low > half || (low == half && (sticky || (mant & 1)))) mant += 1;
  return ldexp((double)(uint64_t)mant, e);
}

// CPython 3.12 builtin sum() over floats with int start (Neumaier), sequential.
struct PySum {
  double f = 0.0, c = 0.0;
  bool started = false;
  __device__ __forceinline__ void add(double x) {
    if (!started) { f = 0.0 + x; started = true; return; }
    double t = f + x;
    if (fabs(f) >= fabs(x)) c += (f - t) + x; else c += (x - t) + f;
    f = t;
  }
  __device__ __forceinline__ double result() const {
    if (!started) return 0.0;
    return (c != 0.0 && isfinite(c)) ? f + c : f;
  }
};

// ---- numpy PCG64 (XSL-RR 128/64) ----
__host__ __device__ __forceinline__ u128 pcg_mult() {
  return (((u128)0x2360ED051FC65DA4ULL) << 64) | 0x4385DF649FCCF645ULL;
}
__device__ __forceinline__ uint64_t pcg_output(u128 s) {
  uint64_t hi = (uint64_t)(s >> 64), lo = (uint64_t)s;
  uint64_t x = hi ^ lo;
  unsigned rot = (unsigned)(hi >> 58);
  return (x >> rot) | (x << ((64 - rot) & 63));
}
// state after `delta` steps (LCG jump-ahead by squaring)
__host__ __device__ inline u128 pcg_advance(u128 state, u128 inc, u128 delta) {
  u128 acc_mult = 1, acc_plus = 0, cur_mult = pcg_mult(), cur_plus = inc;
  while (delta > 0) {
    if (delta & 1) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    delta >>= 1;
  }
  return acc_mult * state + acc_plus;
}

}  // namespace hps
