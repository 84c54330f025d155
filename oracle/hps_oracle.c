/*
 * hps_oracle.c — TEST INFRASTRUCTURE ONLY. A literal, single-threaded-per-plan CPU
 * restatement of the reference scheduler's per-plan path, used (a) as the parity checker of
 * the CUDA kernels in tests/ and __graft_entry__.smoke(), and (b) as bench.py's
 * `cpu_baseline` / `--impl reference` arm ("port"). The product library
 * (paper_2111_10635_b200/) never links or calls this file.
 *
 * Parity is PINNED: tests/test_oracle_golden.py checks every function here bit-for-bit
 * against golden records produced by the reference itself (tests/golden/make_*.py).
 *
 * Every function cites the reference code it restates (`ls/` = /root/reference/pkg/src/
 * layersched). Arithmetic contract: IEEE binary64, no FMA contraction (-ffp-contract=off),
 * Python evaluation order kept operation by operation:
 *   - builtin sum() over floats is Neumaier-compensated in CPython >= 3.12 (used by
 *     build_stages and _CostModel.real_cost);
 *   - numpy (S,C).sum(axis=0) accumulates rows sequentially for C >= 2 and uses numpy's
 *     pairwise summation for C == 1 (ls/provisioner.py:306);
 *   - Python ints are unbounded: per-stage counts can exceed 2^53 near the serial floor, so
 *     totals are kept in 128-bit integers and int/int true division is correctly rounded.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/hps.h"

typedef unsigned __int128 u128;

#define MAXL HPS_MAX_LAYERS
#define MAXT HPS_MAX_TYPES

typedef struct {
  int type, first, last;
  double oct, odt, alpha, beta;
} OStage;

typedef struct {
  double cost, gap;
  int status; /* HPS_ST_* (| HPS_ST_OVERFLOW_FLAG) */
  int num_stages;
  int ps;
  int ncand;  /* number of candidates handed to _best_candidate */
  int k[MAXL];
  int ntotals;
  int tot_type[MAXT + 1];
  int64_t tot_count[MAXT + 1];
  double pipeline_tp, exec_time;
  int nraw;   /* breakpoints before dedup (diagnostic) */
  int nspan;  /* sum over stages of (span+1) for spans <= 4096, plus 2 */
} HpsoResult;

/* ---- Python builtin sum() over floats with int start 0 (CPython 3.12 Neumaier) ---- */
static double py_sum(const double* x, int n) {
  if (n <= 0) return 0.0;
  double f = 0.0 + x[0], c = 0.0; /* int 0 + float: first add is exact */
  for (int i = 1; i < n; i++) {
    double t = f + x[i];
    if (fabs(f) >= fabs(x[i]))
      c += (f - t) + x[i];
    else
      c += (x[i] - t) + f;
    f = t;
  }
  if (c != 0.0 && isfinite(c)) f += c;
  return f;
}

/* numpy pairwise_sum (numpy/_core/src/umath/loops_utils.h.src), 8 accumulators, block 128 */
static double np_pairwise(const double* a, int n) {
  if (n < 8) {
    double res = -0.0;
    for (int i = 0; i < n; i++) res += a[i];
    return res;
  } else if (n <= 128) {
    double r[8];
    int i;
    for (int j = 0; j < 8; j++) r[j] = a[j];
    for (i = 8; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; j++) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; i++) res += a[i];
    return res;
  } else {
    int n2 = n / 2;
    n2 -= n2 % 8;
    return np_pairwise(a, n2) + np_pairwise(a + n2, n - n2);
  }
}

static double pmax(double a, double b) { return (b > a) ? b : a; } /* Python max(a, b) */
static double pmin(double a, double b) { return (b < a) ? b : a; } /* Python min(a, b) */
static double clamp_gap(double g) { return (g > 0.0) ? g : 0.0; }  /* ls/errors.py:36 */

/* Python int/int true division, correctly rounded, for 0 <= n < 2^127, d > 0. */
static double int_true_div(u128 n, int64_t d) {
  if (n < ((u128)1 << 53)) return (double)(uint64_t)n / (double)d;
  u128 q = n / (u128)d, r = n % (u128)d;
  int e = 0; /* value = mant * 2^e */
  u128 mant = q;
  int sticky;
  while ((mant >> 54) == 0) { /* long division: append fractional bits until 55 bits */
    r <<= 1;
    mant = (mant << 1) | (r >= (u128)d ? 1u : 0u);
    if (r >= (u128)d) r -= (u128)d;
    e--;
  }
  sticky = (r != 0);
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

/* ---- build_stages (ls/domain.py:275-328) ---- */
static int build_stages(const HpsInstanceDesc* d, const uint8_t* plan, OStage* st) {
  const int L = d->num_layers;
  int S = 0, start = 0;
  double octs[MAXL], odts[MAXL], al[MAXL], be[MAXL], w[MAXL];
  for (int pos = 1; pos <= L; pos++) {
    if (pos < L && plan[pos] == plan[start]) continue;
    const int t = plan[start], n = pos - start;
    for (int i = 0; i < n; i++) {
      octs[i] = d->oct[t * L + start + i];
      odts[i] = d->odt[t * L + start + i];
      al[i] = d->alpha[t * L + start + i];
      be[i] = d->beta[t * L + start + i];
    }
    OStage* s = &st[S++];
    s->type = t;
    s->first = start;
    s->last = pos - 1;
    s->oct = py_sum(octs, n);
    if (s->oct > 0) {
      for (int i = 0; i < n; i++) w[i] = octs[i] * al[i];
      s->alpha = py_sum(w, n) / s->oct;
    } else {
      s->alpha = py_sum(al, n) / (double)n;
    }
    double odt_sum = py_sum(odts, n);
    if (odt_sum > 0) {
      for (int i = 0; i < n; i++) w[i] = odts[i] * be[i];
      s->beta = py_sum(w, n) / odt_sum;
    } else {
      s->beta = py_sum(be, n) / (double)n;
    }
    s->odt = odts[n - 1];
    start = pos;
  }
  return S;
}

typedef struct {
  const HpsInstanceDesc* d;
  const OStage* st;
  int S;
  double bo, batch, work, limit;
  double price_s[MAXT]; /* price_per_hour / 3600.0  (ls/provisioner.py:209) */
} Model;

/* _stage_et (ls/provisioner.py:144-147); compute_ct/dt (ls/costmodel.py:50-61) */
static double stage_et(const OStage* s, double k, double bo) {
  double ct = (s->oct / bo) * ((1.0 - s->alpha) + s->alpha / k);
  double dt = (s->odt / bo) * ((1.0 - s->beta) + s->beta / k);
  return pmax(ct, dt);
}

/* min_k1 (ls/provisioner.py:80-104). Returns 0, or 1 on InfeasibleError (gap set). */
static int min_k1(const OStage* s, const Model* m, double* out, double* gap) {
  const double budget = m->d->throughput_limit * m->bo;
  double b[2];
  const double works[2] = {s->oct, s->odt}, fracs[2] = {s->alpha, s->beta};
  for (int i = 0; i < 2; i++) {
    if (works[i] == 0) { b[i] = 0.0; continue; }
    double denom = budget - (1.0 - fracs[i]) * works[i];
    if (denom <= 0) {
      *gap = clamp_gap(((1.0 - fracs[i]) * works[i] - budget) / budget);
      return 1;
    }
    b[i] = fracs[i] * works[i] / denom;
  }
  *out = pmax(b[0], b[1]);
  return 0;
}

/* _floor_count (ls/provisioner.py:150-176). Returns 0, or 1 on raise (gap = -headroom). */
static int floor_count(const OStage* s, double tau, double bo, double* req, double* gap) {
  double required = 1.0;
  const double works[2] = {s->oct, s->odt}, fracs[2] = {s->alpha, s->beta};
  for (int i = 0; i < 2; i++) {
    if (works[i] == 0) continue;
    double headroom = tau * bo / works[i] - (1.0 - fracs[i]);
    if (fracs[i] == 0.0) {
      if (headroom >= 0) continue;
      *gap = clamp_gap(-headroom);
      return 1;
    }
    if (headroom <= 0) {
      *gap = clamp_gap(-headroom);
      return 1;
    }
    required = pmax(required, fracs[i] / headroom);
  }
  *req = required;
  return 0;
}

/* _iceil (ls/provisioner.py:75-77) as an exact integer-valued double (Python int) */
static double iceil(double x) {
  double c = ceil(x - 1e-9);
  return c < 1.0 ? 1.0 : c;
}

static u128 dbl_to_u128(double x) { /* exact for integer-valued 1 <= x < 2^127 */
  if (!(x < 0x1p127)) return ~(u128)0 >> 1; /* saturate: such totals exceed any quota */
  int e;
  double m = frexp(x, &e);
  uint64_t mi = (uint64_t)ldexp(m, 53);
  return (e >= 53) ? ((u128)mi << (e - 53)) : ((u128)mi >> (53 - e));
}

/* _counts_at (ls/provisioner.py:179-181) + per-type totals. Returns 0 / 1 (raise). */
static int counts_at(const Model* m, double tau, double* counts, double* gap) {
  for (int s = 0; s < m->S; s++) {
    double r;
    if (floor_count(&m->st[s], tau, m->bo, &r, gap)) return 1;
    counts[s] = iceil(r);
  }
  return 0;
}

/* _CostModel.quota_ok (ls/provisioner.py:251-259) */
static int quota_ok(const Model* m, double tau) {
  double counts[MAXL], g;
  if (counts_at(m, tau, counts, &g)) return 0;
  u128 tot[MAXT] = {0};
  for (int s = 0; s < m->S; s++) tot[m->st[s].type] += dbl_to_u128(counts[s]);
  for (int t = 0; t < m->d->num_types; t++)
    if (tot[t] > (u128)m->d->quota[t]) return 0;
  return 1;
}

/* _serial_floor (ls/provisioner.py:184-193) */
static double serial_floor(const Model* m) {
  double f = 0.0;
  for (int s = 0; s < m->S; s++) {
    const OStage* x = &m->st[s];
    double a = (x->oct / m->bo) * (1.0 - x->alpha), b = (x->odt / m->bo) * (1.0 - x->beta);
    f = pmax(pmax(f, a), b);
  }
  return f;
}

/* _CostModel.real_cost (ls/provisioner.py:230-249) */
static double real_cost(const Model* m, double tau) {
  double ks[MAXL], g, terms[MAXL];
  for (int s = 0; s < m->S; s++) {
    double r;
    if (floor_count(&m->st[s], tau, m->bo, &r, &g)) return INFINITY;
    ks[s] = pmax(1.0, r);
  }
  double et = stage_et(&m->st[0], ks[0], m->bo);
  for (int s = 1; s < m->S; s++) et = pmax(et, stage_et(&m->st[s], ks[s], m->bo));
  if (et <= 0) return 0.0;
  double thr = m->batch / et;
  if (!(thr > m->limit)) return INFINITY;
  for (int s = 0; s < m->S; s++) terms[s] = m->price_s[m->st[s].type] * ks[s];
  double per_second = py_sum(terms, m->S);
  return m->work / thr * per_second;
}

/* _newton_minimize (ls/provisioner.py:317-345); returns 1 and sets *x_out on success */
static int newton_minimize(const Model* m, double lo, double hi, double* x_out) {
  const HpsInstanceDesc* d = m->d;
  double h = pmax(d->fd_step * (hi - lo), 1e-12);
  double x = pmin(hi - h, lo + pmax(h, (hi - lo) * 0.25));
  if (x <= lo + h) return 0;
  for (int it = 0; it < d->newton_max_iters; it++) {
    double fm = real_cost(m, x - h), f0 = real_cost(m, x), fp = real_cost(m, x + h);
    if (!(isfinite(fm) && isfinite(f0) && isfinite(fp))) return 0;
    double d1 = (fp - fm) / (2.0 * h);
    double d2 = (fp - 2.0 * f0 + fm) / (h * h);
    if (fabs(d2) < 1e-18) return 0;
    double step = d1 / d2;
    double xn = x - step;
    if (!isfinite(xn) || xn < lo || xn > hi) return 0;
    if (fabs(xn - x) < d->newton_tol * pmax(1.0, fabs(x))) {
      if (real_cost(m, xn) <= f0 + 1e-12) {
        *x_out = xn;
        return 1;
      }
      return 0;
    }
    x = xn;
  }
  return 0;
}

/* _golden_minimize (ls/provisioner.py:348-371) */
static double golden_minimize(const Model* m, double lo, double hi) {
  if (hi <= lo) return lo;
  const int n = 17;
  double xs[17], vals[17];
  for (int i = 0; i < n; i++) {
    xs[i] = lo + (hi - lo) * (double)i / (double)(n - 1);
    vals[i] = real_cost(m, xs[i]);
  }
  int best = 0;
  for (int i = 1; i < n; i++)
    if (vals[i] < vals[best]) best = i;
  double a = xs[best > 0 ? best - 1 : 0], b = xs[best + 1 < n ? best + 1 : n - 1];
  const double inv_phi = (sqrt(5.0) - 1.0) / 2.0;
  double c = b - inv_phi * (b - a), dd = a + inv_phi * (b - a);
  double fc = real_cost(m, c), fd = real_cost(m, dd);
  for (int it = 0; it < 60; it++) {
    if (fc <= fd) {
      b = dd; dd = c; fd = fc;
      c = b - inv_phi * (b - a);
      fc = real_cost(m, c);
    } else {
      a = c; c = dd; fc = fd;
      dd = a + inv_phi * (b - a);
      fd = real_cost(m, dd);
    }
  }
  return (a + b) / 2.0;
}

static int cmp_double(const void* a, const void* b) {
  double x = *(const double*)a, y = *(const double*)b;
  return (x > y) - (x < y);
}

typedef struct {
  double* cand; /* candidate taus */
  size_t cap;
  double* mat;  /* S x C scratch */
  size_t mcap;
} Scratch;

static void ensure(Scratch* w, size_t ncand, int S) {
  if (ncand > w->cap) {
    w->cap = ncand * 2;
    w->cand = (double*)realloc(w->cand, w->cap * sizeof(double));
  }
  size_t need = (size_t)S * ncand * 5 + ncand * 4;
  if (need > w->mcap) {
    w->mcap = need * 2;
    w->mat = (double*)realloc(w->mat, w->mcap * sizeof(double));
  }
}

/* numpy side_counts of _best_candidate (ls/provisioner.py:277-284) for one element */
static double np_side_count(double tau, double bo, double work, double frac) {
  double headroom = tau * bo / work - (1.0 - frac);
  double c = (headroom > 0) ? frac / headroom : INFINITY;
  if (work == 0) c = 1.0;
  if (frac == 0 && headroom >= 0) c = 1.0;
  return c;
}

static double np_maximum(double a, double b) { /* propagates NaN */
  if (isnan(a) || isnan(b)) return NAN;
  return a > b ? a : b;
}

/* _best_candidate (ls/provisioner.py:262-314). Returns 1 with counts in best_k, else 0. */
static int best_candidate(const Model* m, const double* taus, int C, Scratch* w, int* best_k) {
  const int S = m->S;
  ensure(w, (size_t)C, S);
  double* safe = w->mat;              /* [S][C] */
  double* cost = safe + (size_t)S * C; /* [C] */
  double* col = cost + C;             /* [S] scratch for C==1 pairwise */
  unsigned char okv[1];
  (void)okv;
  int any_ok = 0;
  double best = INFINITY;
  for (int c = 0; c < C; c++) {
    int ok = 1;
    double tau = taus[c];
    double et_max = -INFINITY;
    for (int s = 0; s < S; s++) {
      const OStage* x = &m->st[s];
      double k = np_maximum(np_side_count(tau, m->bo, x->oct, x->alpha),
                            np_side_count(tau, m->bo, x->odt, x->beta));
      k = np_maximum(k, 1.0);
      double cnt = isfinite(k) ? ceil(k - 1e-9) : INFINITY;
      if (!isfinite(cnt)) ok = 0;
      double sf = isfinite(cnt) ? cnt : 1.0;
      safe[(size_t)s * C + c] = sf;
      double ct = (x->oct / m->bo) * ((1.0 - x->alpha) + x->alpha / sf);
      double dt = (x->odt / m->bo) * ((1.0 - x->beta) + x->beta / sf);
      double e = np_maximum(ct, dt);
      et_max = (s == 0) ? e : np_maximum(et_max, e);
    }
    double thr = (et_max > 0) ? m->batch / et_max : INFINITY;
    ok = ok && (thr > m->limit);
    /* per-type quota: members summed in stage order (exact for counts < 2^53) */
    for (int t = 0; t < m->d->num_types && ok; t++) {
      double tot = 0.0;
      int present = 0;
      for (int s = 0; s < S; s++)
        if (m->st[s].type == t) {
          tot = present ? tot + safe[(size_t)s * C + c] : safe[(size_t)s * C + c];
          present = 1;
        }
      if (present && !(tot <= (double)m->d->quota[t])) ok = 0;
    }
    double per_second;
    if (C >= 2) {
      per_second = m->price_s[m->st[0].type] * safe[c];
      for (int s = 1; s < S; s++) per_second += m->price_s[m->st[s].type] * safe[(size_t)s * C + c];
    } else {
      for (int s = 0; s < S; s++) col[s] = m->price_s[m->st[s].type] * safe[(size_t)s * C + c];
      per_second = np_pairwise(col, S);
    }
    cost[c] = ok ? m->work / thr * per_second : INFINITY;
    if (ok) any_ok = 1;
    if (cost[c] < best) best = cost[c];
  }
  if (!any_ok) return 0;
  const double lim = best + 1e-15;
  int have = 0;
  for (int c = 0; c < C; c++) {
    if (!(cost[c] <= lim)) continue;
    /* lexicographically smallest integer vector among ties */
    int smaller = !have;
    if (have) {
      for (int s = 0; s < S; s++) {
        long long v = (long long)safe[(size_t)s * C + c];
        if (v != best_k[s]) { smaller = v < best_k[s]; break; }
      }
    }
    if (smaller) {
      for (int s = 0; s < S; s++) best_k[s] = (int)(long long)safe[(size_t)s * C + c];
      have = 1;
    }
  }
  return 1;
}

/* evaluate (ls/costmodel.py:102-167) restricted to what the scorer returns; totals are in
 * insertion order as built by make_provisioning (ls/domain.py:331-353). */
static void evaluate_final(const Model* m, const int* k, int ps, int ps_type, HpsoResult* r) {
  const HpsInstanceDesc* d = m->d;
  double overall = INFINITY;
  int first = 1;
  for (int s = 0; s < m->S; s++) {
    const OStage* x = &m->st[s];
    double ct = (x->oct / m->bo) * ((1.0 - x->alpha) + x->alpha / (double)k[s]);
    double dt = (x->odt / m->bo) * ((1.0 - x->beta) + x->beta / (double)k[s]);
    double et = pmax(ct, dt);
    double tp = (et > 0) ? m->batch / et : INFINITY;
    overall = first ? tp : pmin(overall, tp);
    first = 0;
  }
  double exec_time = (overall > 0 && overall != INFINITY) ? m->work / overall : 0.0;
  /* totals in insertion order */
  r->ntotals = 0;
  for (int s = 0; s < m->S; s++) {
    int t = m->st[s].type, j;
    for (j = 0; j < r->ntotals; j++)
      if (r->tot_type[j] == t) break;
    if (j == r->ntotals) { r->tot_type[j] = t; r->tot_count[j] = 0; r->ntotals++; }
    r->tot_count[j] += k[s];
  }
  if (ps > 0) {
    int j;
    for (j = 0; j < r->ntotals; j++)
      if (r->tot_type[j] == ps_type) break;
    if (j == r->ntotals) { r->tot_type[j] = ps_type; r->tot_count[j] = 0; r->ntotals++; }
    r->tot_count[j] += ps;
  }
  double per_second = 0.0;
  for (int j = 0; j < r->ntotals; j++)
    per_second += d->price_per_hour[r->tot_type[j]] / 3600.0 * (double)r->tot_count[j];
  r->pipeline_tp = overall;
  r->exec_time = exec_time;
  r->cost = exec_time * per_second;
}

static double penalty_cost(const HpsInstanceDesc* d, double gap) { /* ls/scoring.py:47-50 */
  double mx = d->price_per_hour[0];
  for (int t = 1; t < d->num_types; t++) mx = pmax(mx, d->price_per_hour[t]);
  return 1e6 * mx * (1.0 + pmax(0.0, gap));
}

/* PlanScorer.__call__ (ls/scoring.py:79-101) = provision (ls/provisioner.py:564-584) +
 * evaluate; optimize_k1 body follows ls/provisioner.py:374-483 line by line. */
static void score_plan(const HpsInstanceDesc* d, const uint8_t* plan, Scratch* w, HpsoResult* r) {
  memset(r, 0, sizeof(*r));
  for (int l = 0; l < d->num_layers; l++)
    if (plan[l] >= d->num_types) { r->status = HPS_ST_INVALID; r->cost = NAN; return; }
  OStage st[MAXL];
  Model m;
  m.d = d;
  m.S = build_stages(d, plan, st);
  m.st = st;
  m.bo = (double)d->profile_batch_size;
  m.batch = (double)d->batch_size;
  m.work = (double)(d->epochs * d->total_samples);
  m.limit = d->throughput_limit;
  for (int t = 0; t < d->num_types; t++) m.price_s[t] = d->price_per_hour[t] / 3600.0;
  r->num_stages = m.S;
  const int S = m.S;
  double gap = 0.0;
  int status = HPS_ST_OK, ovf = 0;
  int best_k[MAXL];

  do {
    double k1_floor;
    if (min_k1(&st[0], &m, &k1_floor, &gap)) { status = HPS_ST_MIN_K1; break; }
    double tau_hi = m.batch / d->throughput_limit;
    if (k1_floor > 1.0) tau_hi = pmin(tau_hi, stage_et(&st[0], k1_floor, m.bo));
    double serial = serial_floor(&m);
    if (serial >= tau_hi) {
      gap = clamp_gap((serial - tau_hi) / tau_hi);
      status = HPS_ST_SERIAL;
      break;
    }
    if (!quota_ok(&m, tau_hi)) {
      double counts[MAXL];
      if (counts_at(&m, tau_hi, counts, &gap)) { status = HPS_ST_FLOOR_TAU_HI; break; }
      u128 tot[MAXT] = {0};
      for (int s = 0; s < S; s++) tot[st[s].type] += dbl_to_u128(counts[s]);
      for (int t = 0; t < d->num_types; t++) /* sorted(totals.items()): ascending type id */
        if (tot[t] > (u128)d->quota[t]) {
          gap = clamp_gap(int_true_div(tot[t] - (u128)d->quota[t], d->quota[t]));
          break;
        }
      status = HPS_ST_QUOTA_TAU_HI;
      break;
    }
    double a = serial, b = tau_hi;
    for (int it = 0; it < 60; it++) {
      double mid = (a + b) / 2.0;
      if (quota_ok(&m, mid)) b = mid; else a = mid;
    }
    const double tau_lo = b;
    /* breakpoints (ls/provisioner.py:442-455) */
    size_t nb = 2;
    double mn[MAXL], mx[MAXL];
    for (int s = 0; s < S; s++) {
      double r1, r2, g;
      floor_count(&st[s], tau_hi, m.bo, &r1, &g);
      floor_count(&st[s], tau_lo, m.bo, &r2, &g);
      mn[s] = iceil(r1);
      mx[s] = iceil(r2);
      double span = mx[s] - mn[s];
      if (span <= HPS_BREAKPOINT_LIMIT) nb += (size_t)span + 1;
    }
    ensure(w, nb, S);
    double* cand = w->cand;
    size_t nc = 0;
    cand[nc++] = tau_lo;
    cand[nc++] = tau_hi;
    for (int s = 0; s < S; s++) {
      if (mx[s] - mn[s] > HPS_BREAKPOINT_LIMIT) continue;
      const OStage* x = &st[s];
      for (double k = mn[s]; k <= mx[s]; k += 1.0) {
        double ct = (x->oct / m.bo) * ((1.0 - x->alpha) + x->alpha / k);
        double dt = (x->odt / m.bo) * ((1.0 - x->beta) + x->beta / k);
        double e = np_maximum(ct, dt);
        if (e >= tau_lo && e <= tau_hi) cand[nc++] = e;
      }
    }
    r->nraw = (int)nc;
    r->nspan = (int)nb;
    qsort(cand, nc, sizeof(double), cmp_double);
    size_t u = 0;
    for (size_t i = 0; i < nc; i++)
      if (u == 0 || cand[i] != cand[u - 1]) cand[u++] = cand[i];
    nc = u;
    if (nc > HPS_BREAKPOINT_LIMIT) { /* ls/provisioner.py:456-470 */
      ovf = 1;
      double tau_star;
      if (!newton_minimize(&m, tau_lo, tau_hi, &tau_star)) tau_star = golden_minimize(&m, tau_lo, tau_hi);
      double step = (double)nc / (double)(HPS_BREAKPOINT_LIMIT / 2);
      unsigned char* keep = (unsigned char*)calloc(nc, 1);
      keep[0] = keep[nc - 1] = 1;
      for (int i = 0; i < HPS_BREAKPOINT_LIMIT / 2; i++) keep[(size_t)((double)i * step)] = 1;
      size_t centre = 0;
      double bestd = fabs(cand[0] - tau_star);
      for (size_t i = 1; i < nc; i++) {
        double dd = fabs(cand[i] - tau_star);
        if (dd < bestd) { bestd = dd; centre = i; }
      }
      size_t lo_i = centre >= 256 ? centre - 256 : 0, hi_i = centre + 256 < nc ? centre + 256 : nc;
      for (size_t i = lo_i; i < hi_i; i++) keep[i] = 1;
      size_t v = 0;
      for (size_t i = 0; i < nc; i++)
        if (keep[i]) cand[v++] = cand[i];
      free(keep);
      nc = v;
    }
    r->ncand = (int)nc;
    if (!best_candidate(&m, cand, (int)nc, w, best_k)) {
      gap = 1.0;
      status = HPS_ST_NO_CANDIDATE;
      break;
    }
  } while (0);

  if (status != HPS_ST_OK) {
    r->status = status | (ovf ? HPS_ST_OVERFLOW_FLAG : 0);
    r->gap = gap;
    r->cost = penalty_cost(d, gap);
    return;
  }
  /* add_ps_cores (ls/provisioner.py:486-513) */
  int ps = 0, ps_type = -1;
  if (d->with_ps) {
    long long accel = 0;
    for (int s = 0; s < S; s++)
      if (!d->is_cpu[st[s].type]) accel += best_k[s];
    if (accel != 0) {
      ps_type = -1;
      for (int t = 0; t < d->num_types; t++)
        if (d->is_cpu[t] && (ps_type < 0 || d->price_per_hour[t] < d->price_per_hour[ps_type])) ps_type = t;
      if (ps_type < 0) {
        r->status = HPS_ST_NO_CPU_TYPE;
        r->cost = NAN;
        return;
      }
      ps = (int)ceil(d->ps_cores_per_gpu * (double)accel - 1e-9);
      long long have = 0;
      for (int s = 0; s < S; s++)
        if (st[s].type == ps_type) have += best_k[s];
      long long would = have + ps;
      if (would > d->quota[ps_type]) {
        for (int s = 0; s < S; s++) r->k[s] = best_k[s];  /* the rejected final counts */
        r->status = HPS_ST_PS_QUOTA | (ovf ? HPS_ST_OVERFLOW_FLAG : 0);
        r->gap = clamp_gap((double)(would - d->quota[ps_type]) / (double)d->quota[ps_type]);
        r->cost = penalty_cost(d, r->gap);
        return;
      }
    }
  }
  for (int s = 0; s < S; s++) r->k[s] = best_k[s];
  r->ps = ps;
  evaluate_final(&m, best_k, ps, ps_type, r);
  r->status = HPS_ST_OK | (ovf ? HPS_ST_OVERFLOW_FLAG : 0);
  r->gap = 0.0;
}

/* ------------------------------ exported API ------------------------------ */

int hpso_score(const HpsInstanceDesc* d, const uint8_t* plan, HpsoResult* r) {
  Scratch w = {0};
  score_plan(d, plan, &w, r);
  free(w.cand);
  free(w.mat);
  return 0;
}

int hpso_result_size(void) { return (int)sizeof(HpsoResult); }

typedef struct {
  const HpsInstanceDesc* d;
  const uint8_t* plans;
  int64_t lo, hi;
  double* cost;
  uint8_t* status;
  double* gap;
  int32_t* ps;
  int32_t* k;
  int32_t* nstage;
  int32_t* ncand;
} BatchJob;

static void* batch_worker(void* arg) {
  BatchJob* j = (BatchJob*)arg;
  Scratch w = {0};
  HpsoResult r;
  const int L = j->d->num_layers;
  for (int64_t i = j->lo; i < j->hi; i++) {
    score_plan(j->d, j->plans + (size_t)i * L, &w, &r);
    j->cost[i] = r.cost;
    j->status[i] = (uint8_t)r.status;
    if (j->gap) j->gap[i] = r.gap;
    if (j->ps) j->ps[i] = r.ps;
    if (j->nstage) j->nstage[i] = r.num_stages;
    if (j->ncand) j->ncand[i] = r.ncand;
    if (j->k) {
      for (int s = 0; s < L; s++) j->k[(size_t)i * L + s] = s < r.num_stages ? r.k[s] : 0;
      if ((r.status & 0x7f) != HPS_ST_OK && (r.status & 0x7f) != HPS_ST_PS_QUOTA)
        memset(j->k + (size_t)i * L, 0, sizeof(int32_t) * L);
    }
  }
  free(w.cand);
  free(w.mat);
  return NULL;
}

/* Score n plans on `threads` host threads (contiguous shards). Any output except cost and
 * status may be NULL. */
int hpso_score_batch(const HpsInstanceDesc* d, const uint8_t* plans, int64_t n, int threads,
                     double* cost, uint8_t* status, double* gap, int32_t* ps, int32_t* k,
                     int32_t* nstage, int32_t* ncand) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  pthread_t tid[256];
  BatchJob jobs[256];
  for (int t = 0; t < threads; t++) {
    jobs[t] = (BatchJob){d, plans, n * t / threads, n * (t + 1) / threads, cost, status, gap, ps, k, nstage, ncand};
    pthread_create(&tid[t], NULL, batch_worker, &jobs[t]);
  }
  for (int t = 0; t < threads; t++) pthread_join(tid[t], NULL);
  return 0;
}

/* brute force over [begin, end) of the itertools.product order (ls/baselines.py:63-87) */
typedef struct {
  const HpsInstanceDesc* d;
  uint64_t lo, hi;
  double best;
  uint64_t best_idx, feasible;
} EnumJob;

static void decode(uint64_t idx, int T, int L, uint8_t* plan) {
  for (int l = L - 1; l >= 0; l--) {
    plan[l] = (uint8_t)(idx % (uint64_t)T);
    idx /= (uint64_t)T;
  }
}

static void* enum_worker(void* arg) {
  EnumJob* j = (EnumJob*)arg;
  Scratch w = {0};
  HpsoResult r;
  uint8_t plan[MAXL];
  j->best = INFINITY;
  j->best_idx = UINT64_MAX;
  j->feasible = 0;
  for (uint64_t i = j->lo; i < j->hi; i++) {
    decode(i, j->d->num_types, j->d->num_layers, plan);
    score_plan(j->d, plan, &w, &r);
    if ((r.status & 0x7f) != HPS_ST_OK) continue;
    j->feasible++;
    if (r.cost < j->best) { j->best = r.cost; j->best_idx = i; }
  }
  free(w.cand);
  free(w.mat);
  return NULL;
}

int hpso_enum_argmin(const HpsInstanceDesc* d, uint64_t begin, uint64_t end, int threads,
                     double* best_cost, uint64_t* best_idx, uint64_t* feasible) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  pthread_t tid[256];
  EnumJob jobs[256];
  uint64_t n = end - begin;
  for (int t = 0; t < threads; t++) {
    jobs[t].d = d;
    jobs[t].lo = begin + (uint64_t)((u128)n * t / threads);
    jobs[t].hi = begin + (uint64_t)((u128)n * (t + 1) / threads);
    pthread_create(&tid[t], NULL, enum_worker, &jobs[t]);
  }
  *best_cost = INFINITY;
  *best_idx = UINT64_MAX;
  *feasible = 0;
  for (int t = 0; t < threads; t++) {
    pthread_join(tid[t], NULL);
    *feasible += jobs[t].feasible;
    /* shards are in index order, so strict < keeps the earliest index on ties */
    if (jobs[t].best < *best_cost) { *best_cost = jobs[t].best; *best_idx = jobs[t].best_idx; }
  }
  return 0;
}

/* ---- full-sweep digest (test infrastructure: pins every plan of a sweep, not only the winner)
 * Per plan the outputs the device writes (cost bits, status byte, gap bits, PS cores, stage
 * count, per-stage counts; k and ps are 0 unless status == OK) are chained through splitmix64
 * together with the enumeration index; the digest is the wrapping 64-bit SUM over plans, so it
 * does not depend on the order in which shards or threads visit the plans. tests/sweep_digest.py
 * computes the same function from device outputs. */
static uint64_t smix(uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}

uint64_t hpso_plan_hash(uint64_t idx, double cost, int status, double gap, int ps, int S,
                        const int32_t* k, int L) {
  uint64_t cb, gb;
  memcpy(&cb, &cost, 8);
  memcpy(&gb, &gap, 8);
  const int ok = (status & 0x7f) == HPS_ST_OK;
  uint64_t h = smix(idx);
  h = smix(h ^ cb);
  h = smix(h ^ gb);
  h = smix(h ^ ((uint64_t)(status & 0xff) | ((uint64_t)(ok ? ps : 0) << 8) | ((uint64_t)S << 40)));
  for (int s = 0; s < L; s++) h = smix(h ^ (uint64_t)(uint32_t)((ok && s < S) ? k[s] : 0) ^ ((uint64_t)s << 32));
  return h;
}

typedef struct {
  const HpsInstanceDesc* d;
  uint64_t lo, hi;
  double best;
  uint64_t best_idx, feasible, digest;
  uint64_t by_status[16];
  uint64_t overflow;
} DigestJob;

static void* digest_worker(void* arg) {
  DigestJob* j = (DigestJob*)arg;
  Scratch w = {0};
  HpsoResult r;
  uint8_t plan[MAXL];
  const int L = j->d->num_layers;
  j->best = INFINITY;
  j->best_idx = UINT64_MAX;
  for (uint64_t i = j->lo; i < j->hi; i++) {
    decode(i, j->d->num_types, L, plan);
    score_plan(j->d, plan, &w, &r);
    const int code = r.status & 0x7f;
    j->by_status[code & 15]++;
    if (r.status & HPS_ST_OVERFLOW_FLAG) j->overflow++;
    j->digest += hpso_plan_hash(i, r.cost, r.status, r.gap, r.ps, r.num_stages, r.k, L);
    if (code != HPS_ST_OK) continue;
    j->feasible++;
    if (r.cost < j->best) { j->best = r.cost; j->best_idx = i; }
  }
  free(w.cand);
  free(w.mat);
  return NULL;
}

/* brute force over [begin, end) plus the sweep digest and per-status plan counts
 * (out18: feasible, digest, overflow count, by_status[0..15)) */
int hpso_enum_digest(const HpsInstanceDesc* d, uint64_t begin, uint64_t end, int threads,
                     double* best_cost, uint64_t* best_idx, uint64_t* out18) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  pthread_t tid[256];
  static DigestJob jobs[256];
  const uint64_t n = end - begin;
  for (int t = 0; t < threads; t++) {
    memset(&jobs[t], 0, sizeof(DigestJob));
    jobs[t].d = d;
    jobs[t].lo = begin + (uint64_t)((u128)n * t / threads);
    jobs[t].hi = begin + (uint64_t)((u128)n * (t + 1) / threads);
    pthread_create(&tid[t], NULL, digest_worker, &jobs[t]);
  }
  *best_cost = INFINITY;
  *best_idx = UINT64_MAX;
  memset(out18, 0, 18 * sizeof(uint64_t));
  for (int t = 0; t < threads; t++) {
    pthread_join(tid[t], NULL);
    out18[0] += jobs[t].feasible;
    out18[1] += jobs[t].digest;
    out18[2] += jobs[t].overflow;
    for (int c = 0; c < 15; c++) out18[3 + c] += jobs[t].by_status[c];
    if (jobs[t].best < *best_cost) { *best_cost = jobs[t].best; *best_idx = jobs[t].best_idx; }
  }
  return 0;
}

/* ---- numpy PCG64 + Generator.integers (buffered 32-bit Lemire) replica ---- */
static const u128 PCG_MULT = (((u128)0x2360ED051FC65DA4ULL) << 64) | 0x4385DF649FCCF645ULL;

static uint64_t pcg_next64(u128* state, u128 inc) {
  *state = *state * PCG_MULT + inc;
  uint64_t hi = (uint64_t)(*state >> 64), lo = (uint64_t)*state;
  uint64_t x = hi ^ lo;
  unsigned rot = (unsigned)(hi >> 58);
  return (x >> rot) | (x << ((64 - rot) & 63));
}

/* Generate n consecutive rng.integers(0, T, L) calls into plans[n][L]. The 32-bit buffer
 * (has_uint32) persists across calls, as numpy's PCG64.next32 does. */
int hpso_random_plans(const HpsPcg64* g, int T, int L, int64_t n, uint8_t* plans) {
  u128 state = ((u128)g->state_hi << 64) | g->state_lo, inc = ((u128)g->inc_hi << 64) | g->inc_lo;
  int has = 0;
  uint32_t buf = 0;
  const uint32_t thr = (uint32_t)((0x100000000ULL - (uint64_t)T) % (uint64_t)T);
  for (int64_t i = 0; i < n; i++)
    for (int l = 0; l < L; l++) {
      if (T == 1) { plans[i * L + l] = 0; continue; }
      uint64_t mm;
      do {
        uint32_t u32;
        if (has) { has = 0; u32 = buf; }
        else { uint64_t v = pcg_next64(&state, inc); has = 1; buf = (uint32_t)(v >> 32); u32 = (uint32_t)v; }
        mm = (uint64_t)u32 * (uint64_t)T;
      } while ((uint32_t)mm < thr);
      plans[i * L + l] = (uint8_t)(mm >> 32);
    }
  return 0;
}
