/*
 * hps.h — C ABI of the B200 plan evaluator (HeterPS scheduling hot path, arXiv 2111.10635).
 *
 * Plain pointers and sizes only; no torch or CUDA types cross this boundary (streams are
 * passed as `void*` = cudaStream_t). Every entry point returns an HPS_OK / HPS_E_* code;
 * per-plan infeasibility is DATA (status byte + gap), exactly as the reference treats
 * InfeasibleError inside PlanScorer (ls/scoring.py:98-99).
 *
 * Reference interface each entry point replaces (`ls/` = /root/reference/pkg/src/layersched):
 *   hps_instance_create   PlanScorer.__init__ staging  (ls/scoring.py:61-77) + _CostModel
 *                         constants (ls/provisioner.py:203-210); stage table = build_stages
 *                         aggregates for every (type, first, last) run (ls/domain.py:275-328)
 *   hps_stage_table       build_stages (ls/domain.py:275-328)
 *   hps_score_plans       PlanScorer.__call__ -> provision -> optimize_k1 -> add_ps_cores ->
 *                         evaluate (ls/scoring.py:79-101, ls/provisioner.py:374-513,564-584,
 *                         ls/costmodel.py:102-167), batched over N plans
 *   hps_enum_argmin       brute_force enumeration loop + _better (ls/baselines.py:54-87)
 *                         over an index range [begin, end) of the itertools.product order
 *   hps_random_argmin     random_search non-dedup path (ls/baselines.py:230-282): the plans
 *                         are numpy default_rng(seed).integers(0,T,L), generated in-kernel
 *   hps_report            evaluate (ls/costmodel.py:102-167) per-stage times for given counts
 *   hps_score_plans_static  PlanScorer(mode='staratio'|'stapsratio') -> static_provision ->
 *                         evaluate (ls/provisioner.py:516-561, ls/scoring.py:79-101)
 *   hps_pcg64_*           numpy PCG64 / Generator.integers / Generator.random replicas used
 *                         by the searchers and the policy sampler (ls/policy/network.py:251-262)
 */
#ifndef HPS_H_
#define HPS_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HPS_ABI_VERSION 2
#define HPS_MAX_LAYERS 64
#define HPS_MAX_TYPES 16
#define HPS_BREAKPOINT_LIMIT 4096 /* ls/provisioner.py:49 */

/* call-level return codes (mapped to the reference's exceptions by the Python shim) */
enum {
  HPS_OK = 0,
  HPS_E_INVALID_ARG = 1,    /* InvariantError (ls/errors.py:20) */
  HPS_E_PLAN = 2,           /* PlanValidationError (ls/errors.py:24): id out of range */
  HPS_E_CONFIG = 3,         /* ConfigError (ls/errors.py:8): e.g. T^L does not fit a key */
  HPS_E_CUDA = 4,           /* CUDA runtime failure */
  HPS_E_NO_CPU_TYPE = 5,    /* InvariantError from cheapest_cpu_type (ls/domain.py:163-167) */
  HPS_E_NUMERIC = 6         /* NumericError (ls/errors.py:40) */
};

/* per-plan status byte (which InfeasibleError the reference raises, if any) */
enum {
  HPS_ST_OK = 0,
  HPS_ST_MIN_K1 = 1,         /* min_k1 denominator <= 0            ls/provisioner.py:96-102 */
  HPS_ST_SERIAL = 2,         /* serial floor >= tau_hi              ls/provisioner.py:400-412 */
  HPS_ST_QUOTA_TAU_HI = 3,   /* per-type total > quota at tau_hi    ls/provisioner.py:413-427 */
  HPS_ST_FLOOR_TAU_HI = 4,   /* _floor_count raises at tau_hi       ls/provisioner.py:164-174,414 */
  HPS_ST_NO_CANDIDATE = 5,   /* no candidate tau feasible           ls/provisioner.py:473-477 */
  HPS_ST_PS_QUOTA = 6,       /* PS cores exceed the CPU quota       ls/provisioner.py:507-512 */
  HPS_ST_DEFENSIVE = 7,      /* evaluate() disagrees (unreachable)  ls/provisioner.py:481-482 */
  HPS_ST_NO_CPU_TYPE = 8,    /* accelerator units but no CPU type: the reference raises
                                InvariantError (not data); the shim re-raises it            */
  HPS_ST_INVALID = 9,        /* plan id out of range: PlanValidationError                    */
  HPS_ST_STATIC_NONE = 10,   /* static mode: no ratio multiple within quota meets the limit
                                (InfeasibleError gap=1.0)          ls/provisioner.py:557-561 */
  HPS_ST_OVERFLOW_FLAG = 0x80 /* OR-ed in when the >4096-breakpoint path ran (:456-470)       */
};

typedef struct HpsInstance HpsInstance;

/* Host-side description of one (ModelGraph, ResourceCatalog, JobParams, ProvisionerConfig)
 * instance. Tables are [T][L] row-major: oct[t * L + l] = layers[l].per_type_oct[t]. */
typedef struct HpsInstanceDesc {
  int32_t num_layers;              /* L, 1..HPS_MAX_LAYERS */
  int32_t num_types;               /* T, 1..HPS_MAX_TYPES */
  const double* oct;               /* [T*L] LayerSpec.per_type_oct   ls/domain.py:21-40 */
  const double* odt;               /* [T*L] LayerSpec.per_type_odt */
  const double* alpha;             /* [T*L] LayerSpec.per_type_alpha */
  const double* beta;              /* [T*L] LayerSpec.per_type_beta */
  const double* price_per_hour;    /* [T]   ResourceType.price_per_hour ls/domain.py:114-134 */
  const int64_t* quota;            /* [T]   ResourceType.quota */
  const uint8_t* is_cpu;           /* [T]   ResourceType.is_cpu */
  int64_t total_samples;           /* ModelGraph.total_samples (M)  ls/domain.py:74-111 */
  int64_t epochs;                  /* ModelGraph.epochs */
  int64_t batch_size;              /* ModelGraph.batch_size (B) */
  int64_t profile_batch_size;      /* ModelGraph.profile_batch_size (B_o) */
  double throughput_limit;         /* JobParams.throughput_limit  ls/costmodel.py:39-47 */
  double ps_cores_per_gpu;         /* ProvisionerConfig           ls/provisioner.py:57-72 */
  int32_t newton_max_iters;
  double newton_tol;
  double fd_step;
  int32_t with_ps;                 /* provision(with_ps=...)      ls/provisioner.py:564-584 */
} HpsInstanceDesc;

/* Per-plan outputs, structure of arrays in DEVICE memory. `cost` and `status` are required;
 * the rest may be NULL. k is [n][L] (stage s of plan i at k[i*L+s]; unused slots are 0). */
typedef struct HpsPlanResults {
  double* cost;        /* ScoredPlan.cost: monetary cost, or penalty_cost(gap) */
  uint8_t* status;     /* HPS_ST_* */
  double* gap;         /* InfeasibleError.gap (0 when feasible) */
  int32_t* ps;         /* ProvisioningPlan.ps_cores */
  int32_t* num_stages; /* len(build_stages(plan)) */
  int32_t* k;          /* ProvisioningPlan.per_stage_k; also the rejected counts of an
                          HPS_ST_PS_QUOTA plan (the PS check runs on final counts) */
} HpsPlanResults;

/* Details of an infeasible plan: the values the reference's InfeasibleError text names
 * (ls/provisioner.py:98-101 min_k1, :164-174 _floor_count at tau_hi, :407-411 serial floor,
 * :421-425 quota at tau_hi, :508-511 PS cores). Filled per status; other fields are 0. */
typedef struct HpsExplain {
  int32_t status;       /* HPS_ST_* code the fields describe (the status passed in, masked) */
  int32_t stage;        /* MIN_K1: 0; SERIAL: the (first) stage with the largest serial time;
                           FLOOR_TAU_HI: the first stage whose _floor_count raises */
  int32_t side;         /* MIN_K1 / FLOOR_TAU_HI: 0 computation, 1 communication */
  int32_t serial_side;  /* FLOOR_TAU_HI: 1 when that side has frac == 0 ("serial ... time") */
  int32_t type;         /* QUOTA_TAU_HI: first offending type id; PS_QUOTA: cheapest CPU type */
  int32_t pad;
  uint64_t units_hi;    /* QUOTA_TAU_HI: that type's units at tau_hi (Python int, 128 bits); */
  uint64_t units_lo;    /* PS_QUOTA: the CPU type's units including the PS cores */
  int64_t ps;           /* PS_QUOTA: parameter-server cores */
  double serial;        /* SERIAL: _serial_floor(stages) */
  double tau_hi;        /* SERIAL: tau_hi */
} HpsExplain;

/* Argmin key over a set of plans: (cost, lexicographic rank of the assignment). The rank is
 * the base-T number with layer 0 most significant (= itertools.product index), 128 bits. */
typedef struct HpsArgmin {
  double cost;          /* +inf when nothing qualified */
  uint64_t rank_hi;
  uint64_t rank_lo;
  uint64_t evaluated;   /* plans scored */
  uint64_t feasible;    /* plans with status OK */
  uint32_t status;      /* status of the winner */
  uint32_t flags;       /* bit0: some plan hit HPS_ST_NO_CPU_TYPE, bit1: HPS_ST_INVALID */
} HpsArgmin;

/* numpy PCG64 bit-generator state (np.random.PCG64().state) as four 64-bit words */
typedef struct HpsPcg64 {
  uint64_t state_hi, state_lo, inc_hi, inc_lo;
} HpsPcg64;

int hps_abi_version(void);
const char* hps_error_string(int code);
const char* hps_last_error(void);

int hps_instance_create(const HpsInstanceDesc* desc, HpsInstance** out);
int hps_instance_destroy(HpsInstance* inst);

/* Stage aggregates of run (type t, layers first..last), computed on the device with the
 * reference's Neumaier summation. Host output arrays of length 4: {oct, odt, alpha, beta}. */
int hps_stage_table(HpsInstance* inst, int32_t type_id, int32_t first, int32_t last,
                    double* out4);

/* Score n plans (u8 [n][L] in device memory, ids in [0,T)). Stream-ordered. */
int hps_score_plans(HpsInstance* inst, const uint8_t* d_plans, int64_t n,
                    const HpsPlanResults* d_out, void* stream);

/* Message details of scored plans: d_status / d_k are hps_score_plans outputs for the same
 * plans (k is read for HPS_ST_PS_QUOTA only). One HpsExplain per plan to d_out (device). */
int hps_explain(HpsInstance* inst, const uint8_t* d_plans, const uint8_t* d_status,
                const int32_t* d_k, int64_t n, HpsExplain* d_out, void* stream);

/* Brute force over enumeration indices [begin, end) (T^L must fit 64 bits). feasible_only=1
 * keeps only status-OK plans (ls/baselines.py:83-84); ties go to the smaller index
 * (ls/baselines.py:54-60). Writes one HpsArgmin to d_best (device). */
int hps_enum_argmin(HpsInstance* inst, uint64_t begin, uint64_t end, int32_t feasible_only,
                    HpsArgmin* d_best, void* stream);

/* hps_enum_argmin over all T^L plans with certified subtree pruning: the plans sharing their
 * first `depth` layers form one index range; a lower bound of the cost of every plan in the range
 * (stage counts relaxed to the continuous requirement at the best possible E, quotas ignored)
 * skips ranges that cannot hold a plan costing <= the incumbent, and the rest are swept exactly.
 * Same winner (cost and index, ties included) as hps_enum_argmin(0, T^L, feasible_only = 1);
 * `evaluated` / `feasible` count the swept plans only. incumbent = +inf: the range with the
 * smallest bound is swept first and its winner is the incumbent. Synchronises `stream` twice
 * (the survivor count sizes the sweep). Replaces the brute_force loop, ls/baselines.py:63-87. */
typedef struct HpsPruneStats {
  uint64_t prefixes;       /* T^depth index ranges */
  uint64_t survivors;      /* ranges swept after pruning (besides the incumbent's) */
  uint64_t evaluated;      /* plans scored */
  uint64_t subtree;        /* plans per range, T^(L - depth) */
  double incumbent_cost;   /* cost the bounds were compared with */
  double min_bound;        /* smallest range bound */
  int32_t depth;
  int32_t pad;
} HpsPruneStats;
int hps_enum_argmin_pruned(HpsInstance* inst, int32_t depth, double incumbent, HpsArgmin* d_best,
                           HpsPruneStats* stats, void* stream);

/* Argmin over an explicit plan batch (u8 [n][L] device memory), same key and tie rules as
 * hps_enum_argmin; the rank packs ceil(log2 T) bits per layer (needs bits*L <= 128).
 * Replaces the scoring loop + _better of random_search's dedup path and of any caller that
 * already holds its plans (ls/baselines.py:252-282). */
int hps_plans_argmin(HpsInstance* inst, const uint8_t* d_plans, int64_t n, int32_t feasible_only,
                     HpsArgmin* d_best, void* stream);

/* Random sweep: plan p (p in [first, first+n)) is the p-th call of
 * default_rng(seed).integers(0, T, L) (ls/baselines.py:270-271) from `gen`'s initial state.
 * Penalised plans are included (ls/baselines.py:275-278). Requires a power-of-two T
 * (Lemire never rejects); other T return HPS_E_CONFIG. */
int hps_random_argmin(HpsInstance* inst, const HpsPcg64* gen, uint64_t first, uint64_t n,
                      HpsArgmin* d_best, void* stream);

/* hps_enum_argmin over the arithmetic progression first, first + stride, ... (count indices):
 * rank r of W takes (first = begin + r, stride = W), which deals neighbouring plans — whose
 * provisioning work is correlated — to different GPUs and balances the shards. Same key
 * semantics as hps_enum_argmin (the rank field is the enumeration index). */
int hps_enum_argmin_strided(HpsInstance* inst, uint64_t first, uint64_t stride, uint64_t count,
                            int32_t feasible_only, HpsArgmin* d_best, void* stream);

/* Materialise the random plans of hps_random_argmin into d_plans (u8 [n][L]). */
int hps_random_plans(HpsInstance* inst, const HpsPcg64* gen, uint64_t first, uint64_t n,
                     uint8_t* d_plans, void* stream);

/* evaluate() for n (plan, per-stage k, ps) triples (ls/costmodel.py:102-167). Device
 * outputs: per-stage ct/dt/et/tp [n][L] and per-plan pipeline throughput, total exec time,
 * monetary cost, feasible flag. */
int hps_report(HpsInstance* inst, const uint8_t* d_plans, const int32_t* d_k,
               const int32_t* d_ps, int64_t n, double* d_ct, double* d_dt, double* d_et,
               double* d_tp, double* d_pipeline_tp, double* d_exec_time, double* d_cost,
               uint8_t* d_feasible, void* stream);

/* Static provisioning baselines (ls/provisioner.py:516-561): the smallest multiplier g with
 * 1 accelerator unit per accelerator stage and `cpu_per_gpu` cores per CPU stage that meets
 * the throughput limit within quota; mode HPS_MODE_STAPSRATIO also charges cpu_per_gpu
 * parameter-server cores per accelerator unit on the cheapest CPU type. Same outputs as
 * hps_score_plans; the instance's ProvisionerConfig and with_ps are not used (as in the
 * reference). A catalog without a CPU type gives HPS_ST_NO_CPU_TYPE for every valid plan
 * (ls/provisioner.py:538 raises before the scan). */
enum { HPS_MODE_STARATIO = 1, HPS_MODE_STAPSRATIO = 2 };
int hps_score_plans_static(HpsInstance* inst, const uint8_t* d_plans, int64_t n, int32_t mode,
                           int32_t cpu_per_gpu, const HpsPlanResults* results, void* stream);

/* ---- scheduling policy on the device (K3-K6) -----------------------------------------------
 * Replaces policy_forward / sample_actions / the train() round body / policy_gradient /
 * policy_backward (ls/policy/network.py:147-262, ls/policy/training.py:115-274). */
typedef struct HpsPolicy HpsPolicy;
int hps_policy_create(int32_t num_layers, int32_t feature_dim, int32_t hidden, int32_t num_types,
                      int32_t lstm, int64_t max_plans, const double* features, HpsPolicy** out);
int hps_policy_destroy(HpsPolicy* policy);
/* which: 0 w_cell [D+H][G*H], 1 b_cell, 2 w_out [H][T], 3 b_out; dir 0 host->device, 1 back */
int hps_policy_params(HpsPolicy* policy, int32_t which, int32_t dir, double* host, int64_t n);
/* K4: LSTM/Elman forward at the current parameters; probabilities [L][T] to d_probs (optional) */
int hps_policy_forward(HpsPolicy* policy, double temperature, double* d_probs, void* stream);
/* K3: n plans; plan g, layer t uses draw first_draw + g*L + t of the PCG64 stream, one
 * Generator.random() per Generator.choice(T, p). first_draw = UINT64_MAX reads the policy's
 * device counter (hps_policy_counter) instead. */
int hps_policy_sample(HpsPolicy* policy, const HpsPcg64* gen, uint64_t first_draw, int64_t n,
                      uint8_t* d_plans, void* stream);
/* K6+K5: one REINFORCE round from the G scored plans: best-ever, winsorising, standardising,
 * dlogits in trace order, BPTT, norm cap, update, moving-average baseline, RoundStats row.
 * round = 0 takes the round number from the device counter. Every call advances the counter
 * (round + 1, draws + G*L), so a captured round (CUDA graph) replays as the next round. */
int hps_policy_reinforce(HpsPolicy* policy, const double* d_cost, const uint8_t* d_status,
                         const uint8_t* d_plans, int64_t num_plans, int32_t round,
                         double temperature, double learning_rate, double baseline_rate,
                         double* d_history, uint8_t* d_best_plan, long long* d_best_where,
                         void* stream);
/* Set the device round counter: the next round's number (>= 1) and the draws consumed. */
int hps_policy_counter(HpsPolicy* policy, uint64_t round, uint64_t draws, void* stream);
/* {baseline, best cost, entropy} and {non-finite logits, non-finite params} flags */
int hps_policy_state(HpsPolicy* policy, double* state3, int32_t* flags2);
const char* hps_policy_last_error(void);

/* Number of kernels this library has launched in the process (all entry points, host-side
 * counter incremented at every launch). bench.py reports the difference over its timed region. */
uint64_t hps_launch_count(void);

/* Device counters of an instrumented build (-DHPS_STATS); HPS_E_CONFIG otherwise. */
int hps_stats_read(unsigned long long* out, int n, int reset);

/* FP64 pipe microbenchmark (kind 0: dependent-chain DFMA x8 per thread, 16 flops per loop
 * step per chain pair; kind 1: IEEE division). Used for the roofline denominator. */
int hps_probe_fp64(int kind, double* d_out, int blocks, int threads, int iters, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* HPS_H_ */
