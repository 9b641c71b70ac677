/*
 * cosched.h -- C-ABI of the B200-native exhaustive, model-driven co-location
 * search of Arima et al., "Optimizing Hardware Resource Partitioning and Job
 * Allocations on Modern GPUs under Power Caps" (arXiv 2405.03838).
 *
 * Citations: P:Lnnn = /root/reference/PAPER.md line (section / equation /
 * table named beside it); R# = a reading of the paper listed in DESIGN.md.
 *
 * WHAT IT COMPUTES (one call chain per job queue):
 *   For every set of n_slots jobs of the queue (pairs by default),
 *   every partition state S of the caller's table and every power cap P of
 *   the caller's grid (the search space of Table `search-space`, P:L556-566,
 *   generalised per P:L500/L794), it evaluates the linear model
 *       RPerf_i(S,P) = C(S,P).H(F_i) + sum_{j!=i} D(S,P).J(F_j)
 *   with the basis H, J of Table `functions`, then
 *       Throughput = sum_i RPerf_i, Fairness = min_i RPerf_i,
 *   and keeps the config maximising Throughput (Problem 1) or
 *   Throughput / P (Problem 2) subject to Fairness > alpha
 *   (strict). That is the paper's exhaustive search run for
 *   every set of a queue; the queue-level reductions (best set, best job ->
 *   GPU allocation) are the extension of P:L843 (reading R12).
 *
 * All compute runs in the library's CUDA kernels (sm_100a). There is no CPU
 * fallback: without a usable CUDA device every compute entry point returns
 * COSCHED_E_CUDA.
 *
 * Conventions:
 *  - Every function returns a cosched_status; no exception crosses the ABI.
 *  - Validation happens before any launch; on error no output is modified and
 *    cosched_last_error(h) holds a one-line message.
 *  - "device" pointers are CUDA device (or managed) memory owned by the
 *    caller; "host" pointers are ordinary host memory owned by the caller.
 *  - Sets are unordered job tuples named by their colexicographic id:
 *      pair   (j0<j1):      id = j1*(j1-1)/2 + j0
 *      triple (j0<j1<j2):   id = C(j2,3) + C(j1,2) + j0
 *      solo   (j0):         id = j0
 *    where j are queue POSITIONS 0..n_jobs-1; slot i of the set gets j_i.
 *  - Configs: c = state * n_caps + cap, state in table order, caps ascending.
 *    Ties in the objective resolve to the lowest c (reading R9).
 *  - Handles are not thread-safe. Collective calls (marked COLLECTIVE) must be
 *    made by every rank of the communicator with identical arguments.
 */
#ifndef COSCHED_H
#define COSCHED_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct cosched_ctx* cosched_t;

typedef enum {
  COSCHED_OK = 0,
  COSCHED_INFEASIBLE = 2,           /* non-fatal: nothing satisfies Fairness > alpha */
  COSCHED_E_ARG = 10,               /* bad argument: null pointer, size, objective, alpha < 0, non-finite coefficient */
  COSCHED_E_INVALID_ALLOCATION = 11, /* a state's GPCs < 1 or not summing to gpcs_total, memory option not 0/1,
                                        caps not positive strictly ascending */
  COSCHED_E_UNKNOWN_KEY = 12,       /* state_slice outside [0, n_slices) */
  COSCHED_E_DEGENERATE_PROFILE = 13, /* a job has F1 <= 0.01 % (reading R4) */
  COSCHED_E_RANGE = 14,             /* a counter is NaN/inf, outside [0,100], or F6+F7+F8 > 100 */
  COSCHED_E_STATE = 15,             /* call order violated (e.g. best_set before score_all) */
  COSCHED_E_CUDA = 20,              /* CUDA error or no CUDA device */
  COSCHED_E_NCCL = 21,              /* NCCL missing or failed */
  COSCHED_E_OOM = 22                /* workspace too small */
} cosched_status;

/* The searched space and the fitted model (all host pointers; deep-copied by
 * cosched_create, the caller may free them on return). */
typedef struct {
  int32_t n_slots;            /* jobs per set: 1 solo, 2 pairs, 3 triples ("up to two" in the paper) */
  int32_t gpcs_total;         /* every state's GPC counts sum to this: 7 on A100 under MIG, 8 B200-like */
  int32_t n_states;           /* partition states S, in canonical (= tie-break) order */
  const int32_t* state_gpcs;  /* [n_states][n_slots] GPCs given to each slot, each >= 1 (validation only) */
  const int32_t* state_mem;   /* [n_states] LLC/HBM option: 0 shared, 1 private */
  const int32_t* state_slice; /* [n_states][n_slots] coefficient row used by each slot (reading R1) */
  int32_t n_slices;           /* rows of the coefficient table per cap */
  int32_t n_caps;             /* power caps P */
  const float* caps_w;        /* [n_caps] watts, > 0, strictly ascending */
  const float* coef_c;        /* [n_caps][n_slices][6]  C of P:L458 (scalability) */
  const float* coef_d;        /* [n_caps][n_slices][3]  D of P:L458 (interference) */
  int32_t objective;          /* 1 = Problem 1 (Throughput; pass a one-cap grid for "given P"), 2 = Problem 2 (Throughput/P) */
  float alpha;                /* fairness threshold, >= 0; feasible iff Fairness > alpha */
} cosched_desc;

/* Per-set results of cosched_score_all for this rank's shard
 * [first_set, first_set + n_sets). Device pointers, caller-owned; either may
 * be NULL (then only the queue-level reductions are kept). obj[k] is the best
 * objective of set first_set+k (-inf if no config is feasible); cfg[k] its
 * config id (-1 if none). first_set / n_sets must equal cosched_shard_range. */
typedef struct {
  float* obj;
  int32_t* cfg;
  int64_t first_set;
  int64_t n_sets;
} cosched_out;

/* Validate and deep-copy the description; bind to CUDA device `cuda_device`.
 * Errors: E_ARG, E_INVALID_ALLOCATION, E_UNKNOWN_KEY, E_CUDA. */
cosched_status cosched_create(const cosched_desc* desc, int cuda_device, cosched_t* out_handle);

void cosched_destroy(cosched_t h);

/* Per-handle message of the last error ("" if none). Valid until the next call on h. */
const char* cosched_last_error(cosched_t h);

/* Message for errors that happen before a handle exists (create). */
const char* cosched_last_create_error(void);

/* ---- Limits (all checked; a call outside them returns the status named) ----
 *  - sets per queue <= 2^32 - 2 (set ids are 32-bit in the argmax keys):
 *    pairs up to 92,682 jobs, triples up to 2,954 jobs        -> COSCHED_E_ARG
 *  - n_slots 1..3, n_states <= 128, n_caps <= 64, n_slices <= 32767 (create) -> COSCHED_E_ARG
 *  - greedy allocation: queues up to 2^20 jobs (the taken bitmask of the
 *    one-block scan lives in shared memory; every queue the scorer accepts
 *    fits); per-rank batches below 2^30 keys (CUB int counts), chosen by the
 *    library                                                    -> COSCHED_E_CUDA
 *  - exact allocation: k * n_slots == n_jobs with n_jobs <= 20 (pairs) / 15 (triples)
 *  - node budgeting: integer-watt caps, node_power_w / gcd(caps) <= 12287 -> COSCHED_E_ARG
 *  - the tiled pair scorer covers every queue the set limit allows (fewer than
 *    32768 column tiles); shards are whole colex columns by construction. */

/* ---- multi-GPU (one process per GPU) -------------------------------------
 * The search shards by contiguous set-id range (whole colex columns, i.e. a
 * range of the largest job position) with no data-path exchange; the only
 * exchanges are the argmax all-reduces of cosched_best_set /
 * cosched_best_allocation, done with ncclAllReduce(u64, max) on the
 * library's own communicator. NCCL is loaded at run time (dlopen
 * "libnccl.so.2", the copy torch already loaded when present). Test hook:
 * when the environment variable COSCHED_NCCL_LIB names a library exporting the
 * same six NCCL entry points, that library is loaded instead (read once per
 * process, at the first communicator use); tests/loopback/ provides an
 * in-process stand-in that runs W ranks as W threads on one GPU. */

/* Rank 0: write a 128-byte ncclUniqueId to uid_out (host). E_NCCL if NCCL is unavailable. */
cosched_status cosched_get_unique_id(void* uid_out);

/* COLLECTIVE: create the communicator from rank 0's id (host, 128 bytes).
 * nranks == 1 with uid == NULL resets to single-rank mode without NCCL;
 * nranks == 1 with an id builds a one-rank communicator (every collective of
 * the library then runs through NCCL, as on a multi-GPU node). */
cosched_status cosched_set_comm(cosched_t h, const void* nccl_unique_id, int rank, int nranks);

/* Shard view without a communicator: score as rank `rank` of `nranks` on this
 * one device (collectives then reduce over this process only). Used to test
 * the multi-GPU sharding on a single GPU ("fake ranks"). */
cosched_status cosched_set_shard_view(cosched_t h, int rank, int nranks);

/* This rank's set range for a queue of n_jobs (host only, no CUDA). Rank r of
 * W gets the sets whose largest position lies in [b_r, b_{r+1}). Pairs: the
 * b_r are multiples of 64 (whole column blocks of the pair scorer's 64 x 64
 * tiles) chosen by a DP that minimises the largest modelled scorer time of a
 * rank on a B200 (whole-tile rounds on 296 CTA slots plus the stage-split last
 * round; api.cu pair_block_bounds); a rank may get no sets when n_jobs is
 * small. Solo: b_r the smallest b with b >= r * n_jobs / W. Triples: balanced
 * on the triple scorer's tiles, b_r the smallest b with T(b) >= r * T(n_jobs) / W,
 * where T(b) = sum over planes 1 <= j < b of t(t+1)/2 with t = ceil(j / 64).
 * A pure function of (n_jobs, n_slots, rank, W): identical on every rank. */
cosched_status cosched_shard_range(cosched_t h, int64_t n_jobs, int64_t* first_set, int64_t* n_sets);

/* The same partition without a handle (host only): rank of nranks, sets of n_slots jobs. */
cosched_status cosched_shard_range_for(int64_t n_jobs, int32_t n_slots, int32_t rank, int32_t nranks,
                                       int64_t* first_set, int64_t* n_sets);

/* Host-only helpers (no CUDA): number of sets, colex unranking of a set id
 * into ascending queue positions pos[n_slots], and the packed argmax key
 * used by every reduction: key = (ord(obj) << 32) | (0xFFFFFFFF - set_id'),
 * ord = order-preserving float->u32 map, key 0 = infeasible. */
int64_t cosched_n_sets(int64_t n_jobs, int32_t n_slots);
cosched_status cosched_unrank(int64_t n_jobs, int32_t n_slots, int64_t set_id, int64_t* pos);
uint64_t cosched_pack_key(float obj, int64_t set_id);
void cosched_unpack_key(uint64_t key, float* obj, int64_t* set_id);

/* Bytes of device workspace cosched_score_all needs for n_jobs. */
cosched_status cosched_workspace_size(cosched_t h, int64_t n_jobs, size_t* bytes);

/* Score every set of this rank's shard (async on `cuda_stream`, a
 * cudaStream_t; NULL = legacy default stream).
 *  features_dev: float [n_rows][8], counters F1..F8 in percent (Table `counters`)
 *  jobs_dev:     int32 [n_jobs] row of each queue position, or NULL for row = position
 *  n_rows:       rows of features_dev (validates jobs_dev)
 *  workspace_dev: >= cosched_workspace_size bytes, 256-byte aligned; device
 *                memory the handle uses between its calls (later calls read
 *                this call's results from it). One region of it, the pair
 *                scorer's stage-split merge area, keeps step-tagged entries from
 *                call to call: it is zeroed the first time a handle sees a
 *                workspace pointer, so pass a new pointer (or a new handle) after
 *                writing to the workspace yourself
 *  out:          host struct with device pointers (may be NULL)
 * Steps (all kernels): validate features (E_RANGE / E_DEGENERATE_PROFILE for
 * the first bad queue position, reported at the next synchronising call),
 * basis H, J, projection onto C, D, per-set model evaluation, objective,
 * fairness constraint, per-set argmax, per-shard argmax key.
 * Exactness: out->cfg[k] is the exact FP32 argmax of set k (strict >, lowest
 * config on ties) or a config whose FP32 objective is within tau/2 = 5e-6
 * relative of it, for every valid input; out->obj[k] is the FP32 objective of
 * out->cfg[k] (-inf, cfg -1 iff no config is feasible: feasibility is decided
 * exactly). The tiled scorers compare configs by a fixed-point objective and
 * re-score exactly, in the same call, every set where that could miss the
 * bound (cosched_last_rescored). With the tiled
 * scorers (variant 1, exhaustive mode) the projection's ka / kb rows are not
 * computed in this call; cosched_best_config, cosched_best_allocation and
 * cosched_node_budget project them on the same stream when they first need
 * them (results are identical either way). */
cosched_status cosched_score_all(cosched_t h, const float* features_dev, int64_t n_rows,
                                 const int32_t* jobs_dev, int64_t n_jobs, void* workspace_dev,
                                 size_t workspace_bytes, const cosched_out* out, void* cuda_stream);

/* Synchronise the last score_all and return this rank's best set (no comm).
 * *key is the packed key (0 if no feasible set). Reports deferred validation errors. */
cosched_status cosched_local_best_key(cosched_t h, uint64_t* key);

/* COLLECTIVE (when a communicator is set): the queue's best set = max over
 * ranks of the packed key (ncclAllReduce u64 max), then its best config and
 * objective, re-derived on the GPU by every rank from the set id (every rank
 * holds every job's basis; no further exchange). *cfg and *obj are that set's
 * exact FP32 argmax and its objective (the detail kernel's evaluation). The
 * detail kernel writes the result straight into pinned host memory: one
 * stream synchronisation.
 * COSCHED_INFEASIBLE if no set has a feasible config. */
cosched_status cosched_best_set(cosched_t h, int64_t* set_id, int32_t* cfg, float* obj);

/* cosched_best_set in two halves. _begin enqueues the same work on the stream
 * of the last score_all (the all-reduce when a communicator is set, then the
 * detail kernel, which writes the result into the handle's pinned host buffer)
 * and returns without synchronising, so the caller can record an event after
 * the step's last device work; _end synchronises that stream and returns what
 * cosched_best_set returns. Every _begin must be followed by one _end before
 * the next call on the handle; _end without _begin returns COSCHED_E_STATE. */
cosched_status cosched_best_set_begin(cosched_t h);
cosched_status cosched_best_set_end(cosched_t h, int64_t* set_id, int32_t* cfg, float* obj);

/* The best config of one set of the last scored queue, evaluated on the GPU
 * (any rank, any set, no comm). rperf: host float[n_slots] (may be NULL);
 * throughput / fairness / obj: host (may be NULL). COSCHED_INFEASIBLE (cfg -1)
 * if no config of that set is feasible. */
cosched_status cosched_best_config(cosched_t h, int64_t set_id, int32_t* cfg, float* obj,
                                   float* rperf, float* throughput, float* fairness);

/* COLLECTIVE: job -> GPU allocation over the last scored queue (reading R12):
 * choose k disjoint sets maximising the sum of per-set objectives.
 *  - exact when k * n_slots == n_jobs and n_jobs <= 20 (pairs) / 15 (triples):
 *    every partition of the queue into sets, enumerated lowest-free-job-first
 *    with partners ascending; partitions containing an infeasible set are
 *    skipped; ties -> first in that order;
 *  - greedy otherwise: repeatedly take the feasible set with the largest
 *    (obj, -set_id) whose jobs are all free, the first k taken -- computed on
 *    the GPU by a histogram-batched sorted scan that resolves the sequential
 *    rule exactly in parallel rounds (greedy.cu); locally-dominant rounds over
 *    the shard when a batch exceeds the per-rank capacity.
 * Requires score_all with out != NULL covering the shard.
 * set_ids, cfgs: host arrays of >= k entries; *n_found = sets chosen, in
 * order of formation (exact) or of decreasing key (greedy).
 * COSCHED_INFEASIBLE if no (complete, for exact) allocation exists. */
cosched_status cosched_best_allocation(cosched_t h, int32_t k, int64_t* set_ids, int32_t* cfgs,
                                       double* total_obj, int32_t* n_found);

/* Select the pair scorer: 1 = tiled fast kernel (default), 0 = generic
 * one-thread-per-set kernel (the simple reference the fast one is tested
 * against). Env COSCHED_PAIR_KERNEL=generic selects 0 at create. */
cosched_status cosched_set_variant(cosched_t h, int variant);

/* Search mode of cosched_score_all (and of best_set / best_config /
 * best_allocation, which follow the scored results):
 *   mode 0: the exhaustive search over every (state, cap) -- default;
 *   mode 1: hill climbing over the (state x cap) grid from (start_state,
 *           start_cap), the heuristic P:L664 / L796 suggests for large spaces
 *           (reading R22: steepest ascent over the 4
 *           grid neighbours in config order, strict improvement, local optimum;
 *           an infeasible climb restarts from every other config in canonical
 *           order). Its objective never exceeds the exhaustive one.
 * COSCHED_E_ARG for another mode or a start outside the grid. Marks previous
 * results stale (call cosched_score_all again). */
cosched_status cosched_set_search(cosched_t h, int mode, int32_t start_state, int32_t start_cap);

/* Candidates (set, config) the last cosched_score_all evaluated on this rank:
 * n_sets x n_configs for the exhaustive search, the counted evaluations of
 * the climbs (revisits included) for hill climbing. Synchronises. */
cosched_status cosched_last_search_evals(cosched_t h, int64_t* evals);

/* ---- Worst / proposal / best against a ground truth ----
 *
 * The paper's evaluation: for every set of the last
 * cosched_score_all, the PROPOSAL (the scored cfg) is re-scored by a
 * ground-truth performance model, and BEST / WORST are the largest / smallest
 * ground-truth objective over the configs whose ground-truth Fairness exceeds
 * alpha. The ground truth is SPEC.md's synthetic GPU (`true_rperf`; reading
 * R21) with these constants -- the stand-in for the paper's A100 measurements. */
typedef struct {
  int32_t g_full;        /* GPCs of the unpartitioned chip (the normalisation point) */
  int32_t n_modules;     /* memory modules of the chip */
  int32_t modules[17];   /* private option: modules given to g GPCs, g = 0..16 */
  float w_base, w_gpc;   /* static power and power per GPC at full non-tensor compute (W) */
  float kappa, f_min;    /* tensor power multiplier; minimum throttle factor */
  float p_max;           /* cap of the normalisation run (W) */
} cosched_truth_desc;

typedef struct {
  float* prop_obj;   /* device [n_sets_local] ground-truth objective of the proposal (-inf: no proposal) */
  float* prop_fair;  /* device [n_sets_local] its ground-truth Fairness */
  float* best_obj;   /* device [n_sets_local] best ground-truth objective with true Fairness > alpha (-inf: none) */
  float* worst_obj;  /* device [n_sets_local] worst such objective (-inf: none) */
} cosched_eval_out;

typedef struct {
  int64_t n_compared;            /* sets with a proposal and a truly feasible config (all ranks) */
  int64_t n_violations;          /* of those, proposals whose true Fairness <= alpha */
  double geomean_prop_over_best; /* geometric mean over the compared sets of proposal / best */
  double geomean_worst_over_best;
} cosched_eval_summary;

/* Workspace bytes for cosched_evaluate_truth on this rank's shard. */
cosched_status cosched_evaluate_workspace_size(cosched_t h, int64_t n_jobs, size_t* bytes);

/* COLLECTIVE (sums the summary over ranks). Requires cosched_score_all with out
 * != NULL; features / jobs must be the ones it scored. Outputs are for this
 * rank's shard; every member of out must be non-NULL. Synchronises the stream. COSCHED_E_ARG for
 * invalid constants (g_full < 1 or > 16, n_modules < 1, p_max <= 0,
 * f_min outside (0, 1], a state's GPCs > g_full). */
cosched_status cosched_evaluate_truth(cosched_t h, const cosched_truth_desc* truth, const float* features_dev,
                                      int64_t n_rows, const int32_t* jobs_dev, void* workspace,
                                      size_t workspace_bytes, const cosched_eval_out* out,
                                      cosched_eval_summary* summary, void* cuda_stream);

/* ---- Node-level power budgeting ----------------------
 *
 * The job manager's power budgeting ("sets the power caps", L400, L782,
 * L844): the n_gpus GPUs are grouped into nodes of gpus_per_node consecutive
 * entries, GPU g running set set_ids[g] (e.g. from cosched_best_allocation).
 * Per GPU and cap, thr(p) = the best Throughput over the states whose Fairness
 * > alpha (lowest state on ties); per node one cap per GPU maximising
 *   objective 1: sum_g thr_g(p_g)                 s.t. sum_g P(p_g) <= node_power_w
 *   objective 2: sum_g thr_g(p_g) / sum_g P(p_g)  s.t. the same
 * exactly, by a DP over the total power in units of the caps' gcd (reading
 * R23; caps must be integer watts, node_power_w / gcd <= 12287). Uses the
 * projection of the last cosched_score_all (any rank: every rank projects the
 * whole queue; no collective). Outputs (host): caps_out[n_gpus] cap index,
 * cfgs_out[n_gpus] = state * n_caps + cap, node_obj[n_nodes]; a node with no
 * feasible assignment gets -1 / -1 / -inf. Synchronises the stream. */
cosched_status cosched_node_workspace_size(cosched_t h, int64_t n_gpus, int32_t gpus_per_node, double node_power_w,
                                           size_t* bytes);
cosched_status cosched_node_budget(cosched_t h, int64_t n_gpus, const int64_t* set_ids, int32_t gpus_per_node,
                                   double node_power_w, int32_t objective, void* workspace, size_t workspace_bytes,
                                   int32_t* caps_out, int32_t* cfgs_out, float* node_obj, void* cuda_stream);

/* Record (on = 1) or not (0, the default) the events cosched_last_timings
 * reads: one between the gather and the scorer and one after the scorer. They
 * cost the scorer's launch its overlap with the gather's tail (programmatic
 * dependent launch, ~5 us a step), so timing runs ask for them explicitly. */
cosched_status cosched_set_timing(cosched_t h, int on);

/* Device time (ms, CUDA events on the caller's stream) of the last
 * cosched_score_all: ms[0] = validate + basis + projection, ms[1] = the set
 * scorer (the dominant kernel), ms[2] = the whole call. Synchronises.
 * COSCHED_E_STATE unless that call ran with cosched_set_timing(h, 1). */
cosched_status cosched_last_timings(cosched_t h, float* ms3);

/* Device time of the last step, in ms: from the event cosched_score_all records
 * on its stream before its first kernel to the one cosched_best_set(_begin)
 * records after the best-set detail kernel (the step's last device work; its
 * result is then in pinned host memory). Host-side call latency before the
 * first launch is not included. Synchronises that event. COSCHED_E_STATE unless
 * cosched_score_all was followed by a completed cosched_best_set. */
cosched_status cosched_last_step_ms(cosched_t h, float* ms);

/* Sets of the last cosched_score_all that the tiled scorer flagged for exact
 * re-scoring (instrumentation): those whose packed-objective choice was not
 * provably within tau/2 = 5e-6 relative of the exact FP32 argmax (objective
 * below 6 * n_slots quanta / tau; DESIGN.md §2 "Exactness of the tiled argmax").
 * (Pairs: the sets the tile end flagged, or more than the list holds; triples:
 * the sets the objective scan found.)
 * Every flagged set was re-scored exactly by k_rescore_sets in the same call, so
 * this is a performance counter, not an error. 0 with the generic scorer.
 * Synchronises the stream. */
cosched_status cosched_last_rescored(cosched_t h, int64_t* n_rescored);

/* Rounds of the last greedy cosched_best_allocation (instrumentation). */
int64_t cosched_last_greedy_rounds(cosched_t h);

/* Number of kernels the library launched since create (instrumentation for bench.py). */
int64_t cosched_kernel_launches(cosched_t h);

/* ---- Calibration of the model coefficients ------------
 *
 * The offline step that produces coef_c / coef_d for cosched_create: "we train
 * the model coefficients ... by the well-known least square method",
 * "for each combination of (S, P) independently and separately":
 * the solo-run coefficients C first, then D from co-runs.
 *
 * key = cap * n_slices + slice, i.e. the row of coef_c / coef_d (reading R1).
 *   stage C: per key, C[key] = argmin_c sum (rperf - c . H(F_app))^2 over its solo samples;
 *   stage D: per key, with r = rperf - C[key] . H(F_subject) on its co-run samples,
 *            D[key] = argmin_d sum (r - d . sum_partners J(F_partner))^2  (the summed
 *            partner term of P:L458).
 * Solved in FP64 by the normal equations (Cholesky); a key is rank deficient
 * when a pivot is <= 1e-10 x its column's squared norm (reading R20). Samples
 * are grouped by key with a stable sort, so results are bit-identical run to run
 * and independent of sample order up to FP64 rounding. */
typedef enum {
  COSCHED_FIT_OK = 0,
  COSCHED_FIT_NO_SAMPLES = 1,      /* the key has no samples for this stage (D of a solo-only key: D = 0) */
  COSCHED_FIT_INSUFFICIENT = 2,    /* fewer samples than coefficients (SPEC.md InsufficientSamples) */
  COSCHED_FIT_RANK_DEFICIENT = 3,  /* (SPEC.md RankDeficient) */
  COSCHED_FIT_MISSING_C = 4        /* co-run samples on a key whose C did not fit (SPEC.md MissingScalabilityCoefficients) */
} cosched_fit_status;

typedef struct {
  int32_t n_slices, n_caps;      /* key space: n_slices * n_caps keys */
  int32_t n_partners;            /* partners per co-run sample (n_slots - 1: 1 or 2); ignored if n_corun = 0 */
  int64_t n_apps;                /* profiled applications */
  const float* features;         /* device [n_apps][8] counters F1..F8 (%), validated like cosched_score_all's */
  int64_t n_solo;                /* solo samples (< 2^31) */
  const int32_t* solo_app;       /* device [n_solo] app index */
  const int32_t* solo_key;       /* device [n_solo] key */
  const float* solo_rperf;       /* device [n_solo] measured RPerf (relative to the solo, full-chip, P_max run) */
  int64_t n_corun;               /* co-run samples, one per (run, subject slot) (< 2^31) */
  const int32_t* co_app;         /* device [n_corun] subject app */
  const int32_t* co_partners;    /* device [n_corun][n_partners] the co-located apps */
  const int32_t* co_key;         /* device [n_corun] key of the subject's slice and cap */
  const float* co_rperf;         /* device [n_corun] the subject's measured RPerf */
} cosched_fit_desc;

typedef struct {
  double* coef_c;   /* device [n_caps][n_slices][6] (0 where the key did not fit) */
  double* coef_d;   /* device [n_caps][n_slices][3] (0 where the key did not fit or has no co-runs) */
  int32_t* status;  /* device [n_keys][2] cosched_fit_status of stage C and stage D */
  int64_t* count;   /* device [n_keys][2] samples per key and stage */
  double* rms;      /* device [n_keys][2] RMS residual of the fit (NaN where it did not fit) */
} cosched_fit_out;

/* Workspace (device bytes) cosched_fit needs for this descriptor. */
cosched_status cosched_fit_workspace_size(const cosched_fit_desc* desc, size_t* bytes);

/* Fit C and D for every key on the caller's stream and synchronise it.
 * Returns COSCHED_OK when the inputs are valid (per-key outcomes are in
 * out->status); COSCHED_E_RANGE / COSCHED_E_DEGENERATE_PROFILE for an invalid
 * feature row, COSCHED_E_UNKNOWN_KEY for a key / app index out of range or a
 * non-finite rperf (then out is unspecified; cosched_fit_last_error says which
 * row), COSCHED_E_OOM if workspace_bytes is too small, COSCHED_E_CUDA without a
 * device. Needs no handle and no communicator (a per-node offline step). */
cosched_status cosched_fit(const cosched_fit_desc* desc, void* workspace, size_t workspace_bytes,
                           const cosched_fit_out* out, void* cuda_stream);

/* Message of the last failed cosched_fit in this process. */
const char* cosched_fit_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* COSCHED_H */
