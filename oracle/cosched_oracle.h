/*
 * cosched_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, single-threaded FP64 CPU oracle for the exhaustive
 * model-driven co-location search of Arima et al., arXiv 2405.03838.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it. The product path (include/cosched.h,
 * paper_2405_03838_b200/) never includes, links or calls anything here, and
 * this file shares no code, header, table or constant with it.
 *
 * Citations: P:Lnnn = PAPER.md line, S:Lnnn = SPEC.md line, R# = a reading
 * listed in DESIGN.md ("Readings of the paper").
 *
 * Parity pins: every function below is pinned by tests/test_oracle_*.py
 * against worked examples, closed forms, invariants or brute force; none is
 * "parity unpinned".
 */
#ifndef COSCHED_ORACLE_H
#define COSCHED_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes of the oracle (its own numbering; tests map them). */
enum {
  ORC_OK = 0,
  ORC_INFEASIBLE = 2,           /* no candidate has Fairness > alpha */
  ORC_E_ARG = 10,
  ORC_E_INVALID_ALLOCATION = 11, /* partition table violates its invariants */
  ORC_E_UNKNOWN_KEY = 12,       /* slice id outside the coefficient table */
  ORC_E_DEGENERATE_PROFILE = 13, /* F1 <= 0.01 % */
  ORC_E_RANGE = 14              /* a counter outside [0,100], non-finite, or F6+F7+F8 > 100 */
};

/* The searched space and the model coefficients: Problem 1/2 of P:L378-400,
 * states S and caps P of Table `search-space`, C(S,P)/D(S,P) of
 * the model equation keyed per slot slice (reading R1). */
typedef struct {
  int32_t n_slots;            /* applications per co-located set: 1, 2 or 3 */
  int32_t gpcs_total;         /* every state's GPCs sum to this */
  int32_t n_states;
  const int32_t* state_gpcs;  /* [n_states][n_slots] */
  const int32_t* state_mem;   /* [n_states] 0 shared / 1 private */
  const int32_t* state_slice; /* [n_states][n_slots] coefficient row per slot */
  int32_t n_slices;
  int32_t n_caps;
  const float* caps_w;        /* [n_caps] strictly ascending */
  const float* coef_c;        /* [n_caps][n_slices][6] */
  const float* coef_d;        /* [n_caps][n_slices][3] */
  int32_t objective;          /* 1: Throughput (Problem 1), 2: Throughput / P (Problem 2) */
  float alpha;                /* Fairness > alpha, strict */
} orc_problem;

/* Validation of the problem description (BASELINE.json split invariant). */
int orc_validate_problem(const orc_problem* pb, char* msg, int msglen);

/* Validation of the job features. features is
 * float[n_rows][8]; jobs (may be NULL = identity) is int32[n_jobs] of row ids. */
int orc_validate_features(const float* features, int64_t n_rows, const int32_t* jobs,
                          int64_t n_jobs, char* msg, int msglen);

/* Basis functions of Table `functions`. */
void orc_basis_h(const float f[8], double h[6]);
void orc_basis_j(const float f[8], double j[3]);

/* RPerf of the job in slot `slot` of the set. members: feature rows
 * of the set's jobs in slot order. */
double orc_rperf(const orc_problem* pb, const float* const* members, int slot, int state, int cap);

/* Evaluate every config c = state*n_caps + cap of one set (P:L663 exhaustive
 * search; c order = S:L380 tie order). Any output may be NULL.
 * obj[c], fair[c], thr[c], feasible[c], rperf[c*n_slots + i]. */
void orc_eval_set(const orc_problem* pb, const float* const* members, double* obj, double* fair,
                  double* thr, int32_t* feasible, double* rperf);

/* The best config of one set: argmax of the objective over feasible configs,
 * first in canonical order on ties. cfg = -1 and obj = -inf when no
 * config is feasible (reading R10). Returns ORC_OK or ORC_INFEASIBLE. */
int orc_best_config_members(const orc_problem* pb, const float* const* members, int32_t* cfg,
                            double* obj);

/* Number of sets C(n_jobs, n_slots), by the plain product formula. */
int64_t orc_n_sets(int64_t n_jobs, int n_slots);
/* Hill climbing over the (state x cap) grid from (start_state, start_cap) with the
 * infeasible-start fallback (reading R22). */
int orc_hill_climb(const orc_problem* pb, const float* const* members, int start_state, int start_cap,
                   int32_t* cfg, double* obj, int64_t* evals);
int orc_hill_range(const orc_problem* pb, const float* features, const int32_t* jobs, int64_t n_jobs,
                   int64_t first, int64_t count, int start_state, int start_cap, int32_t* cfg_out,
                   double* obj_out, int64_t* evals_out);

/* Set id -> job positions (ascending) in colex order, by plain enumeration search. */
int orc_unrank(int64_t n_jobs, int n_slots, int64_t set_id, int64_t* pos);

/* Score sets [first, first+count) in colex order: cfg_out[k], obj_out[k]. */
int orc_score_range(const orc_problem* pb, const float* features, const int32_t* jobs,
                    int64_t n_jobs, int64_t first, int64_t count, int32_t* cfg_out, double* obj_out);

/* The best set over all sets (max obj, lowest id on ties); also visits every set. */
int orc_best_set(const orc_problem* pb, const float* features, const int32_t* jobs, int64_t n_jobs,
                 int64_t first, int64_t count, int64_t* set_id, int32_t* cfg, double* obj);

/* Exact allocation (P:L843 extension, reading R12): over every partition of
 * the n_jobs = k*n_slots queue into k sets, enumerated recursively (lowest
 * free job first, partners ascending), maximise the sum of the per-set
 * objectives; matchings with an infeasible set are skipped; first in
 * enumeration order on ties. set_obj[] are the per-set objectives indexed by
 * colex set id (-inf = infeasible). Outputs the winning rank, its set ids in
 * formation order, the total. *n_matchings = how many partitions exist. */
int orc_exact_allocation(int64_t n_jobs, int n_slots, const double* set_obj, int64_t* best_rank,
                         int64_t* set_ids, double* total, int64_t* n_matchings);

/* Greedy allocation: scan feasible sets by (obj desc, id asc), take a set iff
 * all its jobs are free, stop after k. Returns the number taken. */
int64_t orc_greedy_allocation(int64_t n_jobs, int n_slots, const double* set_obj, int64_t k,
                              int64_t* set_ids);

#ifdef __cplusplus
}
#endif
#endif
