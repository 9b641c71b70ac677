/*
 * cosched_oracle.c -- TEST INFRASTRUCTURE ONLY (see cosched_oracle.h).
 *
 * Plain FP64, single-threaded, un-factorised: every function is the
 * definition in the paper written out, in the paper's order and notation.
 * No blocking, no precomputation across sets, no reordering. It reads the
 * same float32 inputs as the CUDA path and shares no code with it.
 */
#include "cosched_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define ORC_EPS_F1 0.01 /* F1 <= 0.01 % is an idle compute pipe, H3 = F2/F1 undefined */

static void set_msg(char* msg, int msglen, const char* text) {
  if (msg && msglen > 0) {
    strncpy(msg, text, (size_t)msglen - 1);
    msg[msglen - 1] = 0;
  }
}

/* S:L160-168 (validate), P:L283 (GPC total), P:L565 (cap menu), P:L382 (alpha). */
int orc_validate_problem(const orc_problem* pb, char* msg, int msglen) {
  char buf[256];
  if (!pb || pb->n_slots < 1 || pb->n_slots > 3 || pb->n_states < 1 || pb->n_slices < 1 ||
      pb->n_caps < 1 || !pb->state_gpcs || !pb->state_mem || !pb->state_slice || !pb->caps_w ||
      !pb->coef_c || !pb->coef_d) {
    set_msg(msg, msglen, "bad sizes or null table");
    return ORC_E_ARG;
  }
  if (pb->objective != 1 && pb->objective != 2) {
    set_msg(msg, msglen, "objective must be 1 or 2");
    return ORC_E_ARG;
  }
  if (!(pb->alpha >= 0.0f) || isinf(pb->alpha)) {
    set_msg(msg, msglen, "alpha must be finite and >= 0");
    return ORC_E_ARG;
  }
  for (int s = 0; s < pb->n_states; s++) {
    int sum = 0;
    for (int i = 0; i < pb->n_slots; i++) {
      int g = pb->state_gpcs[s * pb->n_slots + i];
      if (g < 1) {
        snprintf(buf, sizeof buf, "state %d slot %d: %d GPCs < 1", s, i, g);
        set_msg(msg, msglen, buf);
        return ORC_E_INVALID_ALLOCATION;
      }
      sum += g;
    }
    if (sum != pb->gpcs_total) {
      snprintf(buf, sizeof buf, "state %d: GPCs sum to %d, not %d", s, sum, pb->gpcs_total);
      set_msg(msg, msglen, buf);
      return ORC_E_INVALID_ALLOCATION;
    }
    if (pb->state_mem[s] != 0 && pb->state_mem[s] != 1) {
      snprintf(buf, sizeof buf, "state %d: memory option %d", s, pb->state_mem[s]);
      set_msg(msg, msglen, buf);
      return ORC_E_INVALID_ALLOCATION;
    }
  }
  for (int c = 0; c < pb->n_caps; c++) {
    float w = pb->caps_w[c];
    if (!(w > 0.0f) || isinf(w) || (c > 0 && !(w > pb->caps_w[c - 1]))) {
      snprintf(buf, sizeof buf, "cap %d: %g W not positive / strictly ascending", c, (double)w);
      set_msg(msg, msglen, buf);
      return ORC_E_INVALID_ALLOCATION;
    }
  }
  for (int s = 0; s < pb->n_states; s++)
    for (int i = 0; i < pb->n_slots; i++) {
      int sl = pb->state_slice[s * pb->n_slots + i];
      if (sl < 0 || sl >= pb->n_slices) {
        snprintf(buf, sizeof buf, "state %d slot %d: slice %d not in coefficient table", s, i, sl);
        set_msg(msg, msglen, buf);
        return ORC_E_UNKNOWN_KEY;
      }
    }
  for (long t = 0; t < (long)pb->n_caps * pb->n_slices * 6; t++)
    if (!isfinite(pb->coef_c[t])) {
      set_msg(msg, msglen, "non-finite C coefficient");
      return ORC_E_ARG;
    }
  for (long t = 0; t < (long)pb->n_caps * pb->n_slices * 3; t++)
    if (!isfinite(pb->coef_d[t])) {
      set_msg(msg, msglen, "non-finite D coefficient");
      return ORC_E_ARG;
    }
  set_msg(msg, msglen, "");
  return ORC_OK;
}

/* S:L26-27 (0 <= F_k <= 100, F6+F7+F8 <= 100), S:L54/L87 (F1 > 0.01). The
 * tensor sum is a float sum, (F6+F7)+F8, the precision the kernel decides in. */
int orc_validate_features(const float* features, int64_t n_rows, const int32_t* jobs,
                          int64_t n_jobs, char* msg, int msglen) {
  char buf[256];
  if (n_jobs < 0 || (n_jobs > 0 && !features)) {
    set_msg(msg, msglen, "bad job count");
    return ORC_E_ARG;
  }
  for (int64_t q = 0; q < n_jobs; q++) {
    int64_t row = jobs ? (int64_t)jobs[q] : q;
    if (row < 0 || row >= n_rows) {
      snprintf(buf, sizeof buf, "job %lld: row %lld outside [0,%lld)", (long long)q, (long long)row,
               (long long)n_rows);
      set_msg(msg, msglen, buf);
      return ORC_E_ARG;
    }
    const float* f = features + row * 8;
    for (int k = 0; k < 8; k++)
      if (!(f[k] >= 0.0f && f[k] <= 100.0f)) {
        snprintf(buf, sizeof buf, "job %lld: F%d=%g outside [0,100]", (long long)q, k + 1, (double)f[k]);
        set_msg(msg, msglen, buf);
        return ORC_E_RANGE;
      }
    float tensor = f[5] + f[6];
    tensor = tensor + f[7];
    if (!(tensor <= 100.0f)) {
      snprintf(buf, sizeof buf, "job %lld: F6+F7+F8=%g > 100", (long long)q, (double)tensor);
      set_msg(msg, msglen, buf);
      return ORC_E_RANGE;
    }
    if (!((double)f[0] > ORC_EPS_F1)) {
      snprintf(buf, sizeof buf, "job %lld: F1=%g <= 0.01", (long long)q, (double)f[0]);
      set_msg(msg, msglen, buf);
      return ORC_E_DEGENERATE_PROFILE;
    }
  }
  set_msg(msg, msglen, "");
  return ORC_OK;
}

/* Table `functions`: H1 = F1/100 - H2, H2 = (F6+F7+F8)/100,
 * H3 = F2/F1, H4 = F4/100 (formula as printed, reading R2), H5 = F5/100,
 * H6 = const = 1 (reading R3). */
void orc_basis_h(const float f[8], double h[6]) {
  double F1 = f[0], F2 = f[1], F4 = f[3], F5 = f[4], F6 = f[5], F7 = f[6], F8 = f[7];
  h[1] = (F6 + F7 + F8) / 100.0;
  h[0] = F1 / 100.0 - h[1];
  h[2] = F2 / F1;
  h[3] = F4 / 100.0;
  h[4] = F5 / 100.0;
  h[5] = 1.0;
}

/* Table `functions`: J1 = F3/100, J2 = F4/100, J3 = const = 1. */
void orc_basis_j(const float f[8], double j[3]) {
  j[0] = (double)f[2] / 100.0;
  j[1] = (double)f[3] / 100.0;
  j[2] = 1.0;
}

/* The model, P:L458:
 *   RPerf_i(S,P) = C(S,P) . H(F_i) + sum_{j != i} D(S,P) . J(F_j)
 * with C and D read from the row of slot i's slice at cap P (reading R1).
 * With one slot the sum is empty: the solo model of P:L468. */
double orc_rperf(const orc_problem* pb, const float* const* members, int slot, int state, int cap) {
  int slice = pb->state_slice[state * pb->n_slots + slot];
  const float* C = pb->coef_c + ((long)cap * pb->n_slices + slice) * 6;
  const float* D = pb->coef_d + ((long)cap * pb->n_slices + slice) * 3;
  double h[6], j[3];
  orc_basis_h(members[slot], h);
  double r = 0.0;
  for (int t = 0; t < 6; t++) r += (double)C[t] * h[t];
  for (int l = 0; l < pb->n_slots; l++) {
    if (l == slot) continue;
    orc_basis_j(members[l], j);
    for (int t = 0; t < 3; t++) r += (double)D[t] * j[t];
  }
  return r;
}

/* Exhaustive search over S x P. Throughput = sum_i RPerf_i,
 * Fairness = min_i RPerf_i, feasible iff Fairness > alpha (P:L382,
 * strict, reading R6), objective = Throughput (Problem 1) or
 * Throughput / P (Problem 2; P is the cap, reading R8). */
void orc_eval_set(const orc_problem* pb, const float* const* members, double* obj, double* fair,
                  double* thr, int32_t* feasible, double* rperf) {
  for (int s = 0; s < pb->n_states; s++)
    for (int p = 0; p < pb->n_caps; p++) {
      int c = s * pb->n_caps + p;
      double through = 0.0, fairness = INFINITY;
      for (int i = 0; i < pb->n_slots; i++) {
        double r = orc_rperf(pb, members, i, s, p);
        if (rperf) rperf[(long)c * pb->n_slots + i] = r;
        through += r;
        if (r < fairness) fairness = r;
      }
      double o = pb->objective == 1 ? through : through / (double)pb->caps_w[p];
      if (obj) obj[c] = o;
      if (fair) fair[c] = fairness;
      if (thr) thr[c] = through;
      if (feasible) feasible[c] = fairness > (double)pb->alpha;
    }
}

/* argmax over feasible configs, replacing only on a strictly greater
 * objective so the first config in (state order, cap ascending) wins ties
 * (reading R9). None feasible: cfg -1, obj -inf (reading R10). */
int orc_best_config_members(const orc_problem* pb, const float* const* members, int32_t* cfg,
                            double* obj) {
  int n_cfg = pb->n_states * pb->n_caps;
  double* o = (double*)malloc(sizeof(double) * n_cfg);
  int32_t* f = (int32_t*)malloc(sizeof(int32_t) * n_cfg);
  orc_eval_set(pb, members, o, NULL, NULL, f, NULL);
  double best = -INFINITY;
  int32_t arg = -1;
  for (int c = 0; c < n_cfg; c++)
    if (f[c] && o[c] > best) {
      best = o[c];
      arg = c;
    }
  free(o);
  free(f);
  *cfg = arg;
  *obj = best;
  return arg < 0 ? ORC_INFEASIBLE : ORC_OK;
}

/* Hill climbing over the (state x cap) grid (the
 * heuristic P:L664 names for large spaces, "apply some heuristics here such as
 * the hill-climbing algorithm", and P:L796). Reading R22, after
 * SPEC.md hill_climb (L352-360):
 *   f(c) = objective of config c if Fairness > alpha, else -inf;
 *   climb from (s, p): evaluate the 4 grid neighbours (s-1,p), (s,p-1),
 *   (s,p+1), (s+1,p) that exist -- in increasing config index -- and move to
 *   the first one with the largest f if that is strictly greater than f of the
 *   current config; stop when none is (a local optimum);
 *   if the climb from the start ends infeasible, climb from every other config
 *   in canonical order and return the first climb that ends feasible;
 *   none: cfg -1, obj -inf.
 * evals counts every f evaluation (revisits included). */
static double hc_f(const orc_problem* pb, const float* const* members, int s, int p) {
  double through = 0.0, fairness = INFINITY;
  for (int i = 0; i < pb->n_slots; i++) {
    double r = orc_rperf(pb, members, i, s, p);
    through += r;
    if (r < fairness) fairness = r;
  }
  if (!(fairness > (double)pb->alpha)) return -INFINITY;
  return pb->objective == 1 ? through : through / (double)pb->caps_w[p];
}

static double hc_climb(const orc_problem* pb, const float* const* members, int s, int p, int* cs, int* cp,
                       int64_t* evals) {
  double v = hc_f(pb, members, s, p);
  (*evals)++;
  for (;;) {
    const int ns[4] = {s - 1, s, s, s + 1}, np[4] = {p, p - 1, p + 1, p};
    int bs = -1, bp = -1;
    double bv = v;
    for (int k = 0; k < 4; k++) {
      if (ns[k] < 0 || ns[k] >= pb->n_states || np[k] < 0 || np[k] >= pb->n_caps) continue;
      double w = hc_f(pb, members, ns[k], np[k]);
      (*evals)++;
      if (w > bv) {
        bv = w;
        bs = ns[k];
        bp = np[k];
      }
    }
    if (bs < 0) break;
    s = bs;
    p = bp;
    v = bv;
  }
  *cs = s;
  *cp = p;
  return v;
}

int orc_hill_climb(const orc_problem* pb, const float* const* members, int start_state, int start_cap,
                   int32_t* cfg, double* obj, int64_t* evals) {
  int s, p;
  int64_t ev = 0;
  double v = hc_climb(pb, members, start_state, start_cap, &s, &p, &ev);
  if (v == -INFINITY) {
    const int start = start_state * pb->n_caps + start_cap;
    for (int c = 0; c < pb->n_states * pb->n_caps && v == -INFINITY; c++) {
      if (c == start) continue;
      v = hc_climb(pb, members, c / pb->n_caps, c % pb->n_caps, &s, &p, &ev);
    }
  }
  if (evals) *evals = ev;
  if (v == -INFINITY) {
    *cfg = -1;
    *obj = -INFINITY;
    return ORC_INFEASIBLE;
  }
  *cfg = s * pb->n_caps + p;
  *obj = v;
  return ORC_OK;
}

/* C(n, k) for k in {1, 2, 3}: the number of unordered k-job sets. */
int64_t orc_n_sets(int64_t n_jobs, int n_slots) {
  if (n_jobs < n_slots) return 0;
  if (n_slots == 1) return n_jobs;
  if (n_slots == 2) return n_jobs * (n_jobs - 1) / 2;
  return n_jobs * (n_jobs - 1) * (n_jobs - 2) / 6;
}

/* colex successor of an ascending position tuple: bump the lowest position
 * that can move, reset the ones below it to 0,1,... */
static void colex_next(int64_t* pos, int k) {
  for (int i = 0; i < k; i++) {
    pos[i]++;
    if (i == k - 1 || pos[i] < pos[i + 1]) return;
    pos[i] = i;
  }
}

/* Colex rank of an ascending tuple: sum_i C(pos[i], i+1). */
static int64_t colex_rank(const int64_t* pos, int k) {
  int64_t r = 0;
  for (int i = 0; i < k; i++) r += orc_n_sets(pos[i], i + 1);
  return r;
}

/* Unrank by plain search: the top position is the largest t with
 * C(t, k) <= id; subtract and recurse on the remaining slots. */
int orc_unrank(int64_t n_jobs, int n_slots, int64_t set_id, int64_t* pos) {
  if (n_slots < 1 || n_slots > 3 || set_id < 0 || set_id >= orc_n_sets(n_jobs, n_slots))
    return ORC_E_ARG;
  int64_t rest = set_id;
  for (int i = n_slots - 1; i >= 0; i--) {
    int64_t t = i;
    while (orc_n_sets(t + 1, i + 1) <= rest) t++;
    pos[i] = t;
    rest -= orc_n_sets(t, i + 1);
  }
  return ORC_OK;
}

static int gather(const float* features, const int32_t* jobs, const int64_t* pos, int k,
                  const float** members) {
  for (int i = 0; i < k; i++) {
    int64_t row = jobs ? (int64_t)jobs[pos[i]] : pos[i];
    members[i] = features + row * 8;
  }
  return 0;
}

int orc_score_range(const orc_problem* pb, const float* features, const int32_t* jobs,
                    int64_t n_jobs, int64_t first, int64_t count, int32_t* cfg_out, double* obj_out) {
  int st = orc_validate_problem(pb, NULL, 0);
  if (st) return st;
  if (first < 0 || count < 0 || first + count > orc_n_sets(n_jobs, pb->n_slots)) return ORC_E_ARG;
  if (count == 0) return ORC_OK;
  int64_t pos[3];
  const float* members[3];
  orc_unrank(n_jobs, pb->n_slots, first, pos);
  for (int64_t q = 0; q < count; q++) {
    gather(features, jobs, pos, pb->n_slots, members);
    orc_best_config_members(pb, members, &cfg_out[q], &obj_out[q]);
    colex_next(pos, pb->n_slots);
  }
  return ORC_OK;
}

/* Hill climbing for every set of [first, first + count) (as orc_score_range). */
int orc_hill_range(const orc_problem* pb, const float* features, const int32_t* jobs, int64_t n_jobs,
                   int64_t first, int64_t count, int start_state, int start_cap, int32_t* cfg_out,
                   double* obj_out, int64_t* evals_out) {
  int st = orc_validate_problem(pb, NULL, 0);
  if (st) return st;
  if (start_state < 0 || start_state >= pb->n_states || start_cap < 0 || start_cap >= pb->n_caps) return ORC_E_ARG;
  if (count <= 0) return ORC_OK;
  int64_t pos[3];
  if (orc_unrank(n_jobs, pb->n_slots, first, pos)) return ORC_E_ARG;
  const float* members[3];
  for (int64_t q = 0; q < count; q++) {
    for (int i = 0; i < pb->n_slots; i++) {
      int64_t row = jobs ? (int64_t)jobs[pos[i]] : pos[i];
      members[i] = features + row * 8;
    }
    int64_t ev = 0;
    orc_hill_climb(pb, members, start_state, start_cap, &cfg_out[q], &obj_out[q], &ev);
    if (evals_out) evals_out[q] = ev;
    colex_next(pos, pb->n_slots);
  }
  return ORC_OK;
}

int orc_best_set(const orc_problem* pb, const float* features, const int32_t* jobs, int64_t n_jobs,
                 int64_t first, int64_t count, int64_t* set_id, int32_t* cfg, double* obj) {
  int st = orc_validate_problem(pb, NULL, 0);
  if (st) return st;
  if (first < 0 || count < 0 || first + count > orc_n_sets(n_jobs, pb->n_slots)) return ORC_E_ARG;
  int64_t pos[3];
  const float* members[3];
  double best = -INFINITY;
  int64_t arg = -1;
  int32_t arg_cfg = -1;
  if (count > 0) orc_unrank(n_jobs, pb->n_slots, first, pos);
  for (int64_t q = 0; q < count; q++) {
    int32_t c;
    double o;
    gather(features, jobs, pos, pb->n_slots, members);
    if (orc_best_config_members(pb, members, &c, &o) == ORC_OK && o > best) {
      best = o;
      arg = first + q;
      arg_cfg = c;
    }
    colex_next(pos, pb->n_slots);
  }
  *set_id = arg;
  *cfg = arg_cfg;
  *obj = best;
  return arg < 0 ? ORC_INFEASIBLE : ORC_OK;
}

/* ---- exact allocation: recursive enumeration of all partitions ---------- */

typedef struct {
  int64_t n_jobs;
  int k;
  const double* set_obj;
  int free_[64];
  int64_t chosen[32];
  int n_chosen;
  int64_t rank;
  int64_t best_rank;
  double best_total;
  int64_t best_sets[32];
} alloc_state;

static void alloc_rec(alloc_state* A) {
  int lowest = -1;
  for (int j = 0; j < A->n_jobs; j++)
    if (A->free_[j]) {
      lowest = j;
      break;
    }
  if (lowest < 0) { /* a complete partition: rank A->rank */
    double total = 0.0;
    int ok = 1;
    for (int i = 0; i < A->n_chosen; i++) {
      double o = A->set_obj[A->chosen[i]];
      if (isinf(o) && o < 0) ok = 0;
      total += o;
    }
    if (ok && total > A->best_total) {
      A->best_total = total;
      A->best_rank = A->rank;
      memcpy(A->best_sets, A->chosen, sizeof(int64_t) * A->n_chosen);
    }
    A->rank++;
    return;
  }
  A->free_[lowest] = 0;
  if (A->k == 2) {
    for (int b = lowest + 1; b < A->n_jobs; b++) {
      if (!A->free_[b]) continue;
      int64_t pos[2] = {lowest, b};
      A->free_[b] = 0;
      A->chosen[A->n_chosen++] = colex_rank(pos, 2);
      alloc_rec(A);
      A->n_chosen--;
      A->free_[b] = 1;
    }
  } else { /* k == 3 */
    for (int b = lowest + 1; b < A->n_jobs; b++) {
      if (!A->free_[b]) continue;
      A->free_[b] = 0;
      for (int c = b + 1; c < A->n_jobs; c++) {
        if (!A->free_[c]) continue;
        int64_t pos[3] = {lowest, b, c};
        A->free_[c] = 0;
        A->chosen[A->n_chosen++] = colex_rank(pos, 3);
        alloc_rec(A);
        A->n_chosen--;
        A->free_[c] = 1;
      }
      A->free_[b] = 1;
    }
  }
  A->free_[lowest] = 1;
}

int orc_exact_allocation(int64_t n_jobs, int n_slots, const double* set_obj, int64_t* best_rank,
                         int64_t* set_ids, double* total, int64_t* n_matchings) {
  if ((n_slots != 2 && n_slots != 3) || n_jobs < n_slots || n_jobs % n_slots || n_jobs > 60)
    return ORC_E_ARG;
  alloc_state* A = (alloc_state*)calloc(1, sizeof(alloc_state));
  A->n_jobs = n_jobs;
  A->k = n_slots;
  A->set_obj = set_obj;
  for (int j = 0; j < n_jobs; j++) A->free_[j] = 1;
  A->best_rank = -1;
  A->best_total = -INFINITY;
  alloc_rec(A);
  *best_rank = A->best_rank;
  *total = A->best_total;
  *n_matchings = A->rank;
  int64_t k = n_jobs / n_slots;
  for (int64_t i = 0; i < k; i++) set_ids[i] = A->best_rank >= 0 ? A->best_sets[i] : -1;
  int st = A->best_rank < 0 ? ORC_INFEASIBLE : ORC_OK;
  free(A);
  return st;
}

/* ---- greedy allocation ----------------------------------------------------- */

static const double* g_sort_obj;
static int cmp_greedy(const void* a, const void* b) {
  int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  double ox = g_sort_obj[x], oy = g_sort_obj[y];
  if (ox > oy) return -1;
  if (ox < oy) return 1;
  return x < y ? -1 : (x > y ? 1 : 0);
}

int64_t orc_greedy_allocation(int64_t n_jobs, int n_slots, const double* set_obj, int64_t k,
                              int64_t* set_ids) {
  int64_t n = orc_n_sets(n_jobs, n_slots);
  int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (n > 0 ? n : 1));
  int32_t* members = (int32_t*)malloc(sizeof(int32_t) * (n > 0 ? n : 1) * n_slots);
  int64_t m = 0;
  int64_t pos[3] = {0, 1, 2};
  for (int64_t id = 0; id < n; id++) {
    for (int i = 0; i < n_slots; i++) members[id * n_slots + i] = (int32_t)pos[i];
    if (!(isinf(set_obj[id]) && set_obj[id] < 0)) order[m++] = id;
    colex_next(pos, n_slots);
  }
  g_sort_obj = set_obj;
  qsort(order, (size_t)m, sizeof(int64_t), cmp_greedy);
  char* taken = (char*)calloc((size_t)n_jobs + 1, 1);
  int64_t got = 0;
  for (int64_t q = 0; q < m && got < k; q++) {
    int64_t id = order[q];
    int ok = 1;
    for (int i = 0; i < n_slots; i++)
      if (taken[members[id * n_slots + i]]) ok = 0;
    if (!ok) continue;
    for (int i = 0; i < n_slots; i++) taken[members[id * n_slots + i]] = 1;
    set_ids[got++] = id;
  }
  free(order);
  free(members);
  free(taken);
  return got;
}
