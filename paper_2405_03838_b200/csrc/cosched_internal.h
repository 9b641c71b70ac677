// cosched_internal.h -- shared declarations of the CUDA path (kernels + C-ABI host code).
// Nothing here is shared with oracle/ (the test oracle); see DESIGN.md.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/cosched.h"

namespace cosched {

constexpr int kMaxCaps = 64;
constexpr int kMaxStates = 128;
constexpr int kMaxSlices = 128;
constexpr int kMaxSlots = 3;
// The tiled scorers walk the flattened config space c = state * n_caps + cap in
// stages of kStageCfg consecutive configs; each stage row is kStageRS floats
// (5 float4: odd, so 8 consecutive rows hit distinct shared-memory bank groups).
// 20 keeps the padding of the last stage small (294 configs -> 300, 882 -> 900).
constexpr int kStageCfg = 20;
constexpr int kStageRS = 20;

// Feasibility scale: the projection stores
// K*fl(U - alpha) and K*V with K = 2^80 (exact power-of-two scaling), each
// flushed to 0 when its magnitude is below K*2^-54 = 2^26 (a change of
// < 5.6e-17 in RPerf). Every nonzero operand is then a multiple of 8 (its ulp
// is >= 2^3), so every sum of them -- a fairness margin r'' = K*(RPerf - alpha)
// in the canonical order -- is 0, negative, or >= 8. The packed objective of
// the tiled scorers is a float < 4.0, so the masked key min3(obj, r0'', r1'')
// is the objective exactly when every margin is positive and <= 0 otherwise.
constexpr float kScale = 1208925819614629174706176.0f;       // 2^80
constexpr float kInvScale = 8.2718061255302767e-25f;         // 2^-80
constexpr float kFlushBelow = 67108864.0f;                   // 2^26 (scaled units)
constexpr float kClampAbs = 8.5070591730234616e37f;          // 2^126: sums of three stay finite
constexpr float kPadMargin = -3.4028234663852886e38f;        // -FLT_MAX: padding caps/jobs, infeasible

// Everything a scoring kernel needs about the search space, passed by value
// (kernel parameter space -> constant bank, read with c[0x0][...] operands).
struct SpaceParams {
  int32_t n_slots;
  int32_t n_states;
  int32_t n_slices;
  int32_t n_caps;
  int32_t np;                 // caps padded to a multiple of 4
  int32_t rs;                 // row stride of the projection rows (floats): np, or np+4 when np/4 is even,
                              // so 8 consecutive rows fall in distinct 16-byte shared-memory bank groups
  int64_t n_jobs_pad;         // jobs rounded up to a multiple of 64 (rows of every projection block)
  int32_t n_stages;           // ceil(n_cfg / kStageCfg)
  int32_t n_roles;            // n_slots * (n_slots + 1) operand roles of the gathered layout
  int32_t n_cfg;              // n_states * n_caps
  float alpha;
  int32_t search_mode;        // 0 exhaustive, 1 hill climbing from (hc_state, hc_cap) (R22)
  int32_t hc_state, hc_cap;
  float inv_ncaps;            // 1 / n_caps (FP32 division-free config decode in the tile ends)
  int64_t fast_lo[kMaxSlots], fast_hi[kMaxSlots];  // per slot: job rows of the gathered layout this
                                                    // rank's tiled scorer reads (gather skips the rest)
  float inv_p[kMaxCaps];      // per cap: fl(1/P) (Problem 2) or 1 (Problem 1)
  int16_t slice[kMaxStates][kMaxSlots];  // state -> slice per slot
};

// Exact re-scoring of the sets whose packed-objective choice is not provably
// within tau/2 of the FP32 argmax (device_common.cuh rescore_threshold): the
// tiled scorers' tile ends append the local index of such a set to `list`.
struct RescoreBuf {
  const unsigned* wmm = nullptr;  // [2 * kMaxSlots] per-slot share ranges (the quantum, hence the threshold)
  unsigned* list = nullptr;       // [cap] flagged local set indices (k = set id - first)
  unsigned* n = nullptr;          // [1] number flagged; > cap: every set below the threshold is re-scored
  unsigned cap = 0;
};

// Merge buffer of the pair scorer's stage-split tail (score_pairs.cu): one u64
// per pair of up to `tiles` 64 x 64 tiles.
struct PairMerge {
  unsigned long long* buf = nullptr;
  unsigned* cnt = nullptr;  // per split tile: stage-group units done (the last one resolves the tile)
  int64_t tiles = 0;
  // the handle's side streams: the partial-column units (side) and the
  // stage-split tail units (side2) run concurrently with the whole-tile launch,
  // taking the CTA slots it frees (forked after the gather, joined before the
  // re-scoring pass); null = everything on the caller's stream
  cudaStream_t side = nullptr, side2 = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_join2 = nullptr;
  unsigned epoch = 1;  // 24-bit step tag of the merge entries and tile counters (never 0)
};

// Device-side tables owned by a handle.
struct DeviceTables {
  float* coef_c = nullptr;  // [n_caps][n_slices][6]
  float* coef_d = nullptr;  // [n_caps][n_slices][3]
};

// Workspace layout (carved from the caller's buffer, all 256-byte aligned).
struct Workspace {
  float* ka = nullptr;              // [n_slices][n_jobs_pad][rs] = K*(U - alpha) (flushed/clamped); padding = -FLT_MAX
  float* kb = nullptr;              // [n_slices][n_jobs_pad][rs] = K*V (flushed/clamped);       padding = -FLT_MAX
  float* w = nullptr;               // [n_slots][n_states][n_jobs_pad][rs] throughput share of the job in
                                    //   slot i of state s at cap p, already divided by P (Problem 2):
                                    //   (U[s_i] + sum_{l != i} V[s_l]) * invP; padding = -1e30
  float* hj = nullptr;              // [n_jobs_pad][12] basis H1..H6, J1..J3 per queue position (k_validate)
  float* fast = nullptr;            // [n_roles][n_stages][n_jobs_pad][kStageRS] operands of the tiled scorers
                                    //   along the flattened config axis; the
                                    //   W roles hold fixed-point objective shares ("packed objective")
  unsigned* wmm = nullptr;          // [2 * kMaxSlots] per-slot min / max of w (order-preserving u32)
  unsigned long long* best_key = nullptr;  // [1] shard argmax key
  unsigned long long* err = nullptr;       // [1] first bad job: (pos << 8) | status, ~0 = none
  unsigned long long* job_key = nullptr;   // [n_jobs] greedy per-job best keys
  uint32_t* taken = nullptr;               // [n_jobs] greedy taken marks
  int64_t* alive = nullptr;                // [n_sets_local] greedy alive list
  int64_t* alive2 = nullptr;               // [n_sets_local]
  unsigned long long* picked = nullptr;    // [n_jobs] greedy picked keys
  int64_t* counters = nullptr;             // [16] device counters
  unsigned* hist = nullptr;                // [kHistBins] greedy objective histogram
  unsigned* mm = nullptr;                  // [2] min / max ord(obj)
  unsigned long long* gath = nullptr;      // [nranks * batch_cap] gathered keys (multi-rank)
  unsigned long long* gath_sorted = nullptr;
  void* sort_tmp = nullptr;
  size_t sort_tmp_bytes = 0;
  int64_t batch_cap = 0;                   // keys per rank per greedy batch
  unsigned long long* pipe_ring = nullptr; // greedy pipeline ring (greedy_pipe_ring_bytes)
  int* pipe_cnt = nullptr;                 // [kPipeSlots]
  int* pipe_ctl = nullptr;                 // [kPipeSlots + 4] ring flags, then next / done / stop
  unsigned long long* merge = nullptr;     // [merge_tiles][64 * 64] (PairMerge)
  int64_t merge_tiles = 0;
  unsigned long long* sel_flags = nullptr;  // [1024] k_select_free published tile counts (epoch-tagged)
  unsigned* merge_cnt = nullptr;            // [merge_tiles]: stage-group units done per split tile
  unsigned* rescore_list = nullptr;        // [rescore_cap] (RescoreBuf)
  unsigned* rescore_n = nullptr;           // [1]
  unsigned rescore_cap = 0;
  size_t bytes = 0;
};

constexpr int kHistLog2 = 14;
constexpr int kHistBins = 1 << kHistLog2;  // greedy objective histogram (per-block copy fits shared memory)
size_t workspace_layout(int64_t n_jobs, const SpaceParams& sp, int64_t n_sets_local, int nranks, char* base,
                        Workspace* ws);
// greedy.cu
void launch_obj_minmax(const float* obj, int64_t count, unsigned* mm, cudaStream_t st);
void launch_obj_hist(const float* obj, int64_t count, const unsigned* mm, int nbins, unsigned* hist, cudaStream_t st);
// Greedy-list keys (greedy.cu): ((ord(obj) - base) << 32) | (0xFFFFFFFF - low), low =
// (j1 << 16) | j0 for pairs of queues <= 65536 jobs (packed: the jobs decode with
// two shifts; colex order of (j1, j0) equals set-id order) else the set id. Orders
// exactly like the canonical packed key; a batch sorts only end_bit low bits.
struct GKeyFmt {
  int packed = 0;
  unsigned base = 0;
  int end_bit = 64;
};
GKeyFmt gkey_format(int n_slots, int64_t n_jobs, unsigned base, unsigned long long span_ord);
void launch_keys_in_range(int n_slots, const float* obj, int64_t first, int64_t count, const unsigned* mm, int nbins,
                          int bin_lo, int bin_hi, const uint32_t* taken_bits, unsigned long long* keys,
                          unsigned long long* n_keys, const GKeyFmt& fmt, cudaStream_t st);
// The same keys from the live rows only (free j1 / free pairs j1 < j2, over the free list it builds)
void launch_keys_live(int n_slots, const uint32_t* taken_bits, int64_t n_jobs, int32_t* free_list, int64_t* n_free_dev,
                      int64_t n_free, const float* obj, int64_t first, int64_t count, const unsigned* mm, int bin_lo,
                      int bin_hi, unsigned long long* keys, unsigned long long* n_keys, const GKeyFmt& fmt,
                      cudaStream_t st);
// [lo ord, hi ord) of histogram bins [bin_lo, bin_hi] given the objective range mm = (lo, hi)
void bin_range_ord(unsigned lo, unsigned hi, int bin_lo, int bin_hi, unsigned* u_lo, unsigned long long* width);
// greedy endgame: keys of every feasible set of free jobs (free list built on the device)
void launch_free_sets(int n_slots, const uint32_t* taken_bits, int64_t n_jobs, int32_t* free_list, int64_t* n_free_dev,
                      int64_t n_comb, const float* obj, int64_t first, int64_t count, unsigned long long* keys,
                      unsigned long long* n_keys, const GKeyFmt& fmt, cudaStream_t st);
size_t sort_temp_bytes(int64_t n);
size_t select_temp_bytes(int64_t n);
cudaError_t select_free_keys(int n_slots, void* temp, size_t temp_bytes, const unsigned long long* in,
                             unsigned long long* out, int64_t* n_out, int64_t n, const uint32_t* taken_bits,
                             const GKeyFmt& fmt, cudaStream_t st);
cudaError_t sort_keys_desc(void* temp, size_t temp_bytes, const unsigned long long* in, unsigned long long* out,
                           int64_t n, cudaStream_t st, int end_bit = 64);
// The sequential rule over a sorted list as a whole-GPU producer / consumer
// pipeline (one cooperative launch); ring / ring_cnt / pipe_ctl from the workspace
// (pipe_ctl: kPipeLag ring flags then 4 control words, reset by the launch).
cudaError_t launch_greedy_pipe(int n_slots, const unsigned long long* sorted, int64_t m, int64_t n_jobs,
                               uint32_t* taken_bits, unsigned long long* picks, int64_t* n_picks, int64_t k_max,
                               const GKeyFmt& fmt, unsigned long long* ring, int* ring_cnt, int* ring_flag, int* ctl,
                               cudaStream_t st);
size_t greedy_pipe_ring_bytes();
constexpr int kPipeSlots = 16;  // = kPipeLag in greedy.cu
// picks are written as canonical packed keys (cosched_pack_key); the list length is
// *m_dev when m_dev != NULL (a count produced on the device), else m
void scan_prof_report();  // COSCHED_SCAN_PROF builds: print and reset the scan phase counters
cudaError_t launch_greedy_scan(int n_slots, const unsigned long long* sorted, int64_t m, const int64_t* m_dev,
                               int64_t n_jobs, uint32_t* taken_bits, unsigned long long* picks, int64_t* n_picks,
                               int64_t k_max, const GKeyFmt& fmt, cudaStream_t st, int64_t* scanned = nullptr);
// greedy window select in one launch (greedy.cu k_select_free): the free keys of
// the n keys at in, in order, compacted at out, their number in *m_out; flags:
// kSelMaxTiles words zeroed once per allocation, epoch distinct per launch
cudaError_t launch_select_free(int n_slots, const unsigned long long* in, int64_t n, const uint32_t* taken,
                               unsigned long long* out, int64_t* m_out, unsigned long long* flags, unsigned epoch,
                               const GKeyFmt& fmt, const int64_t* n_picks, int64_t k_max, cudaStream_t st);
int select_tiles(int64_t n);
int64_t pad_jobs(int64_t n_jobs);
// node.cu
size_t node_workspace_bytes(int64_t n_gpus, int32_t n_caps, int32_t U, int32_t gpus_per_node);
int node_enqueue(const SpaceParams& sp, const float* ka, const float* kb, const float* w, const int64_t* set_ids_host,
                 int64_t n_gpus, int32_t gpus_per_node, int32_t U, float unit_w, const int32_t* u, int32_t objective,
                 void* workspace, int32_t* caps_host, int32_t* cfg_host, float* node_obj_host, cudaStream_t st);
// truth.cu
size_t truth_workspace_bytes(int64_t n_jobs, int64_t count);
int truth_enqueue(const cosched_truth_desc* d, const SpaceParams& sp, int objective, const int32_t* gpcs,
                  const int32_t* mem, const float* caps, const float* features, const int32_t* jobs, int64_t n_jobs,
                  int64_t first, int64_t count, const int32_t* prop_cfg, const cosched_eval_out* out, void* workspace,
                  double* sums_dev, cudaStream_t st);
// calib.cu
cosched_status fit_validate_desc(const cosched_fit_desc* d);
size_t fit_workspace_bytes(const cosched_fit_desc* d);
int fit_enqueue(const cosched_fit_desc* d, void* workspace, const cosched_fit_out* out, unsigned long long** err_dev,
                cudaStream_t st);

// ---- kernel launchers (defined in kernels.cu) ------------------------------------
void launch_validate(const float* features, int64_t n_rows, const int32_t* jobs, int64_t n_jobs,
                     unsigned long long* err, float* hj, cudaStream_t st);
void launch_project(const float* hj, int64_t n_jobs, const SpaceParams& sp, const DeviceTables& tb,
                    const unsigned long long* err, float* ka, float* kb, float* w, float* fast, unsigned* wmm,
                    bool with_kakb, cudaStream_t st, cudaEvent_t mid = nullptr);
// the ka / kb rows alone, after a launch_project without them
void launch_project_kakb(const float* hj, int64_t n_jobs, const SpaceParams& sp, const DeviceTables& tb,
                         const unsigned long long* err, float* ka, float* kb, unsigned* wmm, cudaStream_t st,
                         float* w_full = nullptr);
// Hill climbing for sets [first, first+count) (search_mode 1); adds the f evaluations to *evals.
int launch_score_hill(const SpaceParams& sp, int64_t n_jobs, const float* ka, const float* kb, const float* w,
                      int64_t first, int64_t count, float* obj, int32_t* cfg, unsigned long long* best_key,
                      unsigned long long* evals, const unsigned long long* err, cudaStream_t st);
// Scores sets [first, first+count) of the queue; writes obj/cfg (may be null) and atomically
// maxes the packed key into *best_key. Returns the number of kernels launched.
// variant 0: the generic one-thread-per-set kernel (reads ka / kb / w); variant 1: the
// tiled scorers (read the gathered layout and w) plus the exact re-scoring of the
// flagged sets (rb), when tiled_applicable(), else the generic kernel.
int launch_score(const SpaceParams& sp, int64_t n_jobs, const float* ka, const float* kb, const float* w,
                 const float* fast, int64_t first, int64_t count, float* obj, int32_t* cfg, unsigned long long* best_key,
                 const unsigned long long* err, int variant, cudaStream_t st, const RescoreBuf& rb = RescoreBuf(),
                 const PairMerge& merge = PairMerge());
// Whether the tiled scorer takes shard [first, first + count) of an n_jobs queue
// (whole colex columns / planes; pair queues below 32768 column tiles). The one
// place the tiled-or-generic decision is made: score_all projects ka / kb for
// the generic kernel exactly when this is false.
bool tiled_applicable(int n_slots, int64_t n_jobs, int64_t first, int64_t count);
// Per-device, thread-safe opt-in to more than 48 KB of dynamic shared memory
// for `func` (a __global__ function), done once per (function, device, size);
// returns the CUDA error of the opt-in. num_sms(): SMs of the current device.
cudaError_t smem_optin(const void* func, size_t bytes);
int num_sms();

// Programmatic dependent launch (PDL) along the step's kernel chain (validate ->
// project -> gather -> scorer -> re-score -> best detail): a kernel launched with
// launch_pdl may start while its predecessor on the stream drains; it runs its
// prologue (constant tables into shared memory, barrier init) and then waits in
// pdl_wait() until the predecessor has completed and its writes are visible.
// Every such kernel calls pdl_wait() before touching anything an earlier kernel
// of the stream writes, and pdl_launch_dependents() only after it (so at most
// two adjacent kernels overlap). Both are no-ops for a normal launch.
// COSCHED_PDL=0 turns the attribute off (A/B timing).
bool pdl_enabled();
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}
// Step start: err = ~0 (valid), best_key = 0, rescore count = 0, wmm = empty ranges.
void launch_step_init(unsigned long long* err, unsigned long long* best_key, unsigned* rescore_n, unsigned* wmm,
                      cudaStream_t st);
void launch_exact_alloc(int n_slots, int64_t n_jobs, const float* set_obj, int64_t n_match,
                        unsigned long long* best_key, cudaStream_t st);
void launch_exact_unrank(int n_slots, int64_t n_jobs, const unsigned long long* best_key, int64_t* set_ids,
                         cudaStream_t st);
// greedy (locally dominant rounds)
void launch_greedy_init(int n_slots, int64_t n_jobs, const float* obj, int64_t first, int64_t count,
                        int64_t* alive, int64_t* n_alive, cudaStream_t st);
void launch_greedy_propose(int n_slots, int64_t n_jobs, const float* obj, int64_t first, const int64_t* alive,
                           int64_t n_alive, const uint32_t* taken, unsigned long long* job_key, cudaStream_t st);
void launch_greedy_select(int n_slots, int64_t n_jobs, const float* obj, int64_t first, const int64_t* alive,
                          int64_t n_alive, const unsigned long long* job_key, uint32_t* taken,
                          unsigned long long* picked, int64_t* n_picked, cudaStream_t st);
void launch_greedy_mark(int n_slots, const unsigned long long* picked, int64_t from, int64_t to, uint32_t* taken,
                        cudaStream_t st);
void launch_sort_keys_desc(const unsigned long long* keys, int64_t n, unsigned long long* sorted, cudaStream_t st);
void launch_sets_detail(const SpaceParams& sp, const float* ka, const float* kb, const float* w, const int64_t* set_ids,
                        int64_t n,
                        float* out /* [n][4 + kMaxSlots] */, cudaStream_t st);
// detail row of the set named by the device-resident packed key (best set)
void launch_best_detail(const SpaceParams& sp, const float* ka, const float* kb, const float* w,
                        const unsigned long long* key, const unsigned long long* err, unsigned long long* host_out,
                        const float* hj, const DeviceTables* tb, cudaStream_t st);
void launch_greedy_compact(int n_slots, int64_t n_jobs, const int64_t* alive, int64_t n_alive,
                           const uint32_t* taken, int64_t* alive_out, int64_t* n_out, cudaStream_t st);
void launch_greedy_pairs_propose(const float* obj, int64_t first, int64_t c0, int64_t c1, const uint32_t* taken,
                                 unsigned long long* job_key, cudaStream_t st);
void launch_greedy_pairs_select(const unsigned long long* job_key, int64_t n_jobs, unsigned long long* picked,
                                int64_t* n_picked, cudaStream_t st);
void launch_fill_u64(unsigned long long* p, unsigned long long v, int64_t n, cudaStream_t st);
void launch_fill_u32(uint32_t* p, uint32_t v, int64_t n, cudaStream_t st);

// host-side helpers shared by the API (no CUDA)
int64_t n_sets(int64_t n, int k);
// tiles of the triple scorer's planes j2' < j2 (score_triples.cu): the work
// measure the triple shards are balanced on
int64_t triple_tiles_before(int64_t j2);
uint32_t ord_float(float f);
float unord_float(uint32_t o);

}  // namespace cosched
