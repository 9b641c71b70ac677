// api.cu -- host side of the C-ABI declared in include/cosched.h.
//
// Validation, shard ranges, workspace carving, stream ordering and the NCCL
// communicator. Every arithmetic step of the method runs in the kernels of
// kernels.cu / score_pairs.cu; this file only moves arguments, launches and
// reads back the few bytes of each result.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nvtx3/nvToolsExt.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <cmath>
#include <map>
#include <mutex>
#include <numeric>
#include <string>
#include <vector>

#include "cosched_internal.h"

using namespace cosched;

// ---------------------------------------------------------------------------
// NCCL, loaded at run time (the copy torch already loaded when present).
namespace {
typedef struct ncclComm* ncclComm_t;
typedef struct {
  char internal[128];
} ncclUniqueId;
enum { kNcclUint32 = 3, kNcclUint64 = 5, kNcclFloat64 = 8, kNcclSum = 0, kNcclMax = 2, kNcclMin = 3 };
struct NcclApi {
  bool tried = false;
  void* lib = nullptr;
  int (*getUniqueId)(ncclUniqueId*) = nullptr;
  int (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  int (*allReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  int (*commDestroy)(ncclComm_t) = nullptr;
  int (*allGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*getErrorString)(int) = nullptr;
};
NcclApi g_nccl;

bool nccl_load(std::string* why) {
  static std::mutex mu;  // handles of one process may bootstrap from several threads
  std::lock_guard<std::mutex> lk(mu);
  if (!g_nccl.tried) {
    g_nccl.tried = true;
    // COSCHED_NCCL_LIB: another library with the same six entry points (the
    // test-only in-process loopback, tests/loopback/, runs W ranks as W threads
    // on one GPU); read once, at the first communicator use of the process
    const char* alt = getenv("COSCHED_NCCL_LIB");
    void* h = nullptr;
    if (alt && alt[0]) {
      h = dlopen(alt, RTLD_NOW | RTLD_LOCAL);
    } else {
      h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
      if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
      if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    }
    if (h) {
      g_nccl.getUniqueId = (int (*)(ncclUniqueId*))dlsym(h, "ncclGetUniqueId");
      g_nccl.commInitRank = (int (*)(ncclComm_t*, int, ncclUniqueId, int))dlsym(h, "ncclCommInitRank");
      g_nccl.allReduce = (int (*)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t))dlsym(h, "ncclAllReduce");
      g_nccl.commDestroy = (int (*)(ncclComm_t))dlsym(h, "ncclCommDestroy");
      g_nccl.allGather = (int (*)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t))dlsym(h, "ncclAllGather");
      g_nccl.getErrorString = (const char* (*)(int))dlsym(h, "ncclGetErrorString");
      if (g_nccl.getUniqueId && g_nccl.commInitRank && g_nccl.allReduce && g_nccl.commDestroy && g_nccl.allGather)
        g_nccl.lib = h;
    }
  }
  if (!g_nccl.lib && why) *why = "libnccl.so.2 not loadable";
  return g_nccl.lib != nullptr;
}

thread_local std::string g_create_error;

// NVTX range around each C-ABI entry point (header-only NVTX v3: a no-op
// unless a profiler injects itself), so Nsight timelines show the API calls
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};
}  // namespace

struct cosched_ctx {
  int device = 0;
  int n_slots = 2;
  int objective = 2;
  SpaceParams sp{};
  DeviceTables tb{};
  std::string err;
  int variant = 1;
  int64_t launches = 0;
  // small scratch owned by the handle (exact allocation, details)
  float* d_small_obj = nullptr;      // [kSmallSets]
  int32_t* d_small_cfg = nullptr;    // [kSmallSets]
  unsigned long long* d_small_key = nullptr;  // [2]
  int64_t* d_small_ids = nullptr;    // [64]
  float* d_detail = nullptr;         // [kDetailRows][8]
  int64_t* d_detail_ids = nullptr;   // [kDetailRows]
  unsigned long long* h_pinned = nullptr;  // [8] pinned host readback
  // last score_all
  bool scored = false;
  bool kakb_valid = false;    // ka / kb rows (and every w row) of this step's projection present (else ensure_kakb)
  bool best_pending = false;  // cosched_best_set_begin enqueued, _end not yet called
  bool step_timed = false;    // ev[3] recorded after this score_all's best-set detail kernel
  bool timing = false;        // cosched_set_timing: record the prep / score split events
  unsigned merge_epoch = 0;   // step tag of the pair scorer's tail-merge area (PairMerge::epoch)
  const void* merge_init = nullptr;  // workspace merge area zeroed once (its entries carry step tags after)
  bool split_timed = false;   // this score_all recorded them
  int64_t n_jobs = 0;
  int64_t first = 0, n_sets = 0;
  Workspace ws{};
  float* out_obj = nullptr;
  int32_t* out_cfg = nullptr;
  cudaStream_t stream = nullptr;
  // communicator
  ncclComm_t comm = nullptr;
  int rank = 0, nranks = 1;
  int view_nranks = 1;  // shard view without comm (tests)
  int64_t greedy_rounds = 0;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  cudaEvent_t evp[3] = {nullptr, nullptr, nullptr};  // COSCHED_PREP_EVENTS: after step init, validate, projection
  cudaStream_t side = nullptr;                 // partial-column units of the pair scorer (PairMerge)
  cudaStream_t side2 = nullptr;                // its stage-split tail units
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_join2 = nullptr;
  // host copies of the table (ground-truth evaluation)
  std::vector<int32_t> h_gpcs, h_mem;
  std::vector<float> h_caps;
  double* d_sums = nullptr;  // [4] ground-truth summary sums
  static constexpr int kSmallSets = 512;
  static constexpr int kDetailRows = 8192;
};

namespace cosched {

int64_t n_sets(int64_t n, int k) {
  if (n < k || k < 1) return 0;
  if (k == 1) return n;
  if (k == 2) return n * (n - 1) / 2;
  return n * (n - 1) / 2 * (n - 2) / 3;  // exact: n(n-1)/2 * (n-2) is divisible by 3
}

uint32_t ord_float(float f) {
  uint32_t b;
  memcpy(&b, &f, 4);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

float unord_float(uint32_t o) {
  uint32_t b = (o & 0x80000000u) ? (o & 0x7FFFFFFFu) : ~o;
  float f;
  memcpy(&f, &b, 4);
  return f;
}

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

}  // namespace cosched
// Pair shards: whole 64-column blocks of the triangle (the pair scorer's tile
// columns; no shard boundary inside a block, so no partial-column units except
// the queue's ragged last block), chosen by a DP over block boundaries that
// minimises the largest modelled scorer time. The model, in
// rounds of the persistent launch on a B200 (148 SMs x 2 CTAs = 296 slots):
// a rank's whole tiles take floor(tiles / 296) rounds, its last partial round
// of R tiles is split into q stage groups (score_pairs.cu) costing
// ceil(R q / 296) x (ceil(16 / q) + 0.3 [q > 1]) / 16 rounds, and the ragged
// last block's single-row-group units 0.47 of a tile each. A pure function of
// (n_jobs, nranks), identical on every rank; cached.
static const std::vector<int64_t>& pair_block_bounds(int64_t n_jobs, int nranks) {
  static std::mutex mu;
  static std::map<std::pair<int64_t, int>, std::vector<int64_t>> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find({n_jobs, nranks});
  if (it != cache.end()) return it->second;
  constexpr double kSlots = 296.0, kStages = 16.0, kUnit = 0.3, kPartial = 0.47;
  const int64_t nb = (n_jobs + 63) / 64;
  auto tail = [&](int64_t R) {
    if (R <= 0) return 0.0;
    double best = 1e30;
    for (int q = 1; q <= (int)kStages; q++) {
      const double len = std::ceil(R * q / kSlots) * (std::ceil(kStages / q) + (q > 1 ? kUnit : 0.0)) / kStages;
      best = std::min(best, len);
    }
    return best;
  };
  auto rank_time = [&](int64_t B0, int64_t B1) {
    const int64_t tiles = B1 * (B1 + 1) / 2 - B0 * (B0 + 1) / 2;
    const int64_t part = (B1 == nb && n_jobs % 64) ? B1 : 0;  // the ragged block's tiles (as units)
    const int64_t full = tiles - part, rounds = full > (int64_t)kSlots ? full / (int64_t)kSlots : 0;
    return (double)rounds + tail(full - rounds * (int64_t)kSlots) + part * kPartial / kSlots;
  };
  std::vector<int64_t> b(nranks + 1, 0);
  if (nranks == 1 || nb <= 1) {
    for (int r = 1; r <= nranks; r++) b[r] = nb;
  } else {
    // best[r][B]: smallest max time of blocks [0, B) over r ranks (rank order = block order)
    std::vector<std::vector<double>> best(nranks + 1, std::vector<double>(nb + 1, 1e300));
    std::vector<std::vector<int64_t>> arg(nranks + 1, std::vector<int64_t>(nb + 1, 0));
    best[0][0] = 0.0;
    for (int r = 1; r <= nranks; r++)
      for (int64_t B = 0; B <= nb; B++)
        for (int64_t P = 0; P <= B; P++) {
          if (best[r - 1][P] >= 1e300) continue;
          const double v = std::max(best[r - 1][P], rank_time(P, B));
          if (v < best[r][B] - 1e-12) {
            best[r][B] = v;
            arg[r][B] = P;
          }
        }
    b[nranks] = nb;
    for (int r = nranks; r > 0; r--) b[r - 1] = arg[r][b[r]];
  }
  for (auto& x : b) x = std::min<int64_t>(64 * x, n_jobs);
  return cache.emplace(std::make_pair(n_jobs, nranks), std::move(b)).first->second;
}

// Contiguous whole-column shards. Pairs: pair_block_bounds. Triples: balanced
// on the triple scorer's tiles (its time per plane follows the tile count, the
// small planes' diagonal and ragged tiles included), b_r the smallest b with
// tiles_before(b) >= ceil(r * tiles_before(n_jobs) / W). Solo: balanced on sets.
static void shard_bounds(int64_t n_jobs, int k, int rank, int nranks, int64_t* first, int64_t* count) {
  if (k == 2) {
    const std::vector<int64_t>& b = pair_block_bounds(n_jobs, nranks);
    *first = cosched::n_sets(b[rank], 2);
    *count = cosched::n_sets(b[rank + 1], 2) - *first;
    return;
  }
  auto cost = [&](int64_t b) -> int64_t {
    return k == 3 ? cosched::triple_tiles_before(b) : cosched::n_sets(b, k);
  };
  const int64_t total = cost(n_jobs);
  auto boundary = [&](int r) -> int64_t {  // smallest b with cost(b) >= ceil(r * total / W)
    if (r <= 0) return 0;
    if (r >= nranks) return n_jobs;
    __int128 num = (__int128)r * total;
    int64_t target = (int64_t)((num + nranks - 1) / nranks);
    int64_t lo = 0, hi = n_jobs;
    while (lo < hi) {
      int64_t mid = (lo + hi) / 2;
      if (cost(mid) >= target) hi = mid;
      else lo = mid + 1;
    }
    return lo;
  };
  int64_t b0 = boundary(rank), b1 = boundary(rank + 1);
  *first = cosched::n_sets(b0, k);
  *count = cosched::n_sets(b1, k) - *first;
}

namespace cosched {

int64_t pad_jobs(int64_t n_jobs) { return (n_jobs + 63) / 64 * 64; }

size_t workspace_layout(int64_t n_jobs, const SpaceParams& sp, int64_t n_sets_local, int nranks, char* base,
                        Workspace* ws) {
  const int32_t n_slices = sp.n_slices, rs = sp.rs, n_slots = sp.n_slots, n_states = sp.n_states;
  size_t off = 0;
  auto take = [&](size_t bytes) -> char* {
    char* p = base ? base + off : nullptr;
    off += align256(bytes);
    return p;
  };
  const size_t jp = (size_t)pad_jobs(n_jobs);
  size_t proj = jp * n_slices * rs * sizeof(float);
  Workspace w;
  w.ka = (float*)take(proj);
  w.kb = (float*)take(proj);
  w.w = (float*)take(jp * n_slots * n_states * rs * sizeof(float));
  w.hj = (float*)take(jp * 12 * sizeof(float));
  w.fast = (float*)take(jp * sp.n_roles * sp.n_stages * kStageRS * sizeof(float));
  w.wmm = (unsigned*)take(2 * kMaxSlots * sizeof(unsigned));
  w.best_key = (unsigned long long*)take(8);
  w.err = (unsigned long long*)take(8);
  w.counters = (int64_t*)take(16 * 8);  // [8]: keys through the greedy scan (instrumentation)
  w.job_key = (unsigned long long*)take((size_t)n_jobs * 8);
  w.taken = (uint32_t*)take((size_t)n_jobs * 4);
  w.picked = (unsigned long long*)take((size_t)n_jobs * 8 + 8);
  // largest shard of any rank (the greedy's all-gathered batches are padded to it)
  int64_t largest = n_sets_local;
  for (int r = 0; r < nranks; r++) {
    int64_t f, c;
    shard_bounds(n_jobs, n_slots, r, nranks, &f, &c);
    largest = std::max(largest, c);
  }
  w.alive = (int64_t*)take((size_t)largest * 8 + 8);
  w.alive2 = (int64_t*)take((size_t)largest * 8 + 8);
  w.hist = (unsigned*)take((size_t)kHistBins * 4);
  w.mm = (unsigned*)take(16);
  // nranks = 0: no communicator; else the greedy all-gathers per-rank batches.
  // The per-rank batch capacity must be the same on every rank (the switch to
  // the fallback rounds is taken by all ranks or none): it is bounded by the
  // largest shard of any rank, which every rank computes alike.
  // COSCHED_GREEDY_BATCH_CAP (testing knob): a smaller per-rank batch capacity, which
  // forces the locally-dominant-rounds fallback of the multi-rank greedy
  int64_t cap_max = (int64_t)16 << 20;
  if (const char* e = getenv("COSCHED_GREEDY_BATCH_CAP")) cap_max = std::max<int64_t>(1, atoll(e));
  // CUB's sort / select take int item counts: a gathered batch (cap x nranks) stays below 2^30
  cap_max = std::min<int64_t>(cap_max, ((int64_t)1 << 30) / std::max(nranks, 1));
  const int64_t cap = nranks > 0 ? std::min<int64_t>(largest, cap_max) : n_sets_local;
  w.batch_cap = cap;
  const int64_t gathered = nranks > 0 ? cap * nranks : 0;
  w.gath = (unsigned long long*)take((size_t)gathered * 8 + 8);
  w.gath_sorted = (unsigned long long*)take((size_t)gathered * 8 + 8);
  // the longest list a sort / select sees: a batch (<= 64 M keys, greedy_sorted_scan) or a
  // gathered batch -- never the whole shard, which may exceed CUB's int item counts
  const int64_t list_max = std::max<int64_t>(std::min<int64_t>(nranks > 0 ? gathered : n_sets_local, (int64_t)1 << 30), 1);
  w.sort_tmp_bytes = std::max(sort_temp_bytes(list_max), select_temp_bytes(list_max));
  w.sort_tmp = take(w.sort_tmp_bytes);
  // exact re-scoring list of the tiled scorers: normally empty; an
  // overflow re-scores every flagged-range set instead, so the capacity is a
  // memory bound, not a correctness one
  int64_t rcap = (int64_t)1 << 20;
  if (const char* e = getenv("COSCHED_RESCORE_CAP")) rcap = std::max<int64_t>(0, atoll(e));  // testing knob: overflow path
  w.pipe_ring = (unsigned long long*)take(greedy_pipe_ring_bytes());
  w.pipe_cnt = (int*)take(sizeof(int) * kPipeSlots);
  w.pipe_ctl = (int*)take(sizeof(int) * (kPipeSlots + 4));
  w.rescore_cap = (unsigned)std::min<int64_t>(std::max<int64_t>(n_sets_local, 1), rcap);
  w.rescore_list = (unsigned*)take((size_t)std::max<unsigned>(w.rescore_cap, 1u) * 4);
  // the pair scorer's stage-split tail: at most one CTA-slot round of tiles
  // (2 resident CTAs per SM), 32 KB each (pairs only)
  w.merge_tiles = n_slots == 2 ? 2 * (int64_t)num_sms() : 0;
  w.merge = (unsigned long long*)take((size_t)w.merge_tiles * 64 * 64 * 8);
  w.merge_cnt = (unsigned*)take((size_t)std::max<int64_t>(w.merge_tiles, 1) * 4);  // finished units per split tile
  w.sel_flags = (unsigned long long*)take(1024 * 8);  // k_select_free tiles: windows up to 4 M keys
  w.rescore_n = (unsigned*)take(8);
  w.bytes = off;
  if (ws) *ws = w;
  return off;
}

}  // namespace cosched

// ---------------------------------------------------------------------------
static cosched_status fail(cosched_t h, cosched_status st, const std::string& msg) {
  if (h) h->err = msg;
  return st;
}

static cosched_status cuda_fail(cosched_t h, cudaError_t e, const char* where) {
  return fail(h, COSCHED_E_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define CK(call)                                   \
  do {                                             \
    cudaError_t e_ = (call);                       \
    if (e_ != cudaSuccess) return cuda_fail(h, e_, #call); \
  } while (0)

static cosched_status validate_desc(const cosched_desc* d, std::string* msg) {
  char buf[256];
  if (!d || d->n_slots < 1 || d->n_slots > kMaxSlots || d->n_states < 1 || d->n_states > kMaxStates ||
      d->n_slices < 1 || d->n_slices > 32767 || d->n_caps < 1 || d->n_caps > kMaxCaps || !d->state_gpcs ||
      !d->state_mem || !d->state_slice || !d->caps_w || !d->coef_c || !d->coef_d) {
    *msg = "bad sizes (n_slots 1..3, n_states 1..128, n_caps 1..64) or null table";
    return COSCHED_E_ARG;
  }
  if (d->objective != 1 && d->objective != 2) {
    *msg = "objective must be 1 or 2";
    return COSCHED_E_ARG;
  }
  if (!(d->alpha >= 0.0f) || isinf(d->alpha)) {
    *msg = "alpha must be finite and >= 0";
    return COSCHED_E_ARG;
  }
  for (int s = 0; s < d->n_states; s++) {
    long sum = 0;
    for (int i = 0; i < d->n_slots; i++) {
      int g = d->state_gpcs[s * d->n_slots + i];
      if (g < 1) {
        snprintf(buf, sizeof buf, "state %d slot %d: %d GPCs < 1", s, i, g);
        *msg = buf;
        return COSCHED_E_INVALID_ALLOCATION;
      }
      sum += g;
    }
    if (sum != d->gpcs_total) {
      snprintf(buf, sizeof buf, "state %d: GPCs sum to %ld, not %d", s, sum, d->gpcs_total);
      *msg = buf;
      return COSCHED_E_INVALID_ALLOCATION;
    }
    if (d->state_mem[s] != 0 && d->state_mem[s] != 1) {
      snprintf(buf, sizeof buf, "state %d: memory option %d", s, d->state_mem[s]);
      *msg = buf;
      return COSCHED_E_INVALID_ALLOCATION;
    }
  }
  for (int c = 0; c < d->n_caps; c++) {
    float w = d->caps_w[c];
    if (!(w > 0.0f) || isinf(w) || (c > 0 && !(w > d->caps_w[c - 1]))) {
      snprintf(buf, sizeof buf, "cap %d: %g W not positive / strictly ascending", c, (double)w);
      *msg = buf;
      return COSCHED_E_INVALID_ALLOCATION;
    }
  }
  for (int s = 0; s < d->n_states; s++)
    for (int i = 0; i < d->n_slots; i++) {
      int sl = d->state_slice[s * d->n_slots + i];
      if (sl < 0 || sl >= d->n_slices) {
        snprintf(buf, sizeof buf, "state %d slot %d: slice %d not in coefficient table", s, i, sl);
        *msg = buf;
        return COSCHED_E_UNKNOWN_KEY;
      }
    }
  for (long t = 0; t < (long)d->n_caps * d->n_slices * 6; t++)
    if (!isfinite(d->coef_c[t])) {
      *msg = "non-finite C coefficient";
      return COSCHED_E_ARG;
    }
  for (long t = 0; t < (long)d->n_caps * d->n_slices * 3; t++)
    if (!isfinite(d->coef_d[t])) {
      *msg = "non-finite D coefficient";
      return COSCHED_E_ARG;
    }
  return COSCHED_OK;
}

extern "C" {

const char* cosched_last_create_error(void) { return g_create_error.c_str(); }

cosched_status cosched_create(const cosched_desc* d, int cuda_device, cosched_t* out_handle) {
  g_create_error.clear();
  if (!out_handle) {
    g_create_error = "null out_handle";
    return COSCHED_E_ARG;
  }
  *out_handle = nullptr;
  std::string msg;
  cosched_status st = validate_desc(d, &msg);
  if (st != COSCHED_OK) {
    g_create_error = msg;
    return st;
  }
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev <= 0 || cuda_device < 0 || cuda_device >= ndev) {
    g_create_error = std::string("no usable CUDA device: ") + (e != cudaSuccess ? cudaGetErrorString(e) : "index out of range");
    return COSCHED_E_CUDA;
  }
  cosched_ctx* h = new cosched_ctx();
  h->device = cuda_device;
  h->n_slots = d->n_slots;
  h->objective = d->objective;
  h->h_gpcs.assign(d->state_gpcs, d->state_gpcs + (size_t)d->n_states * d->n_slots);
  h->h_mem.assign(d->state_mem, d->state_mem + d->n_states);
  h->h_caps.assign(d->caps_w, d->caps_w + d->n_caps);
  SpaceParams& sp = h->sp;
  sp.n_slots = d->n_slots;
  sp.n_states = d->n_states;
  sp.n_slices = d->n_slices;
  sp.n_caps = d->n_caps;
  sp.np = (d->n_caps + 3) & ~3;
  sp.rs = ((sp.np >> 2) & 1) ? sp.np : sp.np + 4;
  sp.n_jobs_pad = 0;
  sp.inv_ncaps = 1.0f / (float)d->n_caps;
  sp.search_mode = 0;  // exhaustive
  sp.hc_state = sp.hc_cap = 0;

  sp.n_cfg = d->n_states * d->n_caps;
  sp.n_stages = (sp.n_cfg + kStageCfg - 1) / kStageCfg;
  sp.n_roles = sp.n_slots * (sp.n_slots + 1);
  sp.alpha = d->alpha;
  for (int p = 0; p < d->n_caps; p++) {
    float inv = d->objective == 2 ? 1.0f / d->caps_w[p] : 1.0f;
    sp.inv_p[p] = inv;
  }
  for (int s = 0; s < d->n_states; s++)
    for (int i = 0; i < d->n_slots; i++) sp.slice[s][i] = (int16_t)d->state_slice[s * d->n_slots + i];
  const char* v = getenv("COSCHED_PAIR_KERNEL");
  if (v && !strcmp(v, "generic")) h->variant = 0;

  DeviceGuard g(cuda_device);
  size_t nc = (size_t)d->n_caps * d->n_slices;
  bool ok = cudaMalloc(&h->tb.coef_c, nc * 6 * 4) == cudaSuccess &&
            cudaMalloc(&h->tb.coef_d, nc * 3 * 4) == cudaSuccess &&
            cudaMalloc(&h->d_small_obj, cosched_ctx::kSmallSets * 4) == cudaSuccess &&
            cudaMalloc(&h->d_small_cfg, cosched_ctx::kSmallSets * 4) == cudaSuccess &&
            cudaMalloc(&h->d_small_key, 2 * 8) == cudaSuccess &&
            cudaMalloc(&h->d_small_ids, 64 * 8) == cudaSuccess &&
            cudaMalloc(&h->d_detail, (size_t)cosched_ctx::kDetailRows * 8 * 4) == cudaSuccess &&
            cudaMalloc(&h->d_detail_ids, (size_t)cosched_ctx::kDetailRows * 8) == cudaSuccess &&
            cudaMallocHost(&h->h_pinned, 8 * 8) == cudaSuccess && cudaMalloc(&h->d_sums, 4 * 8) == cudaSuccess &&
            cudaEventCreate(&h->ev[0]) == cudaSuccess && cudaEventCreate(&h->ev[1]) == cudaSuccess &&
            cudaEventCreate(&h->ev[2]) == cudaSuccess && cudaEventCreate(&h->ev[3]) == cudaSuccess &&
            cudaStreamCreateWithFlags(&h->side, cudaStreamNonBlocking) == cudaSuccess &&
            cudaStreamCreateWithFlags(&h->side2, cudaStreamNonBlocking) == cudaSuccess &&
            cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming) == cudaSuccess &&
            cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming) == cudaSuccess &&
            cudaEventCreateWithFlags(&h->ev_join2, cudaEventDisableTiming) == cudaSuccess &&
            cudaMemcpy(h->tb.coef_c, d->coef_c, nc * 6 * 4, cudaMemcpyHostToDevice) == cudaSuccess &&
            cudaMemcpy(h->tb.coef_d, d->coef_d, nc * 3 * 4, cudaMemcpyHostToDevice) == cudaSuccess;
  if (!ok) {
    g_create_error = std::string("CUDA allocation/copy failed: ") + cudaGetErrorString(cudaGetLastError());
    cosched_destroy(h);
    return COSCHED_E_CUDA;
  }
  *out_handle = h;
  return COSCHED_OK;
}

void cosched_destroy(cosched_t h) {
  if (!h) return;
  {
    DeviceGuard g(h->device);
    if (h->comm && g_nccl.commDestroy) g_nccl.commDestroy(h->comm);
    cudaFree(h->tb.coef_c);
    cudaFree(h->tb.coef_d);
    cudaFree(h->d_small_obj);
    cudaFree(h->d_small_cfg);
    cudaFree(h->d_small_key);
    cudaFree(h->d_small_ids);
    cudaFree(h->d_detail);
    cudaFree(h->d_detail_ids);
    cudaFree(h->d_sums);
    if (h->h_pinned) cudaFreeHost(h->h_pinned);
    for (int i = 0; i < 4; i++)
      if (h->ev[i]) cudaEventDestroy(h->ev[i]);
    for (auto& e : h->evp)
      if (e) cudaEventDestroy(e);
    if (h->ev_fork) cudaEventDestroy(h->ev_fork);
    if (h->ev_join) cudaEventDestroy(h->ev_join);
    if (h->ev_join2) cudaEventDestroy(h->ev_join2);
    if (h->side) cudaStreamDestroy(h->side);
    if (h->side2) cudaStreamDestroy(h->side2);
  }
  delete h;
}

const char* cosched_last_error(cosched_t h) { return h ? h->err.c_str() : g_create_error.c_str(); }

int64_t cosched_kernel_launches(cosched_t h) { return h ? h->launches : 0; }

int64_t cosched_last_greedy_rounds(cosched_t h) { return h ? h->greedy_rounds : 0; }

cosched_status cosched_last_rescored(cosched_t h, int64_t* n_rescored) {
  if (!h || !n_rescored) return fail(h, COSCHED_E_ARG, "null argument");
  if (!h->scored) return fail(h, COSCHED_E_STATE, "call cosched_score_all first");
  DeviceGuard g(h->device);
  unsigned v = 0;
  CK(cudaMemcpyAsync(&v, h->ws.rescore_n, 4, cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  *n_rescored = (int64_t)v;
  return COSCHED_OK;
}

cosched_status cosched_set_variant(cosched_t h, int variant) {
  if (!h || variant < 0 || variant > 1) return COSCHED_E_ARG;
  h->variant = variant;
  return COSCHED_OK;
}

cosched_status cosched_set_search(cosched_t h, int mode, int32_t start_state, int32_t start_cap) {
  if (!h) return COSCHED_E_ARG;
  if (mode != 0 && mode != 1) return fail(h, COSCHED_E_ARG, "search mode must be 0 (exhaustive) or 1 (hill climb)");
  if (mode == 1 && (start_state < 0 || start_state >= h->sp.n_states || start_cap < 0 || start_cap >= h->sp.n_caps))
    return fail(h, COSCHED_E_ARG, "hill-climb start outside the (state, cap) grid");
  h->sp.search_mode = mode;
  h->sp.hc_state = mode ? start_state : 0;
  h->sp.hc_cap = mode ? start_cap : 0;
  h->scored = false;  // results of the other mode are stale
  return COSCHED_OK;
}

cosched_status cosched_last_search_evals(cosched_t h, int64_t* evals) {
  if (!h || !evals) return COSCHED_E_ARG;
  if (!h->scored) return fail(h, COSCHED_E_STATE, "no cosched_score_all yet");
  if (h->sp.search_mode == 0) {
    *evals = h->n_sets * (int64_t)h->sp.n_cfg;
    return COSCHED_OK;
  }
  unsigned long long v = 0;
  if (cudaMemcpyAsync(&v, h->ws.counters + 7, 8, cudaMemcpyDeviceToHost, h->stream) != cudaSuccess ||
      cudaStreamSynchronize(h->stream) != cudaSuccess)
    return cuda_fail(h, cudaGetLastError(), "last_search_evals");
  *evals = (int64_t)v;
  return COSCHED_OK;
}

// ---- host-only helpers ------------------------------------------------------
int64_t cosched_n_sets(int64_t n_jobs, int32_t n_slots) { return cosched::n_sets(n_jobs, n_slots); }

cosched_status cosched_unrank(int64_t n_jobs, int32_t n_slots, int64_t set_id, int64_t* pos) {
  if (!pos || n_slots < 1 || n_slots > 3 || set_id < 0 || set_id >= cosched::n_sets(n_jobs, n_slots))
    return COSCHED_E_ARG;
  int64_t rest = set_id;
  for (int i = n_slots - 1; i >= 0; i--) {
    // largest t with C(t, i+1) <= rest: binary search over [i, n_jobs)
    int64_t lo = i, hi = n_jobs - 1;
    while (lo < hi) {
      int64_t mid = (lo + hi + 1) / 2;
      if (cosched::n_sets(mid, i + 1) <= rest) lo = mid;
      else hi = mid - 1;
    }
    pos[i] = lo;
    rest -= cosched::n_sets(lo, i + 1);
  }
  return COSCHED_OK;
}

uint64_t cosched_pack_key(float obj, int64_t set_id) {
  return ((uint64_t)ord_float(obj) << 32) | (0xFFFFFFFFull - (uint64_t)(uint32_t)set_id);
}

void cosched_unpack_key(uint64_t key, float* obj, int64_t* set_id) {
  if (key == 0) {
    if (obj) *obj = -INFINITY;
    if (set_id) *set_id = -1;
    return;
  }
  if (obj) *obj = unord_float((uint32_t)(key >> 32));
  if (set_id) *set_id = (int64_t)(0xFFFFFFFFull - (key & 0xFFFFFFFFull));
}

cosched_status cosched_shard_range(cosched_t h, int64_t n_jobs, int64_t* first_set, int64_t* n_sets_out) {
  if (!h || !first_set || !n_sets_out || n_jobs < 0) return fail(h, COSCHED_E_ARG, "bad shard_range arguments");
  shard_bounds(n_jobs, h->n_slots, h->rank, h->comm ? h->nranks : h->view_nranks, first_set, n_sets_out);
  return COSCHED_OK;
}

cosched_status cosched_shard_range_for(int64_t n_jobs, int32_t n_slots, int32_t rank, int32_t nranks,
                                       int64_t* first_set, int64_t* n_sets_out) {
  if (!first_set || !n_sets_out || n_jobs < 0 || n_slots < 1 || n_slots > 3 || nranks < 1 || rank < 0 ||
      rank >= nranks)
    return COSCHED_E_ARG;
  shard_bounds(n_jobs, n_slots, rank, nranks, first_set, n_sets_out);
  return COSCHED_OK;
}

cosched_status cosched_workspace_size(cosched_t h, int64_t n_jobs, size_t* bytes) {
  if (!h || !bytes || n_jobs < 0) return fail(h, COSCHED_E_ARG, "bad workspace_size arguments");
  int64_t first, count;
  shard_bounds(n_jobs, h->n_slots, h->rank, h->comm ? h->nranks : h->view_nranks, &first, &count);
  *bytes = workspace_layout(n_jobs, h->sp, count, h->comm ? h->nranks : 0, nullptr, nullptr);
  return COSCHED_OK;
}

// ---- NCCL ---------------------------------------------------------------------
cosched_status cosched_get_unique_id(void* uid_out) {
  std::string why;
  if (!uid_out) return COSCHED_E_ARG;
  if (!nccl_load(&why)) {
    g_create_error = why;
    return COSCHED_E_NCCL;
  }
  ncclUniqueId id;
  int r = g_nccl.getUniqueId(&id);
  if (r != 0) return COSCHED_E_NCCL;
  memcpy(uid_out, &id, sizeof id);
  return COSCHED_OK;
}

cosched_status cosched_set_comm(cosched_t h, const void* uid, int rank, int nranks) {
  if (!h || nranks < 1 || rank < 0 || rank >= nranks) return fail(h, COSCHED_E_ARG, "bad rank/nranks");
  DeviceGuard g(h->device);
  if (h->comm) {
    g_nccl.commDestroy(h->comm);
    h->comm = nullptr;
  }
  h->scored = false;
  if (nranks == 1 && !uid) {  // single process without NCCL
    h->rank = 0;
    h->nranks = 1;
    h->view_nranks = 1;
    return COSCHED_OK;
  }
  std::string why;
  if (!uid) return fail(h, COSCHED_E_ARG, "null unique id");
  if (!nccl_load(&why)) return fail(h, COSCHED_E_NCCL, why);
  ncclUniqueId id;
  memcpy(&id, uid, sizeof id);
  int r = g_nccl.commInitRank(&h->comm, nranks, id, rank);
  if (r != 0) {
    h->comm = nullptr;
    return fail(h, COSCHED_E_NCCL, std::string("ncclCommInitRank: ") +
                                       (g_nccl.getErrorString ? g_nccl.getErrorString(r) : "error"));
  }
  h->rank = rank;
  h->nranks = nranks;
  h->view_nranks = 1;
  return COSCHED_OK;
}

cosched_status cosched_set_shard_view(cosched_t h, int rank, int nranks) {
  if (!h || nranks < 1 || rank < 0 || rank >= nranks) return fail(h, COSCHED_E_ARG, "bad rank/nranks");
  if (h->comm) return fail(h, COSCHED_E_STATE, "a communicator is set");
  h->rank = rank;
  h->view_nranks = nranks;
  h->scored = false;
  return COSCHED_OK;
}

static cosched_status allreduce_op(cosched_t h, void* dev, size_t count, int dtype, int op) {
  if (!h->comm) return COSCHED_OK;
  int r = g_nccl.allReduce(dev, dev, count, dtype, op, h->comm, h->stream);
  if (r != 0)
    return fail(h, COSCHED_E_NCCL, std::string("ncclAllReduce: ") +
                                       (g_nccl.getErrorString ? g_nccl.getErrorString(r) : "error"));
  return COSCHED_OK;
}

static cosched_status allreduce_max(cosched_t h, void* dev, size_t count, int dtype) {
  if (!h->comm) return COSCHED_OK;
  int r = g_nccl.allReduce(dev, dev, count, dtype, kNcclMax, h->comm, h->stream);
  if (r != 0)
    return fail(h, COSCHED_E_NCCL, std::string("ncclAllReduce: ") +
                                       (g_nccl.getErrorString ? g_nccl.getErrorString(r) : "error"));
  return COSCHED_OK;
}

// ---- scoring --------------------------------------------------------------------
cosched_status cosched_score_all(cosched_t h, const float* features_dev, int64_t n_rows, const int32_t* jobs_dev,
                                 int64_t n_jobs, void* workspace_dev, size_t workspace_bytes, const cosched_out* out,
                                 void* cuda_stream) {
  NvtxRange nvtx_("cosched_score_all");
  if (!h) return COSCHED_E_ARG;
  h->err.clear();
  if (n_jobs < 0 || n_rows < 0 || (n_jobs > 0 && !features_dev) || (!jobs_dev && n_rows < n_jobs))
    return fail(h, COSCHED_E_ARG, "bad features / jobs arguments");
  if (cosched::n_sets(n_jobs, h->n_slots) > 0xFFFFFFFEll)
    return fail(h, COSCHED_E_ARG, "queue too large: more than 2^32-2 sets");
  int64_t first, count;
  shard_bounds(n_jobs, h->n_slots, h->rank, h->comm ? h->nranks : h->view_nranks, &first, &count);
  size_t need = workspace_layout(n_jobs, h->sp, count, h->comm ? h->nranks : 0, nullptr, nullptr);
  if (!workspace_dev || workspace_bytes < need || ((uintptr_t)workspace_dev & 255))
    return fail(h, COSCHED_E_OOM, "workspace missing, misaligned or smaller than cosched_workspace_size");
  float* obj = nullptr;
  int32_t* cfg = nullptr;
  if (out) {
    if (out->first_set != first || out->n_sets != count)
      return fail(h, COSCHED_E_ARG, "out range differs from cosched_shard_range");
    obj = out->obj;
    cfg = out->cfg;
  }
  DeviceGuard g(h->device);
  cudaStream_t st = (cudaStream_t)cuda_stream;
  Workspace ws;
  workspace_layout(n_jobs, h->sp, count, h->comm ? h->nranks : 0, (char*)workspace_dev, &ws);
  h->sp.n_jobs_pad = pad_jobs(n_jobs);
  cudaEventRecord(h->ev[0], st);
  if (ws.merge && ws.merge_tiles > 0 && h->merge_init != (const void*)ws.merge) {
    // the tail-merge area keeps step-tagged entries between calls: zeroed once per workspace
    cudaMemsetAsync(ws.merge, 0, (size_t)ws.merge_tiles * 64 * 64 * sizeof(unsigned long long), st);
    cudaMemsetAsync(ws.merge_cnt, 0, (size_t)ws.merge_tiles * sizeof(unsigned), st);
    h->merge_init = ws.merge;
  }
  launch_step_init(ws.err, ws.best_key, ws.rescore_n, ws.wmm, st);
  h->launches += 1;
  // instrumentation (COSCHED_PREP_EVENTS=1): the prep's parts, printed by
  // cosched_last_timings; the extra events cut the PDL overlap they measure across
  static const bool prep_events = [] {
    const char* e = getenv("COSCHED_PREP_EVENTS");
    return e && e[0] == '1';
  }();
  if (prep_events && !h->evp[0])
    for (auto& e : h->evp) cudaEventCreate(&e);
  if (prep_events) cudaEventRecord(h->evp[0], st);
  {
    // rows of the gathered layout the tiled scorer reads for this shard: the
    // sets' largest positions lie in [c0, c1), every other position below c1
    // (whole-column shards; otherwise every row)
    int64_t c0 = 0, c1 = n_jobs;
    const int ns = h->n_slots;
    auto col_at = [&](int64_t v) {  // smallest c with C(c, ns) >= v
      int64_t lo = 0, hi = n_jobs;
      while (lo < hi) {
        const int64_t mid = (lo + hi) / 2;
        if (cosched::n_sets(mid, ns) >= v) hi = mid;
        else lo = mid + 1;
      }
      return lo;
    };
    if (count > 0) {
      const int64_t a = col_at(first), b = col_at(first + count);
      if (cosched::n_sets(a, ns) == first && cosched::n_sets(b, ns) == first + count) {
        c0 = a;
        c1 = b;
      }
    }
    for (int i = 0; i < kMaxSlots; i++) {
      h->sp.fast_lo[i] = (i == ns - 1) ? c0 : 0;
      h->sp.fast_hi[i] = c1;
    }
  }
  if (n_jobs > 0) {
    launch_validate(features_dev, n_rows, jobs_dev, n_jobs, ws.err, ws.hj, st);
    if (prep_events) cudaEventRecord(h->evp[1], st);
    // the tiled scorers read only the gathered layout and w: ka / kb are
    // projected later, and only if a consumer (detail of arbitrary sets, node
    // budget, exact allocation) asks for them
    const bool tiled = h->variant != 0 && h->sp.search_mode == 0 && tiled_applicable(h->n_slots, n_jobs, first, count);
    h->kakb_valid = !tiled;
    launch_project(ws.hj, n_jobs, h->sp, h->tb, ws.err, ws.ka, ws.kb, ws.w, ws.fast, ws.wmm, !tiled, st,
                   prep_events ? h->evp[2] : nullptr);
    h->launches += 3;
  }
  // prep / score split for cosched_last_timings, only when asked for
  // (cosched_set_timing): an event between the gather and the scorer stops the
  // scorer's launch from overlapping the gather's tail (PDL) -- 5-6 us a step
  if (h->timing) cudaEventRecord(h->ev[1], st);
  if (h->sp.search_mode == 1) {
    launch_fill_u64((unsigned long long*)(ws.counters + 7), 0ull, 1, st);
    h->launches += 1 + launch_score_hill(h->sp, n_jobs, ws.ka, ws.kb, ws.w, first, count, obj, cfg, ws.best_key,
                                         (unsigned long long*)(ws.counters + 7), ws.err, st);
  } else {
    RescoreBuf rb;
    rb.wmm = ws.wmm;
    rb.list = ws.rescore_list;
    rb.n = ws.rescore_n;
    rb.cap = ws.rescore_cap;
    PairMerge pm;
    pm.buf = ws.merge;
    pm.tiles = ws.merge_tiles;
    pm.side = h->side;
    pm.side2 = h->side2;
    pm.cnt = ws.merge_cnt;
    pm.ev_fork = h->ev_fork;
    pm.ev_join = h->ev_join;
    pm.ev_join2 = h->ev_join2;
    h->merge_epoch = (h->merge_epoch + 1u) & 0xFFFFFFu;  // per step, never 0 (the zeroed state)
    if (h->merge_epoch == 0u) h->merge_epoch = 1u;
    pm.epoch = h->merge_epoch;
    h->launches += launch_score(h->sp, n_jobs, ws.ka, ws.kb, ws.w, ws.fast, first, count, obj, cfg, ws.best_key,
                                ws.err, h->variant, st, rb, pm);
  }
  if (h->timing) cudaEventRecord(h->ev[2], st);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(h, e, "score_all launch");
  h->scored = true;
  h->step_timed = false;
  h->split_timed = h->timing;
  h->n_jobs = n_jobs;
  h->first = first;
  h->n_sets = count;
  h->ws = ws;
  h->out_obj = obj;
  h->out_cfg = cfg;
  h->stream = st;
  return COSCHED_OK;
}

static cosched_status deferred_status(cosched_t h, unsigned long long e);

static cosched_status check_deferred(cosched_t h) {
  CK(cudaMemcpyAsync(h->h_pinned, h->ws.err, 8, cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  return deferred_status(h, h->h_pinned[0]);
}

// the validation outcome of the last score_all (err word written by k_validate)
static cosched_status deferred_status(cosched_t h, unsigned long long e) {
  if (e == ~0ull) return COSCHED_OK;
  int code = (int)(e & 0xFF);
  long long pos = (long long)(e >> 8);
  char buf[160];
  const char* what = code == COSCHED_E_RANGE ? "counter NaN/outside [0,100] or F6+F7+F8 > 100"
                     : code == COSCHED_E_DEGENERATE_PROFILE ? "F1 <= 0.01 (degenerate profile)"
                                                            : "row index outside [0, n_rows)";
  snprintf(buf, sizeof buf, "job %lld: %s", pos, what);
  return fail(h, (cosched_status)code, buf);
}

cosched_status cosched_set_timing(cosched_t h, int on) {
  if (!h) return COSCHED_E_ARG;
  h->timing = on != 0;
  return COSCHED_OK;
}

cosched_status cosched_last_timings(cosched_t h, float* ms3) {
  if (!h || !ms3) return fail(h, COSCHED_E_ARG, "null argument");
  if (!h->scored) return fail(h, COSCHED_E_STATE, "call cosched_score_all first");
  if (!h->split_timed) return fail(h, COSCHED_E_STATE, "the last cosched_score_all ran without cosched_set_timing(h, 1)");
  DeviceGuard g(h->device);
  CK(cudaEventSynchronize(h->ev[2]));
  CK(cudaEventElapsedTime(&ms3[0], h->ev[0], h->ev[1]));
  CK(cudaEventElapsedTime(&ms3[1], h->ev[1], h->ev[2]));
  CK(cudaEventElapsedTime(&ms3[2], h->ev[0], h->ev[2]));
  if (h->evp[0] && getenv("COSCHED_PREP_EVENTS")) {
    float a = 0, b = 0, c = 0, d = 0;
    cudaEventElapsedTime(&a, h->ev[0], h->evp[0]);
    cudaEventElapsedTime(&b, h->evp[0], h->evp[1]);
    cudaEventElapsedTime(&c, h->evp[1], h->evp[2]);
    cudaEventElapsedTime(&d, h->evp[2], h->ev[1]);
    fprintf(stderr, "prep: init %.4f validate %.4f project %.4f gather %.4f ms\n", a, b, c, d);
  }
  return COSCHED_OK;
}

cosched_status cosched_last_step_ms(cosched_t h, float* ms) {
  if (!h || !ms) return fail(h, COSCHED_E_ARG, "null argument");
  if (!h->scored || h->best_pending || !h->step_timed)
    return fail(h, COSCHED_E_STATE, "needs cosched_score_all then cosched_best_set");
  DeviceGuard g(h->device);
  CK(cudaEventSynchronize(h->ev[3]));
  CK(cudaEventElapsedTime(ms, h->ev[0], h->ev[3]));
  return COSCHED_OK;
}

cosched_status cosched_local_best_key(cosched_t h, uint64_t* key) {
  if (!h || !key) return fail(h, COSCHED_E_ARG, "null argument");
  if (!h->scored) return fail(h, COSCHED_E_STATE, "call cosched_score_all first");
  DeviceGuard g(h->device);
  cosched_status st = check_deferred(h);
  if (st != COSCHED_OK) return st;
  CK(cudaMemcpyAsync(h->h_pinned, h->ws.best_key, 8, cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  *key = h->h_pinned[0];
  return COSCHED_OK;
}

// The ka / kb rows of the last score_all, if its projection skipped them.
static void ensure_kakb(cosched_t h) {
  if (h->kakb_valid) return;
  if (h->n_jobs > 0) {
    // the tiled step stored only the w rows its own scorer reads: complete them too
    launch_project_kakb(h->ws.hj, h->n_jobs, h->sp, h->tb, h->ws.err, h->ws.ka, h->ws.kb, h->ws.wmm, h->stream,
                        h->ws.w);
    h->launches++;
  }
  h->kakb_valid = true;
}

static cosched_status detail_rows(cosched_t h, const int64_t* ids, int64_t n, std::vector<float>* rows) {
  ensure_kakb(h);
  rows->assign((size_t)n * 8, 0.0f);
  for (int64_t off = 0; off < n; off += cosched_ctx::kDetailRows) {
    int64_t m = std::min<int64_t>(cosched_ctx::kDetailRows, n - off);
    CK(cudaMemcpyAsync(h->d_detail_ids, ids + off, m * 8, cudaMemcpyHostToDevice, h->stream));
    launch_sets_detail(h->sp, h->ws.ka, h->ws.kb, h->ws.w, h->d_detail_ids, m, h->d_detail, h->stream);
    h->launches++;
    CK(cudaMemcpyAsync(rows->data() + off * 8, h->d_detail, m * 8 * 4, cudaMemcpyDeviceToHost, h->stream));
  }
  CK(cudaStreamSynchronize(h->stream));
  return COSCHED_OK;
}

cosched_status cosched_best_set_begin(cosched_t h) {
  NvtxRange nvtx_("cosched_best_set_begin");
  if (!h) return COSCHED_E_ARG;
  if (!h->scored) return fail(h, COSCHED_E_STATE, "call cosched_score_all first");
  DeviceGuard g(h->device);
  // one device -> host round trip: all-reduce the key, decode the winner's config
  // on the device, then read back the validation word, the key and the detail row
  cosched_status st = allreduce_max(h, h->ws.best_key, 1, kNcclUint64);
  if (st != COSCHED_OK) return st;
  // the detail kernel writes the validation word, the key and the row straight
  // into the pinned (mapped) host buffer: no copy on the stream
  launch_best_detail(h->sp, h->ws.ka, h->ws.kb, h->ws.w, h->ws.best_key, h->ws.err, h->h_pinned, h->ws.hj,
                     h->kakb_valid ? nullptr : &h->tb, h->stream);
  h->launches++;
  cudaEventRecord(h->ev[3], h->stream);  // end of the step's device work (cosched_last_step_ms)
  h->best_pending = true;
  h->step_timed = true;
  return COSCHED_OK;
}

cosched_status cosched_best_set_end(cosched_t h, int64_t* set_id, int32_t* cfg, float* obj) {
  NvtxRange nvtx_("cosched_best_set_end");
  if (!h) return COSCHED_E_ARG;
  if (!h->best_pending) return fail(h, COSCHED_E_STATE, "cosched_best_set_end without cosched_best_set_begin");
  h->best_pending = false;
  DeviceGuard g(h->device);
  CK(cudaStreamSynchronize(h->stream));
  cosched_status st = deferred_status(h, h->h_pinned[0]);
  if (st != COSCHED_OK) return st;
  const uint64_t key = h->h_pinned[1];
  float o;
  int64_t sid;
  cosched_unpack_key(key, &o, &sid);
  if (set_id) *set_id = sid;
  if (obj) *obj = o;
  if (cfg) *cfg = -1;
  if (key == 0) return COSCHED_INFEASIBLE;
  // config and objective of the same evaluation: the detail row's exact FP32
  // argmax of the winning set (the key's objective can be the packed-objective
  // choice, within tau/2 of it)
  if (cfg) memcpy(cfg, h->h_pinned + 2, 4);
  if (obj) memcpy(obj, reinterpret_cast<const float*>(h->h_pinned + 2) + 1, 4);
  return COSCHED_OK;
}

cosched_status cosched_best_set(cosched_t h, int64_t* set_id, int32_t* cfg, float* obj) {
  NvtxRange nvtx_("cosched_best_set");
  cosched_status st = cosched_best_set_begin(h);
  if (st != COSCHED_OK) return st;
  return cosched_best_set_end(h, set_id, cfg, obj);
}

cosched_status cosched_best_config(cosched_t h, int64_t set_id, int32_t* cfg, float* obj, float* rperf,
                                   float* throughput, float* fairness) {
  NvtxRange nvtx_("cosched_best_config");
  if (!h) return COSCHED_E_ARG;
  if (!h->scored) return fail(h, COSCHED_E_STATE, "call cosched_score_all first");
  if (set_id < 0 || set_id >= cosched::n_sets(h->n_jobs, h->n_slots)) return fail(h, COSCHED_E_ARG, "set id out of range");
  DeviceGuard g(h->device);
  cosched_status st = check_deferred(h);
  if (st != COSCHED_OK) return st;
  std::vector<float> rows;
  st = detail_rows(h, &set_id, 1, &rows);
  if (st != COSCHED_OK) return st;
  int32_t c;
  memcpy(&c, &rows[0], 4);
  if (cfg) *cfg = c;
  if (obj) *obj = rows[1];
  if (throughput) *throughput = rows[2];
  if (fairness) *fairness = rows[3];
  if (rperf)
    for (int i = 0; i < h->n_slots; i++) rperf[i] = c >= 0 ? rows[4 + i] : NAN;
  return c >= 0 ? COSCHED_OK : COSCHED_INFEASIBLE;
}

// ---- allocation -------------------------------------------------------------------
static int64_t n_partitions(int k, int64_t n) {
  if (n % k) return 0;
  int64_t acc = 1;
  for (int64_t m = n - 1; m > 0; m -= k) acc *= (k == 2) ? m : m * (m - 1) / 2;
  return acc;
}


// Sequential greedy by a sorted scan (greedy.cu). Picks come back in greedy
// order. *fallback = true when a batch would exceed the workspace capacity.
static cosched_status greedy_sorted_scan(cosched_t h, int32_t k, std::vector<unsigned long long>* picks,
                                         bool* fallback) {
  Workspace& ws = h->ws;
  const int ns = h->n_slots;
  const int64_t N = h->n_jobs;
  const int W = h->comm ? h->nranks : 1;
  *fallback = false;
  cudaStream_t s = h->stream;
  h->greedy_rounds = 0;
  // 1. objective range and histogram over every rank's sets
  unsigned init_mm[2] = {0xFFFFFFFFu, 0u};
  CK(cudaMemcpyAsync(ws.mm, init_mm, 8, cudaMemcpyHostToDevice, s));
  launch_obj_minmax(h->out_obj, h->n_sets, ws.mm, s);
  h->launches++;
  cosched_status st = allreduce_op(h, ws.mm, 1, kNcclUint32, kNcclMin);
  if (st != COSCHED_OK) return st;
  st = allreduce_op(h, ws.mm + 1, 1, kNcclUint32, kNcclMax);
  if (st != COSCHED_OK) return st;
  CK(cudaMemsetAsync(ws.hist, 0, (size_t)kHistBins * 4, s));
  launch_obj_hist(h->out_obj, h->n_sets, ws.mm, kHistBins, ws.hist, s);
  h->launches++;
  st = allreduce_op(h, ws.hist, kHistBins, kNcclUint32, kNcclSum);
  if (st != COSCHED_OK) return st;
  std::vector<unsigned> hist(kHistBins);
  unsigned mmh[2];
  CK(cudaMemcpyAsync(hist.data(), ws.hist, (size_t)kHistBins * 4, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(mmh, ws.mm, 8, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  picks->clear();
  if (mmh[0] > mmh[1]) return COSCHED_OK;  // no feasible set anywhere
  // 2. batches of bins, from the top, of ~kBatch keys (global)
  // a batch is a range of objective bins holding ~kBatch feasible sets; only the
  // sets whose jobs are all still free are compacted and sorted
  // batch sizes grow geometrically from 8 M keys (a first batch that already holds
  // the k picks sorts little; deep scans reach 64 M keys per batch after 3 rounds)
  // first batch 1 M keys, doubling (tools/greedy_stats.py on C4: 17.4 M keys sorted
  // in 6 batches against 26.8 M in 3 with an 8 M first batch)
  int64_t batch_keys = (int64_t)64 << 20, batch_first = (int64_t)1 << 20;
  if (const char* e = getenv("COSCHED_GREEDY_BATCH")) batch_keys = batch_first = std::max<int64_t>(1024, atoll(e));
  const int64_t kBatchMax = std::min<int64_t>(ws.batch_cap, batch_keys);
  int64_t kBatch = std::min<int64_t>(kBatchMax, batch_first);
  uint32_t* taken_bits = ws.taken;
  CK(cudaMemsetAsync(taken_bits, 0, (size_t)((N + 31) / 32) * 4, s));
  int64_t* np_dev = ws.counters + 1;
  CK(cudaMemsetAsync(ws.sel_flags, 0, 1024 * 8, s));  // k_select_free epochs start at 1 in this call
  unsigned sel_epoch = 0;
  unsigned long long* nk_dev = (unsigned long long*)(ws.counters + 2);
  CK(cudaMemsetAsync(np_dev, 0, 8, s));
  CK(cudaMemsetAsync(ws.counters + 8, 0, 8, s));
  int bin_hi = kHistBins - 1;
  int64_t n_picks = 0;
  bool endgame = false;
  while (bin_hi >= 0 && n_picks < k && !endgame) {
    // only the sets whose jobs are all free are compacted: size the batch on
    // their expected number, hist x C(n_free, ns) / C(N, ns) (x2 margin across
    // ranks, whose per-rank capacity is bounded; one rank holds every set)
    const int64_t n_free0 = N - (int64_t)ns * n_picks;
    double f_alive = (double)cosched::n_sets(n_free0, ns) / (double)std::max<int64_t>(cosched::n_sets(N, ns), 1);
    if (h->comm) f_alive = std::min(1.0, 2.0 * f_alive);
    f_alive = std::max(f_alive, 1.0 / 64.0);
    const double budget = (double)kBatch / f_alive;
    int bin_lo = bin_hi;
    double acc = hist[bin_hi];
    while (bin_lo > 0 && acc + hist[bin_lo - 1] <= budget) acc += hist[--bin_lo];
    if (acc == 0) {
      bin_hi = bin_lo - 1;
      continue;
    }
    // endgame: every set that can still be picked lies among the free jobs; when
    // there are at most kBatch of them, take them all in one final batch
    // (sets of earlier batches were picked or blocked, so no bin filter is needed)
    const int64_t n_free = N - (int64_t)ns * n_picks;
    const int64_t n_comb = cosched::n_sets(n_free, ns);
    endgame = n_picks > 0 && n_comb <= kBatchMax && n_comb * 8 <= cosched::n_sets(N, ns);  // gathers << a full scan
    // 3. compact this rank's keys in the range (or of the free jobs); gather over ranks; sort; scan.
    // The list keys are relative to the batch's lowest objective (fewer radix bits)
    // and carry the jobs packed for pairs (GKeyFmt)
    CK(cudaMemsetAsync(nk_dev, 0, 8, s));
    GKeyFmt fmt;
    if (endgame) {
      fmt = gkey_format(ns, N, 0u, 1ull << 32);
      launch_free_sets(ns, taken_bits, N, (int32_t*)ws.job_key, ws.counters + 5, n_comb, h->out_obj, h->first,
                       h->n_sets, (unsigned long long*)ws.alive, nk_dev, fmt, s);
      h->launches += 2;
    } else {
      unsigned u_lo;
      unsigned long long width;
      bin_range_ord(mmh[0], mmh[1], bin_lo, bin_hi, &u_lo, &width);
      fmt = gkey_format(ns, N, u_lo, width);
      // once a quarter of the jobs is taken, read only the live rows (free j1, or free j1 < j2)
      if (n_free * 4 <= N * 3) {
        launch_keys_live(ns, taken_bits, N, (int32_t*)ws.job_key, ws.counters + 5, n_free, h->out_obj, h->first,
                         h->n_sets, ws.mm, bin_lo, bin_hi, (unsigned long long*)ws.alive, nk_dev, fmt, s);
        h->launches += 2;
      } else {
        launch_keys_in_range(ns, h->out_obj, h->first, h->n_sets, ws.mm, kHistBins, bin_lo, bin_hi, taken_bits,
                             (unsigned long long*)ws.alive, nk_dev, fmt, s);
        h->launches++;
      }
    }
    int64_t nk = 0;
    CK(cudaMemcpyAsync(&nk, nk_dev, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const unsigned long long* list = (const unsigned long long*)ws.alive;
    unsigned long long* sorted = (unsigned long long*)ws.alive2;
    int64_t m = nk;
    if (h->comm) {  // every rank scans the same gathered list (also with a 1-rank communicator)
      int64_t mx = nk;
      CK(cudaMemcpyAsync(ws.counters + 4, &mx, 8, cudaMemcpyHostToDevice, s));
      st = allreduce_op(h, ws.counters + 4, 1, kNcclUint64, kNcclMax);
      if (st != COSCHED_OK) return st;
      CK(cudaMemcpyAsync(&mx, ws.counters + 4, 8, cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      if (mx > ws.batch_cap) {
        *fallback = true;
        return COSCHED_OK;
      }
      if (mx > nk) CK(cudaMemsetAsync((unsigned long long*)ws.alive + nk, 0, (size_t)(mx - nk) * 8, s));
      int r = g_nccl.allGather(ws.alive, ws.gath, (size_t)mx, kNcclUint64, h->comm, s);
      if (r != 0) return fail(h, COSCHED_E_NCCL, "ncclAllGather failed");
      list = ws.gath;
      sorted = ws.gath_sorted;
      m = mx * W;
    }
    CK(sort_keys_desc(ws.sort_tmp, ws.sort_tmp_bytes, list, sorted, m, s, fmt.end_bit));
    if (getenv("COSCHED_GREEDY_STATS"))
      fprintf(stderr, "greedy batch: bins [%d, %d], %lld keys sorted on %d bits%s\n", bin_lo, bin_hi, (long long)m,
              fmt.end_bit, endgame ? " (endgame)" : "");
    h->launches++;
    if (getenv("COSCHED_GREEDY_PIPE") && atoi(getenv("COSCHED_GREEDY_PIPE")) != 0) {
      // (COSCHED_GREEDY_PIPE=1, measured slower on C4: DESIGN.md §5) the whole sorted
      // batch through the producer / consumer pipeline (one cooperative launch)
      CK(launch_greedy_pipe(ns, sorted, m, N, taken_bits, ws.picked, np_dev, k, fmt, ws.pipe_ring, ws.pipe_cnt,
                            ws.pipe_ctl, ws.pipe_ctl + kPipeSlots, s));
      h->launches += 2;
      h->greedy_rounds++;
      CK(cudaMemcpyAsync(&n_picks, np_dev, 8, cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      if (getenv("COSCHED_GREEDY_STATS")) {
        int surv = 0;
        CK(cudaMemcpy(&surv, ws.pipe_ctl + kPipeSlots + 3, 4, cudaMemcpyDeviceToHost));
        fprintf(stderr, "greedy pipe batch: %lld keys, %d survivors to the consumer, %lld picks\n", (long long)m, surv,
                (long long)n_picks);
      }
      bin_hi = bin_lo - 1;
      kBatch = std::min<int64_t>(kBatchMax, kBatch * 2);
      continue;
    }
    // scan the sorted list in windows of kWin keys: the first window as it is
    // (its keys were free at the batch start), every later window after an
    // order-preserving select of the keys still free (a full-GPU pass over that
    // window only), its count read by the scan from the device -- rounds are
    // enqueued without host round trips; the scan returns at once after k picks.
    // Every key is selected at most once, and only keys free at their window's
    // start reach the one-block scan.
    unsigned long long* S = h->comm ? ws.gath : (unsigned long long*)ws.alive;
    int64_t* cnt_dev = ws.counters + 3;
    // largest window: 256 K keys when picks are dense in the key order (C4: 5,000
    // picks in 5x10^7 sets), 1 M when sparse (C5: 666 in 1.3x10^9) -- fewer
    // select + scan launches for the same survivors (tools/alloc_prof.py: C4
    // 6.9 / 7.4 / 9.1 ms and C5 37.7 / 31.3 / 31.3 ms at 256 K / 1 M / 4 M)
    const double pick_density = (double)k / (double)std::max<int64_t>(cosched::n_sets(N, ns), 1);
    const int64_t kWin = getenv("COSCHED_GREEDY_CHUNK") ? std::max<int64_t>(1024, atoll(getenv("COSCHED_GREEDY_CHUNK")))
                                                       : (pick_density < 1e-5 ? (int64_t)1 << 20 : (int64_t)1 << 18);
    // windows grow from kWin0 (the batch's first keys are all free at its start:
    // the first windows are where the batch's picks happen and block the most)
    const int64_t kWin0 = getenv("COSCHED_GREEDY_WIN0") ? std::max<int64_t>(1024, atoll(getenv("COSCHED_GREEDY_WIN0")))
                                                       : (int64_t)1 << 14;
    static const bool cub_select = [] {  // COSCHED_GREEDY_CUBSELECT=1: CUB's DeviceSelect (A/B timing)
      const char* e = getenv("COSCHED_GREEDY_CUBSELECT");
      return e && e[0] == '1';
    }();
    int r = 0;
    int64_t win = std::min(kWin0, kWin);
    for (int64_t pos = 0; pos < m; pos += win, win = std::min(kWin, 2 * win), r++) {
      const int64_t w = std::min<int64_t>(win, m - pos);
      if (pos == 0) {
        CK(launch_greedy_scan(ns, sorted, w, nullptr, N, taken_bits, ws.picked, np_dev, k, fmt, s, ws.counters + 8));
      } else if (cub_select || select_tiles(w) > 1024) {
        CK(select_free_keys(ns, ws.sort_tmp, ws.sort_tmp_bytes, sorted + pos, S, cnt_dev, w, taken_bits, fmt, s));
        CK(launch_greedy_scan(ns, S, w, cnt_dev, N, taken_bits, ws.picked, np_dev, k, fmt, s, ws.counters + 8));
        h->launches++;
      } else {  // one-launch select (greedy.cu k_select_free)
        CK(launch_select_free(ns, sorted + pos, w, taken_bits, S, cnt_dev, ws.sel_flags, ++sel_epoch, fmt, np_dev, k, s));
        CK(launch_greedy_scan(ns, S, w, cnt_dev, N, taken_bits, ws.picked, np_dev, k, fmt, s, ws.counters + 8));
        h->launches++;
      }
      h->launches++;
      h->greedy_rounds++;
      // a host look at the pick count every 16 windows (windows enqueued after the
      // k-th pick return at once: select and scan both test the count first)
      if ((r & 15) == 15 || pos + win >= m) {
        CK(cudaMemcpyAsync(&n_picks, np_dev, 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (n_picks >= k) break;
      }
    }
    bin_hi = bin_lo - 1;
    kBatch = std::min<int64_t>(kBatchMax, kBatch * 2);
  }
  if (getenv("COSCHED_GREEDY_STATS")) {
    int64_t scanned = 0;
    CK(cudaMemcpyAsync(&scanned, ws.counters + 8, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    fprintf(stderr, "greedy: %lld picks, %lld keys through the scan, %lld windows\n", (long long)n_picks,
            (long long)scanned, (long long)h->greedy_rounds);
    scan_prof_report();
  }
  picks->resize(n_picks);
  if (n_picks) {
    CK(cudaMemcpyAsync(picks->data(), ws.picked, (size_t)n_picks * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
  }
  return COSCHED_OK;
}

cosched_status cosched_best_allocation(cosched_t h, int32_t k, int64_t* set_ids, int32_t* cfgs, double* total_obj,
                                       int32_t* n_found) {
  NvtxRange nvtx_("cosched_best_allocation");
  if (!h || k < 1 || !set_ids) return fail(h, COSCHED_E_ARG, "bad allocation arguments");
  if (!h->scored) return fail(h, COSCHED_E_STATE, "call cosched_score_all first");
  DeviceGuard g(h->device);
  cosched_status st = check_deferred(h);
  if (st != COSCHED_OK) return st;
  const int ns = h->n_slots;
  const int64_t N = h->n_jobs;
  if (n_found) *n_found = 0;
  if (total_obj) *total_obj = 0.0;
  if (ns < 2) return fail(h, COSCHED_E_ARG, "allocation needs n_slots >= 2");
  bool exact = (int64_t)k * ns == N && ((ns == 2 && N <= 20) || (ns == 3 && N <= 15));
  if (exact) {
    ensure_kakb(h);
    // score every set of the (tiny) queue locally: no collective needed
    int64_t all = cosched::n_sets(N, ns);
    launch_fill_u64(h->d_small_key, 0ull, 2, h->stream);
    if (h->sp.search_mode == 1)
      h->launches += 1 + launch_score_hill(h->sp, N, h->ws.ka, h->ws.kb, h->ws.w, 0, all, h->d_small_obj,
                                           h->d_small_cfg, h->d_small_key, (unsigned long long*)(h->ws.counters + 6),
                                           h->ws.err, h->stream);
    else
      // every set of the queue: the generic kernel (the gathered layout holds only this shard's rows)
      h->launches += 1 + launch_score(h->sp, N, h->ws.ka, h->ws.kb, h->ws.w, h->ws.fast, 0, all, h->d_small_obj,
                                      h->d_small_cfg, h->d_small_key, h->ws.err, 0, h->stream);
    int64_t nm = n_partitions(ns, N);
    launch_exact_alloc(ns, N, h->d_small_obj, nm, h->d_small_key + 1, h->stream);
    launch_exact_unrank(ns, N, h->d_small_key + 1, h->d_small_ids, h->stream);
    h->launches += 2;
    std::vector<int64_t> ids(k + 1);
    std::vector<float> objs(all);
    std::vector<int32_t> cf(all);
    CK(cudaMemcpyAsync(ids.data(), h->d_small_ids, (k + 1) * 8, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaMemcpyAsync(h->h_pinned, h->d_small_key + 1, 8, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaMemcpyAsync(objs.data(), h->d_small_obj, all * 4, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaMemcpyAsync(cf.data(), h->d_small_cfg, all * 4, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    uint64_t key = h->h_pinned[0];
    if (key == 0) return COSCHED_INFEASIBLE;
    for (int i = 0; i < k; i++) {
      set_ids[i] = ids[i];
      if (cfgs) cfgs[i] = cf[ids[i]];
    }
    if (total_obj) *total_obj = (double)unord_float((uint32_t)(key >> 32));
    if (n_found) *n_found = k;
    return COSCHED_OK;
  }
  // greedy: sorted scan (greedy.cu); locally-dominant rounds only as a fallback
  if (!h->out_obj) return fail(h, COSCHED_E_STATE, "greedy allocation needs score_all with out->obj");
  {
    std::vector<unsigned long long> picks;
    bool fallback = false;
    st = greedy_sorted_scan(h, k, &picks, &fallback);
    if (st != COSCHED_OK) return st;
    if (!fallback) {
      if (picks.empty()) return COSCHED_INFEASIBLE;
      int64_t take = std::min<int64_t>(k, (int64_t)picks.size());
      std::vector<int64_t> ids(take);
      double tot = 0.0;
      for (int64_t i = 0; i < take; i++) {
        float o;
        cosched_unpack_key(picks[i], &o, &ids[i]);
        set_ids[i] = ids[i];
        tot += (double)o;
      }
      if (cfgs) {
        std::vector<float> rows;
        st = detail_rows(h, ids.data(), take, &rows);
        if (st != COSCHED_OK) return st;
        for (int64_t i = 0; i < take; i++) memcpy(&cfgs[i], &rows[i * 8], 4);
      }
      if (total_obj) *total_obj = tot;
      if (n_found) *n_found = (int32_t)take;
      return COSCHED_OK;
    }
  }
  // fallback: locally dominant rounds over this rank's shard
  Workspace& ws = h->ws;
  int64_t* cnt = ws.counters;  // [0] n_alive, [1] n_picked, [2] n_alive2
  launch_fill_u64((unsigned long long*)cnt, 0ull, 8, h->stream);
  launch_fill_u32(ws.taken, 0u, N, h->stream);
  h->launches += 2;
  int64_t host_cnt[8];
  int64_t n_picked = 0;
  h->greedy_rounds = 0;
  if (ns == 2) {
    // pairs: tile-scan propose + per-job select; picks are identical on every rank
    auto c2 = [](int64_t n) { return n * (n - 1) / 2; };
    int64_t c0 = 0, c1 = 0;
    while (c2(c0 + 1) <= h->first && c0 < N) c0++;
    if (c2(c0) != h->first) c0 = 0;
    c1 = c0;
    while (c1 < N && c2(c1 + 1) <= h->first + h->n_sets) c1++;
    if (h->n_sets > 0) c1 = std::max(c1, c0 + 1);
    for (int round = 0; round < 1000000; round++) {
      launch_fill_u64(ws.job_key, 0ull, N, h->stream);
      launch_greedy_pairs_propose(h->out_obj, h->first, c0, c1, ws.taken, ws.job_key, h->stream);
      h->launches += 2;
      st = allreduce_max(h, ws.job_key, N, kNcclUint64);
      if (st != COSCHED_OK) return st;
      launch_greedy_pairs_select(ws.job_key, N, ws.picked, cnt + 1, h->stream);
      h->launches++;
      CK(cudaMemcpyAsync(host_cnt, cnt, 64, cudaMemcpyDeviceToHost, h->stream));
      CK(cudaStreamSynchronize(h->stream));
      int64_t now = host_cnt[1];
      h->greedy_rounds++;
      if (now == n_picked) break;
      launch_greedy_mark(2, ws.picked, n_picked, now, ws.taken, h->stream);
      h->launches++;
      n_picked = now;
    }
  } else {
  launch_greedy_init(ns, N, h->out_obj, h->first, h->n_sets, ws.alive, cnt + 0, h->stream);
  h->launches += 1;
  int64_t* alive = ws.alive;
  int64_t* alive2 = ws.alive2;
  CK(cudaMemcpyAsync(host_cnt, cnt, 64, cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  int64_t n_alive = host_cnt[0];
  for (int round = 0; round < 1000000; round++) {
    int64_t any_alive = n_alive;
    if (h->nranks > 1) {
      // global termination: max over ranks of the alive count
      CK(cudaMemcpyAsync(cnt + 4, &any_alive, 8, cudaMemcpyHostToDevice, h->stream));
      st = allreduce_max(h, cnt + 4, 1, kNcclUint64);
      if (st != COSCHED_OK) return st;
      CK(cudaMemcpyAsync(&any_alive, cnt + 4, 8, cudaMemcpyDeviceToHost, h->stream));
      CK(cudaStreamSynchronize(h->stream));
    }
    if (any_alive == 0) break;
    h->greedy_rounds++;
    launch_fill_u64(ws.job_key, 0ull, N, h->stream);
    launch_greedy_propose(ns, N, h->out_obj, h->first, alive, n_alive, ws.taken, ws.job_key, h->stream);
    h->launches += 2;
    st = allreduce_max(h, ws.job_key, N, kNcclUint64);
    if (st != COSCHED_OK) return st;
    launch_greedy_select(ns, N, h->out_obj, h->first, alive, n_alive, ws.job_key, ws.taken, ws.picked, cnt + 1,
                         h->stream);
    CK(cudaMemcpyAsync(host_cnt, cnt, 64, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    int64_t now = host_cnt[1];
    launch_greedy_mark(ns, ws.picked, n_picked, now, ws.taken, h->stream);
    h->launches += 2;
    n_picked = now;
    st = allreduce_max(h, ws.taken, N, kNcclUint32);
    if (st != COSCHED_OK) return st;
    launch_fill_u64((unsigned long long*)(cnt + 2), 0ull, 1, h->stream);
    launch_greedy_compact(ns, N, alive, n_alive, ws.taken, alive2, cnt + 2, h->stream);
    h->launches += 2;
    CK(cudaMemcpyAsync(host_cnt, cnt, 64, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    n_alive = host_cnt[2];
    std::swap(alive, alive2);
  }
  }
  // gather picks: per-job key of the set that took it, max over ranks
  launch_fill_u64(ws.job_key, 0ull, N, h->stream);
  h->launches++;
  std::vector<unsigned long long> mine(n_picked);
  if (n_picked) {
    CK(cudaMemcpyAsync(mine.data(), ws.picked, n_picked * 8, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
  }
  std::vector<unsigned long long> all_keys;
  if (h->nranks > 1 && ns != 2) {
    // job_key[j] = key of the set containing j (a set's key lands on each of its jobs)
    std::vector<unsigned long long> jk(N, 0ull);
    for (unsigned long long key : mine) {
      int64_t sid = (int64_t)(0xFFFFFFFFull - (key & 0xFFFFFFFFull));
      int64_t pos[3];
      cosched_unrank(N, ns, sid, pos);
      for (int i = 0; i < ns; i++) jk[pos[i]] = key;
    }
    CK(cudaMemcpyAsync(ws.job_key, jk.data(), N * 8, cudaMemcpyHostToDevice, h->stream));
    st = allreduce_max(h, ws.job_key, N, kNcclUint64);
    if (st != COSCHED_OK) return st;
    CK(cudaMemcpyAsync(jk.data(), ws.job_key, N * 8, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    for (int64_t j = 0; j < N; j++)
      if (jk[j]) all_keys.push_back(jk[j]);
    std::sort(all_keys.begin(), all_keys.end());
    all_keys.erase(std::unique(all_keys.begin(), all_keys.end()), all_keys.end());
    CK(cudaMemcpyAsync(ws.picked, all_keys.data(), all_keys.size() * 8, cudaMemcpyHostToDevice, h->stream));
    n_picked = (int64_t)all_keys.size();
  }
  if (n_picked == 0) return COSCHED_INFEASIBLE;
  // order picks by key, descending = sequential greedy order (on the GPU)
  unsigned long long* sorted = ws.job_key;  // reuse: n_picked <= N / n_slots
  launch_sort_keys_desc(ws.picked, n_picked, sorted, h->stream);
  h->launches++;
  int64_t take = std::min<int64_t>(k, n_picked);
  std::vector<unsigned long long> top(take);
  CK(cudaMemcpyAsync(top.data(), sorted, take * 8, cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  std::vector<int64_t> ids(take);
  double tot = 0.0;
  for (int64_t i = 0; i < take; i++) {
    float o;
    cosched_unpack_key(top[i], &o, &ids[i]);
    set_ids[i] = ids[i];
    tot += (double)o;
  }
  if (cfgs) {
    std::vector<float> rows;
    st = detail_rows(h, ids.data(), take, &rows);
    if (st != COSCHED_OK) return st;
    for (int64_t i = 0; i < take; i++) memcpy(&cfgs[i], &rows[i * 8], 4);
  }
  if (total_obj) *total_obj = tot;
  if (n_found) *n_found = (int32_t)take;
  return COSCHED_OK;
}

// ---- node-level power budgeting (node.cu) ---------------------------------------------
static cosched_status node_units(cosched_t h, int32_t gpus_per_node, double node_power_w, int32_t* U, float* unit,
                                 std::vector<int32_t>* u) {
  long long g = 0;
  std::vector<long long> w(h->h_caps.size());
  for (size_t i = 0; i < h->h_caps.size(); i++) {
    const double c = h->h_caps[i];
    if (c != floor(c) || c < 1) return fail(h, COSCHED_E_ARG, "node budgeting needs integer-watt caps");
    w[i] = (long long)c;
    g = std::gcd(g, w[i]);
  }
  if (!(node_power_w >= 0) || gpus_per_node < 1 || gpus_per_node > 64)
    return fail(h, COSCHED_E_ARG, "bad node budget or gpus_per_node");
  const double units = floor(node_power_w / (double)g + 1e-9);
  if (units > 12287) return fail(h, COSCHED_E_ARG, "node_power_w / gcd(caps) exceeds 12287 budget units");
  *U = (int32_t)units;
  *unit = (float)g;
  u->resize(w.size());
  for (size_t i = 0; i < w.size(); i++) (*u)[i] = (int32_t)(w[i] / g);
  return COSCHED_OK;
}

cosched_status cosched_node_workspace_size(cosched_t h, int64_t n_gpus, int32_t gpus_per_node, double node_power_w,
                                           size_t* bytes) {
  if (!h || !bytes || n_gpus < 1) return COSCHED_E_ARG;
  int32_t U;
  float unit;
  std::vector<int32_t> u;
  cosched_status st = node_units(h, gpus_per_node, node_power_w, &U, &unit, &u);
  if (st != COSCHED_OK) return st;
  *bytes = node_workspace_bytes(n_gpus, h->sp.n_caps, U, gpus_per_node);
  return COSCHED_OK;
}

cosched_status cosched_node_budget(cosched_t h, int64_t n_gpus, const int64_t* set_ids, int32_t gpus_per_node,
                                   double node_power_w, int32_t objective, void* workspace, size_t workspace_bytes,
                                   int32_t* caps_out, int32_t* cfgs_out, float* node_obj, void* cuda_stream) {
  NvtxRange nvtx_("cosched_node_budget");
  if (!h) return COSCHED_E_ARG;
  if (n_gpus < 1 || !set_ids || !caps_out || !cfgs_out || !node_obj || gpus_per_node < 1 ||
      n_gpus % gpus_per_node != 0 || (objective != 1 && objective != 2))
    return fail(h, COSCHED_E_ARG, "bad node budgeting arguments (n_gpus must be a multiple of gpus_per_node)");
  if (!h->scored) return fail(h, COSCHED_E_STATE, "call cosched_score_all first");
  const int64_t total = cosched::n_sets(h->n_jobs, h->n_slots);
  for (int64_t g = 0; g < n_gpus; g++)
    if (set_ids[g] < 0 || set_ids[g] >= total) return fail(h, COSCHED_E_ARG, "set id out of range");
  int32_t U;
  float unit;
  std::vector<int32_t> u;
  cosched_status st = node_units(h, gpus_per_node, node_power_w, &U, &unit, &u);
  if (st != COSCHED_OK) return st;
  if (!workspace || workspace_bytes < node_workspace_bytes(n_gpus, h->sp.n_caps, U, gpus_per_node))
    return fail(h, COSCHED_E_OOM, "workspace too small");
  st = check_deferred(h);
  if (st != COSCHED_OK) return st;
  DeviceGuard g(h->device);
  cudaStream_t s = (cudaStream_t)cuda_stream;
  ensure_kakb(h);
  int n = node_enqueue(h->sp, h->ws.ka, h->ws.kb, h->ws.w, set_ids, n_gpus, gpus_per_node, U, unit, u.data(),
                       objective, workspace, caps_out, cfgs_out, node_obj, s);
  if (n < 0) return cuda_fail(h, cudaGetLastError(), "node_budget launch");
  h->launches += n;
  CK(cudaStreamSynchronize(s));
  return COSCHED_OK;
}

// ---- worst / proposal / best against a ground truth (truth.cu) ------------------------
cosched_status cosched_evaluate_workspace_size(cosched_t h, int64_t n_jobs, size_t* bytes) {
  if (!h || !bytes || n_jobs < 0) return COSCHED_E_ARG;
  int64_t first, count;
  shard_bounds(n_jobs, h->n_slots, h->rank, h->comm ? h->nranks : h->view_nranks, &first, &count);
  *bytes = truth_workspace_bytes(n_jobs, count);
  return COSCHED_OK;
}

cosched_status cosched_evaluate_truth(cosched_t h, const cosched_truth_desc* truth, const float* features_dev,
                                      int64_t n_rows, const int32_t* jobs_dev, void* workspace,
                                      size_t workspace_bytes, const cosched_eval_out* out,
                                      cosched_eval_summary* summary, void* cuda_stream) {
  NvtxRange nvtx_("cosched_evaluate_truth");
  if (!h) return COSCHED_E_ARG;
  if (!truth || !features_dev || !out || !out->prop_obj || !out->prop_fair || !out->best_obj || !out->worst_obj)
    return fail(h, COSCHED_E_ARG, "null argument");
  if (!h->scored || !h->out_cfg) return fail(h, COSCHED_E_STATE, "call cosched_score_all with out first");
  if (truth->g_full < 1 || truth->g_full > 16 || truth->n_modules < 1 || !(truth->p_max > 0.0f) ||
      !(truth->f_min > 0.0f && truth->f_min <= 1.0f) || !(truth->w_gpc >= 0.0f) || !(truth->kappa >= 0.0f))
    return fail(h, COSCHED_E_ARG, "invalid ground-truth constants");
  for (int32_t g : h->h_gpcs)
    if (g > truth->g_full) return fail(h, COSCHED_E_ARG, "a state gives more GPCs than g_full");
  if (!workspace || workspace_bytes < truth_workspace_bytes(h->n_jobs, h->n_sets))
    return fail(h, COSCHED_E_OOM, "workspace too small");
  (void)n_rows;
  DeviceGuard g(h->device);
  cosched_status vs = check_deferred(h);  // the scored features were valid
  if (vs != COSCHED_OK) return vs;
  cudaStream_t st = (cudaStream_t)cuda_stream;
  int n = truth_enqueue(truth, h->sp, h->objective, h->h_gpcs.data(), h->h_mem.data(), h->h_caps.data(), features_dev,
                        jobs_dev, h->n_jobs, h->first, h->n_sets, h->out_cfg, out, workspace, h->d_sums, st);
  if (n < 0) return cuda_fail(h, cudaGetLastError(), "evaluate_truth launch");
  h->launches += n;
  if (h->comm) {
    int r = g_nccl.allReduce(h->d_sums, h->d_sums, 4, kNcclFloat64, kNcclSum, h->comm, st);
    if (r != 0) return fail(h, COSCHED_E_NCCL, "ncclAllReduce (evaluate_truth)");
  }
  double sums[4];
  CK(cudaMemcpyAsync(sums, h->d_sums, sizeof sums, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (summary) {
    summary->n_compared = (int64_t)llround(sums[0]);
    summary->n_violations = (int64_t)llround(sums[3]);
    summary->geomean_prop_over_best = sums[0] > 0 ? exp(sums[1] / sums[0]) : nan("");
    summary->geomean_worst_over_best = sums[0] > 0 ? exp(sums[2] / sums[0]) : nan("");
  }
  return COSCHED_OK;
}

// ---- calibration (calib.cu) -------------------------------------------------------
static thread_local std::string g_fit_error;

const char* cosched_fit_last_error(void) { return g_fit_error.c_str(); }

cosched_status cosched_fit_workspace_size(const cosched_fit_desc* desc, size_t* bytes) {
  if (!bytes) return COSCHED_E_ARG;
  cosched_status st = fit_validate_desc(desc);
  if (st != COSCHED_OK) return st;
  *bytes = fit_workspace_bytes(desc);
  return COSCHED_OK;
}

cosched_status cosched_fit(const cosched_fit_desc* desc, void* workspace, size_t workspace_bytes,
                           const cosched_fit_out* out, void* cuda_stream) {
  NvtxRange nvtx_("cosched_fit");
  g_fit_error.clear();
  cosched_status st = fit_validate_desc(desc);
  if (st != COSCHED_OK) {
    g_fit_error = "invalid descriptor";
    return st;
  }
  if (!out || !out->coef_c || !out->coef_d || !out->status || !out->count || !out->rms) {
    g_fit_error = "null output";
    return COSCHED_E_ARG;
  }
  if (!workspace || workspace_bytes < fit_workspace_bytes(desc)) {
    g_fit_error = "workspace too small";
    return COSCHED_E_OOM;
  }
  int dev = -1;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    g_fit_error = "no usable CUDA device";
    return COSCHED_E_CUDA;
  }
  cudaStream_t stream = (cudaStream_t)cuda_stream;
  unsigned long long* err_dev = nullptr;
  if (fit_enqueue(desc, workspace, out, &err_dev, stream) < 0) {
    g_fit_error = std::string("launch: ") + cudaGetErrorString(cudaGetLastError());
    return COSCHED_E_CUDA;
  }
  unsigned long long e = 0;
  if (cudaMemcpyAsync(&e, err_dev, 8, cudaMemcpyDeviceToHost, stream) != cudaSuccess ||
      cudaStreamSynchronize(stream) != cudaSuccess) {
    g_fit_error = std::string("CUDA: ") + cudaGetErrorString(cudaGetLastError());
    return COSCHED_E_CUDA;
  }
  if (e != ~0ull) {
    const int code = (int)(e & 0xFF);
    const unsigned long long pos = e >> 8;
    if (pos >= (1ull << 40))
      g_fit_error = "sample " + std::to_string(pos - (1ull << 40)) + ": key, app or partner out of range, or rperf not finite";
    else
      g_fit_error = "app " + std::to_string(pos) + ": invalid counters";
    return (cosched_status)code;
  }
  return COSCHED_OK;
}

}  // extern "C"
