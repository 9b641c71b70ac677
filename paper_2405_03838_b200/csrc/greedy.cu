// greedy.cu -- job -> GPU allocation by the sequential greedy rule (DESIGN.md
// R12): repeatedly take the feasible set with the largest (objective, -id)
// whose jobs are all free. Exactly that order is reproduced on the GPU:
//
//   1. histogram of ord(obj) over the feasible sets (64 K bins between the
//      queue's min and max objective) -> descending key ranges ("batches") of
//      ~M keys each;
//   2. per batch: compact the packed keys (ord(obj) << 32 | ~id) of the range,
//      radix-sort them descending (CUB), and
//   3. scan them in order with one resident block: 1024 keys at a time every
//      thread decodes its set and tests its jobs against the taken bitmask in
//      shared memory (parallel filter); one warp then walks the surviving
//      candidates in order and takes each one still free (the sequential rule).
//      The scan stops at k picks; otherwise the next batch continues it.
//
// Multi-GPU: batch ranges come from the all-reduced histogram, each rank's
// compacted keys are all-gathered, so every rank sorts and scans the same list
// and returns identical picks.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_select.cuh>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "cosched_internal.h"
#include "device_common.cuh"

namespace cosched {

__global__ void k_obj_minmax(const float* __restrict__ obj, int64_t count, unsigned* mm /* [0] min ord, [1] max ord */) {
  unsigned lo = 0xFFFFFFFFu, hi = 0u;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < count; k += (int64_t)gridDim.x * blockDim.x) {
    float o = obj[k];
    if (o > -INFINITY) {
      unsigned u = ord_float_d(o);
      lo = u < lo ? u : lo;
      hi = u > hi ? u : hi;
    }
  }
  for (int off = 16; off > 0; off >>= 1) {
    unsigned a = __shfl_xor_sync(0xFFFFFFFFu, lo, off), b = __shfl_xor_sync(0xFFFFFFFFu, hi, off);
    lo = a < lo ? a : lo;
    hi = b > hi ? b : hi;
  }
  if ((threadIdx.x & 31) == 0) {
    if (lo != 0xFFFFFFFFu) atomicMin(&mm[0], lo);
    if (hi) atomicMax(&mm[1], hi);
  }
}

__device__ __forceinline__ int bin_of(unsigned u, unsigned lo, unsigned span, int nbins) {
  return (int)(((unsigned long long)(u - lo) * (unsigned long long)nbins) / ((unsigned long long)span + 1ull));
}

__global__ void k_obj_hist(const float* __restrict__ obj, int64_t count, const unsigned* __restrict__ mm, int nbins,
                           unsigned* hist) {
  const unsigned lo = mm[0], span = mm[1] - mm[0];
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < count; k += (int64_t)gridDim.x * blockDim.x) {
    float o = obj[k];
    if (o > -INFINITY) atomicAdd(&hist[bin_of(ord_float_d(o), lo, span, nbins)], 1u);
  }
}

// keys of the sets whose bin lies in [bin_lo, bin_hi] and whose jobs are all
// still free (sets touching a taken job can never be picked again)
template <int NS>
__global__ void k_keys_in_range(const float* __restrict__ obj, int64_t first, int64_t count,
                                const unsigned* __restrict__ mm, int nbins, int bin_lo, int bin_hi,
                                const uint32_t* __restrict__ taken_bits, unsigned long long* keys,
                                unsigned long long* n_keys) {
  const unsigned lo = mm[0], span = mm[1] - mm[0];
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < count; k += (int64_t)gridDim.x * blockDim.x) {
    float o = obj[k];
    if (!(o > -INFINITY)) continue;
    int b = bin_of(ord_float_d(o), lo, span, nbins);
    if (b < bin_lo || b > bin_hi) continue;
    int64_t j[3];
    unrank_set<NS>(first + k, j);
    bool fr = true;
#pragma unroll
    for (int q = 0; q < NS; q++) fr = fr && !((__ldg(taken_bits + (j[q] >> 5)) >> (j[q] & 31)) & 1u);
    if (!fr) continue;
    unsigned long long at = atomicAdd(n_keys, 1ull);
    keys[at] = pack_key(o, first + k);
  }
}

// The sequential rule over a sorted window of 1024 candidates, resolved in
// parallel: an undecided candidate whose jobs are all still free and that is
// the lowest-index undecided candidate on every one of its jobs cannot be
// blocked by any earlier candidate, so it is taken; candidates touching a job
// just taken are dropped; repeat until the window is decided. The taken set is
// exactly the sequential greedy's, and picks are emitted in window (key) order.
template <int NS>
__global__ void __launch_bounds__(1024, 1)
    k_greedy_scan(const unsigned long long* __restrict__ sorted, int64_t m, int64_t n_jobs, uint32_t* taken_g,
                  unsigned long long* picks, int64_t* n_picks, int64_t k_max) {
  constexpr int CPT = 4;            // candidates per thread: window = 4096 keys
  constexpr int WIN = 1024 * CPT;
  extern __shared__ uint32_t s_dyn[];
  uint32_t* s_taken = s_dyn;                                                    // n_jobs bits
  int32_t* s_first = reinterpret_cast<int32_t*>(s_dyn + ((n_jobs + 31) >> 5));  // n_jobs
  __shared__ int32_t s_wsum[32];
  __shared__ int64_t s_np;
  const int words = (int)((n_jobs + 31) >> 5);
  for (int i = threadIdx.x; i < words; i += blockDim.x) s_taken[i] = taken_g[i];
  for (int i = threadIdx.x; i < n_jobs; i += blockDim.x) s_first[i] = 0x7FFFFFFF;
  if (threadIdx.x == 0) s_np = *n_picks;
  __syncthreads();
  const int t = threadIdx.x;
  unsigned long long nxt[CPT];
#pragma unroll
  for (int u = 0; u < CPT; u++) {
    const int64_t i = (int64_t)t * CPT + u;
    nxt[u] = i < m ? sorted[i] : 0ull;
  }
  for (int64_t base = 0; base < m; base += WIN) {
    if (s_np >= k_max) break;
    unsigned long long key[CPT];
    int32_t jb[CPT][3];
    bool und[CPT], acc[CPT];
#pragma unroll
    for (int u = 0; u < CPT; u++) {
      key[u] = nxt[u];
      const int64_t i2 = base + WIN + (int64_t)t * CPT + u;  // prefetch the next window
      nxt[u] = i2 < m ? sorted[i2] : 0ull;
      acc[u] = false;
      und[u] = false;
      jb[u][0] = jb[u][1] = jb[u][2] = 0;
      if (key[u]) {
        const int64_t sid = (int64_t)(0xFFFFFFFFull - (key[u] & 0xFFFFFFFFull));
        int64_t j[3];
        unrank_set<NS>(sid, j);
        und[u] = true;
#pragma unroll
        for (int q = 0; q < NS; q++) {
          jb[u][q] = (int32_t)j[q];
          und[u] = und[u] && !((s_taken[jb[u][q] >> 5] >> (jb[u][q] & 31)) & 1u);
        }
      }
    }
    bool any = false;
#pragma unroll
    for (int u = 0; u < CPT; u++) any = any || und[u];
    while (__syncthreads_or(any)) {
#pragma unroll
      for (int u = 0; u < CPT; u++)
        if (und[u])
#pragma unroll
          for (int q = 0; q < NS; q++) atomicMin(&s_first[jb[u][q]], t * CPT + u);
      __syncthreads();
      bool take[CPT];
#pragma unroll
      for (int u = 0; u < CPT; u++) {
        take[u] = und[u];
        if (und[u])
#pragma unroll
          for (int q = 0; q < NS; q++) take[u] = take[u] && (s_first[jb[u][q]] == t * CPT + u);
      }
      __syncthreads();
#pragma unroll
      for (int u = 0; u < CPT; u++) {
        if (und[u])
#pragma unroll
          for (int q = 0; q < NS; q++) s_first[jb[u][q]] = 0x7FFFFFFF;  // reset for the next round
        if (take[u]) {
#pragma unroll
          for (int q = 0; q < NS; q++) atomicOr(&s_taken[jb[u][q] >> 5], 1u << (jb[u][q] & 31));
          acc[u] = true;
          und[u] = false;
        }
      }
      __syncthreads();
      any = false;
#pragma unroll
      for (int u = 0; u < CPT; u++) {
        if (und[u])
#pragma unroll
          for (int q = 0; q < NS; q++)
            if ((s_taken[jb[u][q] >> 5] >> (jb[u][q] & 31)) & 1u) und[u] = false;
        any = any || und[u];
      }
    }
    // emit the window's picks in index order (block prefix sum), stopping at k_max
    int cnt = 0;
#pragma unroll
    for (int u = 0; u < CPT; u++) cnt += acc[u];
    int incl = cnt;
    for (int off = 1; off < 32; off <<= 1) {
      const int v = __shfl_up_sync(0xFFFFFFFFu, incl, off);
      if ((t & 31) >= off) incl += v;
    }
    if ((t & 31) == 31) s_wsum[t >> 5] = incl;
    __syncthreads();
    if (t < 32) {
      int v = s_wsum[t];
      for (int off = 1; off < 32; off <<= 1) {
        const int u2 = __shfl_up_sync(0xFFFFFFFFu, v, off);
        if (t >= off) v += u2;
      }
      s_wsum[t] = v;  // inclusive over warps
    }
    __syncthreads();
    const int64_t np0 = s_np;
    int rank = (t >= 32 ? s_wsum[(t >> 5) - 1] : 0) + incl - cnt;
#pragma unroll
    for (int u = 0; u < CPT; u++)
      if (acc[u]) {
        if (np0 + rank < k_max) picks[np0 + rank] = key[u];
        rank++;
      }
    __syncthreads();
    if (t == 0) s_np = (np0 + s_wsum[31] < k_max) ? np0 + s_wsum[31] : k_max;
    __syncthreads();
  }
  for (int i = threadIdx.x; i < words; i += blockDim.x) taken_g[i] = s_taken[i];
  if (threadIdx.x == 0) *n_picks = s_np;
}

// predicate of the order-preserving re-filter between scan chunks
template <int NS>
struct AllJobsFree {
  const uint32_t* bits;
  __device__ __forceinline__ bool operator()(const unsigned long long& key) const {
    if (!key) return false;
    const int64_t sid = (int64_t)(0xFFFFFFFFull - (key & 0xFFFFFFFFull));
    int64_t j[3];
    unrank_set<NS>(sid, j);
    bool fr = true;
#pragma unroll
    for (int q = 0; q < NS; q++) fr = fr && !((bits[j[q] >> 5] >> (j[q] & 31)) & 1u);
    return fr;
  }
};

size_t select_temp_bytes(int64_t n) {
  size_t bytes = 0;
  AllJobsFree<2> pred{nullptr};
  cub::DeviceSelect::If((void*)nullptr, bytes, (const unsigned long long*)nullptr, (unsigned long long*)nullptr,
                        (int64_t*)nullptr, (int)std::max<int64_t>(n, 1), pred);
  size_t b3 = 0;
  AllJobsFree<3> pred3{nullptr};
  cub::DeviceSelect::If((void*)nullptr, b3, (const unsigned long long*)nullptr, (unsigned long long*)nullptr,
                        (int64_t*)nullptr, (int)std::max<int64_t>(n, 1), pred3);
  return std::max(bytes, b3);
}

cudaError_t select_free_keys(int n_slots, void* temp, size_t temp_bytes, const unsigned long long* in,
                             unsigned long long* out, int64_t* n_out, int64_t n, const uint32_t* taken_bits,
                             cudaStream_t st) {
  if (n_slots == 2)
    return cub::DeviceSelect::If(temp, temp_bytes, in, out, n_out, (int)n, AllJobsFree<2>{taken_bits}, st);
  return cub::DeviceSelect::If(temp, temp_bytes, in, out, n_out, (int)n, AllJobsFree<3>{taken_bits}, st);
}

// ---- launchers -------------------------------------------------------------------------
void launch_obj_minmax(const float* obj, int64_t count, unsigned* mm, cudaStream_t st) {
  if (count <= 0) return;
  int64_t blocks = std::min<int64_t>((count + 255) / 256, 148 * 8);
  k_obj_minmax<<<(unsigned)blocks, 256, 0, st>>>(obj, count, mm);
}
void launch_obj_hist(const float* obj, int64_t count, const unsigned* mm, int nbins, unsigned* hist, cudaStream_t st) {
  if (count <= 0) return;
  int64_t blocks = std::min<int64_t>((count + 255) / 256, 148 * 8);
  k_obj_hist<<<(unsigned)blocks, 256, 0, st>>>(obj, count, mm, nbins, hist);
}
void launch_keys_in_range(int n_slots, const float* obj, int64_t first, int64_t count, const unsigned* mm, int nbins,
                          int bin_lo, int bin_hi, const uint32_t* taken_bits, unsigned long long* keys,
                          unsigned long long* n_keys, cudaStream_t st) {
  if (count <= 0) return;
  int64_t blocks = std::min<int64_t>((count + 255) / 256, 148 * 8);
  if (n_slots == 2)
    k_keys_in_range<2><<<(unsigned)blocks, 256, 0, st>>>(obj, first, count, mm, nbins, bin_lo, bin_hi, taken_bits,
                                                          keys, n_keys);
  else
    k_keys_in_range<3><<<(unsigned)blocks, 256, 0, st>>>(obj, first, count, mm, nbins, bin_lo, bin_hi, taken_bits,
                                                          keys, n_keys);
}

size_t sort_temp_bytes(int64_t n) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortKeysDescending((void*)nullptr, bytes, (const unsigned long long*)nullptr,
                                           (unsigned long long*)nullptr, (int)std::max<int64_t>(n, 1));
  return bytes;
}

cudaError_t sort_keys_desc(void* temp, size_t temp_bytes, const unsigned long long* in, unsigned long long* out,
                           int64_t n, cudaStream_t st) {
  return cub::DeviceRadixSort::SortKeysDescending(temp, temp_bytes, in, out, (int)n, 0, 64, st);
}

cudaError_t launch_greedy_scan(int n_slots, const unsigned long long* sorted, int64_t m, int64_t n_jobs,
                               uint32_t* taken_bits, unsigned long long* picks, int64_t* n_picks, int64_t k_max,
                               cudaStream_t st) {
  const size_t smem = (size_t)((n_jobs + 31) / 32) * 4 + (size_t)n_jobs * 4;
  if (n_slots == 2) {
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_greedy_scan<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_greedy_scan<2><<<1, 1024, smem, st>>>(sorted, m, n_jobs, taken_bits, picks, n_picks, k_max);
  } else {
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_greedy_scan<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_greedy_scan<3><<<1, 1024, smem, st>>>(sorted, m, n_jobs, taken_bits, picks, n_picks, k_max);
  }
  return cudaGetLastError();
}

}  // namespace cosched
