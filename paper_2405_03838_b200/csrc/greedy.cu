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
#include <stdio.h>

#include "cosched_internal.h"
#include "device_common.cuh"

namespace cosched {

// Objective arrays are scanned as float4 when the caller's obj pointer is
// 16-byte aligned (then count/4 float4s and a scalar tail), else scalar.
__device__ __forceinline__ int64_t vec4_count(const float* p, int64_t count) {
  return ((reinterpret_cast<uintptr_t>(p) & 15) == 0) ? (count >> 2) : 0;
}
__global__ void k_obj_minmax(const float* __restrict__ obj, int64_t count, unsigned* mm /* [0] min ord, [1] max ord */) {
  unsigned lo = 0xFFFFFFFFu, hi = 0u;
  const int64_t n4 = vec4_count(obj, count), stride = (int64_t)gridDim.x * blockDim.x;
  const float4* o4 = reinterpret_cast<const float4*>(obj);
  auto take = [&](float o) {
    if (o > -INFINITY) {
      const unsigned u = ord_float_d(o);
      lo = u < lo ? u : lo;
      hi = u > hi ? u : hi;
    }
  };
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n4; k += stride) {
    const float4 v = __ldcs(o4 + k);
    take(v.x);
    take(v.y);
    take(v.z);
    take(v.w);
  }
  for (int64_t k = (n4 << 2) + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < count; k += stride) take(obj[k]);
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

// Bins: 2^14 bins of 2^k ord(obj) units each from lo, k the smallest shift
// with ceil((span + 1) / 2^k) <= 2^14: bin(u) = (u - lo) >> k, a bin range is a
// range of u, and binning an element is a subtraction and a shift (the
// histogram pass streams the whole objective array at HBM speed).
__host__ __device__ __forceinline__ int hist_shift(unsigned span) {
  int k = 0;
  while ((((unsigned long long)span + 1ull + (1ull << k) - 1ull) >> k) > (unsigned long long)kHistBins) k++;
  return k;
}
__device__ __forceinline__ unsigned long long bin_start(unsigned lo, unsigned span, int b) {
  return (unsigned long long)lo + ((unsigned long long)b << hist_shift(span));
}

// ---- greedy-list keys (cosched_internal.h GKeyFmt) ----
GKeyFmt gkey_format(int n_slots, int64_t n_jobs, unsigned base, unsigned long long span_ord) {
  GKeyFmt f;
  f.packed = (n_slots == 2 && n_jobs <= 65536) ? 1 : 0;
  f.base = base;
  int bits = 0;
  while (bits < 32 && (span_ord >> bits) > 1ull) bits++;  // ord - base < span_ord <= 2^bits
  if (span_ord > (1ull << bits)) bits++;
  f.end_bit = 32 + (bits > 32 ? 32 : bits);
  return f;
}

void bin_range_ord(unsigned lo, unsigned hi, int bin_lo, int bin_hi, unsigned* u_lo, unsigned long long* width) {
  const int k = hist_shift(hi - lo);
  auto start = [&](int b) { return (unsigned long long)lo + ((unsigned long long)b << k); };
  *u_lo = (unsigned)start(bin_lo);
  *width = start(bin_hi + 1) - start(bin_lo);
}

template <int NS>
__device__ __forceinline__ unsigned long long gkey_make(const GKeyFmt& f, float o, int64_t sid, const int64_t* j) {
  const unsigned low = (NS == 2 && f.packed) ? (((unsigned)j[1] << 16) | (unsigned)j[0]) : (unsigned)sid;
  return ((unsigned long long)(ord_float_d(o) - f.base) << 32) | (0xFFFFFFFFull - low);
}
template <int NS>
__device__ __forceinline__ void gkey_jobs(const GKeyFmt& f, unsigned long long key, int32_t* jb) {
  const unsigned low = 0xFFFFFFFFu - (unsigned)(key & 0xFFFFFFFFull);
  if (NS == 2 && f.packed) {
    jb[0] = (int32_t)(low & 0xFFFFu);
    jb[1] = (int32_t)(low >> 16);
    return;
  }
  int64_t j[3];
  unrank_set<NS>((int64_t)low, j);
#pragma unroll
  for (int q = 0; q < NS; q++) jb[q] = (int32_t)j[q];
}
// the canonical packed key (pack_key) of a greedy-list key whose jobs are jb
template <int NS>
__device__ __forceinline__ unsigned long long gkey_canonical(const GKeyFmt& f, unsigned long long key,
                                                             const int32_t* jb) {
  const float o = unord_float_d((unsigned)(key >> 32) + f.base);
  int64_t sid = (int64_t)(0xFFFFFFFFu - (unsigned)(key & 0xFFFFFFFFull));
  if (NS == 2 && f.packed) sid = c2(jb[1]) + jb[0];
  return pack_key(o, sid);
}

// Histogram privatised per block in shared memory (64 KB), merged with one
// global atomic per nonzero bin and block.
__global__ void __launch_bounds__(1024) k_obj_hist(const float* __restrict__ obj, int64_t count,
                                                   const unsigned* __restrict__ mm, int nbins, unsigned* hist) {
  extern __shared__ unsigned s_hist[];
  for (int i = threadIdx.x; i < kHistBins; i += blockDim.x) s_hist[i] = 0u;
  __syncthreads();
  const unsigned lo = mm[0], span = mm[1] - mm[0];
  const int sh = hist_shift(span);
  const int64_t n4 = vec4_count(obj, count), stride = (int64_t)gridDim.x * blockDim.x;
  const float4* o4 = reinterpret_cast<const float4*>(obj);
  auto take = [&](float o) {
    if (o > -INFINITY) atomicAdd(&s_hist[(ord_float_d(o) - lo) >> sh], 1u);
  };
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n4; k += stride) {
    const float4 v = __ldcs(o4 + k);
    take(v.x);
    take(v.y);
    take(v.z);
    take(v.w);
  }
  for (int64_t k = (n4 << 2) + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < count; k += stride) take(obj[k]);
  __syncthreads();
  for (int i = threadIdx.x; i < kHistBins; i += blockDim.x)
    if (s_hist[i]) atomicAdd(&hist[i], s_hist[i]);
}

// keys of the sets whose bin lies in [bin_lo, bin_hi] and whose jobs are all
// still free (sets touching a taken job can never be picked again). Two phases
// per warp: the cheap range test on every element compacts the in-range
// (id, obj) pairs into a per-warp shared queue; whenever 32 are queued the
// warp decodes them one per lane (colex unranking, taken-bit test) -- so the
// unranking runs at full lane occupancy instead of diverging on every element.
constexpr int kKirWarps = 8;
constexpr int kKirQueue = 32 + 4 * 32;
constexpr int kKirLoads = 4;
constexpr int kKirOut = 256;
template <int NS>
__global__ void __launch_bounds__(32 * kKirWarps) k_keys_in_range(const float* __restrict__ obj, int64_t first,
                                                                 int64_t count, const unsigned* __restrict__ mm,
                                                                 int nbins, int bin_lo, int bin_hi,
                                                                 const uint32_t* __restrict__ taken_bits,
                                                                 unsigned long long* keys,
                                                                 unsigned long long* n_keys, const GKeyFmt fmt) {
  __shared__ int64_t s_id[kKirWarps][kKirQueue];
  __shared__ float s_o[kKirWarps][kKirQueue];
  // per-warp output buffer: the free keys leave in runs of up to kKirOut with
  // one atomicAdd per run (a single global counter takes every batch's keys)
  __shared__ unsigned long long s_out[kKirWarps][kKirOut];
  const unsigned lo = mm[0], span = mm[1] - mm[0];
  const unsigned long long u_lo = bin_start(lo, span, bin_lo), u_hi = bin_start(lo, span, bin_hi + 1);  // [u_lo, u_hi)
  // one 32-bit unsigned compare: u_lo <= hi < 2^32 and u_hi - u_lo <= span + 1 < 2^32;
  // -inf (infeasible) has ord 0x007FFFFF < lo <= u_lo, so it wraps to a large value
  const unsigned r_lo = (unsigned)u_lo, r_w = (unsigned)(u_hi - u_lo);
  // on raw float bits: every feasible objective is > 0 (Fairness > alpha >= 0
  // makes every RPerf, hence Throughput, positive), so the range lies in the
  // positive floats, where ord(o) = bits(o) | 2^31; the infeasible -inf
  // (0xFF800000) lands far above the range after the subtraction
  const unsigned b_lo = r_lo & 0x7FFFFFFFu;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  int64_t* qid = s_id[wib];
  float* qo = s_o[wib];
  int qn = 0;  // warp-uniform queue length
  auto in_range = [&](float o) { return __float_as_uint(o) - b_lo < r_w; };
  unsigned long long* ob = s_out[wib];
  int on = 0;  // warp-uniform output buffer length
  auto flush = [&]() {
    if (on == 0) return;
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(n_keys, (unsigned long long)on);
    base = __shfl_sync(0xFFFFFFFFu, base, 0);
    for (int e = lane; e < on; e += 32) keys[base + e] = ob[e];
    __syncwarp();
    on = 0;
  };
  // decode the 32 queue entries [qn - n, qn) (n <= 32), append the free ones
  auto drain = [&](int n) {
    unsigned long long kk = 0ull;
    bool ok = false;
    if (lane < n) {
      const int64_t sid = qid[qn - n + lane];
      int64_t j[3];
      unrank_set<NS>(sid, j);
      ok = true;
#pragma unroll
      for (int q = 0; q < NS; q++) ok = ok && !((__ldg(taken_bits + (j[q] >> 5)) >> (j[q] & 31)) & 1u);
      if (ok) kk = gkey_make<NS>(fmt, qo[qn - n + lane], sid, j);
    }
    const unsigned m = __ballot_sync(0xFFFFFFFFu, ok);
    if (ok) ob[on + __popc(m & ((1u << lane) - 1u))] = kk;
    on += __popc(m);
    __syncwarp();
    qn -= n;
    if (on > kKirOut - 32) flush();
  };
  auto push = [&](bool hit, float o, int64_t sid) {
    const unsigned m = __ballot_sync(0xFFFFFFFFu, hit);
    if (hit) {
      const int at = qn + __popc(m & ((1u << lane) - 1u));
      qid[at] = sid;
      qo[at] = o;
    }
    qn += __popc(m);
    __syncwarp();
  };
  const int64_t n4 = vec4_count(obj, count);
  const float4* o4 = reinterpret_cast<const float4*>(obj);
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5, nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  // kKirLoads float4 per lane in flight per iteration (memory-level parallelism:
  // the queue bookkeeping serialises iterations of a warp)
  for (int64_t k0 = gw * 32 * kKirLoads; k0 < n4; k0 += nw * 32 * kKirLoads) {
    float4 v[kKirLoads];
#pragma unroll
    for (int u = 0; u < kKirLoads; u++) {
      const int64_t k = k0 + 32 * u + lane;
      v[u] = k < n4 ? __ldcs(o4 + k) : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
    }
#pragma unroll
    for (int u = 0; u < kKirLoads; u++) {
      const int64_t k = k0 + 32 * u + lane;
      const bool h0 = in_range(v[u].x), h1 = in_range(v[u].y), h2 = in_range(v[u].z), h3 = in_range(v[u].w);
      if (!__any_sync(0xFFFFFFFFu, h0 || h1 || h2 || h3)) continue;  // nothing of the warp's 128 in range
      push(h0, v[u].x, first + 4 * k);
      push(h1, v[u].y, first + 4 * k + 1);
      push(h2, v[u].z, first + 4 * k + 2);
      push(h3, v[u].w, first + 4 * k + 3);
      while (qn >= 32) drain(32);
    }
  }
  // scalar tail (< 4 elements, plus everything when obj is not 16-byte aligned)
  for (int64_t t0 = (n4 << 2) + gw * 32; t0 < count; t0 += nw * 32) {
    const int64_t k = t0 + lane;
    const float o = k < count ? obj[k] : -INFINITY;
    push(k < count && in_range(o), o, first + k);
    while (qn >= 32) drain(32);
  }
  if (qn > 0) drain(qn);
  flush();
}

__global__ void k_free_list(const uint32_t* __restrict__ taken_bits, int64_t n_jobs, int32_t* __restrict__ free_list,
                            int64_t* __restrict__ n_free);

// The range pass restricted to live rows: once many jobs are taken, only the
// sets whose two largest jobs are free can be picked, and for fixed (j1, j2)
// (pairs: j1) the sets j0 < j1 are one contiguous run of the objective array.
// A warp walks such runs -- rows enumerated over the ascending free-job list,
// pairs: every free j1, triples: every free pair j1 < j2 -- reads only their
// objectives and emits the in-range keys whose j0 is free too. The data read
// falls with the square (triples: cube) of the free fraction.
template <int NS>
__global__ void __launch_bounds__(32 * kKirWarps) k_keys_live(const int32_t* __restrict__ free_list, int64_t n_rows,
                                                             const float* __restrict__ obj, int64_t first,
                                                             int64_t count, const unsigned* __restrict__ mm,
                                                             int bin_lo, int bin_hi,
                                                             const uint32_t* __restrict__ taken_bits,
                                                             unsigned long long* keys, unsigned long long* n_keys,
                                                             const GKeyFmt fmt) {
  __shared__ unsigned long long s_out[kKirWarps][kKirOut];
  const unsigned lo = mm[0], span = mm[1] - mm[0];
  const unsigned long long u_lo = bin_start(lo, span, bin_lo), u_hi = bin_start(lo, span, bin_hi + 1);
  const unsigned b_lo = (unsigned)u_lo & 0x7FFFFFFFu, r_w = (unsigned)(u_hi - u_lo);  // raw-bits test (k_keys_in_range)
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  unsigned long long* ob = s_out[wib];
  int on = 0;
  auto flush = [&]() {
    if (on == 0) return;
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(n_keys, (unsigned long long)on);
    base = __shfl_sync(0xFFFFFFFFu, base, 0);
    for (int e = lane; e < on; e += 32) keys[base + e] = ob[e];
    __syncwarp();
    on = 0;
  };
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5, nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = gw; r < n_rows; r += nw) {
    int64_t j[3];
    int64_t s0;  // set id of (j0 = 0, j1, j2)
    if (NS == 2) {
      j[1] = free_list[r];
      s0 = c2(j[1]);
    } else {
      int64_t ab[2];
      unrank_set<2>(r, ab);  // the r-th free pair, ascending positions in the free list
      j[1] = free_list[ab[0]];
      j[2] = free_list[ab[1]];
      s0 = c3(j[2]) + c2(j[1]);
    }
    const int64_t lo_i = s0 > first ? s0 : first, hi_i = s0 + j[1] < first + count ? s0 + j[1] : first + count;
    if (lo_i >= hi_i) continue;
    // the row's objectives [lo_i, hi_i) as aligned float4s of the shard's array
    // (a lane takes 4 consecutive elements, elements outside the row are
    // masked), two 512-byte warp loads in flight per step; key order within a
    // batch list does not matter (it is sorted next)
    const int64_t e_lo = lo_i - first, e_hi = hi_i - first;  // element range in obj
    const int64_t mis = (int64_t)((reinterpret_cast<uintptr_t>(obj) >> 2) & 3);
    int64_t b4 = ((e_lo + mis) & ~3ll) - mis;  // first element of the first 16-byte group
    for (; b4 < e_hi; b4 += 2 * 128) {  // warp-uniform
      float v[2][4];
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int64_t e0 = b4 + h * 128 + 4 * lane;
        if (b4 + h * 128 >= e_hi) {  // warp-uniform: past the row
#pragma unroll
          for (int q = 0; q < 4; q++) v[h][q] = -INFINITY;
        } else if (e0 >= 0 && e0 + 3 < count) {
          const float4 f = __ldcs(reinterpret_cast<const float4*>(obj + e0));
          v[h][0] = f.x;
          v[h][1] = f.y;
          v[h][2] = f.z;
          v[h][3] = f.w;
        } else {
#pragma unroll
          for (int q = 0; q < 4; q++) v[h][q] = (e0 + q >= 0 && e0 + q < count) ? obj[e0 + q] : -INFINITY;
        }
      }
#pragma unroll
      for (int h = 0; h < 2; h++)
#pragma unroll
        for (int q = 0; q < 4; q++) {
          const int64_t e = b4 + h * 128 + 4 * lane + q;
          bool ok = false;
          unsigned long long kk = 0ull;
          if (e >= e_lo && e < e_hi && __float_as_uint(v[h][q]) - b_lo < r_w) {
            j[0] = e + first - s0;
            if (!((__ldg(taken_bits + (j[0] >> 5)) >> (j[0] & 31)) & 1u)) {
              ok = true;
              kk = gkey_make<NS>(fmt, v[h][q], e + first, j);
            }
          }
          const unsigned m = __ballot_sync(0xFFFFFFFFu, ok);
          if (m) {
            if (ok) ob[on + __popc(m & ((1u << lane) - 1u))] = kk;
            on += __popc(m);
            __syncwarp();
            if (on > kKirOut - 32) flush();
          }
        }
    }
  }
  flush();
}

void launch_keys_live(int n_slots, const uint32_t* taken_bits, int64_t n_jobs, int32_t* free_list, int64_t* n_free_dev,
                      int64_t n_free, const float* obj, int64_t first, int64_t count, const unsigned* mm, int bin_lo,
                      int bin_hi, unsigned long long* keys, unsigned long long* n_keys, const GKeyFmt& fmt,
                      cudaStream_t st) {
  k_free_list<<<1, 1024, 0, st>>>(taken_bits, n_jobs, free_list, n_free_dev);
  const int64_t rows = n_slots == 2 ? n_free : n_free * (n_free - 1) / 2;
  if (rows <= 0 || count <= 0) return;
  const unsigned blocks = (unsigned)std::min<int64_t>((rows + kKirWarps - 1) / kKirWarps, 148 * 8);
  if (n_slots == 2)
    k_keys_live<2><<<blocks, 32 * kKirWarps, 0, st>>>(free_list, rows, obj, first, count, mm, bin_lo, bin_hi,
                                                      taken_bits, keys, n_keys, fmt);
  else
    k_keys_live<3><<<blocks, 32 * kKirWarps, 0, st>>>(free_list, rows, obj, first, count, mm, bin_lo, bin_hi,
                                                      taken_bits, keys, n_keys, fmt);
}

// Endgame of the greedy: once few jobs are free, the sets that can still be
// picked are exactly the sets of free jobs. Enumerate them directly (colex
// over the ascending free-job list) instead of scanning every set's objective
// again: C(n_free, n_slots) gathers instead of n_sets reads.
__global__ void k_free_list(const uint32_t* __restrict__ taken_bits, int64_t n_jobs, int32_t* __restrict__ free_list,
                            int64_t* __restrict__ n_free) {
  // one block: ordered compaction by warp ballots
  __shared__ int s_base;
  if (threadIdx.x == 0) s_base = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __shared__ int s_cnt[32];
  for (int64_t b0 = 0; b0 < n_jobs; b0 += blockDim.x) {
    const int64_t j = b0 + threadIdx.x;
    const bool fr = j < n_jobs && !((taken_bits[j >> 5] >> (j & 31)) & 1u);
    const unsigned m = __ballot_sync(0xFFFFFFFFu, fr);
    if (lane == 0) s_cnt[w] = __popc(m);
    __syncthreads();
    int off = s_base;
    for (int q = 0; q < w; q++) off += s_cnt[q];
    if (fr) free_list[off + __popc(m & ((1u << lane) - 1u))] = (int32_t)j;
    __syncthreads();
    if (threadIdx.x == 0)
      for (int q = 0; q < nw; q++) s_base += s_cnt[q];
    __syncthreads();
  }
  if (threadIdx.x == 0) *n_free = s_base;
}

template <int NS>
__global__ void k_free_sets(const int32_t* __restrict__ free_list, int64_t n_comb, const float* __restrict__ obj,
                            int64_t first, int64_t count, unsigned long long* keys, unsigned long long* n_keys,
                            const GKeyFmt fmt) {
  const int lane = threadIdx.x & 31;
  // a warp covers 32 consecutive ranks (whole-warp ballots); r0 is this warp's first
  for (int64_t r0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) & ~31ll; r0 < n_comb;
       r0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = r0 + lane;
    bool ok = false;
    unsigned long long kk = 0ull;
    if (r < n_comb) {
      int64_t q[3];
      unrank_set<NS>(r, q);  // ascending positions in the free list
      int64_t sid = 0, jv[3];
#pragma unroll
      for (int i = 0; i < NS; i++) {
        jv[i] = free_list[q[i]];
        sid += (i == 0) ? jv[i] : (i == 1 ? c2(jv[i]) : c3(jv[i]));  // colex rank of the ascending job tuple
      }
      if (sid >= first && sid < first + count) {
        const float o = obj[sid - first];
        if (o > -INFINITY) {
          ok = true;
          kk = gkey_make<NS>(fmt, o, sid, jv);
        }
      }
    }
    const unsigned m = __ballot_sync(0xFFFFFFFFu, ok);
    if (m) {
      unsigned long long base = 0;
      if (lane == 0) base = atomicAdd(n_keys, (unsigned long long)__popc(m));
      base = __shfl_sync(0xFFFFFFFFu, base, 0);
      if (ok) keys[base + __popc(m & ((1u << lane) - 1u))] = kk;
    }
  }
}

void launch_free_sets(int n_slots, const uint32_t* taken_bits, int64_t n_jobs, int32_t* free_list, int64_t* n_free_dev,
                      int64_t n_comb, const float* obj, int64_t first, int64_t count, unsigned long long* keys,
                      unsigned long long* n_keys, const GKeyFmt& fmt, cudaStream_t st) {
  k_free_list<<<1, 1024, 0, st>>>(taken_bits, n_jobs, free_list, n_free_dev);
  if (n_comb <= 0) return;
  const unsigned blocks = (unsigned)std::min<int64_t>((n_comb + 255) / 256, 148 * 8);
  if (n_slots == 2)
    k_free_sets<2><<<blocks, 256, 0, st>>>(free_list, n_comb, obj, first, count, keys, n_keys, fmt);
  else
    k_free_sets<3><<<blocks, 256, 0, st>>>(free_list, n_comb, obj, first, count, keys, n_keys, fmt);
}

// The sequential rule over the sorted keys, window by window (kScanWin keys):
//  1. filter, all threads: every key of the window is decoded (colex
//     unranking) and tested against the taken bitmask (shared memory); keys
//     with a taken job can never be picked (the greedy only takes sets whose
//     jobs are all free) and are dropped;
//  2. the survivors are compacted in key order (block ballots + prefix sum);
//  3. warp 0 walks the survivors in order, 32 at a time: the first survivor
//     of the group whose jobs are all free is taken (it is the sequential
//     rule's next pick: every earlier key was blocked), its jobs are marked,
//     the group's survivors sharing one of them are dropped, repeat. Picks are
//     appended in key order; the scan stops at k_max.
// Only keys still free at their window's start reach the sequential part --
// 21,033 of the 5x10^7 keys of C4 (tools/greedy_stats.py) -- so the scan costs
// about one decode per key. The taken bitmask (n_jobs bits) is the only
// per-job state: any queue the set scorer accepts fits shared memory.
constexpr int kScanThreads = 512, kScanPer = 4, kScanWin = kScanThreads * kScanPer, kScanWarps = kScanThreads / 32;
// k_select_free tiles (the greedy window select, below)
constexpr int kSelThreads = 256, kSelPer = 16, kSelTile = kSelThreads * kSelPer, kSelMaxTiles = 1024;

#ifdef COSCHED_SCAN_PROF
// instrumentation build only: [0] filter cycles, [1] resolution cycles, [2] chunks,
// [3] survivors, [4] picks, [5] launches, [6] whole-kernel cycles
__device__ unsigned long long g_scan_prof[12];
#endif
// a set's jobs in one word (jobs < 2^20, the scan's limit): j0 | j1 << 20 | j2 << 40
template <int NS>
__device__ __forceinline__ unsigned long long jobs_pack(const int32_t* jb) {
  unsigned long long v = (unsigned long long)(uint32_t)jb[0];
  if (NS > 1) v |= (unsigned long long)(uint32_t)jb[1] << 20;
  if (NS > 2) v |= (unsigned long long)(uint32_t)jb[2] << 40;
  return v;
}
template <int NS>
__device__ __forceinline__ void jobs_unpack(unsigned long long v, int32_t* jb) {
#pragma unroll
  for (int q = 0; q < NS; q++) jb[q] = (int32_t)((v >> (20 * q)) & 0xFFFFFu);
}
template <int NS>
__device__ __forceinline__ bool jobs_packed_free(unsigned long long v, const uint32_t* bits) {
  bool fr = true;
#pragma unroll
  for (int q = 0; q < NS; q++) {
    const unsigned j = (unsigned)((v >> (20 * q)) & 0xFFFFFu);
    fr = fr && !((bits[j >> 5] >> (j & 31)) & 1u);
  }
  return fr;
}
template <int NS>
__device__ __forceinline__ bool key_jobs_free(const GKeyFmt& f, unsigned long long key, const uint32_t* bits,
                                              int32_t* jb) {
  gkey_jobs<NS>(f, key, jb);
  bool fr = true;
#pragma unroll
  for (int q = 0; q < NS; q++) fr = fr && !((bits[jb[q] >> 5] >> (jb[q] & 31)) & 1u);
  return fr;
}

template <int NS>
__global__ void __launch_bounds__(kScanThreads, 1)
    k_greedy_scan(const unsigned long long* __restrict__ sorted, int64_t m_host, const int64_t* __restrict__ m_dev,
                  int64_t n_jobs, uint32_t* taken_g, unsigned long long* picks, int64_t* n_picks, int64_t k_max,
                  const GKeyFmt fmt, int64_t* scanned) {
  pdl_wait();  // the previous scan's picks and taken bits, the select's output
  pdl_launch_dependents();
  int64_t np = *n_picks;  // warp 0's running count (uniform in warp 0)
  if (np >= k_max) return;  // uniform: enqueued windows after the k-th pick cost one launch
  const int64_t m = m_dev ? *m_dev : m_host;
  if (scanned && threadIdx.x == 0) atomicAdd((unsigned long long*)scanned, (unsigned long long)m);
  extern __shared__ __align__(16) unsigned long long s_dyn[];
  unsigned long long* s_surv = s_dyn;                          // [kScanWin] survivors of a window
  unsigned long long* s_sj = s_dyn + kScanWin;                 // [kScanWin] their jobs (jobs_pack)
  uint32_t* s_taken = reinterpret_cast<uint32_t*>(s_dyn + 2 * kScanWin);  // n_jobs bits
  __shared__ long long s_np;                                   // picks so far (every resolving warp starts from it)
  __shared__ int s_pidx[kScanWin];                             // survivor index of each pick of a chunk
  __shared__ int s_cnt[kScanPer * (kScanThreads / 32)];
  constexpr int kCntPerLane = kScanPer * (kScanThreads / 32) / 32;  // the prefix pass: counts per lane of warp 0
  __shared__ int s_n;
  __shared__ int s_stop;
  const int words = (int)((n_jobs + 31) >> 5);
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  for (int i = t; i < words; i += kScanThreads) s_taken[i] = taken_g[i];
  if (t == 0) {
    s_stop = 0;
    s_np = np;
  }
  unsigned long long nxt[kScanPer];
#pragma unroll
  for (int u = 0; u < kScanPer; u++) {
    const int64_t i = (int64_t)u * kScanThreads + t;
    nxt[u] = i < m ? sorted[i] : 0ull;
  }
  __syncthreads();
#ifdef COSCHED_SCAN_PROF
  const long long t_k0 = clock64();
  long long t_f = 0, t_r = 0, n_ch = 0, n_sv = 0, np0 = np;
#endif
  for (int64_t base = 0; base < m && !s_stop; base += kScanWin) {
#ifdef COSCHED_SCAN_PROF
    const long long t_c0 = clock64();
#endif
    // 1-2: filter and compact (key order: index u * kScanThreads + t)
    unsigned long long key[kScanPer], jp[kScanPer];
    bool fr[kScanPer];
#pragma unroll
    for (int u = 0; u < kScanPer; u++) {
      key[u] = nxt[u];
      const int64_t i2 = base + kScanWin + (int64_t)u * kScanThreads + t;  // prefetch the next window
      nxt[u] = i2 < m ? sorted[i2] : 0ull;
      int32_t jb[3] = {0, 0, 0};
      fr[u] = key[u] != 0ull && key_jobs_free<NS>(fmt, key[u], s_taken, jb);
      jp[u] = jobs_pack<NS>(jb);
    }
    unsigned bm[kScanPer];
#pragma unroll
    for (int u = 0; u < kScanPer; u++) {
      bm[u] = __ballot_sync(0xFFFFFFFFu, fr[u]);
      if (lane == 0) s_cnt[u * kScanWarps + wid] = __popc(bm[u]);
    }
    __syncthreads();
    if (wid == 0) {  // exclusive prefix over the (u, warp) counts in key order; a lane owns consecutive ones
      int c[kCntPerLane], sum = 0;
#pragma unroll
      for (int r = 0; r < kCntPerLane; r++) {
        c[r] = s_cnt[lane * kCntPerLane + r];
        sum += c[r];
      }
      int incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += v;
      }
      int run = incl - sum;
#pragma unroll
      for (int r = 0; r < kCntPerLane; r++) {
        s_cnt[lane * kCntPerLane + r] = run;
        run += c[r];
      }
      if (lane == 31) s_n = incl;
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kScanPer; u++)
      if (fr[u]) {
        const int at = s_cnt[u * kScanWarps + wid] + __popc(bm[u] & ((1u << lane) - 1u));
        s_surv[at] = key[u];
        s_sj[at] = jp[u];
      }
    __syncthreads();
    const int off = s_n;
#ifdef COSCHED_SCAN_PROF
    const long long t_c1 = clock64();
    t_f += t_c1 - t_c0;
    n_ch++;
    n_sv += off;
#endif
#ifndef COSCHED_SCAN_OLD
    // 3: the sequential rule over the chunk's survivors (all free at the chunk's
    // start, in key order), by warp 0 in batches of 32 x 16: lane l holds
    // survivors l + 32u (u < 16; jobs in registers, a live mask). Each step the
    // smallest live index (one warp min) is the next pick -- every earlier
    // survivor was picked or shares a job with a pick -- and every lane drops its
    // survivors sharing a job with it (branch-free compares): one step per pick,
    // whatever the number of survivors the pick blocks. Between batches the
    // batch's picks are marked taken; the canonical keys are written after the
    // chunk by the whole block.
    np = s_np;  // warps that sat out earlier chunks catch up
    const long long np0 = np;
    if (wid == 0) {
      constexpr int kLs = 16;  // survivors per lane and batch
      for (int b0 = 0; b0 < off && np < k_max; b0 += 32 * kLs) {
        unsigned long long jr[kLs];
        unsigned live = 0u;
#pragma unroll
        for (int u = 0; u < kLs; u++) {  // branch-free: every load of the batch in flight at once
          const int e = b0 + lane + 32 * u;
          jr[u] = s_sj[e < off ? e : 0];
        }
#pragma unroll
        for (int u = 0; u < kLs; u++) {  // taken by an earlier batch of this chunk?
          bool fr = b0 + lane + 32 * u < off;
#pragma unroll
          for (int q = 0; q < NS; q++) {
            const unsigned j = (unsigned)((jr[u] >> (20 * q)) & 0xFFFFFu);
            fr = fr & !((s_taken[j >> 5] >> (j & 31)) & 1u);
          }
          live |= fr ? (1u << u) : 0u;
        }
        const long long npb = np;
#ifdef COSCHED_SCAN_PROF
        const long long t_l0 = clock64();
        long long n_it = 0;
#endif
        while (np < k_max) {
#ifdef COSCHED_SCAN_PROF
          n_it++;
#endif
          const int my = live ? 32 * (__ffs(live) - 1) + lane : 0x7FFFFFFF;
          const int g = __reduce_min_sync(0xFFFFFFFFu, my);
          if (g == 0x7FFFFFFF) break;  // uniform: no live survivor left in the batch
          const unsigned long long pj = s_sj[b0 + g];
          const unsigned p0 = (unsigned)(pj & 0xFFFFFu), p1 = (unsigned)((pj >> 20) & 0xFFFFFu),
                         p2 = (unsigned)((pj >> 40) & 0xFFFFFu);
          unsigned kill = 0u;
#pragma unroll
          for (int u = 0; u < kLs; u++) {  // the pick itself too
            bool c = false;
#pragma unroll
            for (int q = 0; q < NS; q++) {
              const unsigned x = (unsigned)((jr[u] >> (20 * q)) & 0xFFFFFu);
              c = c | (x == p0) | (NS > 1 && x == p1) | (NS > 2 && x == p2);
            }
            kill |= c ? (1u << u) : 0u;
          }
          live &= ~kill;
          if (lane == 0) s_pidx[np - np0] = b0 + g;
          np++;
        }
#ifdef COSCHED_SCAN_PROF
        if (lane == 0) {
          atomicAdd(&g_scan_prof[8], (unsigned long long)(clock64() - t_l0));
          atomicAdd(&g_scan_prof[9], (unsigned long long)n_it);
          atomicAdd(&g_scan_prof[10], 1ull);
        }
#endif
        __syncwarp();
        for (long long i = npb + lane; i < np; i += 32) {  // this batch's picks: taken for the next batches
          int32_t tj[3];
          jobs_unpack<NS>(s_sj[s_pidx[i - np0]], tj);
#pragma unroll
          for (int q = 0; q < NS; q++) atomicOr(&s_taken[tj[q] >> 5], 1u << (tj[q] & 31));
        }
        __syncwarp();
      }
    }
    if (t == 0) s_np = np;
    __syncthreads();
    {
      const long long np1 = s_np;
      for (int i = t; i < (int)(np1 - np0); i += kScanThreads) {  // the chunk's picks, in parallel
        const int g = s_pidx[i];
        int32_t tj[3];
        jobs_unpack<NS>(s_sj[g], tj);
        picks[np0 + i] = gkey_canonical<NS>(fmt, s_surv[g], tj);
      }
      np = np1;
      if (t == 0) s_stop = np1 >= k_max;
    }
#else
    // 3: warp 0 resolves the survivors in order, kRes groups of 32 per step: all
    // their shared-memory loads in flight at once (the step is latency-bound);
    // a pick removes the keys sharing a job from its own and the later groups
    if (wid == 0) {
      constexpr int kRes = 8;
      for (int g = 0; g < off && np < k_max; g += 32 * kRes) {
        unsigned long long kk[kRes];
        int32_t jb[kRes][3];
        unsigned cand[kRes];
#pragma unroll
        for (int r = 0; r < kRes; r++) {
          const int e = g + 32 * r + lane;
          kk[r] = e < off ? s_surv[e] : 0ull;
          jb[r][0] = jb[r][1] = jb[r][2] = -1;
          const bool ok = kk[r] != 0ull && key_jobs_free<NS>(fmt, kk[r], s_taken, jb[r]);
          cand[r] = __ballot_sync(0xFFFFFFFFu, ok);
        }
#pragma unroll
        for (int r = 0; r < kRes; r++) {
          while (cand[r] && np < k_max) {
            const int l = __ffs(cand[r]) - 1;
            int32_t tj[3];
#pragma unroll
            for (int q = 0; q < NS; q++) tj[q] = __shfl_sync(0xFFFFFFFFu, jb[r][q], l);
            const unsigned long long pk = __shfl_sync(0xFFFFFFFFu, kk[r], l);
            if (lane == 0) {
#pragma unroll
              for (int q = 0; q < NS; q++) s_taken[tj[q] >> 5] |= 1u << (tj[q] & 31);
              picks[np] = gkey_canonical<NS>(fmt, pk, tj);
            }
            np++;
#pragma unroll
            for (int r2 = 0; r2 < kRes; r2++) {
              if (r2 < r) continue;
              bool clash = false;
#pragma unroll
              for (int q = 0; q < NS; q++)
#pragma unroll
                for (int q2 = 0; q2 < NS; q2++) clash = clash || (jb[r2][q] == tj[q2]);
              cand[r2] &= ~__ballot_sync(0xFFFFFFFFu, clash);
            }
            __syncwarp();
          }
        }
      }
      if (lane == 0) s_stop = np >= k_max;
    }
#endif
    __syncthreads();  // taken bits and the stop flag are visible to the next window
#ifdef COSCHED_SCAN_PROF
    t_r += clock64() - t_c1;
#endif
  }
#ifdef COSCHED_SCAN_PROF
  if (t == 0) {
    atomicAdd(&g_scan_prof[0], (unsigned long long)t_f);
    atomicAdd(&g_scan_prof[1], (unsigned long long)t_r);
    atomicAdd(&g_scan_prof[2], (unsigned long long)n_ch);
    atomicAdd(&g_scan_prof[3], (unsigned long long)n_sv);
    atomicAdd(&g_scan_prof[5], 1ull);
    atomicAdd(&g_scan_prof[6], (unsigned long long)(clock64() - t_k0));
  }
  if (t == 0) atomicAdd(&g_scan_prof[4], (unsigned long long)(np - np0));
#endif
  for (int i = t; i < words; i += kScanThreads) taken_g[i] = s_taken[i];
  if (t == 0) *n_picks = np;
}

// ---- the sequential rule as a producer / consumer pipeline over the whole GPU ----
// One cooperative launch per sorted batch (all CTAs resident, one per SM).
// Producers (CTAs 1..G-1) claim windows of kPipeWin consecutive keys of the
// sorted list in order, drop the keys with a taken job -- reading the taken
// bitmask the consumer publishes, at most kPipeLag windows stale -- and write
// the survivors, still in key order, to a ring slot. The consumer (warp 0 of
// CTA 0) takes the slots in window order and applies the sequential rule to
// the survivors against its own exact taken bitmask (shared memory): a
// survivor whose jobs are all free is the next pick. Staleness only lets
// extra keys through the filter; the picks are exactly the sequential
// greedy's. The consumer publishes every pick's jobs (global taken bits) and
// its window progress; producers wait when kPipeLag windows ahead.
#ifndef COSCHED_PIPE_PARTS
#define COSCHED_PIPE_PARTS 2
#endif
#ifndef COSCHED_PIPE_AHEAD
#define COSCHED_PIPE_AHEAD 4
#endif
constexpr int kPipeThreads = 512, kPipePer = 16, kPipeSub = kPipeThreads * kPipePer, kPipeParts = COSCHED_PIPE_PARTS;
constexpr int kPipeWin = kPipeSub * kPipeParts, kPipeLag = kPipeSlots;
constexpr int kPipeAhead = COSCHED_PIPE_AHEAD;  // producers run at most this many windows ahead of the consumer

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <int NS>
__global__ void __launch_bounds__(kPipeThreads, 1)
    k_greedy_pipe(const unsigned long long* __restrict__ sorted, int64_t m, int64_t n_jobs, uint32_t* taken_g,
                  unsigned long long* picks, int64_t* n_picks, int64_t k_max, const GKeyFmt fmt,
                  unsigned long long* ring, int* ring_cnt, int* ring_flag, int* ctl /* [0] next, [1] done, [2] stop */) {
  extern __shared__ __align__(16) unsigned long long p_dyn[];
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const int64_t n_win = (m + kPipeWin - 1) / kPipeWin;
  const int words = (int)((n_jobs + 31) >> 5);
  if (blockIdx.x == 0) {
    // ---------------- consumer ----------------
    // warps 1..: loaders -- wait for window w+1's slot and copy its survivors into
    // the shared buffer (w+1) % 2; warp 0: the sequential rule over buffer w % 2,
    // against the exact taken bitmask in shared memory. One barrier per window.
    constexpr int kBuf = kPipeSub;  // survivors staged per window; beyond that warp 0 reads the slot in L2
    unsigned long long* s_buf = p_dyn;                                        // [2][kBuf]
    uint32_t* s_taken = reinterpret_cast<uint32_t*>(p_dyn + 2 * kBuf);       // n_jobs bits
    __shared__ int s_c[2], s_stop_c;
    for (int i = t; i < words; i += kPipeThreads) s_taken[i] = taken_g[i];
    if (t == 0) s_stop_c = 0;
    constexpr int kLoaders = kPipeThreads - 32;
    auto load = [&](int64_t w) {  // loader warps only
      const int slot = (int)(w % kPipeLag);
      if (t == 32)
        while (ld_acquire(ring_flag + slot) != (int)(w + 1)) __nanosleep(32);
      asm volatile("bar.sync 1, %0;" ::"r"(kLoaders));  // loaders only
      const int c = __ldcg(ring_cnt + slot);
      const unsigned long long* src = ring + (size_t)slot * kPipeWin;
      unsigned long long* dst = s_buf + (size_t)(w & 1) * kBuf;
      const int cs = c < kBuf ? c : kBuf;
      for (int e = t - 32; e < cs; e += kLoaders) dst[e] = __ldcg(src + e);
      if (t == 32) {
        s_c[w & 1] = c;
        atomicAdd(ctl + 3, c);  // survivors (instrumentation)
      }
    };
    if (t >= 32 && n_win > 0) load(0);
    __syncthreads();
    int64_t np = *n_picks;
    for (int64_t w = 0; w < n_win; w++) {
      if (wid == 0) {
        const int c = s_c[w & 1];
        const unsigned long long* sv = s_buf + (size_t)(w & 1) * kBuf;
        const unsigned long long* gv = ring + (size_t)(w % kPipeLag) * kPipeWin;
        constexpr int kRes = 8;
        for (int g = 0; g < c && np < k_max; g += 32 * kRes) {
          unsigned long long kk[kRes];
          int32_t jb[kRes][3];
          unsigned cand[kRes];
#pragma unroll
          for (int r = 0; r < kRes; r++) {
            const int e = g + 32 * r + lane;
            kk[r] = e < c ? (e < kBuf ? sv[e] : __ldcg(gv + e)) : 0ull;
            jb[r][0] = jb[r][1] = jb[r][2] = -1;
            const bool ok = kk[r] != 0ull && key_jobs_free<NS>(fmt, kk[r], s_taken, jb[r]);
            cand[r] = __ballot_sync(0xFFFFFFFFu, ok);
          }
#pragma unroll
          for (int r = 0; r < kRes; r++) {
            while (cand[r] && np < k_max) {
              const int l = __ffs(cand[r]) - 1;
              int32_t tj[3];
#pragma unroll
              for (int q = 0; q < NS; q++) tj[q] = __shfl_sync(0xFFFFFFFFu, jb[r][q], l);
              const unsigned long long pk = __shfl_sync(0xFFFFFFFFu, kk[r], l);
              if (lane == 0) {
#pragma unroll
                for (int q = 0; q < NS; q++) {
                  s_taken[tj[q] >> 5] |= 1u << (tj[q] & 31);
                  atomicOr(taken_g + (tj[q] >> 5), 1u << (tj[q] & 31));  // published to the producers
                }
                picks[np] = gkey_canonical<NS>(fmt, pk, tj);
              }
              np++;
#pragma unroll
              for (int r2 = 0; r2 < kRes; r2++) {
                if (r2 < r) continue;
                bool clash = false;
#pragma unroll
                for (int q = 0; q < NS; q++)
#pragma unroll
                  for (int q2 = 0; q2 < NS; q2++) clash = clash || (jb[r2][q] == tj[q2]);
                cand[r2] &= ~__ballot_sync(0xFFFFFFFFu, clash);
              }
              __syncwarp();
            }
          }
        }
        if (lane == 0 && np >= k_max) s_stop_c = 1;
      } else if (w + 1 < n_win) {
        load(w + 1);
      }
      __syncthreads();
      if (t == 0) st_release(ctl + 1, (int)(w + 1));  // window w consumed: its ring slot is free
      if (s_stop_c) break;
    }
    if (t == 0) {
      *n_picks = np;
      st_release(ctl + 2, 1);  // stop: the producers exit
    }
    return;
  }
  // ---------------- producers ----------------
  __shared__ int s_w, s_stop;
  __shared__ int s_cnt[kPipePer * (kPipeThreads / 32)];
  __shared__ int s_n;
  constexpr int kWarps = kPipeThreads / 32, kCntPerLane = kPipePer * kWarps / 32;
  for (;;) {
    if (t == 0) {
      int w = atomicAdd(ctl + 0, 1);
      int stop = ld_acquire(ctl + 2);
      while (!stop && w < n_win && w >= ld_acquire(ctl + 1) + kPipeAhead) {
        __nanosleep(128);
        stop = ld_acquire(ctl + 2);
      }
      s_w = w;
      s_stop = stop;
    }
    __syncthreads();
    const int64_t w = s_w;
    if (s_stop || w >= n_win) return;
    const int slot = (int)(w % kPipeLag);
    unsigned long long* dst = ring + (size_t)slot * kPipeWin;
    int run = 0;  // survivors written so far (block-uniform)
    for (int part = 0; part < kPipeParts; part++) {
    const int64_t base = w * kPipeWin + (int64_t)part * kPipeSub;
    unsigned long long key[kPipePer];
    bool fr[kPipePer];
#pragma unroll
    for (int u = 0; u < kPipePer; u++) {
      const int64_t i = base + (int64_t)u * kPipeThreads + t;
      key[u] = i < m ? __ldg(sorted + i) : 0ull;
    }
#pragma unroll
    for (int u = 0; u < kPipePer; u++) {
      fr[u] = false;
      if (key[u]) {
        int32_t jb[3];
        gkey_jobs<NS>(fmt, key[u], jb);
        bool f = true;
#pragma unroll
        for (int q = 0; q < NS; q++) f = f && !((ld_relaxed_u32(taken_g + (jb[q] >> 5)) >> (jb[q] & 31)) & 1u);
        fr[u] = f;
      }
    }
    unsigned bm[kPipePer];
#pragma unroll
    for (int u = 0; u < kPipePer; u++) {
      bm[u] = __ballot_sync(0xFFFFFFFFu, fr[u]);
      if (lane == 0) s_cnt[u * kWarps + wid] = __popc(bm[u]);
    }
    __syncthreads();
    if (wid == 0) {
      int c[kCntPerLane], sum = 0;
#pragma unroll
      for (int r = 0; r < kCntPerLane; r++) {
        c[r] = s_cnt[lane * kCntPerLane + r];
        sum += c[r];
      }
      int incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += v;
      }
      int run = incl - sum;
#pragma unroll
      for (int r = 0; r < kCntPerLane; r++) {
        s_cnt[lane * kCntPerLane + r] = run;
        run += c[r];
      }
      if (lane == 31) s_n = incl;
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kPipePer; u++)
      if (fr[u]) __stcg(dst + run + s_cnt[u * kWarps + wid] + __popc(bm[u] & ((1u << lane) - 1u)), key[u]);
    run += s_n;
    __syncthreads();  // s_cnt / s_n are rewritten by the next part
    }
    __syncthreads();  // every survivor written before the slot is published
    if (t == 0) {
      ring_cnt[slot] = run;
      __threadfence();
      st_release(ring_flag + slot, (int)(w + 1));
    }
  }
}

// One cooperative launch (all CTAs co-resident: the pipeline spin-waits across CTAs).
cudaError_t launch_greedy_pipe(int n_slots, const unsigned long long* sorted, int64_t m, int64_t n_jobs,
                               uint32_t* taken_bits, unsigned long long* picks, int64_t* n_picks, int64_t k_max,
                               const GKeyFmt& fmt, unsigned long long* ring, int* ring_cnt, int* ring_flag, int* ctl,
                               cudaStream_t st) {
  if (m <= 0) return cudaSuccess;
  if (n_jobs > ((int64_t)1 << 20)) return cudaErrorInvalidValue;
  cudaError_t e = cudaMemsetAsync(ring_flag, 0, sizeof(int) * (kPipeLag + 4), st);  // flags and ctl are contiguous
  if (e != cudaSuccess) return e;
  // consumer: two survivor buffers + the taken bitmask (the producers use none of it)
  const size_t smem = sizeof(unsigned long long) * 2 * kPipeSub + (size_t)((n_jobs + 31) / 32) * 4;
  const void* fn = n_slots == 2 ? (const void*)k_greedy_pipe<2> : (const void*)k_greedy_pipe<3>;
  e = smem_optin(fn, smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, n_slots == 2 ? (const void*)k_greedy_pipe<2>
                                                                       : (const void*)k_greedy_pipe<3>,
                                                kPipeThreads, smem);
  const int64_t windows = (m + kPipeWin - 1) / kPipeWin;
  int grid = (int)std::min<int64_t>((int64_t)num_sms() * std::max(per_sm, 1), windows + 1);
  grid = std::max(grid, 2);
  void* args[] = {(void*)&sorted, (void*)&m, (void*)&n_jobs, (void*)&taken_bits, (void*)&picks, (void*)&n_picks,
                  (void*)&k_max, (void*)&fmt, (void*)&ring, (void*)&ring_cnt, (void*)&ring_flag, (void*)&ctl};
  return cudaLaunchCooperativeKernel(fn, grid, kPipeThreads, args, smem, st);
}

size_t greedy_pipe_ring_bytes() { return sizeof(unsigned long long) * kPipeWin * kPipeLag; }

// predicate of the order-preserving re-filter between scan chunks
// The window select of the greedy scan in one launch: block q keeps, in order,
// the keys of tile q (kSelTile consecutive keys of the sorted batch) whose jobs
// are all free and writes them at its offset in one compacted list. The offset
// is the sum of the earlier tiles' counts, which every block publishes as soon
// as it has counted (tagged with the launch's epoch, so the flags need no reset
// within an allocation); blocks start in index order, so a block only waits for
// counts that are being computed. The last block writes the list length.
template <int NS>
__global__ void __launch_bounds__(kSelThreads) k_select_free(const unsigned long long* __restrict__ in, int64_t n,
                                                             const uint32_t* __restrict__ taken,
                                                             unsigned long long* __restrict__ out, int64_t* m_out,
                                                             unsigned long long* flags, unsigned epoch,
                                                             const GKeyFmt fmt, const int64_t* n_picks,
                                                             int64_t k_max) {
  __shared__ int s_c[kSelPer][kSelThreads / 32];
  __shared__ long long s_off;
  pdl_wait();  // the previous scan's taken bits
  pdl_launch_dependents();
  if (*n_picks >= k_max) {  // windows enqueued after the k-th pick: nothing to select
    if (blockIdx.x == 0 && threadIdx.x == 0) *m_out = 0;
    return;
  }
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const int q = blockIdx.x;
  const int64_t base = (int64_t)q * kSelTile;
  unsigned long long k[kSelPer];
  unsigned bm[kSelPer];
#pragma unroll
  for (int u = 0; u < kSelPer; u++) {
    const int64_t i = base + u * kSelThreads + t;
    k[u] = i < n ? __ldcs(in + i) : 0ull;
  }
#pragma unroll
  for (int u = 0; u < kSelPer; u++) {
    int32_t jb[3];
    const bool f = k[u] != 0ull && key_jobs_free<NS>(fmt, k[u], taken, jb);
    bm[u] = __ballot_sync(0xFFFFFFFFu, f);
    if (lane == 0) s_c[u][wid] = __popc(bm[u]);
  }
  __syncthreads();
  if (wid == 0) {
    // exclusive prefix over the (u, warp) counts in key order: 4 per lane
    constexpr int kPer = kSelPer * (kSelThreads / 32) / 32;
    int* c = &s_c[0][0];
    int v[kPer], sum = 0;
#pragma unroll
    for (int r = 0; r < kPer; r++) {
      v[r] = c[lane * kPer + r];
      sum += v[r];
    }
    int incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int x = __shfl_up_sync(0xFFFFFFFFu, incl, o);
      if (lane >= o) incl += x;
    }
    int run = incl - sum;
#pragma unroll
    for (int r = 0; r < kPer; r++) {
      c[lane * kPer + r] = run;
      run += v[r];
    }
    const int tot = __shfl_sync(0xFFFFFFFFu, incl, 31);
    if (lane == 0) {  // publish this tile's count
      const unsigned long long tag = ((unsigned long long)epoch << 32) | (unsigned)tot;
      asm volatile("st.release.gpu.global.b64 [%0], %1;" ::"l"(flags + q), "l"(tag) : "memory");
    }
    long long off = 0;  // the earlier tiles' counts
    for (int q0 = 0; q0 < q; q0 += 32) {
      long long x = 0;
      if (q0 + lane < q) {
        unsigned long long f;
        do {
          asm volatile("ld.acquire.gpu.global.b64 %0, [%1];" : "=l"(f) : "l"(flags + q0 + lane) : "memory");
        } while ((unsigned)(f >> 32) != epoch);
        x = (long long)(f & 0xFFFFFFFFull);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xFFFFFFFFu, x, o);
      off += x;
    }
    if (lane == 0) {
      s_off = off;
      if (q == (int)gridDim.x - 1) *m_out = off + tot;
    }
  }
  __syncthreads();
  unsigned long long* o = out + s_off;
#pragma unroll
  for (int u = 0; u < kSelPer; u++)
    if ((bm[u] >> lane) & 1u) o[s_c[u][wid] + __popc(bm[u] & ((1u << lane) - 1u))] = k[u];
}

cudaError_t launch_select_free(int n_slots, const unsigned long long* in, int64_t n, const uint32_t* taken,
                               unsigned long long* out, int64_t* m_out, unsigned long long* flags, unsigned epoch,
                               const GKeyFmt& fmt, const int64_t* n_picks, int64_t k_max, cudaStream_t st) {
  const int64_t tiles = (n + kSelTile - 1) / kSelTile;
  if (tiles > kSelMaxTiles) return cudaErrorInvalidValue;
  if (tiles <= 0) return cudaSuccess;
  if (n_slots == 2)
    return launch_pdl(k_select_free<2>, dim3((unsigned)tiles), dim3(kSelThreads), 0, st, in, n, taken, out, m_out,
                      flags, epoch, fmt, n_picks, k_max);
  return launch_pdl(k_select_free<3>, dim3((unsigned)tiles), dim3(kSelThreads), 0, st, in, n, taken, out, m_out, flags,
                    epoch, fmt, n_picks, k_max);
}
int select_tiles(int64_t n) { return (int)((n + kSelTile - 1) / kSelTile); }

template <int NS>
struct AllJobsFree {
  const uint32_t* bits;
  GKeyFmt fmt;
  __device__ __forceinline__ bool operator()(const unsigned long long& key) const {
    if (!key) return false;
    int32_t jb[3];
    return key_jobs_free<NS>(fmt, key, bits, jb);
  }
};

size_t select_temp_bytes(int64_t n) {
  size_t bytes = 0;
  AllJobsFree<2> pred{nullptr, GKeyFmt()};
  cub::DeviceSelect::If((void*)nullptr, bytes, (const unsigned long long*)nullptr, (unsigned long long*)nullptr,
                        (int64_t*)nullptr, (int)std::max<int64_t>(n, 1), pred);
  size_t b3 = 0;
  AllJobsFree<3> pred3{nullptr, GKeyFmt()};
  cub::DeviceSelect::If((void*)nullptr, b3, (const unsigned long long*)nullptr, (unsigned long long*)nullptr,
                        (int64_t*)nullptr, (int)std::max<int64_t>(n, 1), pred3);
  return std::max(bytes, b3);
}

cudaError_t select_free_keys(int n_slots, void* temp, size_t temp_bytes, const unsigned long long* in,
                             unsigned long long* out, int64_t* n_out, int64_t n, const uint32_t* taken_bits,
                             const GKeyFmt& fmt, cudaStream_t st) {
  if (n_slots == 2)
    return cub::DeviceSelect::If(temp, temp_bytes, in, out, n_out, (int)n, AllJobsFree<2>{taken_bits, fmt}, st);
  return cub::DeviceSelect::If(temp, temp_bytes, in, out, n_out, (int)n, AllJobsFree<3>{taken_bits, fmt}, st);
}

// ---- launchers -------------------------------------------------------------------------
void launch_obj_minmax(const float* obj, int64_t count, unsigned* mm, cudaStream_t st) {
  if (count <= 0) return;
  int64_t blocks = std::min<int64_t>((count + 255) / 256, 148 * 8);
  k_obj_minmax<<<(unsigned)blocks, 256, 0, st>>>(obj, count, mm);
}
void launch_obj_hist(const float* obj, int64_t count, const unsigned* mm, int nbins, unsigned* hist, cudaStream_t st) {
  if (count <= 0) return;
  smem_optin((const void*)k_obj_hist, kHistBins * 4);
  int64_t blocks = std::min<int64_t>((count + 1023) / 1024, 148 * 2);
  k_obj_hist<<<(unsigned)blocks, 1024, kHistBins * 4, st>>>(obj, count, mm, nbins, hist);
}
void launch_keys_in_range(int n_slots, const float* obj, int64_t first, int64_t count, const unsigned* mm, int nbins,
                          int bin_lo, int bin_hi, const uint32_t* taken_bits, unsigned long long* keys,
                          unsigned long long* n_keys, const GKeyFmt& fmt, cudaStream_t st) {
  if (count <= 0) return;
  int64_t blocks = std::min<int64_t>((count + 32 * kKirWarps * 4 * kKirLoads - 1) / (32 * kKirWarps * 4 * kKirLoads),
                                     148 * 8);
  if (n_slots == 2)
    k_keys_in_range<2><<<(unsigned)blocks, 32 * kKirWarps, 0, st>>>(obj, first, count, mm, nbins, bin_lo, bin_hi,
                                                                    taken_bits, keys, n_keys, fmt);
  else
    k_keys_in_range<3><<<(unsigned)blocks, 32 * kKirWarps, 0, st>>>(obj, first, count, mm, nbins, bin_lo, bin_hi,
                                                                    taken_bits, keys, n_keys, fmt);
}

size_t sort_temp_bytes(int64_t n) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortKeysDescending((void*)nullptr, bytes, (const unsigned long long*)nullptr,
                                           (unsigned long long*)nullptr, (int)std::max<int64_t>(n, 1));
  return bytes;
}

cudaError_t sort_keys_desc(void* temp, size_t temp_bytes, const unsigned long long* in, unsigned long long* out,
                           int64_t n, cudaStream_t st, int end_bit) {
  return cub::DeviceRadixSort::SortKeysDescending(temp, temp_bytes, in, out, (int)n, 0, end_bit, st);
}

cudaError_t launch_greedy_scan(int n_slots, const unsigned long long* sorted, int64_t m, const int64_t* m_dev,
                               int64_t n_jobs, uint32_t* taken_bits, unsigned long long* picks, int64_t* n_picks,
                               int64_t k_max, const GKeyFmt& fmt, cudaStream_t st, int64_t* scanned) {
  // dynamic shared memory: a window's survivors (64 KB) and the taken bitmask
  // (n_jobs bits; <= 2^20 jobs, far above any queue the set scorer accepts)
  const size_t smem = sizeof(unsigned long long) * 2 * kScanWin + (size_t)((n_jobs + 31) / 32) * 4;
  if (n_jobs > ((int64_t)1 << 20)) return cudaErrorInvalidValue;
  if (n_slots == 2) {
    cudaError_t e = smem_optin((const void*)k_greedy_scan<2>, smem);
    if (e != cudaSuccess) return e;
    e = launch_pdl(k_greedy_scan<2>, dim3(1), dim3(kScanThreads), smem, st, sorted, m, m_dev, n_jobs, taken_bits, picks,
                   n_picks, k_max, fmt, scanned);
    if (e != cudaSuccess) return e;
  } else {
    cudaError_t e = smem_optin((const void*)k_greedy_scan<3>, smem);
    if (e != cudaSuccess) return e;
    e = launch_pdl(k_greedy_scan<3>, dim3(1), dim3(kScanThreads), smem, st, sorted, m, m_dev, n_jobs, taken_bits, picks,
                   n_picks, k_max, fmt, scanned);
    if (e != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

#ifdef COSCHED_SCAN_PROF
void scan_prof_report() {
  unsigned long long v[12];
  cudaMemcpyFromSymbol(v, g_scan_prof, sizeof v);
  fprintf(stderr, "scan prof: pick loop %.3f Mcyc, %llu steps, %llu batches\n", v[8] / 1e6,
          v[9], v[10]);
  fprintf(stderr, "scan prof: filter %.3f Mcyc, resolve %.3f Mcyc, kernel %.3f Mcyc, chunks %llu, survivors %llu, picks %llu, launches %llu\n",
          v[0] / 1e6, v[1] / 1e6, v[6] / 1e6, v[2], v[3], v[4], v[5]);
  unsigned long long z[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  cudaMemcpyToSymbol(g_scan_prof, z, sizeof z);
}
#else
void scan_prof_report() {}
#endif
}  // namespace cosched
