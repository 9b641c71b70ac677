// kernels.cu -- the CUDA path of the co-location search (sm_100a).
//
// Steps: a1 validate features, a2 basis H/J,
// a3 projection onto C/D (the exact factorisation of P:L458), a4-a7 set
// enumeration + model evaluation + objective/fairness + per-set argmax,
// a8 per-shard argmax key, a10 allocation (exact / greedy).
//
// The fast pair scorer lives in score_pairs.cu; this file holds the generic
// scorer (any n_slots, also the reference for the fast one), the per-set
// detail evaluator and the allocation kernels.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <algorithm>
#include <mutex>
#include <set>
#include <tuple>

#include "cosched_internal.h"
#include "device_common.cuh"

namespace cosched {

// ---------------------------------------------------------------------------
// a1: validation (SPEC.md L26-27 ranges, L54/L87 degenerate F1) and a2: the
// basis H, J of every queue position, computed once per job (4
// IEEE divisions) into hj[pos][12] = (H1..H6, J1..J3, 0, 0, 0). One thread per
// queue position; the first bad position wins through an atomicMin on
// (pos << 8 | status).
__global__ void k_validate(const float* __restrict__ F, int64_t n_rows, const int32_t* __restrict__ jobs,
                           int64_t n_jobs, unsigned long long* err, float* __restrict__ hj) {
  int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= n_jobs) return;
  // the inputs were copied before the step began: read and test them before
  // the PDL wait; the err word (reset by k_step_init) and hj after it
  int64_t row = jobs ? (int64_t)jobs[q] : q;
  int code = 0;
  if (row < 0 || row >= n_rows) {
    code = COSCHED_E_ARG;
  } else {
    const float* f = F + row * 8;
    float v[8];
#pragma unroll
    for (int k = 0; k < 8; k++) v[k] = f[k];
#pragma unroll
    for (int k = 0; k < 8; k++)
      if (!(v[k] >= 0.0f && v[k] <= 100.0f)) code = COSCHED_E_RANGE;
    if (!code) {
      float tensor = __fadd_rn(__fadd_rn(v[5], v[6]), v[7]);
      if (!(tensor <= 100.0f)) code = COSCHED_E_RANGE;
      else if (!(v[0] > 0.01f)) code = COSCHED_E_DEGENERATE_PROFILE;
    }
    if (!code) {
      float h[6], j[3];
      basis_hj(v, h, j);
      pdl_wait();
      pdl_launch_dependents();
      float4* o = reinterpret_cast<float4*>(hj + q * 12);
      o[0] = make_float4(h[0], h[1], h[2], h[3]);
      o[1] = make_float4(h[4], h[5], j[0], j[1]);
      o[2] = make_float4(j[2], 0.0f, 0.0f, 0.0f);
    }
  }
  if (code) {
    pdl_wait();
    atomicMin(err, ((unsigned long long)q << 8) | (unsigned long long)code);
  }
}

void launch_validate(const float* features, int64_t n_rows, const int32_t* jobs, int64_t n_jobs,
                     unsigned long long* err, float* hj, cudaStream_t st) {
  if (n_jobs <= 0) return;
  int bs = 256;
  launch_pdl(k_validate, dim3((unsigned)((n_jobs + bs - 1) / bs)), dim3(bs), 0, st, features, n_rows, jobs, n_jobs, err,
             hj);
}

// ---------------------------------------------------------------------------
// a3: projection (the exact factorisation of P:L458). For job n, slice s, cap p:
//   U = C[p][s] . H(F_n),  V = D[p][s] . J(F_n)   (the two dot products of P:L458)
//   ka = K*(U - alpha),   kb = K*V               (exact power-of-two scaling,
//                                                 flushed / clamped: cosched_internal.h)
//   w[slot][state] = (U[s_slot] + sum_{l != slot} V[s_l]) * fl(1/P)
// One function per quantity, shared by the projection and the gather kernels,
// so both compute bit-identical values.
// Padding caps (p >= n_caps) get kPadMargin (-FLT_MAX) so every candidate using them is infeasible.
__device__ __forceinline__ float dot_u(const float c[6], const float h[6]) {
  float u = __fmul_rn(c[0], h[0]);
#pragma unroll
  for (int t = 1; t < 6; t++) u = __fmaf_rn(c[t], h[t], u);
  return u;
}
__device__ __forceinline__ float dot_v(const float d[3], const float j[3]) {
  float v = __fmul_rn(d[0], j[0]);
#pragma unroll
  for (int t = 1; t < 3; t++) v = __fmaf_rn(d[t], j[t], v);
  return v;
}
__device__ __forceinline__ void load_hj(const float* __restrict__ hj, int64_t n, float h[6], float j[3]) {
  const float4* q = reinterpret_cast<const float4*>(hj + n * 12);
  const float4 a = __ldg(q), b = __ldg(q + 1), c = __ldg(q + 2);
  h[0] = a.x; h[1] = a.y; h[2] = a.z; h[3] = a.w; h[4] = b.x; h[5] = b.y;
  j[0] = b.z; j[1] = b.w; j[2] = c.x;
}
__device__ __forceinline__ float flush_clamp(float x) {
  x = fminf(fmaxf(x, -kClampAbs), kClampAbs);  // no overflow in a sum of three, no NaN against the padding
  return fabsf(x) < kFlushBelow ? 0.0f : x;    // nonzero operands are multiples of 8: margins are 0 or >= 8
}

// The coefficient rows one (slot, state or slice, cap) needs, held in registers
// by the lane that owns that column while it loops over jobs.
struct CoefRow {
  float c[6];                   // C[p][slice of the slot]
  float d[kMaxSlots][3];        // D[p][slice]: [0] for a kb row; for a w row D of the other slots, ascending
  float inv_p;
  float wfloor;                 // w row: below this share every config is infeasible (feasibility floor)
};
__device__ __forceinline__ void load_c(CoefRow& r, const SpaceParams& sp, const float* __restrict__ coef_c, int slice,
                                       int p) {
#pragma unroll
  for (int t = 0; t < 6; t++) r.c[t] = __ldg(coef_c + ((int64_t)p * sp.n_slices + slice) * 6 + t);
}
__device__ __forceinline__ void load_d(float d[3], const SpaceParams& sp, const float* __restrict__ coef_d, int slice,
                                       int p) {
#pragma unroll
  for (int t = 0; t < 3; t++) d[t] = __ldg(coef_d + ((int64_t)p * sp.n_slices + slice) * 3 + t);
}
// Bounds of V = D.J over valid features: J = (F3/100, F4/100, 1) with F3, F4 in
// [0, 100] (a1), so J1, J2 in [0, 1] and V lies in [d3 + min(d1,0) + min(d2,0),
// d3 + max(d1,0) + max(d2,0)].
__device__ __forceinline__ float vmax_of(const float d[3]) { return d[2] + fmaxf(d[0], 0.0f) + fmaxf(d[1], 0.0f); }
__device__ __forceinline__ float vmin_of(const float d[3]) { return d[2] + fminf(d[0], 0.0f) + fminf(d[1], 0.0f); }

// w row of (slot, state s) at cap p: C of the slot's slice, D of the other slots' slices.
// Feasibility floor (DESIGN.md §2 "Exactness of the tiled argmax"): a feasible
// config has RPerf_i = U_i[s_i] + sum_{l!=i} V_l[s_i] > alpha, so U_i[s_i] >
// alpha - (NS-1) Vmax[s_i], and w_i = (U_i[s_i] + sum_{l!=i} V_i[s_l]) / P >
// (alpha - (NS-1) Vmax[s_i] + sum_{l!=i} Vmin[s_l]) / P. Shares below that
// (minus a slack far above the FP32 rounding of these O(1) sums) belong to
// infeasible configs only, so they are left out of the quantisation range and
// coded as its bottom: one extreme but valid profile (F1 near 0.01 %, H3 = F2/F1
// up to 10^4) cannot coarsen the packed objective of the whole queue.
__device__ __forceinline__ void load_w_row(CoefRow& r, const SpaceParams& sp, const float* __restrict__ coef_c,
                                           const float* __restrict__ coef_d, int slot, int s, int p) {
  load_c(r, sp, coef_c, sp.slice[s][slot], p);
  float own[3];
  load_d(own, sp, coef_d, sp.slice[s][slot], p);
  const float vmx = vmax_of(own);
  float f = sp.alpha, mag = 1.0f + fabsf(sp.alpha);
  int k = 0;
  for (int l = 0; l < sp.n_slots; l++)
    if (l != slot) {
      load_d(r.d[k], sp, coef_d, sp.slice[s][l], p);
      const float vmn = vmin_of(r.d[k]);
      f = f - vmx + vmn;
      mag += fabsf(vmx) + fabsf(vmn);
      k++;
    }
  r.inv_p = sp.inv_p[p];
  r.wfloor = (f - 1e-3f * mag) * r.inv_p;
}
__device__ __forceinline__ float ka_value(const SpaceParams& sp, const CoefRow& r, const float h[6]) {
  return flush_clamp(__fmul_rn(__fsub_rn(dot_u(r.c, h), sp.alpha), kScale));
}
__device__ __forceinline__ float kb_value(const CoefRow& r, const float j[3]) {
  return flush_clamp(__fmul_rn(dot_v(r.d[0], j), kScale));
}
template <int NS>
__device__ __forceinline__ float w_value(const CoefRow& r, const float h[6], const float j[3]) {
  float acc = dot_u(r.c, h);
#pragma unroll
  for (int k = 0; k + 1 < NS; k++) acc = __fadd_rn(acc, dot_v(r.d[k], j));
  return __fmul_rn(acc, r.inv_p);
}

// Both kernels below: a thread owns a job (its basis in registers, one
// coalesced 48-byte load), loops over the columns of its row (caps or the 20
// configs of a stage) with the columns' coefficient rows broadcast from shared
// memory, and writes the row into a per-warp staging tile; the warp then stores
// its 32 consecutive rows, which are contiguous in global memory, with
// coalesced stores.
constexpr int kProjWarps = 4;
constexpr int kProjJobs = 32 * kProjWarps;

// A warp's 32 staged rows (row stride ld = cols + 1 floats) -> 32 consecutive
// rows of `cols` floats in global memory: one flat coalesced copy, the (row,
// col) of each element advanced incrementally (no division).
__device__ __forceinline__ void flush_rows(const float* stg, int ld, int cols, float* __restrict__ dst, int lane) {
  const int step_r = 32 / cols, step_c = 32 - step_r * cols;
  int r = lane / cols, c = lane - r * cols;
  for (int e = lane; e < 32 * cols; e += 32) {
    dst[e] = stg[r * ld + c];
    r += step_r;
    c += step_c;
    if (c >= cols) {
      c -= cols;
      r++;
    }
  }
}

// Grid (x: blocks of kProjJobs jobs, y: row kind): y < n_slices -> the ka and kb
// rows of slice y; else the w row of (slot, state) = divmod(y - n_slices,
// n_states). The per-slot min/max of w is reduced per block, then one atomic
// per block. Block-uniform branches only; the cap loop has no per-element test.
template <int NS>
__global__ void __launch_bounds__(kProjJobs) k_project_all(const float* __restrict__ hj, int64_t n_jobs,
                                                           const SpaceParams sp, const float* __restrict__ coef_c,
                                                           const float* __restrict__ coef_d,
                                                           const unsigned long long* __restrict__ err,
                                                           float* __restrict__ ka, float* __restrict__ kb,
                                                           float* __restrict__ w, unsigned* wmm, int y0,
                                                           int w_partial) {
  __shared__ CoefRow s_coef[kMaxCaps];
  __shared__ unsigned s_mm[2];
  extern __shared__ float s_stage[];  // [2][kProjWarps][32][rs + 1]
  const int y = blockIdx.y + y0;
  const bool is_w = y >= sp.n_slices;
  const int slot = is_w ? (y - sp.n_slices) / sp.n_states : 0, state = is_w ? (y - sp.n_slices) % sp.n_states : 0;
  for (int p = threadIdx.x; p < sp.n_caps; p += blockDim.x) {
    CoefRow r;
    if (!is_w) {
      load_c(r, sp, coef_c, y, p);
      load_d(r.d[0], sp, coef_d, y, p);
    } else {
      load_w_row(r, sp, coef_c, coef_d, slot, state, p);
    }
    s_coef[p] = r;
  }
  if (threadIdx.x < 2) s_mm[threadIdx.x] = threadIdx.x ? 0u : 0xFFFFFFFFu;
  __syncthreads();
  pdl_wait();  // hj, err and wmm of this step (the prologue above reads constant tables only)
  pdl_launch_dependents();
  if (*err != ~0ull) return;  // invalid input: leave the workspace untouched (uniform per launch)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int rs = sp.rs, ld = rs + 1, nc = sp.n_caps;
  const size_t npad = (size_t)sp.n_jobs_pad;
  unsigned lo = 0xFFFFFFFFu, hi = 0u;
  // blocks loop over job chunks: the coefficient prologue (dependent global
  // loads + a block barrier) is paid once per block, not once per 128 jobs
  for (int64_t chunk = blockIdx.x; chunk * kProjJobs < (int64_t)npad; chunk += gridDim.x) {
  const int64_t n0 = chunk * kProjJobs + warp * 32, n = n0 + lane;
  if (n0 < (int64_t)npad) {
    float* stg_a = s_stage + warp * 32 * ld;
    float* stg_b = s_stage + (kProjWarps + warp) * 32 * ld;
    float* row_a = stg_a + lane * ld;
    float* row_b = stg_b + lane * ld;
    float h[6], j[3];
    const bool job = n < n_jobs;
    if (job) load_hj(hj, n, h, j);
    if (!is_w) {
      if (job) {
        for (int p = 0; p < nc; p++) {
          const CoefRow& r = s_coef[p];
          row_a[p] = ka_value(sp, r, h);
          row_b[p] = kb_value(r, j);
        }
      } else {
        for (int p = 0; p < nc; p++) row_a[p] = row_b[p] = kPadMargin;
      }
      for (int p = nc; p < rs; p++) row_a[p] = row_b[p] = kPadMargin;
      __syncwarp();
      flush_rows(stg_a, ld, rs, ka + ((size_t)y * npad + n0) * rs, lane);
      flush_rows(stg_b, ld, rs, kb + ((size_t)y * npad + n0) * rs, lane);
    } else {
      if (job) {
        for (int p = 0; p < nc; p++) {
          const float v = w_value<NS>(s_coef[p], h, j);
          row_a[p] = v;
          const unsigned uo = ord_float_d(fmaxf(v, s_coef[p].wfloor));  // range of the feasible-capable shares
          lo = uo < lo ? uo : lo;
          hi = uo > hi ? uo : hi;
        }
      } else {
        for (int p = 0; p < nc; p++) row_a[p] = -1e30f;
      }
      for (int p = nc; p < rs; p++) row_a[p] = -1e30f;
      __syncwarp();
      // w_partial (a tiled step): only the rows this rank's scorer reads are stored
      // (the range above still covers every job); ensure_kakb completes the rest
      if (!w_partial || (n0 + 32 > sp.fast_lo[slot] && n0 < sp.fast_hi[slot]))
        flush_rows(stg_a, ld, rs, w + ((((size_t)slot * sp.n_states + state) * npad) + n0) * rs, lane);
    }
    __syncwarp();  // the staging rows are rewritten by the next chunk
  }
  }
  if (!is_w) return;
  for (int off = 16; off > 0; off >>= 1) {
    const unsigned a = __shfl_xor_sync(0xFFFFFFFFu, lo, off), b = __shfl_xor_sync(0xFFFFFFFFu, hi, off);
    lo = a < lo ? a : lo;
    hi = b > hi ? b : hi;
  }
  if (lane == 0) {
    atomicMin(&s_mm[0], lo);
    atomicMax(&s_mm[1], hi);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicMin(&wmm[2 * slot], s_mm[0]);
    atomicMax(&wmm[2 * slot + 1], s_mm[1]);
  }
}

// Gathered layout of the tiled scorers (DESIGN.md "gathered layout" and
// "packed objective"). For slot i of a set and config c = (state s, cap p) the
// operands are laid out along the flattened config axis, per role:
//   role A_i   = ka[s_i(s)][j][p]            (own term minus alpha, scaled)
//   role B_i^l = kb[s_l(s)][j][p], l != i    (this job's interference on slot l)
//   role W_i   = fixed-point share of Throughput[/P]:
//       q = rint(fma(max(w[i][s][j][p], floor), inv_delta, -fl(wmin_i * inv_delta))),
//       inv_delta = (2^25 - 2 - n_slots) / sum_i (wmax_i - wmin_i)   (quant_inv; sum_i q_i < 2^25)
//       floor = the row's feasibility floor (load_w_row), wmin/wmax over the clamped shares
//       W_0 = 0x00800000 + (q << 5); W_last = (q << 5) | (31 - off); others q << 5
//     where off = c mod kStageCfg. The integer sum of a candidate's W's, read
//     as FP32 bits, is a positive normal float below 4.0 that orders like the
//     objective up to one quantum per slot (< 4e-7 relative for the presets)
//     and carries the config's offset in its stage in the low 5 bits.
// Rows are [role][stage][job][kStageRS]; padding (configs >= n_cfg, jobs >=
// n_jobs) gets A = B = kPadMargin (infeasible) and W = 0. Grid (x: blocks of
// kProjJobs jobs, y: role * n_stages + stage). Values are recomputed from hj
// with the projection's own functions (bit-identical to ka / kb / w).
template <int NS>
__global__ void __launch_bounds__(kProjJobs) k_gather_fast(const float* __restrict__ hj,
                                                           const float* __restrict__ coef_c,
                                                           const float* __restrict__ coef_d, const SpaceParams sp,
                                                           int64_t n_jobs, const unsigned long long* __restrict__ err,
                                                           const unsigned* __restrict__ wmm, float* __restrict__ fast) {
  constexpr int ld = kStageCfg + 1;  // odd: the column writes of a warp hit distinct banks
  __shared__ CoefRow s_coef[kStageCfg];
  __shared__ float s_stage[kProjWarps][32 * ld];
  __shared__ float s_nlo, s_inv;
  const int role = blockIdx.y / sp.n_stages, stage = blockIdx.y - role * sp.n_stages;
  const int slot = role / (NS + 1), kind = role % (NS + 1);  // 0 = A, NS = W, else B
  const int ncol = min(kStageCfg, sp.n_cfg - stage * kStageCfg);  // real configs in this stage
  if (threadIdx.x < ncol) {
    const int c = stage * kStageCfg + threadIdx.x, st = c / sp.n_caps, p = c - st * sp.n_caps;
    CoefRow r;
    if (kind == NS) {
      load_w_row(r, sp, coef_c, coef_d, slot, st, p);
    } else if (kind == 0) {
      load_c(r, sp, coef_c, sp.slice[st][slot], p);
    } else {
      const int l = kind - 1 + (kind - 1 >= slot ? 1 : 0);  // the kind-th other slot, ascending
      load_d(r.d[0], sp, coef_d, sp.slice[st][l], p);
    }
    s_coef[threadIdx.x] = r;
  }
  pdl_wait();  // the projection's w range (wmm), hj and err
  pdl_launch_dependents();
  if (threadIdx.x == 0) {
    const float inv = quant_inv<NS>(wmm);
    s_inv = inv;
    s_nlo = -__fmul_rn(unord_float_d(wmm[2 * slot]), inv);
  }
  __syncthreads();
  if (*err != ~0ull) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const size_t npad = (size_t)sp.n_jobs_pad;
  float* row = s_stage[warp] + lane * ld;
  // blocks loop over job chunks (the coefficient prologue once per block)
  for (int64_t chunk = blockIdx.x; chunk * kProjJobs < (int64_t)npad; chunk += gridDim.x) {
  const int64_t n0 = chunk * kProjJobs + warp * 32, n = n0 + lane;
  if (n0 >= (int64_t)npad) break;
  if (n0 + 32 <= sp.fast_lo[slot] || n0 >= sp.fast_hi[slot]) continue;  // rows this rank's scorer never reads
  const bool job = n < n_jobs;
  float h[6], j[3];
  if (job) load_hj(hj, n, h, j);
  const int nreal = job ? ncol : 0;
  if (kind == NS) {
    const float nlo = s_nlo, inv = s_inv;
    const unsigned base = slot == 0 ? 0x00800000u : 0u;
    for (int col = 0; col < nreal; col++) {
      const float qf = rintf(__fmaf_rn(fmaxf(w_value<NS>(s_coef[col], h, j), s_coef[col].wfloor), inv, nlo));
      unsigned bits = ((qf > 0.0f ? (unsigned)qf : 0u) << 5) + base;
      if (slot == NS - 1) bits |= (unsigned)(31 - col);
      row[col] = __uint_as_float(bits);
    }
    for (int col = nreal; col < kStageCfg; col++) row[col] = 0.0f;
  } else if (kind == 0) {
    for (int col = 0; col < nreal; col++) row[col] = ka_value(sp, s_coef[col], h);
    for (int col = nreal; col < kStageCfg; col++) row[col] = kPadMargin;
  } else {
    for (int col = 0; col < nreal; col++) row[col] = kb_value(s_coef[col], j);
    for (int col = nreal; col < kStageCfg; col++) row[col] = kPadMargin;
  }
  __syncwarp();
  static_assert(kStageRS == kStageCfg, "the stage row is exactly the stage's configs");
  flush_rows(s_stage[warp], ld, kStageCfg, fast + (((size_t)role * sp.n_stages + stage) * npad + n0) * kStageRS, lane);
  __syncwarp();  // the staging rows are rewritten by the next chunk
  }
}

__global__ void k_step_init(unsigned long long* err, unsigned long long* best_key, unsigned* rescore_n,
                            unsigned* wmm) {
  if (threadIdx.x < 2 * kMaxSlots) wmm[threadIdx.x] = (threadIdx.x & 1) ? 0u : 0xFFFFFFFFu;
  if (threadIdx.x == 0) {
    *err = ~0ull;
    *best_key = 0ull;
    *rescore_n = 0u;
  }
}

cudaError_t smem_optin(const void* func, size_t bytes) {
  if (bytes <= 48 * 1024) return cudaSuccess;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  static std::mutex mu;
  static std::set<std::tuple<const void*, int, size_t>> done;
  std::lock_guard<std::mutex> lk(mu);
  const auto key = std::make_tuple(func, dev, bytes);
  if (done.count(key)) return cudaSuccess;
  e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) done.insert(key);
  return e;
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("COSCHED_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

int num_sms() {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    return 148;
  return n;
}

void launch_step_init(unsigned long long* err, unsigned long long* best_key, unsigned* rescore_n, unsigned* wmm,
                      cudaStream_t st) {
  k_step_init<<<1, 32, 0, st>>>(err, best_key, rescore_n, wmm);
}

void launch_project(const float* hj, int64_t n_jobs, const SpaceParams& sp, const DeviceTables& tb,
                    const unsigned long long* err, float* ka, float* kb, float* w, float* fast, unsigned* wmm,
                    bool with_kakb, cudaStream_t st, cudaEvent_t mid) {
  if (n_jobs <= 0) return;  // wmm was reset by launch_step_init
  // 2 job chunks of 128 per block (measured on C4: 1 -> 60.4 us, 2 -> 58.9,
  // 4 -> 62.1, 8 -> 75.2 for project + gather; COSCHED_PROJ_CHUNKS overrides)
  const int64_t n_chunks = (sp.n_jobs_pad + kProjJobs - 1) / kProjJobs;
  const char* pc = getenv("COSCHED_PROJ_CHUNKS");
  const int per_block = pc ? std::max(1, atoi(pc)) : 2;
  const unsigned jb = (unsigned)((n_chunks + per_block - 1) / per_block);
  const size_t stage_bytes = (size_t)2 * kProjWarps * 32 * (sp.rs + 1) * sizeof(float);  // <= 70 KB (rs <= 68)
  // ka / kb rows only when a consumer of this step reads them (the tiled
  // scorers read the gathered layout and w); launch_project_kakb adds them later
  const int y0 = with_kakb ? 0 : sp.n_slices;
  const dim3 gp(jb, (unsigned)(sp.n_slices + sp.n_slots * sp.n_states - y0)), gg(jb, (unsigned)(sp.n_roles * sp.n_stages));
  smem_optin((const void*)k_project_all<1>, 72 * 1024);
  smem_optin((const void*)k_project_all<2>, 72 * 1024);
  smem_optin((const void*)k_project_all<3>, 72 * 1024);
  if (sp.n_slots == 1) {
    launch_pdl(k_project_all<1>, gp, dim3(kProjJobs), stage_bytes, st, hj, n_jobs, sp, tb.coef_c, tb.coef_d, err, ka, kb, w, wmm, y0,
               with_kakb ? 0 : 1);
    if (mid) cudaEventRecord(mid, st);
    launch_pdl(k_gather_fast<1>, gg, dim3(kProjJobs), 0, st, hj, tb.coef_c, tb.coef_d, sp, n_jobs, err, wmm, fast);
  } else if (sp.n_slots == 2) {
    launch_pdl(k_project_all<2>, gp, dim3(kProjJobs), stage_bytes, st, hj, n_jobs, sp, tb.coef_c, tb.coef_d, err, ka, kb, w, wmm, y0,
               with_kakb ? 0 : 1);
    if (mid) cudaEventRecord(mid, st);
    launch_pdl(k_gather_fast<2>, gg, dim3(kProjJobs), 0, st, hj, tb.coef_c, tb.coef_d, sp, n_jobs, err, wmm, fast);
  } else {
    launch_pdl(k_project_all<3>, gp, dim3(kProjJobs), stage_bytes, st, hj, n_jobs, sp, tb.coef_c, tb.coef_d, err, ka, kb, w, wmm, y0,
               with_kakb ? 0 : 1);
    if (mid) cudaEventRecord(mid, st);
    launch_pdl(k_gather_fast<3>, gg, dim3(kProjJobs), 0, st, hj, tb.coef_c, tb.coef_d, sp, n_jobs, err, wmm, fast);
  }
}

// The ka / kb rows alone (after a launch_project without them).
void launch_project_kakb(const float* hj, int64_t n_jobs, const SpaceParams& sp, const DeviceTables& tb,
                         const unsigned long long* err, float* ka, float* kb, unsigned* wmm, cudaStream_t st,
                         float* w_full) {
  if (n_jobs <= 0) return;
  const int64_t n_chunks = (sp.n_jobs_pad + kProjJobs - 1) / kProjJobs;
  const unsigned jb = (unsigned)((n_chunks + 1) / 2);
  const size_t stage_bytes = (size_t)2 * kProjWarps * 32 * (sp.rs + 1) * sizeof(float);
  // rows y < n_slices (ka / kb); with w_full also every w row, recomputed bit-identically
  // (the w range it folds into wmm is the one the step already reduced: unchanged)
  const dim3 gp(jb, (unsigned)(sp.n_slices + (w_full ? sp.n_slots * sp.n_states : 0)));
  if (sp.n_slots == 1)
    k_project_all<1><<<gp, kProjJobs, stage_bytes, st>>>(hj, n_jobs, sp, tb.coef_c, tb.coef_d, err, ka, kb, w_full, wmm,
                                                         0, 0);
  else if (sp.n_slots == 2)
    k_project_all<2><<<gp, kProjJobs, stage_bytes, st>>>(hj, n_jobs, sp, tb.coef_c, tb.coef_d, err, ka, kb, w_full, wmm,
                                                         0, 0);
  else
    k_project_all<3><<<gp, kProjJobs, stage_bytes, st>>>(hj, n_jobs, sp, tb.coef_c, tb.coef_d, err, ka, kb, w_full, wmm,
                                                         0, 0);
}

// ---------------------------------------------------------------------------
// a4-a8, generic reference scorer: one thread per set. For each config in
// canonical order (state in table order, caps ascending):
//   r_i'' = ka[j_i][s_i][p] + sum_{l != i} kb[j_l][s_i][p]   (= K*(RPerf_i - alpha))
//   obj   = sum_i w[j_i][i][s][p]                          (= Throughput [/ P])
//   feasible iff every r_i'' > 0  (Fairness > alpha)
// keep the first strictly greater feasible obj.
template <int NS>
__global__ void __launch_bounds__(256) k_score_generic(const SpaceParams sp, int64_t n_jobs,
                                                       const float* __restrict__ ka, const float* __restrict__ kb,
                                                       const float* __restrict__ w,
                                                       int64_t first, int64_t count, float* __restrict__ out_obj,
                                                       int32_t* __restrict__ out_cfg,
                                                       unsigned long long* __restrict__ best_key,
                                                       const unsigned long long* __restrict__ err) {
  if (*err != ~0ull) return;
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  unsigned long long key = 0;
  if (k < count) {
    int64_t sid = first + k;
    int64_t j[3];
    unrank_set<NS>(sid, j);
    float best = -INFINITY;
    int32_t bc = -1;
    for (int s = 0; s < sp.n_states; s++) {
      for (int p = 0; p < sp.n_caps; p++) {
        float r[NS], o;
        eval_cfg<NS>(sp, ka, kb, w, j, s, p, r, &o);
        bool feas = true;
#pragma unroll
        for (int i = 0; i < NS; i++) feas = feas && (r[i] > 0.0f);
        if (feas && o > best) {
          best = o;
          bc = s * sp.n_caps + p;
        }
      }
    }
    if (out_obj) out_obj[k] = bc >= 0 ? best : -INFINITY;
    if (out_cfg) out_cfg[k] = bc;
    key = bc >= 0 ? pack_key(best, sid) : 0ull;
  }
  block_max_key(key, best_key);
}

// NEXT #2: hill climbing per set (R22), one thread per set; evaluations
// counted per block (one atomic per block).
template <int NS>
__global__ void __launch_bounds__(256) k_score_hill(const SpaceParams sp, const float* __restrict__ ka,
                                                    const float* __restrict__ kb, const float* __restrict__ w,
                                                    int64_t first, int64_t count, float* __restrict__ out_obj,
                                                    int32_t* __restrict__ out_cfg,
                                                    unsigned long long* __restrict__ best_key,
                                                    unsigned long long* __restrict__ evals,
                                                    const unsigned long long* __restrict__ err) {
  __shared__ unsigned long long s_ev;
  if (threadIdx.x == 0) s_ev = 0;
  __syncthreads();
  if (*err != ~0ull) return;
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  unsigned long long key = 0;
  if (k < count) {
    const int64_t sid = first + k;
    int64_t j[3];
    unrank_set<NS>(sid, j);
    float o;
    int ev = 0;
    const int c = hill_search<NS>(sp, ka, kb, w, j, sp.hc_state, sp.hc_cap, &o, &ev);
    if (out_obj) out_obj[k] = c >= 0 ? o : -INFINITY;
    if (out_cfg) out_cfg[k] = c;
    key = c >= 0 ? pack_key(o, sid) : 0ull;
    atomicAdd(&s_ev, (unsigned long long)ev);
  }
  block_max_key(key, best_key);
  if (threadIdx.x == 0) atomicAdd(evals, s_ev);
}

int launch_score_hill(const SpaceParams& sp, int64_t n_jobs, const float* ka, const float* kb, const float* w,
                      int64_t first, int64_t count, float* obj, int32_t* cfg, unsigned long long* best_key,
                      unsigned long long* evals, const unsigned long long* err, cudaStream_t st) {
  if (count <= 0) return 0;
  const unsigned grid = (unsigned)((count + 255) / 256);
  if (sp.n_slots == 1)
    k_score_hill<1><<<grid, 256, 0, st>>>(sp, ka, kb, w, first, count, obj, cfg, best_key, evals, err);
  else if (sp.n_slots == 2)
    k_score_hill<2><<<grid, 256, 0, st>>>(sp, ka, kb, w, first, count, obj, cfg, best_key, evals, err);
  else
    k_score_hill<3><<<grid, 256, 0, st>>>(sp, ka, kb, w, first, count, obj, cfg, best_key, evals, err);
  return 1;
}

int launch_score_pairs_fast(const SpaceParams& sp, int64_t n_jobs, const float* w, const float* fast, int64_t first,
                            int64_t count, float* obj, int32_t* cfg, unsigned long long* best_key,
                            const unsigned long long* err, const RescoreBuf& rb, const PairMerge& merge,
                            cudaStream_t st);

int launch_score_triples_fast(const SpaceParams& sp, int64_t n_jobs, const float* w, const float* fast, int64_t first,
                              int64_t count, float* obj, int32_t* cfg, unsigned long long* best_key,
                              const unsigned long long* err, const RescoreBuf& rb, cudaStream_t st);

// ---------------------------------------------------------------------------
// Exact re-scoring after the tiled scorers (RescoreBuf, rescore_threshold in
// device_common.cuh). Which sets: pairs -- the sets the tile end flagged
// (objective below the threshold), listed in rb.list; triples, or a list
// overflow -- a scan of the shard's objectives for the same condition (4 B per
// set); without an objective output only the best key matters, and it is within
// tau/2 of the exact one unless its own objective is below the threshold (then
// every set is re-scored). How: one warp per set evaluates every config in the
// canonical FP32 order of eval_cfg -- margins from the gathered layout
// (bit-identical to ka / kb), objective from w -- and keeps the first strictly
// greater feasible objective, i.e. exactly what k_score_generic computes for
// that set. The new key can only be larger than the tile end's (same
// arithmetic, exact argmax), so an atomicMax keeps best_key right.
template <int NS>
__device__ __forceinline__ void rescore_one(const SpaceParams& sp, const float* __restrict__ fast,
                                            const float* __restrict__ w, int64_t first, int64_t k,
                                            float* __restrict__ out_obj, int32_t* __restrict__ out_cfg, int lane,
                                            unsigned long long* bkey) {
  const int64_t npad = sp.n_jobs_pad, sid = first + k;
  int64_t j[3];
  unrank_set<NS>(sid, j);
  unsigned long long best = 0ull;
  for (int c = lane; c < sp.n_cfg; c += 32) {
    const int g = c / kStageCfg, off = c - g * kStageCfg;
    const int s = c / sp.n_caps, p = c - s * sp.n_caps;
    auto F = [&](int role, int64_t job) {
      return __ldg(fast + (((int64_t)role * sp.n_stages + g) * npad + job) * kStageRS + off);
    };
    bool feas;
    float o;
    if (NS == 2) {  // roles [A0 B0^1 W0 | A1 B1^0 W1]
      const float r0 = __fadd_rn(F(0, j[0]), F(4, j[1]));  // ka[s0][j0] + kb[s0][j1]
      const float r1 = __fadd_rn(F(3, j[1]), F(1, j[0]));  // ka[s1][j1] + kb[s1][j0]
      o = __fadd_rn(__ldg(w_row(w, sp, 0, s, j[0]) + p), __ldg(w_row(w, sp, 1, s, j[1]) + p));
      feas = r0 > 0.0f && r1 > 0.0f;
    } else {  // roles [A0 B0^1 B0^2 W0 | A1 B1^0 B1^2 W1 | A2 B2^0 B2^1 W2]
      const float r0 = __fadd_rn(F(0, j[0]), __fadd_rn(F(5, j[1]), F(9, j[2])));
      const float r1 = __fadd_rn(__fadd_rn(F(4, j[1]), F(10, j[2])), F(1, j[0]));
      const float r2 = __fadd_rn(__fadd_rn(F(8, j[2]), F(6, j[1])), F(2, j[0]));
      o = __fadd_rn(__ldg(w_row(w, sp, 0, s, j[0]) + p),
                    __fadd_rn(__ldg(w_row(w, sp, 1, s, j[1]) + p), __ldg(w_row(w, sp, 2, s, j[2]) + p)));
      feas = r0 > 0.0f && r1 > 0.0f && r2 > 0.0f;
    }
    const unsigned long long kk =
        feas ? (((unsigned long long)ord_float_d(o) << 32) | (0xFFFFFFFFull - (unsigned)c)) : 0ull;
    best = kk > best ? kk : best;
  }
  best = warp_max_u64(best);
  if (lane == 0) {
    const int bc = best ? (int)(0xFFFFFFFFull - (best & 0xFFFFFFFFull)) : -1;
    const float bo = best ? unord_float_d((unsigned)(best >> 32)) : -INFINITY;
    if (out_obj) out_obj[k] = bo;
    if (out_cfg) out_cfg[k] = bc;
    if (bc >= 0) {
      const unsigned long long kk = pack_key(bo, sid);
      *bkey = kk > *bkey ? kk : *bkey;
    }
  }
}

template <int NS>
__global__ void __launch_bounds__(256) k_rescore_sets(const SpaceParams sp, const float* __restrict__ fast,
                                                      const float* __restrict__ w, int64_t first, int64_t count,
                                                      float* __restrict__ out_obj, int32_t* __restrict__ out_cfg,
                                                      unsigned long long* __restrict__ best_key, const RescoreBuf rb,
                                                      const unsigned long long* __restrict__ err) {
  pdl_wait();  // the scorer's outputs and re-score list
  pdl_launch_dependents();
  if (*err != ~0ull) return;
  const float thr = rescore_threshold<NS>(rb.wmm);
  const unsigned n_listed = *rb.n;
  const bool listed = NS == 2 && n_listed <= rb.cap;  // uniform per launch
  if (listed && n_listed == 0u) return;               // the common case: one launch, nothing re-scored
  if (!listed && !out_obj) {
    // only the best key is produced: within tau/2 of the exact one unless its own objective is below thr
    const unsigned long long bk = *best_key;
    if (bk == 0ull || unord_float_d((unsigned)(bk >> 32)) >= thr) return;
  }
  const int lane = threadIdx.x & 31;
  const int64_t wpb = blockDim.x >> 5, gw = blockIdx.x * wpb + (threadIdx.x >> 5), nw = (int64_t)gridDim.x * wpb;
  unsigned long long bkey = 0ull;
  if (listed) {
    for (int64_t e = gw; e < (int64_t)n_listed; e += nw)
      rescore_one<NS>(sp, fast, w, first, (int64_t)rb.list[e], out_obj, out_cfg, lane, &bkey);
  } else if (!out_obj) {
    if (NS == 3 && gw == 0 && lane == 0) atomicAdd(rb.n, (unsigned)count);
    for (int64_t k = gw; k < count; k += nw) rescore_one<NS>(sp, fast, w, first, k, out_obj, out_cfg, lane, &bkey);
  } else {
    // scan: 4 x 32 consecutive objectives per warp and step (coalesced, 512 B in flight per warp)
    for (int64_t base = gw * 128; base < count; base += nw * 128) {
      float o[4];
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const int64_t k = base + u * 32 + lane;
        o[u] = k < count ? out_obj[k] : -INFINITY;
      }
#pragma unroll 1
      for (int u = 0; u < 4; u++) {
        unsigned m = __ballot_sync(0xFFFFFFFFu, o[u] > -INFINITY && o[u] < thr);
        if (NS == 3 && lane == 0 && m) atomicAdd(rb.n, (unsigned)__popc(m));  // triples: count what the scan found
        while (m) {
          const int b = __ffs(m) - 1;
          m &= m - 1;
          rescore_one<NS>(sp, fast, w, first, base + u * 32 + b, out_obj, out_cfg, lane, &bkey);
        }
      }
    }
  }
  block_max_key(bkey, best_key);
}

int launch_rescore(const SpaceParams& sp, const float* w, const float* fast, int64_t first, int64_t count, float* obj,
                   int32_t* cfg, unsigned long long* best_key, const unsigned long long* err, const RescoreBuf& rb,
                   cudaStream_t st) {
  if (!rb.n || count <= 0) return 0;
  // up to 8 resident blocks per SM: enough loads in flight for the scan mode
  unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(8 * 148, (count + 1023) / 1024));
  // pairs re-score only the listed sets (normally none): one wave of blocks, each
  // exits at once on an empty list (a 1,184-block launch costs its block scheduling)
  if (sp.n_slots == 2 && rb.cap > 0) grid = std::min(grid, 148u);
  if (sp.n_slots == 2)
    launch_pdl(k_rescore_sets<2>, dim3(grid), dim3(256), 0, st, sp, fast, w, first, count, obj, cfg, best_key, rb, err);
  else
    launch_pdl(k_rescore_sets<3>, dim3(grid), dim3(256), 0, st, sp, fast, w, first, count, obj, cfg, best_key, rb, err);
  return 1;
}

bool tiled_applicable(int n_slots, int64_t n_jobs, int64_t first, int64_t count) {
  if (n_slots < 2 || count <= 0) return false;
  // whole colex columns (pairs) / planes (triples): first and first + count are C(b, n_slots)
  auto whole = [&](int64_t v) {
    int64_t lo = 0, hi = n_jobs;
    while (lo < hi) {
      const int64_t mid = (lo + hi) / 2;
      if (n_sets(mid, n_slots) >= v) hi = mid;
      else lo = mid + 1;
    }
    return n_sets(lo, n_slots) == v;
  };
  if (!whole(first) || !whole(first + count)) return false;
  return n_slots == 3 || (n_jobs + 63) / 64 < 32768;
}

int launch_score(const SpaceParams& sp, int64_t n_jobs, const float* ka, const float* kb, const float* w,
                 const float* fast, int64_t first, int64_t count, float* obj, int32_t* cfg,
                 unsigned long long* best_key, const unsigned long long* err, int variant, cudaStream_t st,
                 const RescoreBuf& rb, const PairMerge& merge) {
  if (count <= 0) return 0;
  if (variant != 0 && tiled_applicable(sp.n_slots, n_jobs, first, count)) {
    int n = sp.n_slots == 2
                ? launch_score_pairs_fast(sp, n_jobs, w, fast, first, count, obj, cfg, best_key, err, rb, merge, st)
                : launch_score_triples_fast(sp, n_jobs, w, fast, first, count, obj, cfg, best_key, err, rb, st);
    return n + launch_rescore(sp, w, fast, first, count, obj, cfg, best_key, err, rb, st);
  }
  int bs = 256;
  unsigned grid = (unsigned)((count + bs - 1) / bs);
  if (sp.n_slots == 1)
    k_score_generic<1><<<grid, bs, 0, st>>>(sp, n_jobs, ka, kb, w, first, count, obj, cfg, best_key, err);
  else if (sp.n_slots == 2)
    k_score_generic<2><<<grid, bs, 0, st>>>(sp, n_jobs, ka, kb, w, first, count, obj, cfg, best_key, err);
  else
    k_score_generic<3><<<grid, bs, 0, st>>>(sp, n_jobs, ka, kb, w, first, count, obj, cfg, best_key, err);
  return 1;
}

// ---------------------------------------------------------------------------
// Per-set detail (cosched_best_config, winners of best_set / allocation): one
// block per listed set evaluates every config of it, reduces (obj desc, cfg asc)
// and reports the winner's RPerf, Throughput, Fairness in natural units
// (RPerf_i = r_i''/K + alpha).
// out row (8 floats): [0] cfg (int bits, -1 none), [1] obj, [2] thr, [3] fair, [4..] rperf
// set_ids == nullptr: one block for the set named by the packed key *key_src
// (the best set after the all-reduce; key 0 = none -> cfg -1), so best_set
// needs a single device -> host round trip.
// eval_cfg (device_common.cuh) with every operand recomputed from the basis
// rows hj and the coefficient tables by the projection's own functions: the
// same FP32 values in the same canonical order, for steps whose projection
// skipped the ka / kb rows (launch_project with_kakb = false).
template <int NS>
__device__ __forceinline__ void eval_cfg_hj(const SpaceParams& sp, const float* __restrict__ s_hj,
                                            const float* __restrict__ coef_c, const float* __restrict__ coef_d,
                                            int s, int p, float* r, float* o) {
  // s_hj: the set's basis rows, slot i at s_hj + 12 i (shared memory)
  float h[NS][6], jv[NS][3];
#pragma unroll
  for (int i = 0; i < NS; i++) {
#pragma unroll
    for (int t = 0; t < 6; t++) h[i][t] = s_hj[12 * i + t];
#pragma unroll
    for (int t = 0; t < 3; t++) jv[i][t] = s_hj[12 * i + 6 + t];
  }
  auto KA = [&](int slot_of_slice, int i) {
    CoefRow cr;
    load_c(cr, sp, coef_c, sp.slice[s][slot_of_slice], p);
    return ka_value(sp, cr, h[i]);
  };
  auto KB = [&](int slot_of_slice, int i) {
    CoefRow cr;
    load_d(cr.d[0], sp, coef_d, sp.slice[s][slot_of_slice], p);
    return kb_value(cr, jv[i]);
  };
  auto WV = [&](int slot) {
    CoefRow cr;
    load_w_row(cr, sp, coef_c, coef_d, slot, s, p);
    return w_value<NS>(cr, h[slot], jv[slot]);
  };
  if (NS == 1) {
    r[0] = KA(0, 0);
    *o = WV(0);
  } else if (NS == 2) {
    r[0] = __fadd_rn(KA(0, 0), KB(0, 1));
    r[1] = __fadd_rn(KA(1, 1), KB(1, 0));
    *o = __fadd_rn(WV(0), WV(1));
  } else {
    r[0] = __fadd_rn(KA(0, 0), __fadd_rn(KB(0, 1), KB(0, 2)));
    r[1] = __fadd_rn(__fadd_rn(KA(1, 1), KB(1, 2)), KB(1, 0));
    r[2] = __fadd_rn(__fadd_rn(KA(2, 2), KB(2, 1)), KB(2, 0));
    *o = __fadd_rn(WV(0), __fadd_rn(WV(1), WV(2)));
  }
}

template <bool HJ>
__device__ __forceinline__ void eval_any(const SpaceParams& sp, const float* __restrict__ ka,
                                         const float* __restrict__ kb, const float* __restrict__ w,
                                         const float* __restrict__ s_hj, const float* __restrict__ coef_c,
                                         const float* __restrict__ coef_d, const int64_t* j, int s, int p, float* r,
                                         float* u) {
  if (HJ) {
    if (sp.n_slots == 1) eval_cfg_hj<1>(sp, s_hj, coef_c, coef_d, s, p, r, u);
    else if (sp.n_slots == 2) eval_cfg_hj<2>(sp, s_hj, coef_c, coef_d, s, p, r, u);
    else eval_cfg_hj<3>(sp, s_hj, coef_c, coef_d, s, p, r, u);
  } else {
    if (sp.n_slots == 1) eval_cfg<1>(sp, ka, kb, w, j, s, p, r, u);
    else if (sp.n_slots == 2) eval_cfg<2>(sp, ka, kb, w, j, s, p, r, u);
    else eval_cfg<3>(sp, ka, kb, w, j, s, p, r, u);
  }
}

// One block per set: every config evaluated once (a config per thread per
// pass), the block's max key (objective desc, config asc) found by a warp
// then block reduction, and the thread that evaluated the winner writes its
// RPerf / Throughput / Fairness -- no second evaluation. HJ: operands from the
// basis rows (staged in shared memory) and the coefficient tables.
template <bool HJ>
__global__ void __launch_bounds__(512) k_sets_detail(const SpaceParams sp, const float* __restrict__ ka,
                                                     const float* __restrict__ kb, const float* __restrict__ w,
                                                     const int64_t* __restrict__ set_ids,
                                                     const unsigned long long* __restrict__ key_src, float* out_all,
                                                     const unsigned long long* __restrict__ err,
                                                     unsigned long long* hdr, const float* __restrict__ hj,
                                                     const float* __restrict__ coef_c,
                                                     const float* __restrict__ coef_d) {
  __shared__ unsigned long long s_key[32];
  __shared__ float s_hj[3 * 12];
  pdl_wait();  // (launch_best_detail) the step's best key and outputs
  pdl_launch_dependents();
  float* out = out_all + (int64_t)blockIdx.x * 8;
  int64_t set_id;
  if (set_ids) {
    set_id = set_ids[blockIdx.x];
  } else {
    const unsigned long long kk = *key_src;
    if (hdr && threadIdx.x == 0) {  // best mode: validation word and key next to the row
      hdr[0] = *err;
      hdr[1] = kk;
    }
    if (kk == 0ull) {
      if (threadIdx.x == 0) {
        out[0] = __int_as_float(-1);
        out[1] = -INFINITY;
        out[2] = out[3] = 0.0f;
      }
      return;
    }
    set_id = (int64_t)(0xFFFFFFFFull - (kk & 0xFFFFFFFFull));
  }
  int64_t j[3];
  if (sp.n_slots == 1) unrank_set<1>(set_id, j);
  else if (sp.n_slots == 2) unrank_set<2>(set_id, j);
  else unrank_set<3>(set_id, j);
  if (HJ) {
    if (threadIdx.x < 12 * sp.n_slots) s_hj[threadIdx.x] = hj[j[threadIdx.x / 12] * 12 + threadIdx.x % 12];
    __syncthreads();
  }
  unsigned long long key = 0;
  float br[3] = {0.0f, 0.0f, 0.0f}, bu = 0.0f;  // the thread's best config's values
  if (sp.search_mode == 1) {  // the hill climb's choice (R22), not the exhaustive argmax
    if (threadIdx.x == 0) {
      float o;
      int ev = 0, c;
      if (sp.n_slots == 1) c = hill_search<1>(sp, ka, kb, w, j, sp.hc_state, sp.hc_cap, &o, &ev);
      else if (sp.n_slots == 2) c = hill_search<2>(sp, ka, kb, w, j, sp.hc_state, sp.hc_cap, &o, &ev);
      else c = hill_search<3>(sp, ka, kb, w, j, sp.hc_state, sp.hc_cap, &o, &ev);
      if (c >= 0) {
        key = ((unsigned long long)ord_float_d(o) << 32) | (0xFFFFFFFFull - (unsigned)c);
        eval_any<HJ>(sp, ka, kb, w, s_hj, coef_c, coef_d, j, c / sp.n_caps, c % sp.n_caps, br, &bu);
      }
    }
  } else {
    for (int c = threadIdx.x; c < sp.n_cfg; c += blockDim.x) {
      const int s = c / sp.n_caps, p = c % sp.n_caps;
      float r[3], u;
      eval_any<HJ>(sp, ka, kb, w, s_hj, coef_c, coef_d, j, s, p, r, &u);
      bool feas = true;
      for (int i = 0; i < sp.n_slots; i++) feas = feas && (r[i] > 0.0f);
      const unsigned long long kk =
          feas ? (((unsigned long long)ord_float_d(u) << 32) | (0xFFFFFFFFull - (unsigned)c)) : 0ull;
      if (kk > key) {
        key = kk;
        bu = u;
        br[0] = r[0];
        br[1] = r[1];
        br[2] = r[2];
      }
    }
  }
  const unsigned long long mine = key;
  key = warp_max_u64(key);
  if ((threadIdx.x & 31) == 0) s_key[threadIdx.x >> 5] = key;
  __syncthreads();
  if (threadIdx.x < 32) {
    const int nw = (blockDim.x + 31) >> 5;
    unsigned long long v = threadIdx.x < nw ? s_key[threadIdx.x] : 0ull;
    v = warp_max_u64(v);
    if (threadIdx.x == 0) s_key[0] = v;
  }
  __syncthreads();
  const unsigned long long m = s_key[0];
  if (m == 0ull) {
    if (threadIdx.x == 0) {
      out[0] = __int_as_float(-1);
      out[1] = -INFINITY;
      out[2] = out[3] = 0.0f;
    }
    return;
  }
  if (mine != m) return;  // exactly one thread holds the winning (unique) key
  const int c = (int)(0xFFFFFFFFull - (m & 0xFFFFFFFFull));
  float thr = 0.0f, fair = INFINITY;
  for (int i = 0; i < sp.n_slots; i++) {
    const float rp = __fmaf_rn(br[i], kInvScale, sp.alpha);
    out[4 + i] = rp;
    thr = (i == 0) ? rp : __fadd_rn(thr, rp);
    fair = fminf(fair, rp);
  }
  out[0] = __int_as_float(c);
  out[1] = bu;
  out[2] = thr;
  out[3] = fair;
}

void launch_sets_detail(const SpaceParams& sp, const float* ka, const float* kb, const float* w, const int64_t* set_ids,
                        int64_t n, float* out, cudaStream_t st) {
  if (n <= 0) return;
  k_sets_detail<false><<<(unsigned)n, 256, 0, st>>>(sp, ka, kb, w, set_ids, nullptr, out, nullptr, nullptr, nullptr,
                                                   nullptr, nullptr);
}

void launch_best_detail(const SpaceParams& sp, const float* ka, const float* kb, const float* w,
                        const unsigned long long* key, const unsigned long long* err, unsigned long long* host_out,
                        const float* hj, const DeviceTables* tb, cudaStream_t st) {
  // host_out is pinned host memory (UVA-mapped): [0] validation word, [1] key,
  // [2..5] the detail row -- the kernel writes it directly, no copy. tb != NULL:
  // operands from hj and the coefficient tables (no ka / kb this step)
  const int64_t* no_ids = nullptr;
  const float* no_tab = nullptr;
  // one config per thread (one round of the evaluation's dependent loads): the
  // best set's detail is the step's last kernel
  const unsigned nt = (unsigned)std::min(512, std::max(32, (sp.n_cfg + 31) / 32 * 32));
  if (tb)
    launch_pdl(k_sets_detail<true>, dim3(1), dim3(nt), 0, st, sp, ka, kb, w, no_ids, key,
               reinterpret_cast<float*>(host_out + 2), err, host_out, hj, tb->coef_c, tb->coef_d);
  else
    launch_pdl(k_sets_detail<false>, dim3(1), dim3(nt), 0, st, sp, ka, kb, w, no_ids, key,
               reinterpret_cast<float*>(host_out + 2), err, host_out, no_tab, no_tab, no_tab);
}

// Rank sort of a short list of unique keys, descending: position of key i =
// number of keys greater than it (the greedy picks, <= n_jobs / n_slots).
__global__ void k_sort_keys_desc(const unsigned long long* __restrict__ keys, int64_t n,
                                 unsigned long long* __restrict__ sorted) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  unsigned long long k = keys[i];
  int64_t pos = 0;
  for (int64_t t = 0; t < n; t++) pos += keys[t] > k;
  sorted[pos] = k;
}

void launch_sort_keys_desc(const unsigned long long* keys, int64_t n, unsigned long long* sorted, cudaStream_t st) {
  if (n <= 0) return;
  k_sort_keys_desc<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(keys, n, sorted);
}

// ---------------------------------------------------------------------------
// a10 exact allocation: one thread per partition rank. Rank digits, most
// significant first: level i picks the d_i-th partner (pairs) or partner pair
// (triples, lexicographic) among the free jobs above the lowest free job --
// the enumeration order of DESIGN.md R12. W = sum of per-set objectives in
// formation order (FP32); partitions with an infeasible set are skipped.
__device__ __forceinline__ int nth_set_bit(uint32_t m, int n) {
  for (int i = 0; i < n; i++) m &= m - 1;
  return __ffs(m) - 1;
}

__device__ bool decode_partition(int n_slots, int n_jobs, int64_t rank, int64_t* ids) {
  int k = n_jobs / n_slots;
  // place values
  int64_t place[16];
  int64_t acc = 1;
  for (int i = k - 1; i >= 0; i--) {
    place[i] = acc;
    int m = n_jobs - 1 - n_slots * i;
    int64_t radix = n_slots == 2 ? m : (int64_t)m * (m - 1) / 2;
    acc *= radix;
  }
  if (rank >= acc) return false;
  uint32_t freem = (n_jobs >= 32) ? 0xFFFFFFFFu : ((1u << n_jobs) - 1u);
  for (int i = 0; i < k; i++) {
    int m = n_jobs - 1 - n_slots * i;
    int64_t radix = n_slots == 2 ? m : (int64_t)m * (m - 1) / 2;
    int64_t d = (rank / place[i]) % radix;
    int a = __ffs(freem) - 1;
    freem &= ~(1u << a);
    if (n_slots == 2) {
      int b = nth_set_bit(freem, (int)d);
      freem &= ~(1u << b);
      ids[i] = (int64_t)b * (b - 1) / 2 + a;
    } else {
      int x = 0;
      int64_t dd = d;
      while (dd >= m - 1 - x) {
        dd -= m - 1 - x;
        x++;
      }
      int y = x + 1 + (int)dd;
      int b = nth_set_bit(freem, x), c = nth_set_bit(freem, y);
      freem &= ~(1u << b);
      freem &= ~(1u << c);
      ids[i] = (int64_t)c * (c - 1) * (c - 2) / 6 + (int64_t)b * (b - 1) / 2 + a;
    }
  }
  return true;
}

__global__ void k_exact_alloc(int n_slots, int n_jobs, const float* __restrict__ set_obj, int64_t n_match,
                              unsigned long long* best_key) {
  unsigned long long key = 0;
  int64_t ids[16];
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n_match;
       r += (int64_t)gridDim.x * blockDim.x) {
    if (!decode_partition(n_slots, n_jobs, r, ids)) continue;
    int k = n_jobs / n_slots;
    float w = 0.0f;
    bool ok = true;
    for (int i = 0; i < k; i++) {
      float o = set_obj[ids[i]];
      ok = ok && (o > -INFINITY);
      w = (i == 0) ? o : __fadd_rn(w, o);
    }
    if (ok) {
      unsigned long long kk = ((unsigned long long)ord_float_d(w) << 32) | (0xFFFFFFFFull - (uint64_t)r);
      key = kk > key ? kk : key;
    }
  }
  block_max_key(key, best_key);
}

void launch_exact_alloc(int n_slots, int64_t n_jobs, const float* set_obj, int64_t n_match,
                        unsigned long long* best_key, cudaStream_t st) {
  int bs = 256;
  int64_t blocks = (n_match + bs - 1) / bs;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  k_exact_alloc<<<(unsigned)blocks, bs, 0, st>>>(n_slots, (int)n_jobs, set_obj, n_match, best_key);
}

__global__ void k_exact_unrank(int n_slots, int n_jobs, const unsigned long long* best_key, int64_t* set_ids) {
  unsigned long long key = *best_key;
  int k = n_jobs / n_slots;
  if (key == 0) {
    for (int i = 0; i < k; i++) set_ids[i] = -1;
    set_ids[k] = -1;
    return;
  }
  int64_t rank = (int64_t)(0xFFFFFFFFull - (key & 0xFFFFFFFFull));
  decode_partition(n_slots, n_jobs, rank, set_ids);
  set_ids[k] = rank;
}

void launch_exact_unrank(int n_slots, int64_t n_jobs, const unsigned long long* best_key, int64_t* set_ids,
                         cudaStream_t st) {
  k_exact_unrank<<<1, 1, 0, st>>>(n_slots, (int)n_jobs, best_key, set_ids);
}

// ---------------------------------------------------------------------------
// a10 greedy allocation as locally-dominant rounds. With unique keys
// (obj, -set_id), a set that is the best remaining set of every one of its
// jobs is taken by the sequential greedy too, so iterating
//   propose: job_key[j] = max key over alive sets with all jobs free
//   select:  take every alive set whose key equals job_key of all its jobs
// until nothing is taken reproduces the sequential greedy's full pick set.
__global__ void k_greedy_init(int n_slots, const float* __restrict__ obj, int64_t first, int64_t count,
                              int64_t* alive, int64_t* n_alive) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= count) return;
  if (obj[k] > -INFINITY) {
    int64_t at = (int64_t)atomicAdd((unsigned long long*)n_alive, 1ull);
    alive[at] = first + k;
  }
}

void launch_greedy_init(int n_slots, int64_t n_jobs, const float* obj, int64_t first, int64_t count, int64_t* alive,
                        int64_t* n_alive, cudaStream_t st) {
  (void)n_jobs;
  if (count <= 0) return;
  k_greedy_init<<<(unsigned)((count + 255) / 256), 256, 0, st>>>(n_slots, obj, first, count, alive, n_alive);
}

template <int NS>
__device__ __forceinline__ bool all_free(int64_t sid, const uint32_t* taken, int64_t* j) {
  unrank_set<NS>(sid, j);
  bool ok = true;
#pragma unroll
  for (int i = 0; i < NS; i++) ok = ok && (taken[j[i]] == 0);
  return ok;
}

template <int NS>
__global__ void k_greedy_propose(const float* __restrict__ obj, int64_t first, const int64_t* __restrict__ alive,
                                 int64_t n_alive, const uint32_t* __restrict__ taken,
                                 unsigned long long* job_key) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n_alive) return;
  int64_t sid = alive[k];
  int64_t j[3];
  if (!all_free<NS>(sid, taken, j)) return;
  unsigned long long key = pack_key(obj[sid - first], sid);
#pragma unroll
  for (int i = 0; i < NS; i++)
    if (job_key[j[i]] < key) atomicMax(&job_key[j[i]], key);
}

template <int NS>
__global__ void k_greedy_select(const float* __restrict__ obj, int64_t first, const int64_t* __restrict__ alive,
                                int64_t n_alive, const unsigned long long* __restrict__ job_key, uint32_t* taken,
                                unsigned long long* picked, int64_t* n_picked) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n_alive) return;
  int64_t sid = alive[k];
  int64_t j[3];
  if (!all_free<NS>(sid, taken, j)) return;
  unsigned long long key = pack_key(obj[sid - first], sid);
  bool win = true;
#pragma unroll
  for (int i = 0; i < NS; i++) win = win && (job_key[j[i]] == key);
  if (!win) return;
  int64_t at = (int64_t)atomicAdd((unsigned long long*)n_picked, 1ull);
  picked[at] = key;
}

// Marks are applied in a separate pass so that `select` reads a consistent taken[].
template <int NS>
__global__ void k_greedy_mark(const unsigned long long* __restrict__ picked, int64_t from, int64_t to,
                              uint32_t* taken) {
  int64_t k = from + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= to) return;
  int64_t sid = (int64_t)(0xFFFFFFFFull - (picked[k] & 0xFFFFFFFFull));
  int64_t j[3];
  unrank_set<NS>(sid, j);
#pragma unroll
  for (int i = 0; i < NS; i++) taken[j[i]] = 1;
}

void launch_greedy_propose(int n_slots, int64_t n_jobs, const float* obj, int64_t first, const int64_t* alive,
                           int64_t n_alive, const uint32_t* taken, unsigned long long* job_key, cudaStream_t st) {
  (void)n_jobs;
  if (n_alive <= 0) return;
  unsigned g = (unsigned)((n_alive + 255) / 256);
  if (n_slots == 1) k_greedy_propose<1><<<g, 256, 0, st>>>(obj, first, alive, n_alive, taken, job_key);
  else if (n_slots == 2) k_greedy_propose<2><<<g, 256, 0, st>>>(obj, first, alive, n_alive, taken, job_key);
  else k_greedy_propose<3><<<g, 256, 0, st>>>(obj, first, alive, n_alive, taken, job_key);
}

void launch_greedy_select(int n_slots, int64_t n_jobs, const float* obj, int64_t first, const int64_t* alive,
                          int64_t n_alive, const unsigned long long* job_key, uint32_t* taken,
                          unsigned long long* picked, int64_t* n_picked, cudaStream_t st) {
  (void)n_jobs;
  if (n_alive <= 0) return;
  unsigned g = (unsigned)((n_alive + 255) / 256);
  if (n_slots == 1) k_greedy_select<1><<<g, 256, 0, st>>>(obj, first, alive, n_alive, job_key, taken, picked, n_picked);
  else if (n_slots == 2) k_greedy_select<2><<<g, 256, 0, st>>>(obj, first, alive, n_alive, job_key, taken, picked, n_picked);
  else k_greedy_select<3><<<g, 256, 0, st>>>(obj, first, alive, n_alive, job_key, taken, picked, n_picked);
}

void launch_greedy_mark(int n_slots, const unsigned long long* picked, int64_t from, int64_t to, uint32_t* taken,
                        cudaStream_t st) {
  if (to <= from) return;
  unsigned g = (unsigned)((to - from + 255) / 256);
  if (n_slots == 1) k_greedy_mark<1><<<g, 256, 0, st>>>(picked, from, to, taken);
  else if (n_slots == 2) k_greedy_mark<2><<<g, 256, 0, st>>>(picked, from, to, taken);
  else k_greedy_mark<3><<<g, 256, 0, st>>>(picked, from, to, taken);
}

template <int NS>
__global__ void k_greedy_compact(const int64_t* __restrict__ alive, int64_t n_alive, const uint32_t* __restrict__ taken,
                                 int64_t* alive_out, int64_t* n_out) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n_alive) return;
  int64_t sid = alive[k];
  int64_t j[3];
  if (!all_free<NS>(sid, taken, j)) return;
  int64_t at = (int64_t)atomicAdd((unsigned long long*)n_out, 1ull);
  alive_out[at] = sid;
}

void launch_greedy_compact(int n_slots, int64_t n_jobs, const int64_t* alive, int64_t n_alive, const uint32_t* taken,
                           int64_t* alive_out, int64_t* n_out, cudaStream_t st) {
  (void)n_jobs;
  if (n_alive <= 0) return;
  unsigned g = (unsigned)((n_alive + 255) / 256);
  if (n_slots == 1) k_greedy_compact<1><<<g, 256, 0, st>>>(alive, n_alive, taken, alive_out, n_out);
  else if (n_slots == 2) k_greedy_compact<2><<<g, 256, 0, st>>>(alive, n_alive, taken, alive_out, n_out);
  else k_greedy_compact<3><<<g, 256, 0, st>>>(alive, n_alive, taken, alive_out, n_out);
}

// ---------------------------------------------------------------------------
// Greedy rounds for pairs without atomics per set: the shard's per-set
// objectives form the upper triangle of an N x N matrix stored column by
// column (colex: column j1 holds rows 0..j1-1 contiguously). A block scans a
// 64 x 64 tile with coalesced column segments, reduces row and column maxima
// of the free-pair keys in shared memory and issues one atomicMax per row and
// column of the tile. Selection is then per job (O(N)): a pair is taken iff it
// is the best free pair of both its jobs. Every rank derives the same picks
// from the all-reduced job_key, so no taken[] exchange is needed.
__global__ void __launch_bounds__(256) k_greedy_pairs_propose(const float* __restrict__ obj, int64_t first,
                                                              int64_t c0, int64_t c1, int64_t jt0, int64_t base,
                                                              int64_t n_tiles, const uint32_t* __restrict__ taken,
                                                              unsigned long long* job_key) {
  __shared__ unsigned long long s_row[4][64];
  __shared__ unsigned long long s_col[64];
  const int64_t t = blockIdx.x;
  if (t >= n_tiles) return;
  int64_t u = t + base;
  int64_t J = (int64_t)((sqrt(8.0 * (double)u + 1.0) - 1.0) * 0.5);
  while (J * (J + 1) / 2 > u) J--;
  while ((J + 1) * (J + 2) / 2 <= u) J++;
  const int64_t I = u - J * (J + 1) / 2;
  const int lane_row = threadIdx.x & 63, cg = threadIdx.x >> 6;
  const int64_t j0 = I * 64 + lane_row;
  if (threadIdx.x < 64) s_col[threadIdx.x] = 0ull;
  __syncthreads();
  const bool row_free = j0 < c1 && taken[j0] == 0;
  unsigned long long rbest = 0ull;
  for (int k = 0; k < 16; k++) {
    const int cl = cg + 4 * k;
    const int64_t j1 = J * 64 + cl;
    unsigned long long kk = 0ull;
    if (row_free && j0 < j1 && j1 >= c0 && j1 < c1 && taken[j1] == 0) {
      const int64_t sid = j1 * (j1 - 1) / 2 + j0;
      const float o = obj[sid - first];
      if (o > -INFINITY) kk = pack_key(o, sid);
    }
    rbest = kk > rbest ? kk : rbest;
    unsigned long long cm = warp_max_u64(kk);  // a warp = 32 rows of one column
    if ((threadIdx.x & 31) == 0 && cm) atomicMax(&s_col[cl], cm);
  }
  s_row[cg][lane_row] = rbest;
  __syncthreads();
  if (threadIdx.x < 64) {
    unsigned long long r = s_row[0][threadIdx.x];
    for (int q = 1; q < 4; q++) r = s_row[q][threadIdx.x] > r ? s_row[q][threadIdx.x] : r;
    const int64_t jr = I * 64 + threadIdx.x;
    if (r && job_key[jr] < r) atomicMax(&job_key[jr], r);
    const unsigned long long c = s_col[threadIdx.x];
    const int64_t jc = J * 64 + threadIdx.x;
    if (c && job_key[jc] < c) atomicMax(&job_key[jc], c);
  }
}

__global__ void k_greedy_pairs_select(const unsigned long long* __restrict__ job_key, int64_t n_jobs,
                                      unsigned long long* picked, int64_t* n_picked) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n_jobs) return;
  const unsigned long long key = job_key[j];
  if (!key) return;
  const int64_t sid = (int64_t)(0xFFFFFFFFull - (key & 0xFFFFFFFFull));
  int64_t jj[2];
  unrank_set<2>(sid, jj);
  if (jj[0] != j) return;  // the lower job of the pair decides
  if (job_key[jj[1]] != key) return;
  int64_t at = (int64_t)atomicAdd((unsigned long long*)n_picked, 1ull);
  picked[at] = key;
}

void launch_greedy_pairs_propose(const float* obj, int64_t first, int64_t c0, int64_t c1, const uint32_t* taken,
                                 unsigned long long* job_key, cudaStream_t st) {
  if (c1 <= c0) return;
  int64_t jt0 = c0 / 64, jt1 = (c1 - 1) / 64;
  int64_t base = jt0 * (jt0 + 1) / 2;
  int64_t n_tiles = (jt1 + 1) * (jt1 + 2) / 2 - base;
  k_greedy_pairs_propose<<<(unsigned)n_tiles, 256, 0, st>>>(obj, first, c0, c1, jt0, base, n_tiles, taken, job_key);
}

void launch_greedy_pairs_select(const unsigned long long* job_key, int64_t n_jobs, unsigned long long* picked,
                                int64_t* n_picked, cudaStream_t st) {
  if (n_jobs <= 0) return;
  k_greedy_pairs_select<<<(unsigned)((n_jobs + 255) / 256), 256, 0, st>>>(job_key, n_jobs, picked, n_picked);
}

// ---------------------------------------------------------------------------
__global__ void k_fill_u64(unsigned long long* p, unsigned long long v, int64_t n) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k < n) p[k] = v;
}
__global__ void k_fill_u32(uint32_t* p, uint32_t v, int64_t n) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k < n) p[k] = v;
}
void launch_fill_u64(unsigned long long* p, unsigned long long v, int64_t n, cudaStream_t st) {
  if (n > 0) k_fill_u64<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(p, v, n);
}
void launch_fill_u32(uint32_t* p, uint32_t v, int64_t n, cudaStream_t st) {
  if (n > 0) k_fill_u32<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(p, v, n);
}

}  // namespace cosched
