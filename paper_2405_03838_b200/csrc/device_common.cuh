// device_common.cuh -- small device helpers of the CUDA path.
#pragma once
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

namespace cosched {

// Table `functions` in FP32, IEEE division (no fast-math):
//   H = (F1/100 - H2, (F6+F7+F8)/100, F2/F1, F4/100, F5/100, 1),  J = (F3/100, F4/100, 1)
__device__ __forceinline__ void basis_hj(const float* __restrict__ f, float h[6], float j[3]) {
  float f1 = f[0], f2 = f[1], f3 = f[2], f4 = f[3], f5 = f[4];
  float tensor = __fadd_rn(__fadd_rn(f[5], f[6]), f[7]);
  h[1] = __fdiv_rn(tensor, 100.0f);
  h[0] = __fsub_rn(__fdiv_rn(f1, 100.0f), h[1]);
  h[2] = __fdiv_rn(f2, f1);
  h[3] = __fdiv_rn(f4, 100.0f);
  h[4] = __fdiv_rn(f5, 100.0f);
  h[5] = 1.0f;
  j[0] = __fdiv_rn(f3, 100.0f);
  j[1] = __fdiv_rn(f4, 100.0f);
  j[2] = 1.0f;
}

// Projection rows (slice-major, padded; see Workspace in cosched_internal.h)
template <typename SP>
__device__ __forceinline__ const float* ka_row(const float* __restrict__ base, const SP& sp, int slice, int64_t job) {
  return base + ((int64_t)slice * sp.n_jobs_pad + job) * sp.rs;
}
template <typename SP>
__device__ __forceinline__ const float* w_row(const float* __restrict__ base, const SP& sp, int slot, int state,
                                              int64_t job) {
  return base + (((int64_t)slot * sp.n_states + state) * sp.n_jobs_pad + job) * sp.rs;
}

// One candidate (set j[], state s, cap p) in the canonical FP32 evaluation
// order shared by every scorer (generic, tiled pairs, tiled triples, detail):
//   pairs:   r0 = ka0 + kb1,              r1 = ka1 + kb0,              o = w0 + w1
//   triples: r0 = ka0 + (kb1 + kb2),      r1 = (ka1 + kb2) + kb0,
//            r2 = (ka2 + kb1) + kb0,      o  = w0 + (w1 + w2)
// (kaX = ka[s_slot][j_X], kbX = kb[s_slot][j_X] for the slot being scored.)
template <int NS, typename SP>
__device__ __forceinline__ void eval_cfg(const SP& sp, const float* __restrict__ ka, const float* __restrict__ kb,
                                         const float* __restrict__ w, const int64_t* j, int s, int p, float* r,
                                         float* o) {
  if (NS == 1) {
    r[0] = ka_row(ka, sp, sp.slice[s][0], j[0])[p];
    *o = w_row(w, sp, 0, s, j[0])[p];
  } else if (NS == 2) {
    const int s0 = sp.slice[s][0], s1 = sp.slice[s][1];
    r[0] = __fadd_rn(ka_row(ka, sp, s0, j[0])[p], ka_row(kb, sp, s0, j[1])[p]);
    r[1] = __fadd_rn(ka_row(ka, sp, s1, j[1])[p], ka_row(kb, sp, s1, j[0])[p]);
    *o = __fadd_rn(w_row(w, sp, 0, s, j[0])[p], w_row(w, sp, 1, s, j[1])[p]);
  } else {
    const int s0 = sp.slice[s][0], s1 = sp.slice[s][1], s2 = sp.slice[s][2];
    r[0] = __fadd_rn(ka_row(ka, sp, s0, j[0])[p], __fadd_rn(ka_row(kb, sp, s0, j[1])[p], ka_row(kb, sp, s0, j[2])[p]));
    r[1] = __fadd_rn(__fadd_rn(ka_row(ka, sp, s1, j[1])[p], ka_row(kb, sp, s1, j[2])[p]), ka_row(kb, sp, s1, j[0])[p]);
    r[2] = __fadd_rn(__fadd_rn(ka_row(ka, sp, s2, j[2])[p], ka_row(kb, sp, s2, j[1])[p]), ka_row(kb, sp, s2, j[0])[p]);
    *o = __fadd_rn(w_row(w, sp, 0, s, j[0])[p], __fadd_rn(w_row(w, sp, 1, s, j[1])[p], w_row(w, sp, 2, s, j[2])[p]));
  }
}

// ---- hill climbing over the (state x cap) grid (NEXT #2; R22) ----
// f(c) = objective of config c if every margin is positive (Fairness > alpha), else -inf,
// in the canonical FP32 order of eval_cfg.
template <int NS, typename SP>
__device__ __forceinline__ float hc_value(const SP& sp, const float* __restrict__ ka, const float* __restrict__ kb,
                                          const float* __restrict__ w, const int64_t* j, int s, int p) {
  float r[NS], o;
  eval_cfg<NS>(sp, ka, kb, w, j, s, p, r, &o);
  bool feas = true;
#pragma unroll
  for (int i = 0; i < NS; i++) feas = feas && (r[i] > 0.0f);
  return feas ? o : -INFINITY;
}

// Steepest ascent from (*s, *p): the existing 4-neighbours in increasing config
// index, move to the first largest if strictly better; stop at a local optimum.
template <int NS, typename SP>
__device__ float hc_climb(const SP& sp, const float* __restrict__ ka, const float* __restrict__ kb,
                          const float* __restrict__ w, const int64_t* j, int* s_io, int* p_io, int* evals) {
  int s = *s_io, p = *p_io;
  float v = hc_value<NS>(sp, ka, kb, w, j, s, p);
  (*evals)++;
  for (;;) {
    int bs = -1, bp = -1;
    float bv = v;
#pragma unroll
    for (int k = 0; k < 4; k++) {
      const int ns = s + (k == 0 ? -1 : (k == 3 ? 1 : 0)), np = p + (k == 1 ? -1 : (k == 2 ? 1 : 0));
      if (ns < 0 || ns >= sp.n_states || np < 0 || np >= sp.n_caps) continue;
      const float u = hc_value<NS>(sp, ka, kb, w, j, ns, np);
      (*evals)++;
      if (u > bv) {
        bv = u;
        bs = ns;
        bp = np;
      }
    }
    if (bs < 0) break;
    s = bs;
    p = bp;
    v = bv;
  }
  *s_io = s;
  *p_io = p;
  return v;
}

// The search of R22: climb from the start; if that ends infeasible, climb from every
// other config in canonical order until one ends feasible. Returns cfg (-1: none).
template <int NS, typename SP>
__device__ int hill_search(const SP& sp, const float* __restrict__ ka, const float* __restrict__ kb,
                           const float* __restrict__ w, const int64_t* j, int s0, int p0, float* obj, int* evals) {
  int s = s0, p = p0;
  float v = hc_climb<NS>(sp, ka, kb, w, j, &s, &p, evals);
  if (v == -INFINITY) {
    const int start = s0 * sp.n_caps + p0;
    for (int c = 0; c < sp.n_cfg && v == -INFINITY; c++) {
      if (c == start) continue;
      s = c / sp.n_caps;
      p = c - s * sp.n_caps;
      v = hc_climb<NS>(sp, ka, kb, w, j, &s, &p, evals);
    }
  }
  *obj = v;
  return v == -INFINITY ? -1 : s * sp.n_caps + p;
}

// order-preserving float -> u32 (larger float <=> larger u32; -0 < +0)
__device__ __forceinline__ uint32_t ord_float_d(float f) {
  uint32_t b = __float_as_uint(f);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

__device__ __forceinline__ float unord_float_d(uint32_t o) {
  uint32_t b = (o & 0x80000000u) ? (o & 0x7FFFFFFFu) : ~o;
  return __uint_as_float(b);
}

// ---- packed objective of the tiled scorers ----
// Inverse quantum inv = (2^25 - 2 - NS) / sum_i (wmax_i - wmin_i) from the
// per-slot ranges wmm (order-preserving u32, k_project_all); 0 when every share
// is equal (then every packed objective ties and the canonical order decides).
template <int NS>
__device__ __forceinline__ float quant_inv(const unsigned* __restrict__ wmm) {
  float span = 0.0f;
#pragma unroll
  for (int i = 0; i < NS; i++) span += unord_float_d(wmm[2 * i + 1]) - unord_float_d(wmm[2 * i]);
  return span > 0.0f ? (float)(33554430 - NS) / span : 0.0f;
}

// Exactness bound of the packed argmax (DESIGN.md §2 "Exactness of the tiled
// argmax"). Each slot's code q = rint(fma(w, inv, -fl(lo*inv))) is within 1.5
// quanta of inv*w + const_slot (one FMA rounding <= 1 below 2^25, rint 0.5), so a
// candidate's packed key is within 1.5*NS quanta of inv*(sum of its FP32 shares)
// + const, and the config the max picks has a true FP32 objective at most
// 3*NS/inv below the set's FP32 maximum. Sets whose chosen objective O satisfies
// 3*NS/inv > (tau/2)*O, i.e. O < 6*NS/(tau*inv), are re-scored exactly
// (k_rescore_sets): every reported choice is within tau/2 = 5e-6 relative of the
// exact FP32 argmax's objective, whatever the input.
constexpr float kTauObj = 1e-5f;  // BASELINE.json north_star: objectives within 1e-5 relative
template <int NS>
__device__ __forceinline__ float rescore_threshold(const unsigned* __restrict__ wmm) {
  const float inv = quant_inv<NS>(wmm);
  return inv > 0.0f ? (6.0f * NS / kTauObj) / inv : 0.0f;
}

// Packed argmax key: larger objective first, then lower set id. Unique per set.
__device__ __forceinline__ unsigned long long pack_key(float obj, int64_t sid) {
  return ((unsigned long long)ord_float_d(obj) << 32) | (0xFFFFFFFFull - (unsigned long long)(uint32_t)sid);
}

__device__ __forceinline__ int64_t c2(int64_t n) { return n * (n - 1) / 2; }
// PDL (cosched_internal.h launch_pdl): wait for the predecessor kernel's
// completion and memory; allow the successor to launch
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ int64_t c3(int64_t n) { return n * (n - 1) * (n - 2) / 6; }

// colex unranking: set id -> ascending queue positions. FP32 root estimates
// (within +-2 of the answer for ids < 2^53) corrected by exact integer tests.
template <int NS>
__device__ __forceinline__ void unrank_set(int64_t id, int64_t* j) {
  if (NS == 1) {
    j[0] = id;
  } else if (NS == 2) {
    int64_t b = (int64_t)((1.0f + sqrtf(1.0f + 8.0f * (float)id)) * 0.5f);
    while (b > 1 && c2(b) > id) b--;
    while (c2(b + 1) <= id) b++;
    j[1] = b;
    j[0] = id - c2(b);
  } else {
    int64_t c = (int64_t)cbrtf(6.0f * (float)id) + 1;
    while (c > 2 && c3(c) > id) c--;
    while (c3(c + 1) <= id) c++;
    int64_t rest = id - c3(c);
    int64_t b = (int64_t)((1.0f + sqrtf(1.0f + 8.0f * (float)rest)) * 0.5f);
    while (b > 1 && c2(b) > rest) b--;
    while (c2(b + 1) <= rest) b++;
    j[2] = c;
    j[1] = b;
    j[0] = rest - c2(b);
  }
}

__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long w = __shfl_xor_sync(0xFFFFFFFFu, v, o);
    v = w > v ? w : v;
  }
  return v;
}

// Block-wide max of a per-thread key, then one atomicMax per block. The max of
// unique keys does not depend on the order, so the result is deterministic.
__device__ __forceinline__ void block_max_key(unsigned long long key, unsigned long long* dst) {
  __shared__ unsigned long long s_part[32];
  key = warp_max_u64(key);
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) s_part[w] = key;
  __syncthreads();
  if (w == 0) {
    int nw = (blockDim.x + 31) >> 5;
    unsigned long long v = lane < nw ? s_part[lane] : 0ull;
    v = warp_max_u64(v);
    if (lane == 0 && v) atomicMax(dst, v);
  }
}

}  // namespace cosched
