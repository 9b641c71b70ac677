// truth.cu -- worst / proposal / best evaluation of the search's choices against
// a ground-truth performance model, sm_100a.
//
// PAPER.md §5.2.2 L752 ("The worst/best chooses one partitioning/allocation state
// (S) from those meet the fairness constraint"), L777 (the geometric means of
// worst, proposal and best), evaluated here for every set of the queue: the
// proposal is the search's choice (cosched_score_all's cfg), scored by the
// ground truth; best / worst are the extremes of the ground-truth objective
// over the configs whose ground-truth fairness exceeds alpha.
//
// The ground truth is SPEC.md's synthetic GPU (`true_rperf`, L430-470) with
// caller-given constants -- a stand-in for the A100 measurements the paper
// uses (reading R21). For the apps co-located on state (g_i, memory option) at
// cap P (c_i = F1/100, b_i = F3/100, t_i = (F6+F7+F8)/F1):
//   draw = w_base + w_gpc sum_i g_i c_i (1 + kappa t_i)
//   thr  = clamp((P - w_base) / (draw - w_base), f_min, 1) if draw > P else 1
//   r_i  = min(1, (g_i / g_full) thr / c_i, mem_i / b_i)      (b term only if b_i > 0)
//   mem_i = modules(g_i) / n_modules (private) | b_i or b_i / sum b (shared)
// normalised by the app alone on the full chip (g_full, shared) at P_max.
// FP32, one thread per set.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "cosched_internal.h"
#include "device_common.cuh"

namespace cosched {

namespace {

struct TruthParams {
  int32_t n_slots, n_states, n_caps, objective;
  float alpha;
  float g_full, n_modules, w_base, w_gpc, kappa, f_min, p_max;
  float modules[17];                    // by GPC count 0..16
  int8_t gpcs[kMaxStates][kMaxSlots];
  int8_t mem[kMaxStates];
  float caps[kMaxCaps];
  float inv_caps[kMaxCaps];
};

__device__ __forceinline__ float raw_rperf(const TruthParams& q, const float* c, const float* b, const float* t,
                                           const int* g, int n, int mem, float P, int i) {
  float draw = q.w_base;
  float bsum = 0.0f;
  for (int k = 0; k < n; k++) {
    draw = __fmaf_rn(q.w_gpc * (float)g[k], c[k] * (1.0f + q.kappa * t[k]), draw);
    bsum += b[k];
  }
  float thr = 1.0f;
  if (draw > P) thr = fminf(fmaxf((P - q.w_base) / fmaxf(draw - q.w_base, 1e-12f), q.f_min), 1.0f);
  float r = fminf(1.0f, ((float)g[i] / q.g_full) * thr / c[i]);
  if (b[i] > 0.0f) {
    const float memv = mem ? q.modules[g[i]] / q.n_modules : (bsum <= 1.0f ? b[i] : b[i] / fmaxf(bsum, 1e-12f));
    r = fminf(r, memv / b[i]);
  }
  return r;
}

// per queue position: (c, b, t, baseline) of its app
__global__ void k_truth_jobs(const float* __restrict__ F, const int32_t* __restrict__ jobs, int64_t n_jobs,
                             const TruthParams q, float4* __restrict__ jp) {
  const int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (n >= n_jobs) return;
  const int64_t row = jobs ? (int64_t)jobs[n] : n;
  const float* f = F + row * 8;
  const float c = f[0] / 100.0f, b = f[2] / 100.0f;
  const float t = f[0] > 0.0f ? (f[5] + f[6] + f[7]) / f[0] : 0.0f;
  const int g = (int)q.g_full;
  const float base = raw_rperf(q, &c, &b, &t, &g, 1, 0, q.p_max, 0);
  jp[n] = make_float4(c, b, t, base);
}

template <int NS>
__global__ void __launch_bounds__(256) k_truth_sets(const TruthParams q, const float4* __restrict__ jp, int64_t first,
                                                    int64_t count, const int32_t* __restrict__ prop_cfg,
                                                    float* __restrict__ prop_obj, float* __restrict__ prop_fair,
                                                    float* __restrict__ best_obj, float* __restrict__ worst_obj,
                                                    double* __restrict__ part) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};  // n_compared, sum log(prop/best), sum log(worst/best), violations
  if (k < count) {
    int64_t j[3];
    unrank_set<NS>(first + k, j);
    float c[NS], b[NS], t[NS], base[NS];
#pragma unroll
    for (int i = 0; i < NS; i++) {
      const float4 v = jp[j[i]];
      c[i] = v.x;
      b[i] = v.y;
      t[i] = v.z;
      base[i] = v.w;
    }
    const int pc = prop_cfg[k];
    float best = -INFINITY, worst = INFINITY, po = -INFINITY, pf = -INFINITY;
    // hoisted per set: c_eff, the sum of bandwidth demands, reciprocals
    float ceff[NS], inv_c[NS], inv_b[NS], inv_base[NS], bsum = 0.0f;
#pragma unroll
    for (int i = 0; i < NS; i++) {
      ceff[i] = c[i] * (1.0f + q.kappa * t[i]);
      inv_c[i] = 1.0f / c[i];
      inv_b[i] = b[i] > 0.0f ? 1.0f / b[i] : 0.0f;
      inv_base[i] = 1.0f / base[i];
      bsum += b[i];
    }
    for (int s = 0; s < q.n_states; s++) {
      // per state: the power draw and, per slot, the compute scale and the
      // memory-bound ceiling (independent of the cap)
      float draw = q.w_base, kc[NS], rcap[NS];
#pragma unroll
      for (int i = 0; i < NS; i++) draw = __fmaf_rn(q.w_gpc * (float)q.gpcs[s][i], ceff[i], draw);
      const float inv_ded = 1.0f / fmaxf(draw - q.w_base, 1e-12f);
#pragma unroll
      for (int i = 0; i < NS; i++) {
        const int g = q.gpcs[s][i];
        kc[i] = ((float)g / q.g_full) * inv_c[i];
        float cap = 1.0f;
        if (b[i] > 0.0f) {
          const float memv = q.mem[s] ? q.modules[g] / q.n_modules : (bsum <= 1.0f ? b[i] : b[i] / fmaxf(bsum, 1e-12f));
          cap = fminf(cap, memv * inv_b[i]);
        }
        rcap[i] = cap;
      }
      for (int p = 0; p < q.n_caps; p++) {
        const float P = q.caps[p];
        const float thr = draw > P ? fminf(fmaxf((P - q.w_base) * inv_ded, q.f_min), 1.0f) : 1.0f;
        float sum = 0.0f, fair = INFINITY;
#pragma unroll
        for (int i = 0; i < NS; i++) {
          const float r = fminf(rcap[i], kc[i] * thr) * inv_base[i];
          sum += r;
          fair = fminf(fair, r);
        }
        const float o = q.objective == 2 ? sum * q.inv_caps[p] : sum;
        if (fair > q.alpha) {
          best = fmaxf(best, o);
          worst = fminf(worst, o);
        }
        if (s * q.n_caps + p == pc) {
          po = o;
          pf = fair;
        }
      }
    }
    prop_obj[k] = po;
    prop_fair[k] = pf;
    best_obj[k] = best;
    worst_obj[k] = best > -INFINITY ? worst : -INFINITY;
    if (pc >= 0 && best > -INFINITY) {
      acc[0] = 1.0;
      acc[1] = log((double)po / (double)best);
      acc[2] = log((double)worst / (double)best);
      acc[3] = pf > q.alpha ? 0.0 : 1.0;
    }
  }
  // fixed-order block reduction -> one partial per block (deterministic)
  __shared__ double s_part[8][4];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int r = 0; r < 4; r++) {
    double v = acc[r];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xFFFFFFFFu, v, o);
    if (lane == 0) s_part[w][r] = v;
  }
  __syncthreads();
  if (threadIdx.x < 4) {
    double v = 0.0;
    for (int q2 = 0; q2 < 8; q2++) v += s_part[q2][threadIdx.x];
    part[blockIdx.x * 4 + threadIdx.x] = v;
  }
}

__global__ void k_truth_sum(const double* __restrict__ part, int64_t n_blocks, double* __restrict__ out) {
  // one block of 4 warps: warp r sums column r in a fixed order
  const int r = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double v = 0.0;
  for (int64_t b = lane; b < n_blocks; b += 32) v += part[b * 4 + r];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xFFFFFFFFu, v, o);
  if (lane == 0) out[r] = v;
}

}  // namespace

size_t truth_workspace_bytes(int64_t n_jobs, int64_t count) {
  return ((size_t)n_jobs * 16 + 255) / 256 * 256 + ((size_t)((count + 255) / 256) * 4 * 8 + 255) / 256 * 256 + 64;
}

int truth_enqueue(const cosched_truth_desc* d, const SpaceParams& sp, int objective, const int32_t* gpcs,
                  const int32_t* mem, const float* caps, const float* features, const int32_t* jobs, int64_t n_jobs,
                  int64_t first, int64_t count, const int32_t* prop_cfg, const cosched_eval_out* out, void* workspace,
                  double* sums_dev, cudaStream_t st) {
  TruthParams q;
  memset(&q, 0, sizeof q);
  q.n_slots = sp.n_slots;
  q.n_states = sp.n_states;
  q.n_caps = sp.n_caps;
  q.objective = objective;
  q.alpha = sp.alpha;
  q.g_full = (float)d->g_full;
  q.n_modules = (float)d->n_modules;
  q.w_base = d->w_base;
  q.w_gpc = d->w_gpc;
  q.kappa = d->kappa;
  q.f_min = d->f_min;
  q.p_max = d->p_max;
  for (int g = 0; g <= 16; g++) q.modules[g] = (float)d->modules[g];
  for (int s = 0; s < sp.n_states; s++) {
    for (int i = 0; i < sp.n_slots; i++) q.gpcs[s][i] = (int8_t)gpcs[s * sp.n_slots + i];
    q.mem[s] = (int8_t)mem[s];
  }
  for (int p = 0; p < sp.n_caps; p++) {
    q.caps[p] = caps[p];
    q.inv_caps[p] = 1.0f / caps[p];
  }
  char* base = (char*)workspace;
  float4* jp = (float4*)base;
  double* part = (double*)(base + ((size_t)n_jobs * 16 + 255) / 256 * 256);
  int launches = 0;
  k_truth_jobs<<<(unsigned)((n_jobs + 255) / 256), 256, 0, st>>>(features, jobs, n_jobs, q, jp);
  launches++;
  const int64_t blocks = (count + 255) / 256;
  if (count > 0) {
    if (sp.n_slots == 1)
      k_truth_sets<1><<<(unsigned)blocks, 256, 0, st>>>(q, jp, first, count, prop_cfg, out->prop_obj, out->prop_fair,
                                                        out->best_obj, out->worst_obj, part);
    else if (sp.n_slots == 2)
      k_truth_sets<2><<<(unsigned)blocks, 256, 0, st>>>(q, jp, first, count, prop_cfg, out->prop_obj, out->prop_fair,
                                                        out->best_obj, out->worst_obj, part);
    else
      k_truth_sets<3><<<(unsigned)blocks, 256, 0, st>>>(q, jp, first, count, prop_cfg, out->prop_obj, out->prop_fair,
                                                        out->best_obj, out->worst_obj, part);
    launches++;
  }
  k_truth_sum<<<1, 128, 0, st>>>(part, blocks, sums_dev);
  launches++;
  return cudaGetLastError() == cudaSuccess ? launches : -1;
}

}  // namespace cosched
