// node.cu -- node-level power budgeting across the GPUs of a node (SURVEY.md
// §8(f) NEXT #4), sm_100a.
//
// The job manager sets each GPU's power cap under a node
// budget (L782, L844). Reading R23: for the set allocated to GPU g,
//   thr_g(p) = max over states with Fairness > alpha of Throughput   (lowest state on ties)
// and per node one cap per GPU maximising sum_g thr_g(p_g) (Problem 1) or
// sum_g thr_g(p_g) / sum_g P(p_g) (Problem 2) subject to sum_g P(p_g) <= P_node:
// a multiple-choice knapsack over integer-watt caps, solved exactly by a DP over
// the total power in units of the caps' gcd (one block per node, threads over
// the budget axis, decisions kept for the backtrack).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "cosched_internal.h"
#include "device_common.cuh"

namespace cosched {

namespace {

// Block per GPU: thr of every config (-inf if infeasible) in shared memory, then
// per cap the best state.
template <int NS>
__global__ void k_node_frontier(const SpaceParams sp, const float* __restrict__ ka, const float* __restrict__ kb,
                                const float* __restrict__ w, const int64_t* __restrict__ set_ids,
                                float* __restrict__ front, int32_t* __restrict__ front_state) {
  extern __shared__ float s_thr[];  // [n_cfg]
  const int g = blockIdx.x;
  int64_t j[3];
  unrank_set<NS>(set_ids[g], j);
  for (int c = threadIdx.x; c < sp.n_cfg; c += blockDim.x) {
    const int s = c / sp.n_caps, p = c - s * sp.n_caps;
    float r[NS], o;
    eval_cfg<NS>(sp, ka, kb, w, j, s, p, r, &o);
    bool feas = true;
    float thr = 0.0f;
#pragma unroll
    for (int i = 0; i < NS; i++) {
      feas = feas && r[i] > 0.0f;
      const float rp = __fmaf_rn(r[i], kInvScale, sp.alpha);  // RPerf = margin / K + alpha
      thr = i == 0 ? rp : __fadd_rn(thr, rp);
    }
    s_thr[c] = feas ? thr : -INFINITY;
  }
  __syncthreads();
  for (int p = threadIdx.x; p < sp.n_caps; p += blockDim.x) {
    float best = -INFINITY;
    int arg = -1;
    for (int s = 0; s < sp.n_states; s++) {
      const float v = s_thr[s * sp.n_caps + p];
      if (v > best) {
        best = v;
        arg = s;
      }
    }
    front[(int64_t)g * sp.n_caps + p] = best;
    front_state[(int64_t)g * sp.n_caps + p] = arg;
  }
}

struct NodeParams {
  int32_t gpus, n_caps, U, objective;
  float unit_w;
  int32_t u[kMaxCaps];
};

__global__ void __launch_bounds__(1024) k_node_dp(const NodeParams q, const float* __restrict__ front,
                                                  const int32_t* __restrict__ front_state,
                                                  int8_t* __restrict__ choice, int32_t* __restrict__ caps_out,
                                                  int32_t* __restrict__ cfg_out, float* __restrict__ node_obj) {
  extern __shared__ float s_dp[];  // [2][U + 1]
  __shared__ float s_val[32];
  __shared__ int s_arg[32];
  const int node = blockIdx.x, U = q.U;
  float* cur = s_dp;
  float* nxt = s_dp + (U + 1);
  for (int b = threadIdx.x; b <= U; b += blockDim.x) cur[b] = b == 0 ? 0.0f : -INFINITY;
  __syncthreads();
  int8_t* ch = choice + (int64_t)node * q.gpus * (U + 1);
  for (int g = 0; g < q.gpus; g++) {
    const float* f = front + ((int64_t)node * q.gpus + g) * q.n_caps;
    for (int b = threadIdx.x; b <= U; b += blockDim.x) {
      float best = -INFINITY;
      int arg = -1;
      for (int p = 0; p < q.n_caps; p++) {
        const float fp = f[p];
        if (fp == -INFINITY || q.u[p] > b) continue;
        const float v = __fadd_rn(cur[b - q.u[p]], fp);  // sum in GPU order
        if (v > best) {  // strict: the lowest cap wins ties
          best = v;
          arg = p;
        }
      }
      nxt[b] = best;
      ch[(int64_t)g * (U + 1) + b] = (int8_t)arg;
    }
    __syncthreads();
    float* t = cur;
    cur = nxt;
    nxt = t;
  }
  // argmax over the total power (lowest total on ties)
  float bv = -INFINITY;
  int bb = -1;
  for (int b = threadIdx.x; b <= U; b += blockDim.x) {
    float v = cur[b];
    if (q.objective == 2) v = b > 0 ? v / ((float)b * q.unit_w) : -INFINITY;
    if (v > bv) {
      bv = v;
      bb = b;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const float v2 = __shfl_down_sync(0xFFFFFFFFu, bv, o);
    const int b2 = __shfl_down_sync(0xFFFFFFFFu, bb, o);
    if (v2 > bv || (v2 == bv && b2 >= 0 && (bb < 0 || b2 < bb))) {
      bv = v2;
      bb = b2;
    }
  }
  if ((threadIdx.x & 31) == 0) {
    s_val[threadIdx.x >> 5] = bv;
    s_arg[threadIdx.x >> 5] = bb;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    bv = -INFINITY;
    bb = -1;
    for (int k = 0; k < (int)(blockDim.x >> 5); k++)
      if (s_val[k] > bv || (s_val[k] == bv && s_arg[k] >= 0 && (bb < 0 || s_arg[k] < bb))) {
        bv = s_val[k];
        bb = s_arg[k];
      }
    node_obj[node] = bv;
    int b = bb;
    for (int g = q.gpus - 1; g >= 0; g--) {
      const int64_t gi = (int64_t)node * q.gpus + g;
      if (bv == -INFINITY) {
        caps_out[gi] = -1;
        cfg_out[gi] = -1;
        continue;
      }
      const int p = ch[(int64_t)g * (U + 1) + b];
      caps_out[gi] = p;
      cfg_out[gi] = front_state[gi * q.n_caps + p] * q.n_caps + p;
      b -= q.u[p];
    }
  }
}

}  // namespace

size_t node_workspace_bytes(int64_t n_gpus, int32_t n_caps, int32_t U, int32_t gpus_per_node) {
  const int64_t n_nodes = n_gpus / gpus_per_node;
  auto al = [](size_t b) { return (b + 255) / 256 * 256; };
  return al((size_t)n_gpus * 8) + al((size_t)n_gpus * n_caps * 4) * 2 + al((size_t)n_nodes * gpus_per_node * (U + 1)) +
         al((size_t)n_gpus * 4) * 2 + al((size_t)n_nodes * 4);
}

int node_enqueue(const SpaceParams& sp, const float* ka, const float* kb, const float* w, const int64_t* set_ids_host,
                 int64_t n_gpus, int32_t gpus_per_node, int32_t U, float unit_w, const int32_t* u, int32_t objective,
                 void* workspace, int32_t* caps_host, int32_t* cfg_host, float* node_obj_host, cudaStream_t st) {
  const int64_t n_nodes = n_gpus / gpus_per_node;
  auto al = [](size_t b) { return (b + 255) / 256 * 256; };
  char* p = (char*)workspace;
  int64_t* d_ids = (int64_t*)p;
  p += al((size_t)n_gpus * 8);
  float* d_front = (float*)p;
  p += al((size_t)n_gpus * sp.n_caps * 4);
  int32_t* d_fstate = (int32_t*)p;
  p += al((size_t)n_gpus * sp.n_caps * 4);
  int8_t* d_choice = (int8_t*)p;
  p += al((size_t)n_nodes * gpus_per_node * (U + 1));
  int32_t* d_caps = (int32_t*)p;
  p += al((size_t)n_gpus * 4);
  int32_t* d_cfg = (int32_t*)p;
  p += al((size_t)n_gpus * 4);
  float* d_obj = (float*)p;
  if (cudaMemcpyAsync(d_ids, set_ids_host, n_gpus * 8, cudaMemcpyHostToDevice, st) != cudaSuccess) return -1;
  const size_t fsm = (size_t)sp.n_cfg * 4;
  if (sp.n_slots == 1)
    k_node_frontier<1><<<(unsigned)n_gpus, 256, fsm, st>>>(sp, ka, kb, w, d_ids, d_front, d_fstate);
  else if (sp.n_slots == 2)
    k_node_frontier<2><<<(unsigned)n_gpus, 256, fsm, st>>>(sp, ka, kb, w, d_ids, d_front, d_fstate);
  else
    k_node_frontier<3><<<(unsigned)n_gpus, 256, fsm, st>>>(sp, ka, kb, w, d_ids, d_front, d_fstate);
  NodeParams q;
  q.gpus = gpus_per_node;
  q.n_caps = sp.n_caps;
  q.U = U;
  q.objective = objective;
  q.unit_w = unit_w;
  for (int i = 0; i < sp.n_caps; i++) q.u[i] = u[i];
  const size_t dsm = (size_t)2 * (U + 1) * 4;
  smem_optin((const void*)k_node_dp, dsm);
  k_node_dp<<<(unsigned)n_nodes, 1024, dsm, st>>>(q, d_front, d_fstate, d_choice, d_caps, d_cfg, d_obj);
  if (cudaMemcpyAsync(caps_host, d_caps, n_gpus * 4, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaMemcpyAsync(cfg_host, d_cfg, n_gpus * 4, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaMemcpyAsync(node_obj_host, d_obj, n_nodes * 4, cudaMemcpyDeviceToHost, st) != cudaSuccess)
    return -1;
  return cudaGetLastError() == cudaSuccess ? 2 : -1;
}

}  // namespace cosched
