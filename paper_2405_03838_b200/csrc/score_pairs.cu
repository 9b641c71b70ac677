// score_pairs.cu -- the fast pair scorer (SURVEY.md §8(a) a4-a8 for n_slots = 2), sm_100a.
//
// Work: for every pair (j0 < j1) of this rank's column range and every config
// c = (state s, cap p):
//   r0'' = ka[s0][j0][p] + kb[s0][j1][p]      (= K*(RPerf_0 - alpha))
//   r1'' = ka[s1][j1][p] + kb[s1][j0][p]
//   o    = w[0][s][j0][p] + w[1][s][j1][p]    (= Throughput [/P])
//   x    = min3(o, r0'', r1'')                (= o when Fairness > alpha, <= 0 otherwise)
// and the per-pair argmax of x over configs (first config on ties).
//
// Design (DESIGN.md §5 "Pair scorer"):
//  - persistent CTAs walk 64x64 tiles of the pair triangle (column tiles in
//    ascending order); each thread owns a 4x4 register micro-tile of pairs
//    (j0 = tx + 16a, j1 = ty + 16b: lanes hold consecutive j0, so the per-pair
//    output writes coalesce);
//  - per state, the tile's operand rows -- 6 blocks of 64 jobs x rs floats,
//    contiguous in the slice-major projection layout -- land in shared memory
//    with 6 TMA bulk copies (cp.async.bulk + mbarrier complete_tx), double
//    buffered so the next state streams in while this one is scored; the row
//    stride rs puts 8 consecutive rows in distinct 16-byte bank groups;
//  - per 4 caps: float4 LDS operands, FADD2 for r0'', r1'', o (1.5 per
//    candidate), one FMNMX3 for the masked objective and half an FMNMX3 for the
//    running max (the ALU pipe, 64 lanes/clk/SM, binds: profiles/r01/microbench*);
//  - the argmax index is tracked per group of 4G caps (FSETP + 2 predicated
//    moves per group) and resolved exactly at tile end by re-evaluating the
//    winning group from L2 with float4 loads (first max within the group,
//    strict > across groups = canonical order).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "cosched_internal.h"
#include "device_common.cuh"
#include "tile_common.cuh"

namespace cosched {

namespace {

constexpr int kTile = 64;      // pairs per tile side
constexpr int kThreads = 256;  // 16 x 16 threads, 4 x 4 pairs each
constexpr int kM = 4;          // micro-tile side
constexpr int kBgRow = kTile + 4;  // (4*ty + tx) mod 32: the group-end LDS/STS of a warp hit distinct banks

struct PairGrid {
  int64_t n_jobs;
  int64_t c0, c1;     // column (largest position) range of this shard: j1 in [c0, c1)
  int64_t n_tiles;
  int64_t base;       // tiles before the first column tile: jt0*(jt0+1)/2
  int64_t first_set;  // output index offset
  int groups_per_state;
};

__device__ __forceinline__ void tile_coords(const PairGrid& g, int64_t t, int64_t* I, int64_t* J) {
  // tiles are ordered column tile J ascending, row tile I = 0..J; cum(J) = J(J+1)/2 - base
  int64_t u = t + g.base;
  int64_t j = (int64_t)((sqrt(8.0 * (double)u + 1.0) - 1.0) * 0.5);
  while (j * (j + 1) / 2 > u) j--;
  while ((j + 1) * (j + 2) / 2 <= u) j++;
  *J = j;
  *I = u - j * (j + 1) / 2;
}

// Stage layout (floats): blocks [A0][B0][W0][A1][B1][W1], each kTile rows x rs.
//  A0 = ka[s0][I-rows], B0 = kb[s1][I-rows], W0 = w[slot 0][s][I-rows]
//  A1 = ka[s1][J-rows], B1 = kb[s0][J-rows], W1 = w[slot 1][s][J-rows]
__device__ __forceinline__ void issue_stage(float* stage, uint64_t* bar, const SpaceParams& sp,
                                            const float* __restrict__ ka, const float* __restrict__ kb,
                                            const float* __restrict__ w, int64_t I, int64_t J, int s) {
  const int s0 = sp.slice[s][0], s1 = sp.slice[s][1];
  const int blk = kTile * sp.rs;
  const unsigned bytes = (unsigned)blk * 4u;
  mbar_arrive_expect_tx(bar, 6u * bytes);
  const int64_t r0 = I * kTile, r1 = J * kTile;
  tma_bulk_g2s(stage + 0 * blk, ka_row(ka, sp, s0, r0), bytes, bar);
  tma_bulk_g2s(stage + 1 * blk, ka_row(kb, sp, s1, r0), bytes, bar);
  tma_bulk_g2s(stage + 2 * blk, w_row(w, sp, 0, s, r0), bytes, bar);
  tma_bulk_g2s(stage + 3 * blk, ka_row(ka, sp, s1, r1), bytes, bar);
  tma_bulk_g2s(stage + 4 * blk, ka_row(kb, sp, s0, r1), bytes, bar);
  tma_bulk_g2s(stage + 5 * blk, w_row(w, sp, 1, s, r1), bytes, bar);
}

}  // namespace

// NP = padded cap count known at compile time (0 = runtime): static row strides
// turn every operand load into an LDS with an immediate offset.
template <int NP, int G>
__global__ void __launch_bounds__(kThreads, 2)
    k_score_pairs_tiled(const SpaceParams sp, const PairGrid g, const float* __restrict__ ka,
                        const float* __restrict__ kb, const float* __restrict__ w, float* __restrict__ out_obj,
                        int32_t* __restrict__ out_cfg, unsigned long long* __restrict__ best_key,
                        const unsigned long long* __restrict__ err) {
  extern __shared__ __align__(128) float smem[];
  __shared__ __align__(8) uint64_t bars[2];
  if (*err != ~0ull) return;
  constexpr int kRS = NP ? (((NP >> 2) & 1) ? NP : NP + 4) : 0;
  const int rs = NP ? kRS : sp.rs;
  const int stage_floats = 6 * kTile * rs;
  // thread -> (tx, ty): a warp covers 4 j0 rows x 8 j1 rows, so each float4
  // operand load is one 128-byte shared-memory wavefront (j0 rows broadcast to
  // 8 lanes, 8 consecutive j1 rows in distinct bank groups)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int tx = ((warp & 3) << 2) | (lane & 3), ty = ((warp >> 2) << 3) | (lane >> 2);
  const int rs4 = rs >> 2;
  const int gps = NP ? (NP >> 2) / G : g.groups_per_state;
  unsigned long long key = 0;

  int64_t t = blockIdx.x;
  if (t >= g.n_tiles) {
    block_max_key(0ull, best_key);
    return;
  }
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    mbar_fence_init();
  }
  __syncthreads();
  int64_t I, J;
  tile_coords(g, t, &I, &J);
  int s = 0, buf = 0;
  unsigned phase[2] = {0u, 0u};
  if (threadIdx.x == 0) issue_stage(smem, &bars[0], sp, ka, kb, w, I, J, 0);

  // per pair, in shared memory ([j1 local][j0 local], padded rows): the best
  // masked objective so far and its group (state << 4 | group-in-state); read
  // and written once per group, which keeps the register file for operands.
  float* sbest = smem + 2 * stage_floats;
  int16_t* sbg = reinterpret_cast<int16_t*>(sbest + kTile * kBgRow);
  for (int e = threadIdx.x; e < kTile * kBgRow; e += kThreads) {
    sbest[e] = 0.0f;  // feasible masked objectives are > 0
    sbg[e] = -1;
  }
  __syncthreads();  // the owners of each pair read these at their first group end

  while (true) {
    // prefetch the next (tile, state) into the other buffer
    int64_t nt = t, nI = I, nJ = J;
    int ns = s + 1;
    if (ns == sp.n_states) {
      ns = 0;
      nt = t + gridDim.x;
      if (nt < g.n_tiles) tile_coords(g, nt, &nI, &nJ);
    }
    const bool has_next = nt < g.n_tiles;
    if (has_next && threadIdx.x == 0) issue_stage(smem + (buf ^ 1) * stage_floats, &bars[buf ^ 1], sp, ka, kb, w, nI, nJ, ns);
    mbar_wait(&bars[buf], phase[buf]);
    phase[buf] ^= 1u;

    const float4* st4 = reinterpret_cast<const float4*>(smem + buf * stage_floats);
    const int blk4 = kTile * rs4;
    const float4* A0 = st4 + 0 * blk4 + tx * rs4;
    const float4* B0 = st4 + 1 * blk4 + tx * rs4;
    const float4* W0 = st4 + 2 * blk4 + tx * rs4;
    const float4* A1 = st4 + 3 * blk4 + ty * rs4;
    const float4* B1 = st4 + 4 * blk4 + ty * rs4;
    const float4* W1 = st4 + 5 * blk4 + ty * rs4;
    const int row16 = 16 * rs4;  // float4s between rows r and r+16

#pragma unroll
    for (int grp = 0; grp < gps; grp++) {
      float m[kM][kM];
#pragma unroll
      for (int qq = 0; qq < G; qq++) {
        const int q = grp * G + qq;
        float4 a1[kM], b1[kM], w1[kM];
#pragma unroll
        for (int b = 0; b < kM; b++) {
          a1[b] = A1[b * row16 + q];
          b1[b] = B1[b * row16 + q];
          w1[b] = W1[b * row16 + q];
        }
#pragma unroll
        for (int a = 0; a < kM; a++) {
          const float4 a0 = A0[a * row16 + q];
          const float4 b0 = B0[a * row16 + q];
          const float4 w0 = W0[a * row16 + q];
#pragma unroll
          for (int b = 0; b < kM; b++) {
            const float4 r0 = add4(a0, b1[b]);
            const float4 r1 = add4(a1[b], b0);
            const float4 o = add4(w0, w1[b]);
            const float x0 = min3f(o.x, r0.x, r1.x);
            const float x1 = min3f(o.y, r0.y, r1.y);
            const float x2 = min3f(o.z, r0.z, r1.z);
            const float x3 = min3f(o.w, r0.w, r1.w);
            if (qq == 0)
              m[a][b] = fmaxf(max3f(x0, x1, x2), x3);
            else
              m[a][b] = max3f(max3f(m[a][b], x0, x1), x2, x3);
          }
        }
      }
      const int16_t gidx = (int16_t)((s << 4) | grp);
#pragma unroll
      for (int a = 0; a < kM; a++)
#pragma unroll
        for (int b = 0; b < kM; b++) {
          const int e = (ty + 16 * b) * kBgRow + tx + 16 * a;
          if (m[a][b] > sbest[e]) {
            sbest[e] = m[a][b];
            sbg[e] = gidx;
          }
        }
    }

    if (s == sp.n_states - 1) {
      // ---- tile end: park (best group, group index) per pair in the stage
      // buffer just consumed, then resolve the winning groups with a rolled loop
      // (low register pressure) in which a warp owns 32 consecutive j0 of one
      // column: the obj/cfg writes are 128-byte coalesced.
      __syncthreads();  // every pair's group index is in sbg
      for (int e = threadIdx.x; e < kTile * kTile; e += kThreads) {
        const int rj = e >> 6, ri = e & 63;
        const int64_t j0 = I * kTile + ri;
        const int64_t j1 = J * kTile + rj;
        const int gb = sbg[rj * kBgRow + ri];  // read and reset every slot, valid or not
        sbg[rj * kBgRow + ri] = -1;
        sbest[rj * kBgRow + ri] = 0.0f;
        if (!(j0 < j1 && j1 < g.n_jobs && j1 >= g.c0 && j1 < g.c1)) continue;
        float bo = -INFINITY;
        int bc = -1;
        if (gb >= 0) {
          const int sg = gb >> 4;
          const int q0 = (gb & 15) * G;
          const int sl0 = sp.slice[sg][0], sl1 = sp.slice[sg][1];
          const float4* pa0 = reinterpret_cast<const float4*>(ka_row(ka, sp, sl0, j0)) + q0;
          const float4* pb1 = reinterpret_cast<const float4*>(ka_row(kb, sp, sl0, j1)) + q0;
          const float4* pa1 = reinterpret_cast<const float4*>(ka_row(ka, sp, sl1, j1)) + q0;
          const float4* pb0 = reinterpret_cast<const float4*>(ka_row(kb, sp, sl1, j0)) + q0;
          const float4* pw0 = reinterpret_cast<const float4*>(w_row(w, sp, 0, sg, j0)) + q0;
          const float4* pw1 = reinterpret_cast<const float4*>(w_row(w, sp, 1, sg, j1)) + q0;
#pragma unroll
          for (int c = 0; c < G; c++) {
            const float4 r0 = add4(__ldg(pa0 + c), __ldg(pb1 + c));
            const float4 r1 = add4(__ldg(pa1 + c), __ldg(pb0 + c));
            const float4 o = add4(__ldg(pw0 + c), __ldg(pw1 + c));
            const float rr0[4] = {r0.x, r0.y, r0.z, r0.w};
            const float rr1[4] = {r1.x, r1.y, r1.z, r1.w};
            const float oo[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
            for (int q = 0; q < 4; q++)
              if (rr0[q] > 0.0f && rr1[q] > 0.0f && oo[q] > bo) {  // padding caps have r'' = -1e30
                bo = oo[q];
                bc = sg * sp.n_caps + 4 * (q0 + c) + q;
              }
          }
        }
        const int64_t sid = j1 * (j1 - 1) / 2 + j0;
        const int64_t k = sid - g.first_set;
        if (out_obj) out_obj[k] = bo;
        if (out_cfg) out_cfg[k] = bc;
        if (bc >= 0) {
          const unsigned long long kk = pack_key(bo, sid);
          key = kk > key ? kk : key;
        }
      }
    }

    __syncthreads();  // everyone is done with `buf` before it is refilled
    if (!has_next) break;
    t = nt;
    I = nI;
    J = nJ;
    s = ns;
    buf ^= 1;
  }
  block_max_key(key, best_key);
}

static int g_num_sms = 0;

template <int NP, int G>
static int launch_tiled(const SpaceParams& sp, const PairGrid& g, const float* ka, const float* kb, const float* w,
                        float* obj, int32_t* cfg, unsigned long long* best_key, const unsigned long long* err,
                        cudaStream_t st) {
  size_t smem = (size_t)2 * 6 * kTile * sp.rs * sizeof(float) + (size_t)kTile * kBgRow * (sizeof(float) + sizeof(int16_t));
  static size_t configured = 0;
  if (smem > configured) {
    cudaFuncSetAttribute(k_score_pairs_tiled<NP, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    configured = smem;
  }
  if (!g_num_sms) {
    int dev;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_score_pairs_tiled<NP, G>, kThreads, smem);
  if (per_sm < 1) per_sm = 1;
  int64_t grid = (int64_t)g_num_sms * per_sm;
  if (grid > g.n_tiles) grid = g.n_tiles;
  if (grid < 1) grid = 1;
  k_score_pairs_tiled<NP, G><<<(unsigned)grid, kThreads, smem, st>>>(sp, g, ka, kb, w, obj, cfg, best_key, err);
  return 1;
}

int launch_score_pairs_fast(const SpaceParams& sp, int64_t n_jobs, const float* ka, const float* kb, const float* w,
                            int64_t first, int64_t count, float* obj, int32_t* cfg, unsigned long long* best_key,
                            const unsigned long long* err, cudaStream_t st) {
  // column range of the shard; shards are whole columns (cosched_shard_range)
  auto c2 = [](int64_t n) { return n * (n - 1) / 2; };
  auto col_at = [&](int64_t v) {  // smallest c with C(c,2) >= v
    int64_t c = (int64_t)((1.0 + sqrt(1.0 + 8.0 * (double)v)) * 0.5);
    while (c > 0 && c2(c - 1) >= v) c--;
    while (c2(c) < v) c++;
    return c;
  };
  int64_t c0 = col_at(first), c1 = col_at(first + count);
  if (c2(c0) != first || c2(c1) != first + count || c1 > n_jobs || (sp.np >> 2) > 16 ||
      (size_t)2 * 6 * kTile * sp.rs * 4 > 180 * 1024) {
    return launch_score(sp, n_jobs, ka, kb, w, first, count, obj, cfg, best_key, err, 0, st);
  }
  PairGrid g;
  g.n_jobs = n_jobs;
  g.c0 = c0;
  g.c1 = c1;
  g.first_set = first;
  int64_t jt0 = c0 / kTile, jt1 = (c1 - 1) / kTile;
  g.base = jt0 * (jt0 + 1) / 2;
  g.n_tiles = (jt1 + 1) * (jt1 + 2) / 2 - g.base;
  const int chunks = sp.np >> 2;
  // compile-time cap counts for the preset grids (c10 -> 12, c21 -> 24, A100 -> 8)
  switch (sp.np) {
    case 8:
      g.groups_per_state = 1;
      return launch_tiled<8, 2>(sp, g, ka, kb, w, obj, cfg, best_key, err, st);
    case 12:
      g.groups_per_state = 1;
      return launch_tiled<12, 3>(sp, g, ka, kb, w, obj, cfg, best_key, err, st);
    case 16:
      g.groups_per_state = 2;
      return launch_tiled<16, 2>(sp, g, ka, kb, w, obj, cfg, best_key, err, st);
    case 24:
      g.groups_per_state = 2;
      return launch_tiled<24, 3>(sp, g, ka, kb, w, obj, cfg, best_key, err, st);
    default:
      break;
  }
  if (chunks % 3 == 0) {
    g.groups_per_state = chunks / 3;
    return launch_tiled<0, 3>(sp, g, ka, kb, w, obj, cfg, best_key, err, st);
  }
  if (chunks % 2 == 0) {
    g.groups_per_state = chunks / 2;
    return launch_tiled<0, 2>(sp, g, ka, kb, w, obj, cfg, best_key, err, st);
  }
  g.groups_per_state = chunks;
  return launch_tiled<0, 1>(sp, g, ka, kb, w, obj, cfg, best_key, err, st);
}

}  // namespace cosched
