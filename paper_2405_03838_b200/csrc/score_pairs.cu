// score_pairs.cu -- the fast pair scorer (SURVEY.md §8(a) a4-a8 for n_slots = 2), sm_100a.
//
// Work: for every pair (j0 < j1) of this rank's column range and every config
// c = (state s, cap p):
//   r0'' = ka[s0][j0][p] + kb[s0][j1][p]      (= K*(RPerf_0 - alpha))
//   r1'' = ka[s1][j1][p] + kb[s1][j0][p]
//   o    = W0[c][j0] + W1[c][j1]              (integer: fixed-point Throughput[/P]
//                                              with the config's stage offset in the low 5 bits)
//   x    = min3(float_bits(o), r0'', r1'')    (> 0 iff Fairness > alpha)
// and the per-pair argmax of x: configs are walked in stages of 20 (kStageCfg)
// along the flattened axis c = state * n_caps + cap (no cap padding); the stage
// of the best x is kept per pair, its offset comes back from x's low bits, and
// the winner's exact FP32 objective is read back at tile end.
//
// Design (DESIGN.md §5 "Pair scorer"):
//  - persistent CTAs (two per SM, 8 warps each, 128 registers per thread) walk 64x64
//    tiles of the pair triangle; each thread owns a 4x4 register micro-tile
//    (j0 = tx + 16a, j1 = ty + 16b); a warp covers 4 j0 x 8 j1 rows, so every
//    float4 operand load is one shared-memory wavefront;
//  - per stage, the tile's operand rows (6 roles x 64 jobs x 20 floats,
//    contiguous in the gathered layout) land in shared memory by 6 TMA bulk
//    copies (cp.async.bulk + mbarrier complete_tx), double buffered;
//  - per 4 caps and pair: 2 FADD2 (r0'', r1''), 4 IMAD (o, FMA pipe),
//    4 FMNMX3 (masked objective) + 2 FMNMX3 (running max): ALU 1.5 per
//    candidate, FMA pipe 2 -- the mix that measured fastest in
//    tools/microbench/inner.cu;
//  - per stage and pair one FSETP + 2 predicated moves; per tile and pair the
//    exact FP32 objective of the chosen config (2 loads + 1 FADD), resolved by
//    the thread that owns the pair with all its loads in flight (tile end);
//  - the last round's tiles (whole tiles mod CTA slots) are split along the
//    config axis into stage-group units (k_score_pairs_tiled<2, 4, true>) on a
//    side stream, enqueued next to the whole-tile launch; the last unit of a tile
//    resolves it from the step-tagged merge entries; the queue's ragged last
//    column block runs as 16-row units (<2, 1, false>) on another side stream;
//  - the whole-tile launch is PDL-launched behind the gather (its prologue
//    overlaps the gather's tail).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#include "cosched_internal.h"
#include "device_common.cuh"
#include "tile_common.cuh"

namespace cosched {

namespace {

constexpr int kTile = 64;      // pairs per tile side
constexpr int kThreads = 256;  // 16 x 16 threads, 4 x 4 pairs each
constexpr int kM = 4;          // micro-tile side
constexpr int kBgRow = kTile + 4;  // (4*ty + tx) mod 32: a warp's per-pair state accesses hit distinct banks

struct PairGrid {
  int64_t n_jobs;
  int64_t c0, c1;     // column (largest position) range of this shard: j1 in [c0, c1)
  int64_t n_tiles;
  int64_t base;       // tiles before the first column tile: jt0*(jt0+1)/2
  int64_t first_set;  // output index offset
  int64_t t0;         // first tile of this launch (NB = 4: whole tiles t0 .. t0 + n_units - 1)
  int64_t n_units;    // work units of this launch: a unit is a tile's j1 row groups [b0, b0 + NB)
  // NB < 4: up to 3 segments of units, segment s covering tiles seg_t0[s]...,
  // seg_per[s] units per tile starting at row group seg_b[s], units
  // [seg_end[s-1], seg_end[s]) of the launch
  int n_seg;
  int64_t seg_t0[3], seg_end[3];
  int seg_per[3], seg_b[3];
  unsigned one;       // runtime 1: keeps the integer adds on the FMA pipe (IMAD)
  // stage-split launches (SPLIT): unit u = stage group u % n_sg of whole tile
  // t0 + u / n_sg; group q covers stages [q n_stages / n_sg, (q + 1) n_stages / n_sg).
  // Each unit folds its best masked key per pair into merge[u / n_sg][j1 local][j0 local]
  // as (key bits << 32 | ~stage) by atomicMax; k_pairs_merge_finish resolves them.
  int n_sg;
  unsigned long long* merge;
  unsigned* cnt;  // non-null: per split tile, units done; the last unit resolves the tile (no finish launch)
  unsigned epoch;  // 24-bit step tag of the merge entries and counters (no reset between steps)
};

// Stage-split merge entry: [step epoch : 24][best masked key bits : 32][255 - stage : 8].
// atomicMax keeps this step's entries over any earlier step's (larger epoch), then
// the largest key, then the lowest stage (the canonical first maximum); the merge
// area is never reset between steps (zeroed once per workspace, api.cu).
__device__ __forceinline__ unsigned long long merge_entry(unsigned epoch, unsigned key_bits, int stage) {
  return ((unsigned long long)(epoch & 0xFFFFFFu) << 40) | ((unsigned long long)key_bits << 8) |
         (unsigned long long)(255 - stage);
}
// Count one finished unit of a split tile, [epoch : 24][count : 8]: the first
// unit of this step restarts the count. Returns the count after this unit.
__device__ __forceinline__ unsigned tile_count_up(unsigned* c, unsigned epoch) {
  const unsigned ep = epoch & 0xFFFFFFu;
  unsigned cur = atomicAdd(c, 0u), nv;
  while (true) {
    nv = (cur >> 8) == ep ? cur + 1u : ((ep << 8) | 1u);
    const unsigned prev = atomicCAS(c, cur, nv);
    if (prev == cur) break;
    cur = prev;
  }
  return nv & 0xFFu;
}

__device__ __forceinline__ void tile_coords(const PairGrid& g, int64_t t, int64_t* I, int64_t* J) {
  // tiles are ordered column tile J ascending, row tile I = 0..J; cum(J) = J(J+1)/2 - base
  int64_t u = t + g.base;
  int64_t j = (int64_t)((sqrt(8.0 * (double)u + 1.0) - 1.0) * 0.5);
  while (j * (j + 1) / 2 > u) j--;
  while ((j + 1) * (j + 2) / 2 <= u) j++;
  *J = j;
  *I = u - j * (j + 1) / 2;
}

// Work unit u of a launch with NB row groups (of 16 j1 rows) per unit -> tile
// (I, J) and its first row group b0. NB = 4: whole tiles.
// last stage + 1 of stage-split unit u (recomputed from u: no loop-carried register)
__device__ __forceinline__ int split_stage_hi(const PairGrid& g, int n_stages, int64_t u) {
  return ((int)u % g.n_sg + 1) * n_stages / g.n_sg;
}

template <int NB, bool SPLIT>
__device__ __forceinline__ void unit_coords(const PairGrid& g, int n_stages, int64_t u, int64_t* I, int64_t* J,
                                            int* b0, int* s_lo, int* s_hi) {
  *s_lo = 0;
  *s_hi = n_stages;
  if (SPLIT) {  // < 2^31 units (at most one round of CTA slots)
    const int t = (int)u / g.n_sg;
    const int q = (int)u - t * g.n_sg;
    tile_coords(g, g.t0 + t, I, J);
    *b0 = 0;
    *s_lo = q * n_stages / g.n_sg;
    *s_hi = (q + 1) * n_stages / g.n_sg;
    return;
  }
  if (NB == kM) {
    tile_coords(g, g.t0 + u, I, J);
    *b0 = 0;
    return;
  }
  int q = 0;
  while (q + 1 < g.n_seg && u >= g.seg_end[q]) q++;
  const int64_t v = u - (q ? g.seg_end[q - 1] : 0);
  tile_coords(g, g.seg_t0[q] + v / g.seg_per[q], I, J);
  *b0 = g.seg_b[q] + (int)(v % g.seg_per[q]) * NB;
}

// Stage layout (floats): role blocks [A0][B0][W0][A1][B1][W1], each kTile rows x
// kStageRS, copied from fast[role][g][row0 .. row0+63][*] (contiguous 7 KB).
__device__ __forceinline__ void issue_stage(float* stage, uint64_t* bar, const SpaceParams& sp,
                                            const float* __restrict__ fast, int64_t I, int64_t J, int g) {
  constexpr int blk = kTile * kStageRS;
  constexpr unsigned bytes = (unsigned)blk * 4u;
  mbar_arrive_expect_tx(bar, 6u * bytes);
#pragma unroll
  for (int role = 0; role < 6; role++) {
    const int64_t row0 = (role < 3 ? I : J) * kTile;
    const float* src = fast + (((int64_t)role * sp.n_stages + g) * sp.n_jobs_pad + row0) * kStageRS;
    tma_bulk_g2s(stage + role * blk, src, bytes, bar);
  }
}

}  // namespace

__device__ __forceinline__ void merge_finish_part(const SpaceParams& sp, const PairGrid& g, const float* __restrict__ w,
                                                  float* __restrict__ out_obj, int32_t* __restrict__ out_cfg,
                                                  const RescoreBuf& rb, unsigned long long* mg, int64_t I, int64_t J,
                                                  int e0, float thr, unsigned long long* key);

// The scorer's work for one CTA: units t0, t0 + stride, ... of the launch
// described by g (whole tiles, stage-split units or row-group units).
template <int MINB, int NB, bool SPLIT>
__device__ __forceinline__ void pairs_body(const SpaceParams& sp, const PairGrid& g, const float* __restrict__ w,
                                           const float* __restrict__ fast, float* __restrict__ out_obj,
                                           int32_t* __restrict__ out_cfg, unsigned long long* __restrict__ best_key,
                                           const unsigned long long* __restrict__ err, const RescoreBuf& rb,
                                           int64_t t0, int64_t stride) {
  extern __shared__ __align__(128) float smem[];
  __shared__ __align__(8) uint64_t bars[2];
  __shared__ float s_thr;  // exact re-scoring threshold (rescore_threshold)
  __shared__ int s_last;   // SPLIT: this unit finished its tile
  constexpr int rs = kStageRS, rs4 = kStageRS / 4, chunks = kStageCfg / 4;
  constexpr int stage_floats = 6 * kTile * rs;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // lane bits: a quad (4 consecutive lanes) spans 2 values of tx and 2 of ty, so
  // every LDS.128 of an operand row costs 2 shared wavefronts (4 when a quad
  // reads 4 different rows: tools/microbench/lds.cu)
  const int tx = ((warp & 3) << 2) | (((lane >> 2) & 1) << 1) | (lane & 1);
  const int ty = ((warp >> 2) << 3) | ((lane >> 3) << 1) | ((lane >> 1) & 1);
  const unsigned one = g.one;
  unsigned long long key = 0;

  int64_t t = t0;  // work unit
  if (t >= g.n_units) {
    pdl_wait();
    if (*err == ~0ull) block_max_key(0ull, best_key);
    return;
  }
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    mbar_fence_init();
  }
  // per pair ([j1 local][j0 local], padded rows): state of the best masked key
  // (written when a state improves) and, at tile end, the key itself
  float* sbest = smem + 2 * stage_floats;
  int16_t* sbg = reinterpret_cast<int16_t*>(sbest + kTile * kBgRow);
  for (int e = threadIdx.x; e < kTile * kBgRow; e += kThreads) sbg[e] = -1;
  // the prologue above touches shared memory only: it overlaps the gather's tail (PDL)
  pdl_wait();
  pdl_launch_dependents();
  if (*err != ~0ull) return;  // uniform
  if (threadIdx.x == 0) s_thr = rescore_threshold<2>(rb.wmm);
  __syncthreads();
  int64_t I, J;
  int b0, s_lo, s_hi;  // stages [s_lo, s_hi) of the unit (the whole config axis unless SPLIT)
  unit_coords<NB, SPLIT>(g, sp.n_stages, t, &I, &J, &b0, &s_lo, &s_hi);
  int s = s_lo, buf = 0;
  (void)s_hi;
  unsigned phase = 0u;  // bit b = parity of the next wait on bars[b]
  if (threadIdx.x == 0) issue_stage(smem, &bars[0], sp, fast, I, J, s_lo);

  float breg[kM][NB];
#pragma unroll
  for (int a = 0; a < kM; a++)
#pragma unroll
    for (int b = 0; b < NB; b++) breg[a][b] = 0.0f;  // feasible masked keys are > 0

  while (true) {
    // prefetch the next (tile, state) into the other buffer
    int64_t nt = t, nI = I, nJ = J;
    int ns = s + 1, nb0 = b0, ns_lo = 0, ns_hi = 0;
    if (ns == (SPLIT ? split_stage_hi(g, sp.n_stages, t) : sp.n_stages)) {
      nt = t + stride;
      if (nt < g.n_units) unit_coords<NB, SPLIT>(g, sp.n_stages, nt, &nI, &nJ, &nb0, &ns_lo, &ns_hi);
      ns = SPLIT ? ns_lo : 0;
    }
    const bool has_next = nt < g.n_units;
    if (has_next && threadIdx.x == 0)
      issue_stage(smem + (buf ^ 1) * stage_floats, &bars[buf ^ 1], sp, fast, nI, nJ, ns);
    mbar_wait(&bars[buf], (phase >> buf) & 1u);
    phase ^= 1u << buf;

    const float4* st4 = reinterpret_cast<const float4*>(smem + buf * stage_floats);
    const int blk4 = kTile * rs4;
    const float4* A0 = st4 + 0 * blk4 + tx * rs4;
    const float4* B0 = st4 + 1 * blk4 + tx * rs4;
    const uint4* W0 = reinterpret_cast<const uint4*>(st4 + 2 * blk4 + tx * rs4);
    const float4* A1 = st4 + 3 * blk4 + (ty + 16 * b0) * rs4;
    const float4* B1 = st4 + 4 * blk4 + (ty + 16 * b0) * rs4;
    const uint4* W1 = reinterpret_cast<const uint4*>(st4 + 5 * blk4 + (ty + 16 * b0) * rs4);
    const int row16 = 16 * rs4;  // float4s between rows r and r+16

    float m[kM][NB];
#pragma unroll
    for (int q = 0; q < chunks; q++) {
      float4 a1[NB], b1[NB];
      uint4 w1[NB];
#pragma unroll
      for (int b = 0; b < NB; b++) {
        a1[b] = A1[b * row16 + q];
        b1[b] = B1[b * row16 + q];
        w1[b] = W1[b * row16 + q];
      }
#pragma unroll
      for (int a = 0; a < kM; a++) {
        const float4 a0 = A0[a * row16 + q];
        const float4 b0 = B0[a * row16 + q];
        const uint4 w0 = W0[a * row16 + q];
#pragma unroll
        for (int b = 0; b < NB; b++) {
          const float4 r0 = add4(a0, b1[b]);
          const float4 r1 = add4(a1[b], b0);
          const float x0 = min3f(__uint_as_float(imad_add(w0.x, one, w1[b].x)), r0.x, r1.x);
          const float x1 = min3f(__uint_as_float(imad_add(w0.y, one, w1[b].y)), r0.y, r1.y);
          const float x2 = min3f(__uint_as_float(imad_add(w0.z, one, w1[b].z)), r0.z, r1.z);
          const float x3 = min3f(__uint_as_float(imad_add(w0.w, one, w1[b].w)), r0.w, r1.w);
          if (q == 0)
            m[a][b] = fmaxf(max3f(x0, x1, x2), x3);
          else
            m[a][b] = max3f(max3f(m[a][b], x0, x1), x2, x3);
        }
      }
    }
#pragma unroll
    for (int a = 0; a < kM; a++)
      for (int b = 0; b < NB; b++)
        if (m[a][b] > breg[a][b]) {  // strict: the first stage wins ties (canonical order)
          breg[a][b] = m[a][b];
          sbg[(ty + 16 * (b0 + b)) * kBgRow + tx + 16 * a] = (int16_t)s;
        }

    if (SPLIT && s == split_stage_hi(g, sp.n_stages, t) - 1) {
      // ---- unit end: fold this stage group's best key per pair into the merge
      // buffer (max key, then lowest stage = the canonical first maximum); the
      // entries are the thread's own (no barrier), infeasible-only pairs skip
      // park the keys in shared memory (unrolled stores), merge them in a rolled loop
#pragma unroll
      for (int a = 0; a < kM; a++)
#pragma unroll
        for (int b = 0; b < NB; b++) {
          sbest[(ty + 16 * b) * kBgRow + tx + 16 * a] = breg[a][b];
          breg[a][b] = 0.0f;
        }
      unsigned long long* mg = g.merge + ((int)t / g.n_sg) * (kTile * kTile);
#pragma unroll 1
      for (int ab = 0; ab < kM * NB; ab++) {
        const int a = ab & 3, b = ab >> 2;
        const int e = (ty + 16 * b) * kBgRow + tx + 16 * a;
        const float m = sbest[e];
        if (m > 0.0f)
          atomicMax(mg + (ty + 16 * b) * kTile + tx + 16 * a, merge_entry(g.epoch, __float_as_uint(m), sbg[e]));
        sbg[e] = -1;
      }
      if (g.cnt) {
        // the tile's last unit to finish resolves it (threadfence reduction):
        // every unit's merge atomics are visible before its count
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) s_last = tile_count_up(g.cnt + (int)t / g.n_sg, g.epoch) == (unsigned)g.n_sg;
        __syncthreads();
        if (s_last) {
          __threadfence();
#pragma unroll 1
          for (int q = 0; q < 4; q++)
            merge_finish_part(sp, g, w, out_obj, out_cfg, rb, mg, I, J, q * (kTile * kTile / 4), s_thr, &key);
        }
      }
    }
    if (!SPLIT && s == sp.n_stages - 1) {
      // ---- tile end, owner first: each thread resolves its own 4 x 4 pairs with
      // all 32 w loads in flight, parks (objective, config) in shared memory; a
      // rolled loop then writes them with 128-byte coalesced stores (r01's
      // resolve-in-the-store-loop, 4 pairs' loads per pass: 3.030 -> 3.022 ms on C4).
      // A positive fairness margin is >= 8 (kScale, cosched_internal.h) and a
      // packed key is < 4.0, so the best masked key of a feasible pair is never
      // clipped: its low bits are the stage offset of the argmax, and the
      // reported objective is the exact FP32 w0 + w1 of that config (2 loads).
      const int jI = (int)(I * kTile), jJ = (int)(J * kTile);
      const int c_lo = (int)g.c0, c_hi = (int)g.c1;
      const int rsz = sp.rs, npad = (int)sp.n_jobs_pad, w1base = sp.n_states * npad;
      int cc[kM][NB];
      float f0[kM][NB], f1[kM][NB];
#pragma unroll
      for (int a = 0; a < kM; a++)
#pragma unroll
        for (int b = 0; b < NB; b++) {
          const int e = (ty + 16 * (b0 + b)) * kBgRow + tx + 16 * a;
          const int j0 = jI + tx + 16 * a, j1 = jJ + ty + 16 * (b0 + b);
          const int sg = sbg[e];  // this thread's own entry
          const unsigned kbits = __float_as_uint(breg[a][b]);
          breg[a][b] = 0.0f;
          const bool ok = j0 < j1 && j1 >= c_lo && j1 < c_hi;
          const int c = sg * kStageCfg + 31 - (int)(kbits & 31u);
          cc[a][b] = (ok && sg >= 0 && c < sp.n_cfg) ? c : (ok ? -1 : -2);
          f0[a][b] = f1[a][b] = 0.0f;
          if (cc[a][b] >= 0) {
            const int st = (int)__fmul_rn((float)c + 0.5f, sp.inv_ncaps), p = c - st * sp.n_caps;
            f0[a][b] = __ldg(w + (int64_t)(st * npad + j0) * rsz + p);
            f1[a][b] = __ldg(w + (int64_t)(w1base + st * npad + j1) * rsz + p);
          }
        }
#pragma unroll
      for (int a = 0; a < kM; a++)
#pragma unroll
        for (int b = 0; b < NB; b++) {
          const int e = (ty + 16 * (b0 + b)) * kBgRow + tx + 16 * a;
          sbest[e] = cc[a][b] >= 0 ? __fadd_rn(f0[a][b], f1[a][b]) : -INFINITY;
          sbg[e] = (int16_t)cc[a][b];
        }
      __syncthreads();
      const float thr = s_thr;
#pragma unroll 4
      for (int e = 16 * kTile * b0 + threadIdx.x; e < 16 * kTile * (b0 + NB); e += kThreads) {
        const int rj = e >> 6, ri = e & 63;  // a warp writes 32 consecutive j0 of one column
        const int bc = sbg[rj * kBgRow + ri];
        const float bo = sbest[rj * kBgRow + ri];
        sbg[rj * kBgRow + ri] = -1;
        if (bc == -2) continue;
        const int j0 = jI + ri, j1 = jJ + rj;
        const int64_t sid = (((int64_t)j1 * (j1 - 1)) >> 1) + j0;
        const int64_t k = sid - g.first_set;
        if (out_obj) out_obj[k] = bo;
        if (out_cfg) out_cfg[k] = bc;
        if (bc >= 0) {
          const unsigned long long kk = pack_key(bo, sid);
          key = kk > key ? kk : key;
          if (bo < thr) {  // not provably within tau/2 of the FP32 argmax: exact re-score
            const unsigned at = atomicAdd(rb.n, 1u);
            if (at < rb.cap) rb.list[at] = (unsigned)k;
          }
        }
      }
    }

    __syncthreads();  // everyone is done with `buf` (and the per-pair state) before reuse
    if (!has_next) break;
    t = nt;
    I = nI;
    J = nJ;
    b0 = nb0;
    s = ns;
    buf ^= 1;
  }
  block_max_key(key, best_key);
}

template <int MINB, int NB, bool SPLIT>
__global__ void __launch_bounds__(kThreads, MINB)
    k_score_pairs_tiled(const SpaceParams sp, const PairGrid g, const float* __restrict__ w,
                        const float* __restrict__ fast, float* __restrict__ out_obj, int32_t* __restrict__ out_cfg,
                        unsigned long long* __restrict__ best_key, const unsigned long long* __restrict__ err,
                        const RescoreBuf rb) {
  pairs_body<MINB, NB, SPLIT>(sp, g, w, fast, out_obj, out_cfg, best_key, err, rb, blockIdx.x, gridDim.x);
}


// Resolution of the stage-split tiles (four blocks per tile): per pair the merged
// (best masked key, first stage) gives the config -- stage and the key's low
// bits, as in the tile end -- and the exact FP32 objective w0 + w1 of it; the
// merge entries are reset for the next step. Writes obj / cfg, the rescore flag
// and the block's best key.
// Resolution of pairs [e0, e0 + 1024) of a stage-split tile (256 threads, 4
// pairs each, all loads in flight): per pair the merged (best masked key, first
// stage) gives the config -- stage and the key's low bits, as in the tile end --
// and the exact FP32 objective w0 + w1 of it; the merge entries are reset for the
// next step. Writes obj / cfg and the rescore flag; folds the best key into *key.
__device__ __forceinline__ void merge_finish_part(const SpaceParams& sp, const PairGrid& g, const float* __restrict__ w,
                                                  float* __restrict__ out_obj, int32_t* __restrict__ out_cfg,
                                                  const RescoreBuf& rb, unsigned long long* mg, int64_t I, int64_t J,
                                                  int e0, float thr, unsigned long long* key) {
  const int rsz = sp.rs, npad = (int)sp.n_jobs_pad, w1base = sp.n_states * npad;
  constexpr int kPer = 4;
  int c_[kPer];
  float f0[kPer], f1[kPer];
#pragma unroll
  for (int u = 0; u < kPer; u++) {
    const int e = e0 + u * 256 + threadIdx.x, rj = e >> 6, ri = e & 63;
    const int64_t j0 = I * kTile + ri, j1 = J * kTile + rj;
    const unsigned long long v = __ldcg(mg + e);  // L2: written by other CTAs' atomics
    const bool ok = j0 < j1 && j1 >= g.c0 && j1 < g.c1;
    c_[u] = ok ? -1 : -2;
    f0[u] = f1[u] = 0.0f;
    if (ok && (unsigned)(v >> 40) == (g.epoch & 0xFFFFFFu)) {  // a feasible stage group wrote it this step
      const int sg = 255 - (int)(v & 0xFFu);
      const int c = sg * kStageCfg + 31 - (int)((v >> 8) & 31u);
      c_[u] = c;
      const int st = (int)__fmul_rn((float)c + 0.5f, sp.inv_ncaps), p = c - st * sp.n_caps;
      f0[u] = __ldg(w + (int64_t)(st * npad + (int)j0) * rsz + p);
      f1[u] = __ldg(w + (int64_t)(w1base + st * npad + (int)j1) * rsz + p);
    }
  }
#pragma unroll
  for (int u = 0; u < kPer; u++) {
    if (c_[u] == -2) continue;
    const int e = e0 + u * 256 + threadIdx.x, rj = e >> 6, ri = e & 63;
    const int64_t j0 = I * kTile + ri, j1 = J * kTile + rj;
    const int c = c_[u];
    const float bo = c >= 0 ? __fadd_rn(f0[u], f1[u]) : -INFINITY;
    const int64_t sid = ((j1 * (j1 - 1)) >> 1) + j0, k = sid - g.first_set;
    if (out_obj) out_obj[k] = bo;
    if (out_cfg) out_cfg[k] = c;
    if (c >= 0) {
      const unsigned long long kk = pack_key(bo, sid);
      *key = kk > *key ? kk : *key;
      if (bo < thr) {
        const unsigned at = atomicAdd(rb.n, 1u);
        if (at < rb.cap) rb.list[at] = (unsigned)k;
      }
    }
  }
}

// Resolution of the stage-split tiles by a separate launch (four blocks per tile)
// when the units do not resolve their tiles themselves (PairGrid::cnt null).
__global__ void __launch_bounds__(256) k_pairs_merge_finish(const SpaceParams sp, const PairGrid g,
                                                             const float* __restrict__ w, float* __restrict__ out_obj,
                                                             int32_t* __restrict__ out_cfg,
                                                             unsigned long long* __restrict__ best_key,
                                                             const unsigned long long* __restrict__ err,
                                                             const RescoreBuf rb) {
  if (*err != ~0ull) return;
  int64_t I, J;
  tile_coords(g, g.t0 + blockIdx.x, &I, &J);
  unsigned long long key = 0ull;
  merge_finish_part(sp, g, w, out_obj, out_cfg, rb, g.merge + (int64_t)blockIdx.x * (kTile * kTile), I, J,
                    blockIdx.y * (kTile * kTile / 4), rescore_threshold<2>(rb.wmm), &key);
  block_max_key(key, best_key);
}

// Precondition: tiled_applicable(2, n_jobs, first, count) (kernels.cu), i.e. the
// shard is whole colex columns and the queue has < 32768 column tiles.
int launch_score_pairs_fast(const SpaceParams& sp, int64_t n_jobs, const float* w, const float* fast, int64_t first,
                            int64_t count, float* obj, int32_t* cfg, unsigned long long* best_key,
                            const unsigned long long* err, const RescoreBuf& rb, const PairMerge& merge,
                            cudaStream_t st) {
  // column range of the shard; shards are whole columns (cosched_shard_range)
  auto c2 = [](int64_t n) { return n * (n - 1) / 2; };
  auto col_at = [&](int64_t v) {  // smallest c with C(c,2) >= v
    int64_t c = (int64_t)((1.0 + sqrt(1.0 + 8.0 * (double)v)) * 0.5);
    while (c > 0 && c2(c - 1) >= v) c--;
    while (c2(c) < v) c++;
    return c;
  };
  const int64_t c0 = col_at(first), c1 = col_at(first + count);
  PairGrid g;
  g.n_jobs = n_jobs;
  g.c0 = c0;
  g.c1 = c1;
  g.first_set = first;
  g.one = 1u;
  int64_t jt0 = c0 / kTile, jt1 = (c1 - 1) / kTile;
  g.base = jt0 * (jt0 + 1) / 2;
  g.n_tiles = (jt1 + 1) * (jt1 + 2) / 2 - g.base;
  constexpr size_t smem = (size_t)2 * 6 * kTile * kStageRS * sizeof(float) +
                          (size_t)kTile * kBgRow * (sizeof(float) + sizeof(int16_t));
  const char* fs = getenv("COSCHED_PAIR_SPLIT");  // testing knob: stage groups of the tail split (1 = none)
  const int forced_split = fs ? atoi(fs) : 0;
  const char* mb = getenv("COSCHED_PAIR_MINB");
  const int minb = (mb && mb[0] == '1') ? 1 : 2;
  smem_optin((const void*)k_score_pairs_tiled<1, 4, false>, smem);
  smem_optin((const void*)k_score_pairs_tiled<2, 4, false>, smem);
  smem_optin((const void*)k_score_pairs_tiled<2, 4, true>, smem);
  smem_optin((const void*)k_score_pairs_tiled<2, 1, false>, smem);
  const int g_num_sms = num_sms();
  int per_sm = 0;
  if (minb == 1) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_score_pairs_tiled<1, 4, false>, kThreads, smem);
  else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_score_pairs_tiled<2, 4, false>, kThreads, smem);
  if (per_sm < 1) per_sm = 1;
  const int64_t slots = (int64_t)g_num_sms * per_sm;
  // Partial column blocks: the shard's first and last column blocks hold only
  // the 16-row j1 groups [lo0, 4) and [0, hi1) of its columns (a shard boundary
  // inside a block, or the queue's ragged end); their tiles go to a unit launch
  // that evaluates only those groups. The other tiles run whole.
  const int lo0 = (int)((c0 - jt0 * kTile) / 16), hi1 = (int)((c1 - jt1 * kTile + 15) / 16);
  struct Seg {
    int64_t t0, n;  // tiles [t0, t0 + n)
    int groups, b;  // row groups [b, b + groups) of each
  };
  Seg segs[3];
  int n_seg = 0;
  int64_t fa = 0, fb = g.n_tiles;  // whole tiles [fa, fb)
  if (minb == 2) {
    if (jt0 == jt1) {
      if (hi1 - lo0 < kM) {
        segs[n_seg++] = {0, g.n_tiles, hi1 - lo0, lo0};
        fb = fa;
      }
    } else {
      if (lo0 > 0) {
        segs[n_seg++] = {0, jt0 + 1, kM - lo0, lo0};
        fa = jt0 + 1;
      }
      if (hi1 < kM) {
        segs[n_seg++] = {g.n_tiles - (jt1 + 1), jt1 + 1, hi1, 0};
        fb = g.n_tiles - (jt1 + 1);
      }
    }
  }
  // Tail: whole-tile rounds leave slots - R CTAs idle for a
  // whole tile time in the last round (R = whole tiles mod slots), which is what
  // limits strong scaling once a rank has few tiles. The last R tiles are split
  // along the config axis instead: n_sg = min(n_stages, slots / R) units per
  // tile, each scoring a contiguous group of stages of the whole tile and
  // folding its per-pair best into the merge buffer; k_pairs_merge_finish then
  // resolves those tiles. A stage group costs its share of the tile's per-stage
  // work (TMA, barriers, bodies), unlike a row-group split, which pays every
  // stage of the tile. COSCHED_PAIR_SPLIT = n forces n stage groups (1 = none).
  const int64_t n_full = fb - fa;
  const int64_t R = n_full > slots ? n_full % slots : n_full;
  // groups per tile: minimise the tail's length in stage times,
  // ceil(R q / slots) rounds of units of ceil(n_stages / q) stages plus a unit's
  // fixed cost (the merge atomics and the pipeline start, ~0.3 of a stage,
  // measured on C4); q = 1 keeps whole tiles. Ties keep fewer, larger units.
  int n_sg = 1;
  if (R > 0 && merge.buf && minb == 2 && R <= merge.tiles && sp.n_stages <= 255) {  // stage in 8 bits
    auto tail_len = [&](int q) {
      return (double)((R * q + slots - 1) / slots) * ((sp.n_stages + q - 1) / q + (q > 1 ? 0.3 : 0.0));
    };
    double best = tail_len(1);
    for (int q = 2; q <= sp.n_stages; q++)
      if (tail_len(q) < best - 1e-9) {
        best = tail_len(q);
        n_sg = q;
      }
    if (forced_split > 0) n_sg = std::min(forced_split, sp.n_stages);
  }
  const int64_t n_whole = n_sg > 1 ? n_full - R : n_full;
  int launches = 0;
  g.epoch = merge.epoch;
  g.cnt = nullptr;
  // partial-column units (side stream) and stage-split tail units (side2): both
  // are enqueued at once next to the whole-tile launch, so their CTAs take the
  // slots it frees in its last round (no launch gap); the tail units resolve
  // their tiles themselves (last unit per tile, PairGrid::cnt).
  // COSCHED_PAIR_TAIL_CONC=0: tail units and a finish launch on the caller's stream.
  const char* tc = getenv("COSCHED_PAIR_TAIL_CONC");
  const bool conc = n_sg > 1 && !(tc && tc[0] == '0') && merge.side2 && merge.cnt && merge.ev_join2 && merge.ev_fork;
  const bool fork_side = n_seg > 0 && merge.side && merge.ev_fork && merge.ev_join;
  if (fork_side || conc) cudaEventRecord(merge.ev_fork, st);
  cudaStream_t ust = st, sst = st;
  if (fork_side) {
    cudaStreamWaitEvent(merge.side, merge.ev_fork, 0);
    ust = merge.side;
  }
  if (conc) {
    cudaStreamWaitEvent(merge.side2, merge.ev_fork, 0);
    sst = merge.side2;
  }
  if (n_whole > 0) {
    launches++;
    g.t0 = fa;
    g.n_units = n_whole;
    g.n_seg = 0;
    const int64_t grid = n_whole < slots ? n_whole : slots;
    if (minb == 1)
      launch_pdl(k_score_pairs_tiled<1, 4, false>, dim3((unsigned)grid), dim3(kThreads), smem, st, sp, g, w, fast, obj,
                 cfg, best_key, err, rb);
    else
      launch_pdl(k_score_pairs_tiled<2, 4, false>, dim3((unsigned)grid), dim3(kThreads), smem, st, sp, g, w, fast, obj,
                 cfg, best_key, err, rb);
  }
  if (n_sg > 1) {
    launches += conc ? 1 : 2;  // the merge entries and tile counts carry the step's epoch: no reset
    g.t0 = fa + n_whole;
    g.n_units = R * n_sg;
    g.n_sg = n_sg;
    g.merge = merge.buf;
    g.cnt = conc ? merge.cnt : nullptr;
    g.n_seg = 0;
    const int64_t grid = g.n_units < slots ? g.n_units : slots;
    k_score_pairs_tiled<2, 4, true><<<(unsigned)grid, kThreads, smem, sst>>>(sp, g, w, fast, obj, cfg, best_key, err, rb);
    if (!conc) k_pairs_merge_finish<<<dim3((unsigned)R, 4), 256, 0, st>>>(sp, g, w, obj, cfg, best_key, err, rb);
    g.cnt = nullptr;
  }
  if (n_seg > 0) {
    launches++;
    int64_t end = 0;
    for (int q = 0; q < n_seg; q++) {
      const int per = segs[q].groups;  // single-row-group units
      end += segs[q].n * per;
      g.seg_t0[q] = segs[q].t0;
      g.seg_end[q] = end;
      g.seg_per[q] = per;
      g.seg_b[q] = segs[q].b;
    }
    g.n_seg = n_seg;
    g.t0 = 0;
    g.n_units = end;
    const int64_t grid = end < slots ? end : slots;
    k_score_pairs_tiled<2, 1, false><<<(unsigned)grid, kThreads, smem, ust>>>(sp, g, w, fast, obj, cfg, best_key, err, rb);
  }
  if (fork_side) {
    cudaEventRecord(merge.ev_join, merge.side);
    cudaStreamWaitEvent(st, merge.ev_join, 0);
  }
  if (conc) {
    cudaEventRecord(merge.ev_join2, merge.side2);
    cudaStreamWaitEvent(st, merge.ev_join2, 0);
  }
  return launches;
}

}  // namespace cosched
