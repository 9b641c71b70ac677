// score_triples.cu -- the fast triple scorer (SURVEY.md §8(a) a4-a8 for n_slots = 3), sm_100a.
//
// For every triple j0 < j1 < j2 of this rank's plane range (j2 in [c0, c1)) and
// every config c (state s with slot slices s0, s1, s2; cap p), in the canonical
// order of eval_cfg<3> (device_common.cuh):
//   r0'' = ka[s0][j0] + P0,  P0 = kb[s0][j1] + kb[s0][j2]
//   r1'' = P1 + kb[s1][j0],  P1 = ka[s1][j1] + kb[s1][j2]
//   r2'' = P2 + kb[s2][j0],  P2 = ka[s2][j2] + kb[s2][j1]
//   o    = W0[j0] + Q,       Q  = W1[j1] + W2[j2]        (integer packed objective)
//   x    = min3(float_bits(o), r0'', min(r1'', r2''))
// The partner partials P0, P1, P2, Q depend on (j1, j2) only: they are built once
// per tile and stage in shared memory and reused by all 64 j0 rows, so a
// candidate costs 3 FP32 adds (FADD2), 1 integer add (IMAD, FMA pipe) and 2.5 ALU
// ops (FMNMX + FMNMX3 + half an FMNMX3 for the running max).
//
// Tiles: fixed j2, a block of 64 j1 (b) and a block of 64 j0 (a <= b); 256
// threads, 4 x 4 (j0 x j1) micro-tiles, two resident blocks per SM. Configs are
// walked in stages of 20 along the flattened axis (gathered layout, roles
// [A0 B01 B02 W0 | A1 B10 B12 W1 | A2 B20 B21 W2]); per stage 8 role blocks of
// 64 rows and 4 single j2 rows land by TMA bulk copies, double buffered. The
// stage of each triple's best key is tracked; the offset comes back from the
// key's low bits and the winner's exact FP32 objective is read back at tile end.
// The stage body is specialised per tile shape (tstage_body<DIAG, NBV>): diagonal
// tiles skip the never-valid a > b entries, last-j1-block tiles the row groups
// at or above j2.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#include "cosched_internal.h"
#include "device_common.cuh"
#include "tile_common.cuh"

namespace cosched {

namespace {

constexpr int kTT = 64;         // tile side (j0 and j1)
constexpr int kTThreads = 256;  // 16 x 16 threads, 4 x 4 sets each
constexpr int kTM = 4;
constexpr int kTBgRow = kTT + 4;

struct TripleGrid {
  int64_t n_jobs;
  int64_t c0, c1;  // plane range: j2 in [c0, c1)
  int64_t cum0;    // tiles before plane c0
  int64_t n_tiles;
  int64_t first_set;
  unsigned one;    // runtime 1 for IMAD
  int pair_major;  // tile order (ttile_coords): 1 block pair major (default), 0 plane major
};

// tiles of the planes j2' < j2: plane j has B(j) = ceil(j/64) j1-blocks and B(B+1)/2 tiles
__host__ __device__ __forceinline__ int64_t tiles_before(int64_t j2) {
  if (j2 <= 1) return 0;
  const int64_t n = (j2 - 1) / kTT, rem = (j2 - 1) - kTT * n;
  return 32 * n * (n + 1) * (n + 2) / 3 + rem * (n + 1) * (n + 2) / 2;
}

__device__ __forceinline__ void ttile_coords_planes(const TripleGrid& g, int64_t t, int64_t* j2, int64_t* b, int64_t* a) {
  int64_t lo = g.c0, hi = g.c1 - 1;  // largest plane with tiles_before(plane) - cum0 <= t
  while (lo < hi) {
    int64_t mid = (lo + hi + 1) / 2;
    if (tiles_before(mid) - g.cum0 <= t) lo = mid;
    else hi = mid - 1;
  }
  *j2 = lo;
  const int64_t u = t - (tiles_before(lo) - g.cum0);
  int64_t bb = (int64_t)((sqrt(8.0 * (double)u + 1.0) - 1.0) * 0.5);
  while (bb * (bb + 1) / 2 > u) bb--;
  while ((bb + 1) * (bb + 2) / 2 <= u) bb++;
  *b = bb;
  *a = u - bb * (bb + 1) / 2;
}

// Tile order: block pair (b, a) major, the rank's planes j2 inner -- tiles
// running at the same time read the same (a, b) operand blocks of the gathered
// layout (1.8 MB of TMA source for all 45 stages) and differ only in their
// single j2 rows, so the operands stay in L2 under the 10.65 GB output stream
// (plane-major order cycled the whole 177 MB layout through L2). Plane j2 has
// tiles (a <= b) for b < ceil(j2 / 64), i.e. j2 > 64 b.
__device__ __forceinline__ void ttile_coords(const TripleGrid& g, int64_t t, int64_t* j2, int64_t* b, int64_t* a) {
  if (g.pair_major) {
    for (int64_t bb = 0;; bb++) {
      const int64_t lo = g.c0 > 64 * bb + 1 ? g.c0 : 64 * bb + 1;
      const int64_t n = g.c1 > lo ? g.c1 - lo : 0;  // planes with block bb
      const int64_t cnt = (bb + 1) * n;
      if (t < cnt) {
        *b = bb;
        if (g.pair_major == 2) {  // b, then j2, then a: a row's runs (all a) are written together
          *a = t % (bb + 1);
          *j2 = lo + t / (bb + 1);
        } else {
          *a = t / n;
          *j2 = lo + t % n;
        }
        return;
      }
      t -= cnt;
    }
  }
  ttile_coords_planes(g, t, j2, b, a);
}

// Stage (floats): role blocks 0..7 of kTT rows x kStageRS (j0 rows for roles
// 0-3, j1 rows for roles 4-7), then the 4 single j2 rows of roles 8-11.
__device__ __forceinline__ void issue_tstage(float* stage, uint64_t* bar, const SpaceParams& sp,
                                             const float* __restrict__ fast, int64_t a, int64_t b, int64_t j2,
                                             int g) {
  constexpr int blk = kTT * kStageRS;
  constexpr unsigned bytes = (unsigned)blk * 4u, rowb = (unsigned)kStageRS * 4u;
  mbar_arrive_expect_tx(bar, 8u * bytes + 4u * rowb);
#pragma unroll
  for (int role = 0; role < 8; role++) {
    const int64_t row0 = (role < 4 ? a : b) * kTT;
    tma_bulk_g2s(stage + role * blk, fast + (((int64_t)role * sp.n_stages + g) * sp.n_jobs_pad + row0) * kStageRS,
                 bytes, bar);
  }
  float* rows = stage + 8 * blk;
#pragma unroll
  for (int k = 0; k < 4; k++)
    tma_bulk_g2s(rows + k * kStageRS,
                 fast + (((int64_t)(8 + k) * sp.n_stages + g) * sp.n_jobs_pad + j2) * kStageRS, rowb, bar);
}

// Partner partials of a landed stage, in place over its j1 blocks:
// P1 -> [4], P0 -> [5], P2 -> [6], Q -> [7] (canonical order of eval_cfg<3>).
__device__ __forceinline__ void tstage_partials(float* st) {
  constexpr int rs4 = kStageRS / 4, blk4 = kTT * rs4;  // float4 per role block
  float4* s4 = reinterpret_cast<float4*>(st);
  const float4* rows = s4 + 8 * blk4;  // the 4 single j2 rows (rs4 float4 each)
  for (int e = threadIdx.x; e < blk4; e += kTThreads) {
    const int c = e % rs4;
    const float4 r0 = rows[c], r1 = rows[rs4 + c], r2 = rows[2 * rs4 + c], r3 = rows[3 * rs4 + c];
    s4[4 * blk4 + e] = add4(s4[4 * blk4 + e], r2);  // P1 = ka[s1][j1] + kb[s1][j2]
    s4[5 * blk4 + e] = add4(s4[5 * blk4 + e], r1);  // P0 = kb[s0][j1] + kb[s0][j2]
    s4[6 * blk4 + e] = add4(r0, s4[6 * blk4 + e]);  // P2 = ka[s2][j2] + kb[s2][j1]
    const uint4 q = reinterpret_cast<const uint4*>(s4)[7 * blk4 + e];
    const uint4 w2 = make_uint4(__float_as_uint(r3.x), __float_as_uint(r3.y), __float_as_uint(r3.z),
                                __float_as_uint(r3.w));
    reinterpret_cast<uint4*>(s4)[7 * blk4 + e] = make_uint4(q.x + w2.x, q.y + w2.y, q.z + w2.z, q.w + w2.w);  // Q
  }
}

// One stage of a tile: every (j0, j1) entry of the thread's 4 x 4 micro-tile
// (j0 = 64 A + tx + 16 a, j1 = 64 B + ty + 16 b) against the stage's configs.
// DIAG skips the entries a > b; only the row groups b < NBV are evaluated.
template <bool DIAG, int NBV>
__device__ __forceinline__ void tstage_body(const float* st, int tx, int ty, unsigned one, int s,
                                            float (&breg)[kTM][kTM], int16_t* sbg) {
  constexpr int rs4 = kStageRS / 4, chunks = kStageCfg / 4;
  const float4* st4 = reinterpret_cast<const float4*>(st);
  constexpr int blk4 = kTT * rs4;
  const float4* A0 = st4 + 0 * blk4 + tx * rs4;
  const float4* B01 = st4 + 1 * blk4 + tx * rs4;
  const float4* B02 = st4 + 2 * blk4 + tx * rs4;
  const uint4* W0 = reinterpret_cast<const uint4*>(st4 + 3 * blk4 + tx * rs4);
  const float4* P1 = st4 + 4 * blk4 + ty * rs4;
  const float4* P0 = st4 + 5 * blk4 + ty * rs4;
  const float4* P2 = st4 + 6 * blk4 + ty * rs4;
  const uint4* Q = reinterpret_cast<const uint4*>(st4 + 7 * blk4 + ty * rs4);
  constexpr int row16 = 16 * rs4;

  float m[kTM][kTM];
#pragma unroll
  for (int q = 0; q < chunks; q++) {
    float4 p0[NBV], p1[NBV], p2[NBV];
    uint4 qv[NBV];
#pragma unroll
    for (int b = 0; b < NBV; b++) {
      p0[b] = P0[b * row16 + q];
      p1[b] = P1[b * row16 + q];
      p2[b] = P2[b * row16 + q];
      qv[b] = Q[b * row16 + q];
    }
#pragma unroll
    for (int a = 0; a < kTM; a++) {
      if (DIAG && a >= NBV) continue;  // a > b for every evaluated b
      const float4 a0 = A0[a * row16 + q];
      const float4 b01 = B01[a * row16 + q];
      const float4 b02 = B02[a * row16 + q];
      const uint4 w0 = W0[a * row16 + q];
#pragma unroll
      for (int b = 0; b < NBV; b++) {
        if (DIAG && a > b) continue;
        const float4 r0 = add4(a0, p0[b]);
        const float4 r1 = add4(p1[b], b01);
        const float4 r2 = add4(p2[b], b02);
        const float x0 = min3f(__uint_as_float(imad_add(w0.x, one, qv[b].x)), r0.x, fminf(r1.x, r2.x));
        const float x1 = min3f(__uint_as_float(imad_add(w0.y, one, qv[b].y)), r0.y, fminf(r1.y, r2.y));
        const float x2 = min3f(__uint_as_float(imad_add(w0.z, one, qv[b].z)), r0.z, fminf(r1.z, r2.z));
        const float x3 = min3f(__uint_as_float(imad_add(w0.w, one, qv[b].w)), r0.w, fminf(r1.w, r2.w));
        if (q == 0)
          m[a][b] = fmaxf(max3f(x0, x1, x2), x3);
        else
          m[a][b] = max3f(max3f(m[a][b], x0, x1), x2, x3);
      }
    }
  }
#pragma unroll
  for (int a = 0; a < kTM; a++)
#pragma unroll
    for (int b = 0; b < NBV; b++) {
      if (DIAG && a > b) continue;
      if (m[a][b] > breg[a][b]) {
        breg[a][b] = m[a][b];
        sbg[(ty + 16 * b) * kTBgRow + tx + 16 * a] = (int16_t)s;
      }
    }
}

}  // namespace

template <int MINB>
__global__ void __launch_bounds__(kTThreads, MINB)
    k_score_triples_tiled(const SpaceParams sp, const TripleGrid g, const float* __restrict__ w,
                          const float* __restrict__ fast, float* __restrict__ out_obj, int32_t* __restrict__ out_cfg,
                          unsigned long long* __restrict__ best_key, const unsigned long long* __restrict__ err) {
  extern __shared__ __align__(128) float smem[];
  __shared__ __align__(8) uint64_t bars[2];
  constexpr int rs = kStageRS, rs4 = kStageRS / 4, chunks = kStageCfg / 4;
  constexpr int stage_floats = 8 * kTT * rs + 4 * rs;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // lane bits: a quad (4 consecutive lanes) spans 2 values of tx and 2 of ty, so
  // every LDS.128 of an operand row costs 2 shared wavefronts (4 when a quad
  // reads 4 different rows: tools/microbench/lds.cu)
  const int tx = ((warp & 3) << 2) | (((lane >> 2) & 1) << 1) | (lane & 1);
  const int ty = ((warp >> 2) << 3) | ((lane >> 3) << 1) | ((lane >> 1) & 1);
  const unsigned one = g.one;
  unsigned long long key = 0;

  float* sbest = smem + 2 * stage_floats;
  int16_t* sbg = reinterpret_cast<int16_t*>(sbest + kTT * kTBgRow);
  for (int e = threadIdx.x; e < kTT * kTBgRow; e += kTThreads) sbg[e] = -1;
  int64_t t = blockIdx.x;
  if (t >= g.n_tiles) {
    pdl_wait();
    if (*err == ~0ull) block_max_key(0ull, best_key);
    return;
  }
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    mbar_fence_init();
  }
  // the prologue touches shared memory only: it overlaps the gather's tail (PDL)
  pdl_wait();
  pdl_launch_dependents();
  if (*err != ~0ull) return;  // uniform
  __syncthreads();
  int64_t J2, B, A;
  ttile_coords(g, t, &J2, &B, &A);
  int s = 0, buf = 0;
  unsigned phase[2] = {0u, 0u};
  if (threadIdx.x == 0) issue_tstage(smem, &bars[0], sp, fast, A, B, J2, 0);
  // stage pipeline: the partials of stage s+1 are built at the end of stage s,
  // so one barrier per stage publishes them and frees the buffer of stage s
  mbar_wait(&bars[0], phase[0]);
  phase[0] ^= 1u;
  tstage_partials(smem);
  __syncthreads();

  float breg[kTM][kTM];
#pragma unroll
  for (int a = 0; a < kTM; a++)
#pragma unroll
    for (int b = 0; b < kTM; b++) breg[a][b] = 0.0f;

  while (true) {
    int64_t nt = t, nJ2 = J2, nB = B, nA = A;
    int ns = s + 1;
    if (ns == sp.n_stages) {
      ns = 0;
      nt = t + gridDim.x;
      if (nt < g.n_tiles) ttile_coords(g, nt, &nJ2, &nB, &nA);
    }
    const bool has_next = nt < g.n_tiles;
    if (has_next && threadIdx.x == 0)
      issue_tstage(smem + (buf ^ 1) * stage_floats, &bars[buf ^ 1], sp, fast, nA, nB, nJ2, ns);

    float* st = smem + buf * stage_floats;  // landed, partials built (previous iteration)

    // tile shape (uniform per block): on the diagonal (a == b) the micro-tile
    // entries a > b are never valid (j0 - j1 >= 1) and are skipped; in the last
    // j1 block of the plane only the first ceil((j2 - 64 b) / 16) row groups hold
    // j1 < j2
    const int nbv_raw = (int)((J2 - B * kTT + 15) >> 4);
    const int nbv = nbv_raw > kTM ? kTM : (nbv_raw < 1 ? 1 : nbv_raw);
    const int shape = (A == B ? 4 : 0) + nbv - 1;
    switch (shape) {
      case 0: tstage_body<false, 1>(st, tx, ty, one, s, breg, sbg); break;
      case 1: tstage_body<false, 2>(st, tx, ty, one, s, breg, sbg); break;
      case 2: tstage_body<false, 3>(st, tx, ty, one, s, breg, sbg); break;
      case 3: tstage_body<false, 4>(st, tx, ty, one, s, breg, sbg); break;
      case 4: tstage_body<true, 1>(st, tx, ty, one, s, breg, sbg); break;
      case 5: tstage_body<true, 2>(st, tx, ty, one, s, breg, sbg); break;
      case 6: tstage_body<true, 3>(st, tx, ty, one, s, breg, sbg); break;
      default: tstage_body<true, 4>(st, tx, ty, one, s, breg, sbg); break;
    }

    if (s == sp.n_stages - 1) {
#pragma unroll
      for (int a = 0; a < kTM; a++)
#pragma unroll
        for (int b = 0; b < kTM; b++) {
          sbest[(ty + 16 * b) * kTBgRow + tx + 16 * a] = breg[a][b];
          breg[a][b] = 0.0f;
        }
      __syncthreads();
      // kPass sets per pass with all their loads in flight. Never clipped (positive
      // margins >= 8 > packed key, cosched_internal.h): the key's low bits give
      // the argmax config; its exact FP32 objective in the canonical order
      // w0 + (w1 + w2)
      constexpr int kPass = 4;
      const int jA = (int)(A * kTT), jB = (int)(B * kTT), j2 = (int)J2;
      const bool plane_ok = J2 < g.n_jobs && J2 >= g.c0 && J2 < g.c1;  // uniform per tile
      const int rsz = sp.rs, npad = (int)sp.n_jobs_pad, sl = sp.n_states * npad;
      const int64_t sid2 = (int64_t)j2 * (j2 - 1) * (j2 - 2) / 6;  // colex offset of the plane
#pragma unroll 1
      for (int e0 = 0; e0 < kTT * kTT; e0 += kPass * kTThreads) {
        float f0[kPass], f1[kPass], f2[kPass];
        int c_[kPass];
#pragma unroll
        for (int u = 0; u < kPass; u++) {
          const int e = e0 + u * kTThreads + threadIdx.x;
          const int rj = e >> 6, ri = e & 63;
          const int j0 = jA + ri, j1 = jB + rj;
          const int sg = sbg[rj * kTBgRow + ri];
          const unsigned kbits = __float_as_uint(sbest[rj * kTBgRow + ri]);
          sbg[rj * kTBgRow + ri] = -1;  // every slot, valid or not
          const bool ok = plane_ok && j0 < j1 && j1 < j2;
          const int c = sg * kStageCfg + (31 - (int)(kbits & 31u));
          c_[u] = (ok && sg >= 0 && c < sp.n_cfg) ? c : (ok ? -1 : -2);
          f0[u] = f1[u] = f2[u] = 0.0f;
          if (c_[u] >= 0) {
            // exact FP32 decode of c / n_caps (see score_pairs.cu); w rows < 2^31
            const int st_ = (int)__fmul_rn((float)c + 0.5f, sp.inv_ncaps), p = c - st_ * sp.n_caps;
            const int r = st_ * npad;
            f0[u] = __ldg(w + (int64_t)(r + j0) * rsz + p);
            f1[u] = __ldg(w + (int64_t)(sl + r + j1) * rsz + p);
            f2[u] = __ldg(w + (int64_t)(2 * sl + r + j2) * rsz + p);
          }
        }
#pragma unroll
        for (int u = 0; u < kPass; u++) {
          if (c_[u] == -2) continue;
          const int e = e0 + u * kTThreads + threadIdx.x;
          const int rj = e >> 6, ri = e & 63;  // a warp writes 32 consecutive j0
          const int j0 = jA + ri, j1 = jB + rj;
          const int bc = c_[u];
          const float bo = bc >= 0 ? __fadd_rn(f0[u], __fadd_rn(f1[u], f2[u])) : -INFINITY;
          const int64_t sid = sid2 + (((int64_t)j1 * (j1 - 1)) >> 1) + j0;
          const int64_t k = sid - g.first_set;
          if (out_obj) out_obj[k] = bo;
          if (out_cfg) out_cfg[k] = bc;
          if (bc >= 0) {
            const unsigned long long kk = pack_key(bo, sid);
            key = kk > key ? kk : key;
          }
        }
      }
    }

    // next stage: wait for its data and build its partials before the barrier
    if (has_next) {
      mbar_wait(&bars[buf ^ 1], phase[buf ^ 1]);
      phase[buf ^ 1] ^= 1u;
      tstage_partials(smem + (buf ^ 1) * stage_floats);
    }
    __syncthreads();
    if (!has_next) break;
    t = nt;
    J2 = nJ2;
    B = nB;
    A = nA;
    s = ns;
    buf ^= 1;
  }
  block_max_key(key, best_key);
}

// Host view of the tile count, for work-balanced triple shards (api.cu shard_bounds).
int64_t triple_tiles_before(int64_t j2) { return tiles_before(j2); }

// Precondition: tiled_applicable(3, n_jobs, first, count) (kernels.cu): whole planes.
// The exact re-scoring pass (k_rescore_sets) finds the sets to re-score by a
// scan of the objectives: a flag in this kernel's tile end pushes it past 128
// registers (spills in every stage body).
int launch_score_triples_fast(const SpaceParams& sp, int64_t n_jobs, const float* w, const float* fast, int64_t first,
                              int64_t count, float* obj, int32_t* cfg, unsigned long long* best_key,
                              const unsigned long long* err, const RescoreBuf& rb, cudaStream_t st) {
  auto c3 = [](int64_t n) { return n * (n - 1) * (n - 2) / 6; };
  auto plane_at = [&](int64_t v) {  // smallest c with C(c,3) >= v
    int64_t c = (int64_t)cbrt(6.0 * (double)v);
    while (c > 0 && c3(c - 1) >= v) c--;
    while (c3(c) < v) c++;
    return c;
  };
  const int64_t c0 = plane_at(first), c1 = plane_at(first + count);
  TripleGrid g;
  g.n_jobs = n_jobs;
  g.c0 = c0;
  g.c1 = c1;
  g.first_set = first;
  g.one = 1u;
  g.cum0 = tiles_before(c0);
  g.n_tiles = tiles_before(c1) - g.cum0;
  const char* to = getenv("COSCHED_TRIPLE_ORDER");  // A/B: 0 = r01 plane major, 1 = (b, a, j2), 2 = (b, j2, a)
  g.pair_major = to ? atoi(to) : 2;
  constexpr size_t smem = (size_t)2 * (8 * kTT * kStageRS + 4 * kStageRS) * sizeof(float) +
                          (size_t)kTT * kTBgRow * (sizeof(float) + sizeof(int16_t));
  const char* mb = getenv("COSCHED_TRIPLE_MINB");
  const int minb = (mb && mb[0] == '1') ? 1 : 2;
  smem_optin((const void*)k_score_triples_tiled<1>, smem);
  smem_optin((const void*)k_score_triples_tiled<2>, smem);
  const int g_tri_sms = num_sms();
  int per_sm = 0;
  if (minb == 1) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_score_triples_tiled<1>, kTThreads, smem);
  else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_score_triples_tiled<2>, kTThreads, smem);
  if (per_sm < 1) per_sm = 1;
  int64_t grid = (int64_t)g_tri_sms * per_sm;
  if (grid > g.n_tiles) grid = g.n_tiles;
  if (grid < 1) grid = 1;
  if (minb == 1)
    launch_pdl(k_score_triples_tiled<1>, dim3((unsigned)grid), dim3(kTThreads), smem, st, sp, g, w, fast, obj, cfg,
               best_key, err);
  else
    launch_pdl(k_score_triples_tiled<2>, dim3((unsigned)grid), dim3(kTThreads), smem, st, sp, g, w, fast, obj, cfg,
               best_key, err);
  return 1;
}

}  // namespace cosched
