// Microbenchmark: the greedy scan's pick loop (greedy.cu, resolution step 3) on
// synthetic survivors: n survivors with random pair jobs among `nj` jobs, all
// resolved by the pick loop; reports cycles per step.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o resolve2 resolve2.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int NS>
__device__ __forceinline__ bool jobs_clash(unsigned long long a, unsigned long long b) {
  bool c = false;
#pragma unroll
  for (int q = 0; q < NS; q++) {
    const unsigned x = (unsigned)((a >> (20 * q)) & 0xFFFFFu);
#pragma unroll
    for (int r = 0; r < NS; r++) c = c || (x == (unsigned)((b >> (20 * r)) & 0xFFFFFu));
  }
  return c;
}
__global__ void k(int off, int nj, long long* out, int* sink, int variant) {
  __shared__ __align__(16) int s_wmin[2][16];
  __shared__ unsigned long long s_sj[2048];
  __shared__ int s_pidx[2048];
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  for (int i = t; i < 2048; i += blockDim.x) {
    unsigned h = (unsigned)i * 2654435761u;
    unsigned a = (h >> 8) % nj, b = (h >> 3) % nj;
    if (a == b) b = (b + 1) % nj;
    s_sj[i] = (unsigned long long)a | ((unsigned long long)b << 20);
  }
  if (t < 32) s_wmin[t >> 4][t & 15] = 0x7FFFFFFF;
  __syncthreads();
  const int nrw = (off + 127) / 128;
  long long np = 0, c0 = clock64(), steps = 0;
  if (wid < nrw) {
    unsigned long long jr[4];
    unsigned live = 0u;
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const int e = 4 * t + u;
      jr[u] = e < off ? s_sj[e] : 0ull;
      if (e < off) live |= 1u << u;
    }
    int buf = 0;
    while (np < 1000000) {
      steps++;
      const int my = live ? 4 * t + (__ffs(live) - 1) : 0x7FFFFFFF;
      const int wm = __reduce_min_sync(0xFFFFFFFFu, my);
      if (lane == 0) s_wmin[buf][wid] = wm;
      asm volatile("bar.sync 1, %0;" ::"r"(nrw * 32) : "memory");
      const int4* o4 = reinterpret_cast<const int4*>(s_wmin[buf]);
      const int4 a = o4[0], b = o4[1], c = o4[2], d = o4[3];
      const int g = min(min(min(min(a.x, a.y), min(a.z, a.w)), min(min(b.x, b.y), min(b.z, b.w))),
                        min(min(min(c.x, c.y), min(c.z, c.w)), min(min(d.x, d.y), min(d.z, d.w))));
      if (g == 0x7FFFFFFF) break;
      const unsigned long long pj = s_sj[g];
      if (variant == 0) {
#pragma unroll
        for (int u = 0; u < 4; u++)
          if (((live >> u) & 1u) && jobs_clash<2>(jr[u], pj)) live &= ~(1u << u);
      } else {
        const unsigned p0 = (unsigned)(pj & 0xFFFFF), p1 = (unsigned)((pj >> 20) & 0xFFFFF);
        unsigned kill = 0;
#pragma unroll
        for (int u = 0; u < 4; u++) {
          const unsigned x0 = (unsigned)(jr[u] & 0xFFFFF), x1 = (unsigned)((jr[u] >> 20) & 0xFFFFF);
          kill |= ((x0 == p0) | (x0 == p1) | (x1 == p0) | (x1 == p1)) ? (1u << u) : 0u;
        }
        live &= ~kill;
      }
      if (t == 0) s_pidx[np] = g;
      np++;
      buf ^= 1;
    }
  }
  const long long c1 = clock64();
  if (t == 0) {
    out[0] = c1 - c0;
    out[1] = steps;
    out[2] = np;
  }
  sink[t] = (int)np + s_pidx[t & 7];
}
int main() {
  long long* d;
  int* sink;
  cudaMalloc(&d, 24);
  cudaMalloc(&sink, 4096 * 4);
  for (int variant = 0; variant < 2; variant++)
    for (int off : {128, 384, 1024, 2048})
      for (int nj : {64, 1000, 10000}) {
        k<<<1, 512>>>(off, nj, d, sink, variant);
        long long h[3];
        cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
        printf("variant %d survivors %4d jobs %5d: picks %lld steps %lld, %.1f cycles / step\n", variant, off, nj, h[2],
               h[1], (double)h[0] / h[1]);
      }
  return 0;
}
