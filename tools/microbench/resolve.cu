// Microbenchmark: the per-step latency of the greedy scan's pick loop pieces on one SM.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o resolve resolve.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int mode, int nw, int iters, long long* out, int* sink) {
  __shared__ __align__(16) int s_w[2][16];
  __shared__ unsigned long long s_j[2048];
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  for (int i = t; i < 2048; i += blockDim.x) s_j[i] = i * 7 + 3;
  if (t < 32) s_w[t >> 4][t & 15] = 0x7FFFFFFF;
  __syncthreads();
  if (wid >= nw) return;
  int acc = t, buf = 0;
  const long long c0 = clock64();
  for (int it = 0; it < iters; it++) {
    int my = (acc * 2654435761u) >> 20;
    int wm = my;
    if (mode & 1) wm = __reduce_min_sync(0xFFFFFFFFu, my);
    if (lane == 0) s_w[buf][wid] = wm;
    if (mode & 2) asm volatile("bar.sync 1, %0;" ::"r"(nw * 32) : "memory");
    else __syncwarp();
    int g = wm;
    if (mode & 4) {
      const int4* o4 = reinterpret_cast<const int4*>(s_w[buf]);
      const int4 a = o4[0], b = o4[1], c = o4[2], d = o4[3];
      g = min(min(min(min(a.x, a.y), min(a.z, a.w)), min(min(b.x, b.y), min(b.z, b.w))),
              min(min(min(c.x, c.y), min(c.z, c.w)), min(min(d.x, d.y), min(d.z, d.w))));
    }
    if (mode & 8) {
      const unsigned long long pj = s_j[g & 2047];
      acc += (int)(pj & 0xFF);
    } else {
      acc += g & 0xFF;
    }
    buf ^= 1;
  }
  const long long c1 = clock64();
  if (t == 0) out[0] = (c1 - c0);
  sink[t] = acc;
}
int main() {
  long long* d;
  int* sink;
  cudaMalloc(&d, 8);
  cudaMalloc(&sink, 4096 * 4);
  const int iters = 20000;
  for (int nw = 1; nw <= 16; nw *= 4)
    for (int mode = 0; mode < 16; mode++) {
      k<<<1, 512>>>(mode, nw, iters, d, sink);
      long long c;
      cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
      printf("warps %2d  redux %d  bar %d  min16 %d  lds %d : %.1f cycles / step\n", nw, mode & 1, (mode >> 1) & 1,
             (mode >> 2) & 1, (mode >> 3) & 1, (double)c / iters);
    }
  return 0;
}
