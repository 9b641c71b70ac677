// Microbenchmark: the pair scorer's inner-loop instruction mix (FADD2 x6,
// FMNMX3 x6 per pair per 4 caps, 4x4 pairs per thread) from registers only,
// at several warps/SM, to separate the loop's own issue limit from the
// shared-memory / synchronisation overheads of the real kernel.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float min3f(float a, float b, float c) {
  float r; asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c)); return r;
}
__device__ __forceinline__ float max3f(float a, float b, float c) {
  float r; asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c)); return r;
}
__device__ __forceinline__ float4 add4s(float4 a, float4 b) {
  return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z), __fadd_rn(a.w, b.w));
}
__device__ __forceinline__ float4 add4(float4 a, float4 b) {
  float2 lo = __fadd2_rn(make_float2(a.x, a.y), make_float2(b.x, b.y));
  float2 hi = __fadd2_rn(make_float2(a.z, a.w), make_float2(b.z, b.w));
  return make_float4(lo.x, lo.y, hi.x, hi.y);
}

__device__ __forceinline__ unsigned imad1(unsigned a, unsigned one, unsigned b) {
  unsigned r; asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(one), "r"(b)); return r;
}

template <int MI, int MJ, int MINB, int MODE>
__global__ void __launch_bounds__(256, MINB) kinner(const float4* __restrict__ in, float* out, int iters, unsigned one) {
  float4 a0[MI], b0[MI], w0[MI], a1[MJ], b1[MJ], w1[MJ];
  for (int i = 0; i < MI; i++) { a0[i] = in[threadIdx.x % 7 + i]; b0[i] = in[i + 1]; w0[i] = in[i + 2]; }
  for (int i = 0; i < MJ; i++) { a1[i] = in[i + 3]; b1[i] = in[i + 4]; w1[i] = in[threadIdx.x % 5 + i]; }
  float m[MI][MJ];
  for (int a = 0; a < MI; a++) for (int b = 0; b < MJ; b++) m[a][b] = 0.f;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int a = 0; a < MI; a++) {
#pragma unroll
      for (int b = 0; b < MJ; b++) {
        const float4 r0 = MODE == 1 ? add4s(a0[a], b1[b]) : add4(a0[a], b1[b]);
        const float4 r1 = MODE == 1 ? add4s(a1[b], b0[a]) : add4(a1[b], b0[a]);
        float4 o;
        if (MODE == 3) {  // integer objective on the FMA-heavy pipe (IMAD with a runtime one)
          o.x = __uint_as_float(imad1(__float_as_uint(w0[a].x), one, __float_as_uint(w1[b].x)));
          o.y = __uint_as_float(imad1(__float_as_uint(w0[a].y), one, __float_as_uint(w1[b].y)));
          o.z = __uint_as_float(imad1(__float_as_uint(w0[a].z), one, __float_as_uint(w1[b].z)));
          o.w = __uint_as_float(imad1(__float_as_uint(w0[a].w), one, __float_as_uint(w1[b].w)));
        } else {
          o = MODE >= 1 ? add4s(w0[a], w1[b]) : add4(w0[a], w1[b]);
        }
        const float x0 = min3f(o.x, r0.x, r1.x), x1 = min3f(o.y, r0.y, r1.y);
        const float x2 = min3f(o.z, r0.z, r1.z), x3 = min3f(o.w, r0.w, r1.w);
        m[a][b] = max3f(max3f(m[a][b], x0, x1), x2, x3);
      }
    }
    // perturb operands so nothing is loop-invariant (1 FADD2 per row/col per iteration)
#pragma unroll
    for (int a = 0; a < MI; a++) a0[a] = add4(a0[a], w0[a]);
#pragma unroll
    for (int b = 0; b < MJ; b++) b1[b] = add4(b1[b], w1[b]);
  }
  float s = 0;
  for (int a = 0; a < MI; a++) for (int b = 0; b < MJ; b++) s += m[a][b];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MI, int MJ, int MINB, int MODE>
void run(int warps_per_sm, int nsm, const float4* in, float* out) {
  int threads = 256;
  int blocks = nsm * warps_per_sm * 32 / threads;
  int iters = 2000;
  kinner<MI, MJ, MINB, MODE><<<blocks, threads>>>(in, out, 10, 1u);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kinner<MI, MJ, MINB, MODE><<<blocks, threads>>>(in, out, iters, 1u);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double cands = (double)blocks * threads * iters * MI * MJ * 4;
  printf("MODE=%d MI=%d MJ=%d minB=%d warps/SM=%2d: %.3f ms, %.3g cand/s, %.1f cand/clk/SM @1.9GHz\n", MODE, MI, MJ, MINB, warps_per_sm, ms,
         cands / (ms * 1e-3), cands / (ms * 1e-3) / nsm / 1.9e9);
}

int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  float4* in; float* out;
  cudaMalloc(&in, 64 * sizeof(float4)); cudaMemset(in, 0, 64 * sizeof(float4));
  cudaMalloc(&out, 148 * 2048 * 4 * 4);
  for (int rep = 0; rep < 2; rep++) {
    run<4, 4, 1, 0>(8, nsm, in, out);
    run<4, 4, 1, 2>(8, nsm, in, out);
    run<4, 4, 1, 3>(8, nsm, in, out);
    run<4, 4, 2, 0>(16, nsm, in, out);
    run<4, 4, 2, 2>(16, nsm, in, out);
    run<4, 4, 2, 3>(16, nsm, in, out);
  }
  return 0;
}
