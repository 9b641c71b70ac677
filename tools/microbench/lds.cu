// Microbenchmark: shared-memory wavefronts per warp-wide LDS.128 / LDS.64 for
// the lane -> row patterns a register micro-tile scorer can use (rows of 20
// floats, the pair scorer's stage layout). Timing gives loads/clk/SM; run under
// ncu for l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld per instruction.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ int row_of(int pat, int lane) {
  switch (pat) {
    case 0: return 0;                            // broadcast
    case 1: return lane & 3;                     // 4 rows, period 4 (tx of the scorer)
    case 2: return lane >> 2;                    // 8 rows, 4 consecutive lanes each (ty)
    case 3: return lane;                         // 32 rows
    case 4: return lane >> 3;                    // 4 rows, 8 consecutive lanes each
    case 5: return lane & 7;                     // 8 rows, period 8
    case 6: return lane >> 4;                    // 2 rows
    case 7: return (lane >> 3) | ((lane & 1) << 2);  // 8 rows mixed
    default: return lane & 1;                    // 2 rows, period 2
  }
}

template <int PAT, int W>  // W = 4 (LDS.128) or 2 (LDS.64) or 1 (LDS.32)
__global__ void __launch_bounds__(256) klds(float* out, int iters) {
  __shared__ __align__(16) float s[64 * 20 + 64];
  for (int i = threadIdx.x; i < 64 * 20 + 64; i += blockDim.x) s[i] = (float)i;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int base = row_of(PAT, lane) * 20;
  float acc = 0.f;
  int q = 0;
#pragma unroll 1
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int u = 0; u < 16; u++) {
      const int off = base + ((q + u) % 5) * 4;
      if (W == 4) {
        float4 v = *reinterpret_cast<const float4*>(s + off);
        acc += (v.x + v.y) + (v.z + v.w);
      } else if (W == 2) {
        float2 v = *reinterpret_cast<const float2*>(s + off);
        acc += v.x + v.y;
      } else {
        acc += s[off];
      }
    }
    q = (q + 1) % 5;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int PAT, int W>
void run(int nsm, float* out) {
  const int blocks = nsm * 4, iters = 4000;
  klds<PAT, W><<<blocks, 256>>>(out, 10);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  klds<PAT, W><<<blocks, 256>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double warp_loads = (double)blocks * 8 * iters * 16;
  printf("PAT=%d LDS.%d: %.3f ms, %.3f warp-loads/clk/SM @1.965GHz\n", PAT, 32 * W, ms,
         warp_loads / (ms * 1e-3) / nsm / 1.965e9);
}

int main() {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  cudaMalloc(&out, nsm * 4 * 256 * 4);
  run<0, 4>(nsm, out);
  run<1, 4>(nsm, out);
  run<2, 4>(nsm, out);
  run<3, 4>(nsm, out);
  run<4, 4>(nsm, out);
  run<5, 4>(nsm, out);
  run<6, 4>(nsm, out);
  run<7, 4>(nsm, out);
  run<8, 4>(nsm, out);
  run<1, 2>(nsm, out);
  run<2, 2>(nsm, out);
  run<5, 2>(nsm, out);
  run<1, 1>(nsm, out);
  run<2, 1>(nsm, out);
  return 0;
}
