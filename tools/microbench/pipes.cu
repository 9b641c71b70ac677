// Microbenchmark: per-SM issue throughput of the FP32/INT instructions the
// pair scorer's inner loop is built from (FADD, FADD2, FMNMX, FMNMX3, FSETP,
// FSEL, LOP3, IADD3, predicated FMNMX), alone and in mixes.
// Prints warp-instructions per SM clock per SM (4.0 = one per SMSP per clock).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITERS 4096
#define CH 8

template <int OP>
__global__ void __launch_bounds__(1024) kbench(float* out, float seed, long long* cyc) {
  float a[CH], b[CH];
  float2 p[CH], q[CH];
  unsigned u[CH];
#pragma unroll
  for (int i = 0; i < CH; i++) {
    a[i] = seed * (threadIdx.x + i);
    b[i] = seed + i;
    p[i] = make_float2(a[i], b[i]);
    q[i] = make_float2(b[i], a[i]);
    u[i] = __float_as_uint(a[i]);
  }
  float k = seed * 0.5f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < CH; i++) {
      if (OP == 0) asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(b[i]));
      if (OP == 1) p[i] = __fadd2_rn(p[i], q[i]);
      if (OP == 2) { asm volatile("max.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(b[i])); asm volatile("min.f32 %0, %0, %1;" : "+f"(b[i]) : "f"(a[i])); }
      if (OP == 3) asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(b[i]), "f"(k));
      if (OP == 4) asm volatile("{.reg .pred p; setp.gt.f32 p, %0, %1; selp.f32 %0, %1, %0, p;}" : "+f"(a[i]) : "f"(b[i]));
      if (OP == 5) asm volatile("lop3.b32 %0, %0, %1, %2, 0xE8;" : "+r"(u[i]) : "r"(__float_as_uint(b[i])), "r"(0x80000000u));
      if (OP == 6) asm volatile("add.u32 %0, %0, %1;" : "+r"(u[i]) : "r"(__float_as_uint(b[i])));
      if (OP == 7) asm volatile("{.reg .pred p; setp.gt.f32 p, %0, %2; @p max.f32 %0, %0, %1;}" : "+f"(a[i]) : "f"(b[i]), "f"(k));
      if (OP == 8) { // mix A: FADD + 2 FSETP + predicated FMNMX
        asm volatile("{.reg .pred p; .reg .f32 t; add.rn.f32 t, %1, %2; setp.gt.f32 p, %1, %3; setp.gt.and.f32 p, %2, %3, p; @p max.f32 %0, %0, t;}"
                     : "+f"(a[i]) : "f"(b[i]), "f"(p[i].x), "f"(k));
      }
      if (OP == 9) { // mix B per 2 cands: 3 FADD2, 2 FMNMX, 2 LOP3, 1 FMNMX3
        float2 r0 = __fadd2_rn(p[i], q[i]);
        float2 r1 = __fadd2_rn(q[i], make_float2(b[i], k));
        float2 th = __fadd2_rn(r0, r1);
        float f0 = fminf(r0.x, r1.x), f1 = fminf(r0.y, r1.y);
        unsigned x0, x1;
        asm volatile("lop3.b32 %0, %1, %2, %3, 0xB8;" : "=r"(x0) : "r"(__float_as_uint(th.x)), "r"(__float_as_uint(f0)), "r"(0x80000000u));
        asm volatile("lop3.b32 %0, %1, %2, %3, 0xB8;" : "=r"(x1) : "r"(__float_as_uint(th.y)), "r"(__float_as_uint(f1)), "r"(0x80000000u));
        asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(__uint_as_float(x0)), "f"(__uint_as_float(x1)));
        p[i] = r0; q[i] = th;
      }
      if (OP == 10) asm volatile("{.reg .pred p; setp.gt.f32 p, %0, %1; setp.gt.and.f32 p, %1, %2, p; selp.f32 %0, %1, %0, p;}" : "+f"(a[i]) : "f"(b[i]), "f"(k));
      if (OP == 11) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(b[i]), "f"(k));
      if (OP == 12) { // FADD + FMNMX alternating (dual-pipe?)
        asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(k));
        asm volatile("max.f32 %0, %0, %1;" : "+f"(b[i]) : "f"(k));
      }
      if (OP == 13) { // FSETP feeding a predicated FADD
        asm volatile("{.reg .pred p; setp.gt.f32 p, %0, %2; @p add.rn.f32 %0, %0, %1;}" : "+f"(a[i]) : "f"(b[i]), "f"(k));
      }
    }
  }
  long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < CH; i++) s += a[i] + b[i] + p[i].x + p[i].y + q[i].x + __uint_as_float(u[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// SASS instructions per chain-iteration (counted from cuobjdump of this file)
static const char* names[] = {"FADD", "FADD2", "FMNMX", "FMNMX3", "FSETP+FSEL", "LOP3", "IADD",
                              "FSETP+@P FMNMX", "mixA(FADD,2FSETP,@P FMNMX)", "mixB(3FADD2,2FMNMX,2LOP3,FMNMX3)",
                              "2FSETP+FSEL", "FFMA", "FADD||FMNMX", "FSETP+@P FADD"};
static const double ninstr[] = {1, 1, 2, 1, 2, 1, 1, 2, 4, 8, 3, 1, 2, 2};

template <int OP>
void run(int nsm, float* out, long long* cyc) {
  int threads = 1024, blocks = nsm;
  kbench<OP><<<blocks, threads>>>(out, 1.0001f, cyc);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kbench<OP><<<blocks, threads>>>(out, 1.0001f, cyc);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long h[1024]; cudaMemcpy(h, cyc, blocks * sizeof(long long), cudaMemcpyDeviceToHost);
  double mx = 0; for (int i = 0; i < blocks; i++) mx = h[i] > mx ? h[i] : mx;
  double winstr = (double)threads / 32 * ITERS * CH * ninstr[OP];
  double ipc = winstr / mx;
  double ghz = mx / (ms * 1e6);
  printf("%-40s warp-instr/clk/SM = %6.3f  (lane-ops/clk/SM = %6.1f)  kernel %.3f ms, clk ~%.0f MHz\n",
         names[OP], ipc, ipc * 32, ms, ghz * 1000);
}

int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  float* out; long long* cyc;
  cudaMalloc(&out, nsm * 1024 * 4); cudaMalloc(&cyc, nsm * 8);
  run<0>(nsm, out, cyc); run<1>(nsm, out, cyc); run<2>(nsm, out, cyc); run<3>(nsm, out, cyc);
  run<4>(nsm, out, cyc); run<5>(nsm, out, cyc); run<6>(nsm, out, cyc); run<7>(nsm, out, cyc);
  run<8>(nsm, out, cyc); run<9>(nsm, out, cyc); run<10>(nsm, out, cyc); run<11>(nsm, out, cyc);
  run<12>(nsm, out, cyc); run<13>(nsm, out, cyc);
  printf("SMs=%d\n", nsm);
  return 0;
}
