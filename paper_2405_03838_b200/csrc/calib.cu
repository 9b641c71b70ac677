// calib.cu -- calibration of the model coefficients on the GPU (SURVEY.md §8(f)
// NEXT #1), sm_100a.
//
// PAPER.md §4.3: "we apply the least square method (or curve fitting)
// for each combination of (S, P) independently and separately"; §5.1.3
// L660-661: C from solo runs first, then D from co-runs. L795: "the
// calibration of coefficients would be time consuming if the numbers of P and
// S would increase" -- here every key is fitted in parallel.
//
// Per key (slice, cap) -- key = cap * n_slices + slice, the row of coef_c/coef_d:
//   stage C: X = H(F_app) (6 columns), y = measured rperf of the key's solo samples
//   stage D: X = sum_{partners} J(F_partner) (3 columns),
//            y = rperf - C[key] . H(F_subject) on the key's co-run samples
// solved by the normal equations G c = X^T y in FP64 (Cholesky). Samples are
// grouped by key with a stable radix sort, so every reduction runs in a fixed
// order: results are bit-identical run to run. The RMS of the residuals is a
// second pass over the samples (no cancellation in y^T y - c^T X^T y).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <cub/cub.cuh>

#include "cosched_internal.h"

namespace cosched {

namespace {

constexpr int kFitThreads = 256;
constexpr double kPivotTol = 1e-10;  // DESIGN.md reading: pivot <= 1e-10 * column norm^2 -> rank deficient

// a2 in FP64: H = (F1/100 - H2, (F6+F7+F8)/100, F2/F1, F4/100, F5/100, 1), J = (F3/100, F4/100, 1)
__device__ __forceinline__ void basis64(const float* f, double h[6], double j[3]) {
  const double F1 = f[0], F2 = f[1], F3 = f[2], F4 = f[3], F5 = f[4];
  h[1] = ((double)f[5] + (double)f[6] + (double)f[7]) / 100.0;
  h[0] = F1 / 100.0 - h[1];
  h[2] = F2 / F1;
  h[3] = F4 / 100.0;
  h[4] = F5 / 100.0;
  h[5] = 1.0;
  j[0] = F3 / 100.0;
  j[1] = F4 / 100.0;
  j[2] = 1.0;
}

// Validate every app's counters (same rules as k_validate) and store its FP64 basis.
__global__ void k_fit_basis(const float* __restrict__ F, int64_t n_apps, double* __restrict__ Hd,
                            double* __restrict__ Jd, unsigned long long* err) {
  const int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (a >= n_apps) return;
  float v[8];
#pragma unroll
  for (int k = 0; k < 8; k++) v[k] = F[a * 8 + k];
  int code = 0;
#pragma unroll
  for (int k = 0; k < 8; k++)
    if (!(v[k] >= 0.0f && v[k] <= 100.0f)) code = COSCHED_E_RANGE;
  if (!code) {
    const float tensor = __fadd_rn(__fadd_rn(v[5], v[6]), v[7]);
    if (!(tensor <= 100.0f)) code = COSCHED_E_RANGE;
    else if (!(v[0] > 0.01f)) code = COSCHED_E_DEGENERATE_PROFILE;
  }
  if (code) {
    atomicMin(err, ((unsigned long long)a << 8) | (unsigned long long)code);
    return;
  }
  double h[6], j[3];
  basis64(v, h, j);
#pragma unroll
  for (int t = 0; t < 6; t++) Hd[a * 6 + t] = h[t];
#pragma unroll
  for (int t = 0; t < 3; t++) Jd[a * 3 + t] = j[t];
}

// Sort keys of the samples (+ the sample index as the payload); checks indices.
__global__ void k_fit_keys(const int32_t* __restrict__ app, const int32_t* __restrict__ partners, int n_partners,
                           const int32_t* __restrict__ key, const float* __restrict__ y, int64_t n, int64_t n_apps,
                           int32_t n_keys, int32_t* __restrict__ keys_out, int32_t* __restrict__ idx_out,
                           unsigned long long* err) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t k = key[i], a = app[i];
  bool bad = k < 0 || k >= n_keys || a < 0 || a >= n_apps || !isfinite(y[i]);
  for (int l = 0; l < n_partners; l++) {
    const int32_t b = partners[i * n_partners + l];
    bad = bad || b < 0 || b >= n_apps;
  }
  // out-of-range sample: reported after the 2^40 offset so feature errors (position = app) win
  if (bad) atomicMin(err, ((unsigned long long)(i + (1ll << 40)) << 8) | (unsigned long long)COSCHED_E_UNKNOWN_KEY);
  keys_out[i] = bad ? 0 : k;
  idx_out[i] = (int32_t)i;
}

__global__ void k_fit_offsets(const int32_t* __restrict__ sorted, int64_t n, int32_t n_keys, int64_t* __restrict__ off) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k > n_keys) return;
  int64_t lo = 0, hi = n;  // first position with sorted[pos] >= k
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (sorted[mid] < k) lo = mid + 1;
    else hi = mid;
  }
  off[k] = lo;
}

// One design row and target of sample i for stage NC (6: C, 3: D).
template <int NC>
__device__ __forceinline__ void fit_row(int64_t i, const int32_t* __restrict__ app, const int32_t* __restrict__ partners,
                                        int n_partners, const float* __restrict__ y, const double* __restrict__ Hd,
                                        const double* __restrict__ Jd, const double* __restrict__ Ck, double x[NC],
                                        double* t) {
  const int64_t a = app[i];
  if (NC == 6) {
#pragma unroll
    for (int c = 0; c < 6; c++) x[c] = Hd[a * 6 + c];
    *t = (double)y[i];
  } else {
#pragma unroll
    for (int c = 0; c < NC; c++) x[c] = 0.0;
    for (int l = 0; l < n_partners; l++) {
      const int64_t b = partners[i * n_partners + l];
#pragma unroll
      for (int c = 0; c < NC; c++) x[c] += Jd[b * 3 + c];
    }
    double pred = 0.0;
#pragma unroll
    for (int c = 0; c < 6; c++) pred += Ck[c] * Hd[a * 6 + c];
    *t = (double)y[i] - pred;
  }
}

// Deterministic block sum of NV doubles per thread (fixed shuffle tree, then warp 0).
template <int NV>
__device__ __forceinline__ void block_sum(double v[NV], double* out) {
  __shared__ double s_part[kFitThreads / 32][NV];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < NV; q++) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[q] += __shfl_down_sync(0xFFFFFFFFu, v[q], o);
    if (lane == 0) s_part[w][q] = v[q];
  }
  __syncthreads();
  if (threadIdx.x < NV) {
    double s = 0.0;
    for (int k = 0; k < kFitThreads / 32; k++) s += s_part[k][threadIdx.x];
    out[threadIdx.x] = s;
  }
  __syncthreads();
}

// Block per key: the Gram matrix (upper triangle, row-major) and X^T y.
template <int NC>
__global__ void __launch_bounds__(kFitThreads) k_fit_gram(const int32_t* __restrict__ idx, const int64_t* __restrict__ off,
                                                          const int32_t* __restrict__ app,
                                                          const int32_t* __restrict__ partners, int n_partners,
                                                          const float* __restrict__ y, const double* __restrict__ Hd,
                                                          const double* __restrict__ Jd, const double* __restrict__ C,
                                                          double* __restrict__ gram) {
  constexpr int NT = NC * (NC + 1) / 2, NV = NT + NC;
  const int k = blockIdx.x;
  double acc[NV];
#pragma unroll
  for (int q = 0; q < NV; q++) acc[q] = 0.0;
  double Ck[6];
  if (NC == 3) {
#pragma unroll
    for (int c = 0; c < 6; c++) Ck[c] = C[(int64_t)k * 6 + c];
  }
  for (int64_t p = off[k] + threadIdx.x; p < off[k + 1]; p += kFitThreads) {
    double x[NC], t;
    fit_row<NC>(idx[p], app, partners, n_partners, y, Hd, Jd, Ck, x, &t);
    int q = 0;
#pragma unroll
    for (int r = 0; r < NC; r++)
#pragma unroll
      for (int c = r; c < NC; c++) acc[q++] += x[r] * x[c];
#pragma unroll
    for (int r = 0; r < NC; r++) acc[NT + r] += x[r] * t;
  }
  block_sum<NV>(acc, gram + (int64_t)k * NV);
}

// Thread per key: Cholesky of G, status, solve.
template <int NC>
__global__ void k_fit_solve(const double* __restrict__ gram, const int64_t* __restrict__ off, int32_t n_keys,
                            const int32_t* __restrict__ c_status, double* __restrict__ coef,
                            int32_t* __restrict__ status, int64_t* __restrict__ count) {
  constexpr int NT = NC * (NC + 1) / 2, NV = NT + NC;
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n_keys) return;
  const int64_t n = off[k + 1] - off[k];
  count[(int64_t)k * 2] = n;
  int st = COSCHED_FIT_OK;
  double G[NC][NC], b[NC], L[NC][NC];
  const double* g = gram + (int64_t)k * NV;
  int q = 0;
  for (int r = 0; r < NC; r++)
    for (int c = r; c < NC; c++) G[r][c] = G[c][r] = g[q++];
  for (int r = 0; r < NC; r++) b[r] = g[NT + r];
  if (n == 0) st = COSCHED_FIT_NO_SAMPLES;
  else if (c_status && c_status[(int64_t)k * 2] != COSCHED_FIT_OK) st = COSCHED_FIT_MISSING_C;
  else if (n < NC) st = COSCHED_FIT_INSUFFICIENT;
  if (st == COSCHED_FIT_OK) {
    for (int r = 0; r < NC && st == COSCHED_FIT_OK; r++) {
      double d = G[r][r];
      for (int c = 0; c < r; c++) d -= L[r][c] * L[r][c];
      if (!(d > kPivotTol * G[r][r])) {  // also catches an all-zero column (0 > 0 is false)
        st = COSCHED_FIT_RANK_DEFICIENT;
        break;
      }
      L[r][r] = sqrt(d);
      for (int i = r + 1; i < NC; i++) {
        double s = G[i][r];
        for (int c = 0; c < r; c++) s -= L[i][c] * L[r][c];
        L[i][r] = s / L[r][r];
      }
    }
  }
  double x[NC];
  for (int r = 0; r < NC; r++) x[r] = 0.0;
  if (st == COSCHED_FIT_OK) {
    double z[NC];
    for (int r = 0; r < NC; r++) {  // L z = b
      double s = b[r];
      for (int c = 0; c < r; c++) s -= L[r][c] * z[c];
      z[r] = s / L[r][r];
    }
    for (int r = NC - 1; r >= 0; r--) {  // L^T x = z
      double s = z[r];
      for (int c = r + 1; c < NC; c++) s -= L[c][r] * x[c];
      x[r] = s / L[r][r];
    }
  }
  for (int r = 0; r < NC; r++) coef[(int64_t)k * NC + r] = x[r];
  status[(int64_t)k * 2] = st;
}

// Block per key: RMS of the residuals at the fitted coefficients.
template <int NC>
__global__ void __launch_bounds__(kFitThreads) k_fit_rms(const int32_t* __restrict__ idx, const int64_t* __restrict__ off,
                                                         const int32_t* __restrict__ app,
                                                         const int32_t* __restrict__ partners, int n_partners,
                                                         const float* __restrict__ y, const double* __restrict__ Hd,
                                                         const double* __restrict__ Jd, const double* __restrict__ C,
                                                         const double* __restrict__ coef,
                                                         const int32_t* __restrict__ status, double* __restrict__ rms,
                                                         double* __restrict__ scratch) {
  const int k = blockIdx.x;
  double acc[1] = {0.0};
  double Ck[6], ck[NC];
  if (NC == 3) {
#pragma unroll
    for (int c = 0; c < 6; c++) Ck[c] = C[(int64_t)k * 6 + c];
  }
#pragma unroll
  for (int c = 0; c < NC; c++) ck[c] = coef[(int64_t)k * NC + c];
  const bool ok = status[(int64_t)k * 2] == COSCHED_FIT_OK;
  if (ok) {
    for (int64_t p = off[k] + threadIdx.x; p < off[k + 1]; p += kFitThreads) {
      double x[NC], t;
      fit_row<NC>(idx[p], app, partners, n_partners, y, Hd, Jd, Ck, x, &t);
      double r = t;
#pragma unroll
      for (int c = 0; c < NC; c++) r -= ck[c] * x[c];
      acc[0] += r * r;
    }
  }
  block_sum<1>(acc, scratch + k);
  if (threadIdx.x == 0) {
    const int64_t n = off[k + 1] - off[k];
    rms[(int64_t)k * 2] = ok ? sqrt(scratch[k] / (double)n) : nan("");
  }
}

__global__ void k_fit_store(const double* __restrict__ coef, int32_t n_keys, int NC, double* __restrict__ out) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e < (int64_t)n_keys * NC) out[e] = coef[e];
}

inline size_t al(size_t b) { return (b + 255) & ~(size_t)255; }

struct FitWs {
  double *Hd, *Jd, *gram, *coef_c, *coef_d, *scratch;
  int32_t *s_keys, *s_keys_sorted, *s_idx, *s_idx_sorted;
  int32_t *c_keys, *c_keys_sorted, *c_idx, *c_idx_sorted;
  int64_t *off_s, *off_c;
  unsigned long long* err;
  void* sort_tmp;
  size_t sort_bytes, bytes;
};

size_t fit_layout(const cosched_fit_desc* d, char* base, FitWs* w) {
  const int64_t nk = (int64_t)d->n_slices * d->n_caps;
  size_t off = 0;
  auto take = [&](size_t b) -> char* {
    char* p = base ? base + off : nullptr;
    off += al(b);
    return p;
  };
  FitWs f;
  f.Hd = (double*)take((size_t)d->n_apps * 6 * 8 + 8);
  f.Jd = (double*)take((size_t)d->n_apps * 3 * 8 + 8);
  f.gram = (double*)take((size_t)nk * 27 * 8);
  f.coef_c = (double*)take((size_t)nk * 6 * 8);
  f.coef_d = (double*)take((size_t)nk * 3 * 8);
  f.scratch = (double*)take((size_t)nk * 8);
  const size_t ns = (size_t)d->n_solo * 4 + 4, nc = (size_t)d->n_corun * 4 + 4;
  f.s_keys = (int32_t*)take(ns);
  f.s_keys_sorted = (int32_t*)take(ns);
  f.s_idx = (int32_t*)take(ns);
  f.s_idx_sorted = (int32_t*)take(ns);
  f.c_keys = (int32_t*)take(nc);
  f.c_keys_sorted = (int32_t*)take(nc);
  f.c_idx = (int32_t*)take(nc);
  f.c_idx_sorted = (int32_t*)take(nc);
  f.off_s = (int64_t*)take((size_t)(nk + 1) * 8);
  f.off_c = (int64_t*)take((size_t)(nk + 1) * 8);
  f.err = (unsigned long long*)take(8);
  size_t sb = 0, sb2 = 0;
  cub::DeviceRadixSort::SortPairs((void*)nullptr, sb, (const int32_t*)nullptr, (int32_t*)nullptr,
                                  (const int32_t*)nullptr, (int32_t*)nullptr, (int)std::max<int64_t>(d->n_solo, 1));
  cub::DeviceRadixSort::SortPairs((void*)nullptr, sb2, (const int32_t*)nullptr, (int32_t*)nullptr,
                                  (const int32_t*)nullptr, (int32_t*)nullptr, (int)std::max<int64_t>(d->n_corun, 1));
  f.sort_bytes = std::max(sb, sb2);
  f.sort_tmp = take(f.sort_bytes);
  f.bytes = off;
  if (w) *w = f;
  return off;
}

__global__ void k_fill_err(unsigned long long* e) { *e = ~0ull; }

}  // namespace

cosched_status fit_validate_desc(const cosched_fit_desc* d) {
  if (!d) return COSCHED_E_ARG;
  if (d->n_slices < 1 || d->n_caps < 1 || (int64_t)d->n_slices * d->n_caps > (1 << 24)) return COSCHED_E_ARG;
  if (d->n_apps < 0 || d->n_solo < 0 || d->n_corun < 0 || d->n_solo >= (1ll << 31) || d->n_corun >= (1ll << 31))
    return COSCHED_E_ARG;
  if (d->n_apps > 0 && !d->features) return COSCHED_E_ARG;
  if (d->n_solo > 0 && (!d->solo_app || !d->solo_key || !d->solo_rperf)) return COSCHED_E_ARG;
  if (d->n_corun > 0 && (!d->co_app || !d->co_key || !d->co_rperf || d->n_partners < 1 || d->n_partners > 2 ||
                         !d->co_partners))
    return COSCHED_E_ARG;
  return COSCHED_OK;
}

size_t fit_workspace_bytes(const cosched_fit_desc* d) { return fit_layout(d, nullptr, nullptr); }

// Enqueue the whole fit on `st`; returns the number of kernels launched (or -1 on a launch error).
int fit_enqueue(const cosched_fit_desc* d, void* workspace, const cosched_fit_out* out, unsigned long long** err_dev,
                cudaStream_t st) {
  FitWs w;
  fit_layout(d, (char*)workspace, &w);
  *err_dev = w.err;
  const int32_t nk = d->n_slices * d->n_caps;
  int launches = 0;
  k_fill_err<<<1, 1, 0, st>>>(w.err);
  launches++;
  if (d->n_apps > 0) {
    k_fit_basis<<<(unsigned)((d->n_apps + 255) / 256), 256, 0, st>>>(d->features, d->n_apps, w.Hd, w.Jd, w.err);
    launches++;
  }
  const int kb = 8;
  auto group = [&](const int32_t* app, const int32_t* partners, int np, const int32_t* key, const float* y, int64_t n,
                   int32_t* keys, int32_t* keys_sorted, int32_t* idx, int32_t* idx_sorted, int64_t* offs) {
    if (n > 0) {
      k_fit_keys<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(app, partners, np, key, y, n, d->n_apps, nk, keys, idx,
                                                             w.err);
      int bits = 1;
      while ((1ll << bits) < nk) bits++;
      size_t tb = w.sort_bytes;
      cub::DeviceRadixSort::SortPairs(w.sort_tmp, tb, keys, keys_sorted, idx, idx_sorted, (int)n, 0, bits, st);
      launches += 2 + 2 * ((bits + 7) / 8);
    }
    k_fit_offsets<<<(unsigned)((nk + 1 + 255) / 256), 256, 0, st>>>(keys_sorted, n, nk, offs);
    launches++;
  };
  (void)kb;
  group(d->solo_app, nullptr, 0, d->solo_key, d->solo_rperf, d->n_solo, w.s_keys, w.s_keys_sorted, w.s_idx,
        w.s_idx_sorted, w.off_s);
  group(d->co_app, d->co_partners, d->n_partners, d->co_key, d->co_rperf, d->n_corun, w.c_keys, w.c_keys_sorted,
        w.c_idx, w.c_idx_sorted, w.off_c);
  // stage C (solo runs)
  k_fit_gram<6><<<nk, kFitThreads, 0, st>>>(w.s_idx_sorted, w.off_s, d->solo_app, nullptr, 0, d->solo_rperf, w.Hd,
                                            w.Jd, nullptr, w.gram);
  k_fit_solve<6><<<(nk + 127) / 128, 128, 0, st>>>(w.gram, w.off_s, nk, nullptr, w.coef_c, out->status, out->count);
  k_fit_rms<6><<<nk, kFitThreads, 0, st>>>(w.s_idx_sorted, w.off_s, d->solo_app, nullptr, 0, d->solo_rperf, w.Hd,
                                           w.Jd, nullptr, w.coef_c, out->status, out->rms, w.scratch);
  // stage D (co-run residuals of C)
  k_fit_gram<3><<<nk, kFitThreads, 0, st>>>(w.c_idx_sorted, w.off_c, d->co_app, d->co_partners, d->n_partners,
                                            d->co_rperf, w.Hd, w.Jd, w.coef_c, w.gram);
  k_fit_solve<3><<<(nk + 127) / 128, 128, 0, st>>>(w.gram, w.off_c, nk, out->status, w.coef_d, out->status + 1,
                                                   out->count + 1);
  k_fit_rms<3><<<nk, kFitThreads, 0, st>>>(w.c_idx_sorted, w.off_c, d->co_app, d->co_partners, d->n_partners,
                                           d->co_rperf, w.Hd, w.Jd, w.coef_c, w.coef_d, out->status + 1, out->rms + 1,
                                           w.scratch);
  k_fit_store<<<(unsigned)((nk * 6 + 255) / 256), 256, 0, st>>>(w.coef_c, nk, 6, out->coef_c);
  k_fit_store<<<(unsigned)((nk * 3 + 255) / 256), 256, 0, st>>>(w.coef_d, nk, 3, out->coef_d);
  launches += 8;
  return cudaGetLastError() == cudaSuccess ? launches : -1;
}

}  // namespace cosched
