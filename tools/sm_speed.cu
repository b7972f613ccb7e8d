// Is per-SM gather throughput systematically uneven on B200?  Every CTA (one
// per SM) runs the same amount of random fp64 gathers over a 3.4 MB vector
// (configs[1]'s x); prints per-SM time for several repetitions and the
// correlation between repetitions.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/sm_speed tools/sm_speed.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include <algorithm>

__global__ void __launch_bounds__(512, 1) gather_kernel(const double* x, int n, int iters, unsigned seed,
                                                       unsigned long long* out, double* sink) {
  unsigned long long t0 = 0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  unsigned s = seed * 2654435761u + blockIdx.x * 977u + threadIdx.x * 131u + 1u;
  double acc = 0.0;
  for (int it = 0; it < iters; ++it) {
    int idx[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      s = s * 1664525u + 1013904223u;
      idx[j] = (s >> 8) % n;
    }
    double v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = x[idx[j]];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc += v[j];
  }
  __syncthreads();
  unsigned long long t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (acc == 1234.5) sink[0] = acc;
  if (threadIdx.x == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    out[blockIdx.x * 3 + 0] = smid;
    out[blockIdx.x * 3 + 1] = t0;
    out[blockIdx.x * 3 + 2] = t1;
  }
}

int main() {
  const int n = 430000, G = 148, reps = 6, iters = 400;
  double* x;
  double* sink;
  unsigned long long* out;
  cudaMalloc(&x, n * sizeof(double));
  cudaMemset(x, 0, n * sizeof(double));
  cudaMalloc(&sink, 8);
  cudaMalloc(&out, G * 3 * 8);
  std::vector<std::vector<double>> bysm(reps, std::vector<double>(256, 0.0));
  for (int r = 0; r < reps + 1; ++r) {
    gather_kernel<<<G, 512>>>(x, n, iters, r, out, sink);
    std::vector<unsigned long long> h(G * 3);
    cudaMemcpy(h.data(), out, G * 3 * 8, cudaMemcpyDeviceToHost);
    if (r == 0) continue;  // warm-up
    unsigned long long tmin = ~0ull;
    for (int b = 0; b < G; ++b) tmin = std::min(tmin, h[b * 3 + 1]);
    double mn = 1e30, mx = 0, sum = 0;
    for (int b = 0; b < G; ++b) {
      const double us = (h[b * 3 + 2] - h[b * 3 + 1]) / 1e3;
      bysm[r - 1][h[b * 3]] = us;
      mn = std::min(mn, us), mx = std::max(mx, us), sum += us;
    }
    printf("rep %d: per-CTA us min %.1f mean %.1f max %.1f (gathers/CTA %d)\n", r, mn, sum / G, mx, 512 * 8 * iters);
  }
  // correlation across reps by SM
  for (int r = 1; r < reps; ++r) {
    double sa = 0, sb = 0, saa = 0, sbb = 0, sab = 0;
    int k = 0;
    for (int s = 0; s < 256; ++s)
      if (bysm[0][s] > 0 && bysm[r][s] > 0) {
        const double a = bysm[0][s], b = bysm[r][s];
        sa += a, sb += b, saa += a * a, sbb += b * b, sab += a * b, ++k;
      }
    const double cov = sab / k - sa / k * sb / k;
    const double corr = cov / std::sqrt((saa / k - sa / k * sa / k) * (sbb / k - sb / k * sb / k));
    printf("corr(rep0, rep%d) over %d SMs = %.3f\n", r, k, corr);
  }
  printf("smid: times (rep0..)\n");
  for (int s = 0; s < 256; ++s)
    if (bysm[0][s] > 0) {
      printf("%3d:", s);
      for (int r = 0; r < reps; ++r) printf(" %.1f", bysm[r][s]);
      printf("\n");
    }
  return 0;
}
