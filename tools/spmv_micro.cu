// Microbenchmark of fp64 CSR SpMV strategies on B200 (design calibration for
// the hx engine).  Reads a CSR matrix dumped by tools/spmv_micro.py:
//   int64 m, n, nnz; int32 row_ptr[m+1]; int32 col[nnz]; double val[nnz]
// and times y = A x for several kernels and L1/shared carve-outs.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e = (x);                                                        \
    if (e != cudaSuccess) {                                                     \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));         \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

// V1: thread per row, sequential (CSR scalar)
__global__ void k_scalar(int m, const int* __restrict__ rp, const int* __restrict__ ci, const double* __restrict__ v,
                         const double* __restrict__ x, double* __restrict__ y) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    double s = 0.0;
    const int e = rp[i + 1];
    for (int p = rp[i]; p < e; ++p) s += v[p] * __ldg(x + ci[p]);
    y[i] = s;
  }
}

// V2: VEC lanes per row (CSR vector), gathers through L1 (__ldg) or L2 (__ldcg)
template <int VEC, bool L2ONLY>
__global__ void k_vector(int m, const int* __restrict__ rp, const int* __restrict__ ci, const double* __restrict__ v,
                         const double* __restrict__ x, double* __restrict__ y) {
  const int lane = threadIdx.x % VEC;
  const int groups = gridDim.x * blockDim.x / VEC;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) / VEC; i < m; i += groups) {
    double s = 0.0;
    const int e = rp[i + 1];
#pragma unroll 4
    for (int p = rp[i] + lane; p < e; p += VEC) s += v[p] * (L2ONLY ? __ldcg(x + ci[p]) : __ldg(x + ci[p]));
#pragma unroll
    for (int o = VEC / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o, VEC);
    if (lane == 0) y[i] = s;
  }
}

// V3: nnz-chunk per warp, products in registers, segmented by row via smem
// row starts (rows <= 64 nnz), 8 entries per lane.
__global__ void k_chunk(int ntask, const int4* __restrict__ tasks, const int* __restrict__ rp,
                        const int* __restrict__ ci, const double* __restrict__ v, const double* __restrict__ x,
                        double* __restrict__ y) {
  __shared__ double prod[8][256];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* pr = prod[w];
  for (int t = blockIdx.x * 8 + w; t < ntask; t += gridDim.x * 8) {
    const int4 tk = tasks[t];
    const int p0 = tk.z, len = tk.w - tk.z;
    double g[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int q = j * 32 + lane;
      g[j] = q < len ? v[p0 + q] * __ldg(x + ci[p0 + q]) : 0.0;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) pr[j * 32 + lane] = g[j];
    __syncwarp();
    const int r = tk.x + lane;
    if (r < tk.y) {
      double s = 0.0;
      const int a = rp[r] - p0, b = rp[r + 1] - p0;
      for (int q = a; q < b; ++q) s += pr[q];
      y[r] = s;
    }
    __syncwarp();
  }
}

int main(int argc, char** argv) {
  FILE* f = fopen(argv[1], "rb");
  long long m, n, nnz;
  fread(&m, 8, 1, f);
  fread(&n, 8, 1, f);
  fread(&nnz, 8, 1, f);
  std::vector<int> rp(m + 1), ci(nnz);
  std::vector<double> v(nnz);
  fread(rp.data(), 4, m + 1, f);
  fread(ci.data(), 4, nnz, f);
  fread(v.data(), 8, nnz, f);
  fclose(f);
  // tasks for k_chunk: rows packed to <= 256 nnz and <= 32 rows (rows > 256 unsupported here)
  std::vector<int4> tasks;
  for (int r = 0; r < m;) {
    int r0 = r, used = 0;
    while (r < m && r - r0 < 32 && used + (rp[r + 1] - rp[r]) <= 256) used += rp[r + 1] - rp[r], ++r;
    if (r == r0) ++r;
    tasks.push_back(int4{r0, r, rp[r0], rp[r]});
  }
  int *drp, *dci;
  double *dv, *dx, *dy;
  int4* dt;
  CK(cudaMalloc(&drp, (m + 1) * 4));
  CK(cudaMalloc(&dci, nnz * 4));
  CK(cudaMalloc(&dv, nnz * 8));
  CK(cudaMalloc(&dx, n * 8));
  CK(cudaMalloc(&dy, m * 8));
  CK(cudaMalloc(&dt, tasks.size() * 16));
  CK(cudaMemcpy(drp, rp.data(), (m + 1) * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dci, ci.data(), nnz * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dv, v.data(), nnz * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dt, tasks.data(), tasks.size() * 16, cudaMemcpyHostToDevice));
  std::vector<double> hx(n);
  for (long long j = 0; j < n; ++j) hx[j] = 1.0 + (j % 7) * 0.25;
  CK(cudaMemcpy(dx, hx.data(), n * 8, cudaMemcpyHostToDevice));
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](const char* name, auto launch) {
    for (int i = 0; i < 3; ++i) launch();
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    for (int i = 0; i < 50; ++i) launch();
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double us = ms * 1e3 / 50;
    printf("%-34s %8.2f us  %7.1f GB/s(12nnz+8m+8n)\n", name, us, (12.0 * nnz + 8.0 * m + 8.0 * n) / us / 1e3);
  };
  const int blocks = sms * 8;
  timeit("scalar 256t", [&] { k_scalar<<<(m + 255) / 256, 256>>>(m, drp, dci, dv, dx, dy); });
  timeit("vector2 L1", [&] { k_vector<2, false><<<blocks, 256>>>(m, drp, dci, dv, dx, dy); });
  timeit("vector4 L1", [&] { k_vector<4, false><<<blocks, 256>>>(m, drp, dci, dv, dx, dy); });
  timeit("vector8 L1", [&] { k_vector<8, false><<<blocks, 256>>>(m, drp, dci, dv, dx, dy); });
  timeit("vector16 L1", [&] { k_vector<16, false><<<blocks, 256>>>(m, drp, dci, dv, dx, dy); });
  timeit("vector32 L1", [&] { k_vector<32, false><<<blocks, 256>>>(m, drp, dci, dv, dx, dy); });
  timeit("vector4 L2only", [&] { k_vector<4, true><<<blocks, 256>>>(m, drp, dci, dv, dx, dy); });
  timeit("vector8 L2only", [&] { k_vector<8, true><<<blocks, 256>>>(m, drp, dci, dv, dx, dy); });
  for (int carve : {0, 25, 50, 100}) {
    CK(cudaFuncSetAttribute(k_vector<8, false>, cudaFuncAttributePreferredSharedMemoryCarveout, carve));
    char nm[64];
    snprintf(nm, 64, "vector8 L1 carve%d", carve);
    timeit(nm, [&] { k_vector<8, false><<<blocks, 256>>>(m, drp, dci, dv, dx, dy); });
  }
  const int nt = static_cast<int>(tasks.size());
  timeit("chunk256 regs+smem", [&] { k_chunk<<<sms * 4, 256>>>(nt, dt, drp, dci, dv, dx, dy); });
  timeit("chunk256 regs+smem x2 grid", [&] { k_chunk<<<sms * 8, 256>>>(nt, dt, drp, dci, dv, dx, dy); });
  // pure streaming reference: copy val (bandwidth roof)
  timeit("stream: copy 12nnz bytes", [&] {
    cudaMemcpyAsync(dy, dv, std::min<long long>(m, nnz) * 8, cudaMemcpyDeviceToDevice);
  });
  return 0;
}
