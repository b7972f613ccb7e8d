// Random fp64 gather throughput on B200: L2-resident global vector (the
// current SpMV gather path) vs the same vector spread over a thread-block
// cluster's distributed shared memory (ld.shared::cluster after mapa).
// Every thread issues G independent random gathers per round (8 in flight,
// like the SpMV engine), R rounds; gathers/s over the whole grid.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dsmem_micro tools/dsmem_micro.cu
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdio>

namespace cg = cooperative_groups;

constexpr int kThreads = 512;
constexpr int kInFlight = 8;

__device__ __forceinline__ unsigned hash(unsigned x) {
  x ^= x >> 16;
  x *= 0x7feb352dU;
  x ^= x >> 15;
  x *= 0x846ca68bU;
  x ^= x >> 16;
  return x;
}

template <int F>
__global__ void __launch_bounds__(kThreads, 1) gather_global(const double* v, unsigned n, int rounds, double* out) {
  unsigned s = hash(blockIdx.x * kThreads + threadIdx.x + 1);
  double acc = 0.0;
  for (int r = 0; r < rounds; ++r) {
    double t[F];
#pragma unroll
    for (int k = 0; k < F; ++k) {
      s = hash(s + k);
      t[k] = __ldca(v + (s % n));
    }
#pragma unroll
    for (int k = 0; k < F; ++k) acc += t[k];
  }
  if (acc == 12345.678) out[0] = acc;
}

// Cache-operator variants of the same random gather (K: 0 .cg, 1
// L1::no_allocate, 2 .nc (read-only path; only valid for data the kernel
// never writes), 3 .lu / last use)
template <int F, int K>
__global__ void __launch_bounds__(kThreads, 1) gather_op(const double* v, unsigned n, int rounds, double* out) {
  unsigned s = hash(blockIdx.x * kThreads + threadIdx.x + 1);
  double acc = 0.0;
  for (int r = 0; r < rounds; ++r) {
    double t[F];
#pragma unroll
    for (int k = 0; k < F; ++k) {
      s = hash(s + k);
      const double* p = v + (s % n);
      if constexpr (K == 0) t[k] = __ldcg(p);
      else if constexpr (K == 1) asm volatile("ld.global.L1::no_allocate.f64 %0, [%1];" : "=d"(t[k]) : "l"(p));
      else if constexpr (K == 2) t[k] = __ldg(p);
      else t[k] = __ldlu(p);
    }
#pragma unroll
    for (int k = 0; k < F; ++k) acc += t[k];
  }
  if (acc == 12345.678) out[0] = acc;
}

// The same gathers plus the stream tasks' shared-memory traffic: every
// product stored to a per-warp buffer, then read back lane-per-row (stride
// `rowlen`, the bank pattern of the row sums).
template <int F>
__global__ void __launch_bounds__(kThreads, 1) gather_plus_smem(const double* v, unsigned n, int rounds, int rowlen,
                                                                double* out) {
  __shared__ double buf[kThreads / 32][F * 32];
  double* st = buf[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31;
  unsigned s = hash(blockIdx.x * kThreads + threadIdx.x + 1);
  double acc = 0.0;
  for (int r = 0; r < rounds; ++r) {
    double t[F];
#pragma unroll
    for (int k = 0; k < F; ++k) {
      s = hash(s + k);
      t[k] = __ldca(v + (s % n));
    }
#pragma unroll
    for (int k = 0; k < F; ++k) st[k * 32 + lane] = t[k];
    __syncwarp();
    const int base = (lane * rowlen) % (F * 32);
    for (int k = 0; k < F; ++k) acc += st[(base + k) % (F * 32)];
    __syncwarp();
  }
  if (acc == 12345.678) out[0] = acc;
}

// slice = elements per CTA; cluster = CTAs per cluster (runtime dims)
__global__ void __launch_bounds__(kThreads, 1) gather_dsmem(const double* v, unsigned slice, int rounds, double* out) {
  extern __shared__ double sm[];
  cg::cluster_group cl = cg::this_cluster();
  const unsigned rank = cl.block_rank(), csize = cl.num_blocks();
  for (unsigned i = threadIdx.x; i < slice; i += kThreads) sm[i] = v[rank * slice + i];
  cl.sync();
  unsigned s = hash(blockIdx.x * kThreads + threadIdx.x + 7);
  const unsigned n = slice * csize;
  double acc = 0.0;
  for (int r = 0; r < rounds; ++r) {
    double t[kInFlight];
#pragma unroll
    for (int k = 0; k < kInFlight; ++k) {
      s = hash(s + k);
      const unsigned e = s % n;
      const double* p = cl.map_shared_rank(sm + (e % slice), e / slice);
      t[k] = *p;
    }
#pragma unroll
    for (int k = 0; k < kInFlight; ++k) acc += t[k];
  }
  cl.sync();
  if (acc == 12345.678) out[0] = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const unsigned n = 430000;  // configs[1] x (430k doubles = 3.44 MB)
  double *v, *out;
  cudaMalloc(&v, sizeof(double) * 1100000);
  cudaMalloc(&out, 8);
  cudaMemset(v, 0, sizeof(double) * 1100000);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int rounds = 200;
  auto report = [&](const char* name, int ctas, float ms) {
    const double g = static_cast<double>(ctas) * kThreads * rounds * kInFlight;
    printf("%-34s ctas %4d: %.3f ms, %.1f G gathers/s (%.2f per SM per ns)\n", name, ctas, ms, g / ms / 1e6,
           g / ms / 1e6 / ctas);
  };
  auto run_g = [&](auto kern, int f, const char* name) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      kern<<<sms, kThreads>>>(v, n, rounds * kInFlight / f, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep) report(name, sms, ms);
    }
  };
  run_g(gather_global<4>, 4, "global, 4 in flight / thread");
  run_g(gather_global<8>, 8, "global, 8 in flight / thread");
  run_g(gather_global<16>, 16, "global, 16 in flight / thread");
  run_g(gather_global<32>, 32, "global, 32 in flight / thread");
  run_g(gather_op<8, 0>, 8, "ld.global.cg, 8 in flight");
  run_g(gather_op<8, 1>, 8, "ld.global.L1::no_allocate, 8");
  run_g(gather_op<8, 2>, 8, "ld.global.nc (read-only), 8");
  run_g(gather_op<8, 3>, 8, "ld.global.lu, 8");
  for (int rowlen : {1, 8, 20}) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      gather_plus_smem<8><<<sms, kThreads>>>(v, n, rounds, rowlen, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      char name[80];
      snprintf(name, sizeof name, "global + smem products (row stride %d)", rowlen);
      if (rep) report(name, sms, ms);
    }
  }
  cudaFuncSetAttribute(gather_dsmem, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(gather_dsmem, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  for (int csize : {8, 16}) {
    const unsigned vec = csize == 16 ? 430000u : 200000u;  // 16: all of x; 8: the 200k random-column part
    const unsigned slice = (vec + csize - 1) / csize;
    const size_t smem = slice * sizeof(double);
    int clusters = 0;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = csize;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(csize);
    cudaOccupancyMaxActiveClusters(&clusters, gather_dsmem, &cfg);
    const int ctas = clusters * csize;
    cfg.gridDim = dim3(ctas);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      cudaError_t err = cudaLaunchKernelEx(&cfg, gather_dsmem, (const double*)v, slice, rounds, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (err != cudaSuccess || cudaGetLastError() != cudaSuccess) {
        printf("cluster %d launch failed: %s\n", csize, cudaGetErrorString(err));
        break;
      }
      char name[80];
      snprintf(name, sizeof name, "DSMEM cluster %d (%u KB/CTA, %d clusters)", csize, static_cast<unsigned>(smem / 1024),
               clusters);
      if (rep) report(name, ctas, ms);
    }
  }
  return 0;
}
