// Where does the SpMV engine lose against the random-gather ceiling?  Synthetic
// stream of 2.43M random column indices into a 430k fp64 vector (configs[1]
// sizes); every warp walks 256-nnz chunks w, w + W, ... like the engine's
// tasks, kLoads = 8 per lane, and adds one ingredient at a time:
//   A  idx/val coalesced loads + gathers, products summed in registers
//   B  A + products through the per-warp shared buffer, lane-per-row sums (rows of 20)
//   C  B + a per-row epilogue (3 coalesced loads, 2 stores per row, 2 rows per lane)
//   D  C with the next chunk's idx/val loaded before this chunk's gathers (the engine's pipeline)
//   F  C with idx/val staged in shared memory by bulk copies (cp.async.bulk +
//      mbarrier, the next chunk's issued before this chunk's gathers): no
//      registers hold the next chunk
//   G  F with three stages and the next chunk's gathers issued before this
//      chunk's sums (gathers of two chunks in flight per warp)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/engine_micro tools/engine_micro.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

constexpr int kThreads = 512, kLoads = 8, kChunk = 32 * kLoads, kRowLen = 20;

template <int MODE>
__global__ void __launch_bounds__(kThreads, 1) engine(const int* __restrict__ idx, const double* __restrict__ val,
                                                      const double* __restrict__ x, int nnz,
                                                      const double* __restrict__ ein, double* __restrict__ eout,
                                                      int rounds, double* out) {
  __shared__ double stage[kThreads / 32][kChunk];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int W = gridDim.x * (kThreads / 32), gw = blockIdx.x * (kThreads / 32) + warp;
  const int nchunks = nnz / kChunk;
  double* st = stage[warp];
  double acc = 0.0;
  for (int r = 0; r < rounds; ++r) {
    int ci[kLoads];
    double cv[kLoads];
    int c = gw;
    if (MODE == 3 && c < nchunks)
#pragma unroll
      for (int j = 0; j < kLoads; ++j) ci[j] = __ldg(idx + c * kChunk + j * 32 + lane), cv[j] = __ldg(val + c * kChunk + j * 32 + lane);
    for (; c < nchunks; c += W) {
      const int base = c * kChunk;
      if (MODE != 3) {
#pragma unroll
        for (int j = 0; j < kLoads; ++j) ci[j] = __ldg(idx + base + j * 32 + lane), cv[j] = __ldg(val + base + j * 32 + lane);
      }
      int ni[kLoads];
      double nv[kLoads];
      if (MODE == 3) {
        const int nb = (c + W < nchunks ? c + W : c) * kChunk;
#pragma unroll
        for (int j = 0; j < kLoads; ++j) ni[j] = __ldg(idx + nb + j * 32 + lane), nv[j] = __ldg(val + nb + j * 32 + lane);
      }
      // rows of kRowLen: 256 / 20 -> 12 rows per chunk (lane < 12 owns one; no second row here)
      const int rows = kChunk / kRowLen;
      double e0 = 0, e1 = 0, e2 = 0;
      const int row = c * rows + lane;
      if (MODE >= 2 && lane < rows) e0 = __ldcg(ein + row), e1 = __ldcg(ein + row + 7), e2 = __ldg(ein + row + 13);
#pragma unroll
      for (int j = 0; j < kLoads; ++j) cv[j] *= __ldca(x + ci[j]);
      if (MODE == 0) {
#pragma unroll
        for (int j = 0; j < kLoads; ++j) acc += cv[j];
      } else {
#pragma unroll
        for (int j = 0; j < kLoads; ++j) st[j * 32 + lane] = cv[j];
        __syncwarp();
        if (lane < rows) {
          double s = 0.0;
          for (int q = lane * kRowLen; q < (lane + 1) * kRowLen; ++q) s += st[q];
          if (MODE >= 2) {
            const double v = e0 - 0.5 * (s + e2);
            eout[row] = v < 0 ? 0 : v;
            eout[row + 1000000] = e1 * v;
          }
          acc += s;
        }
        __syncwarp();
      }
      if (MODE == 3) {
#pragma unroll
        for (int j = 0; j < kLoads; ++j) ci[j] = ni[j], cv[j] = nv[j];
      }
    }
  }
  if (acc == 12345.678) out[0] = acc;
}

// E: sliced-ELL -- lane = row, a slice of 32 rows stored k-major (entry k of
// the 32 rows contiguous), rows of kRowLen; products summed in registers in
// ascending k, the next 8 entries' idx/val preloaded; per-row epilogue as C.
__global__ void __launch_bounds__(kThreads, 1) engine_sell(const int* __restrict__ idx, const double* __restrict__ val,
                                                           const double* __restrict__ x, int nnz,
                                                           const double* __restrict__ ein, double* __restrict__ eout,
                                                           int rounds, double* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int W = gridDim.x * (kThreads / 32), gw = blockIdx.x * (kThreads / 32) + warp;
  constexpr int kSlice = 32 * kRowLen;
  const int nslices = nnz / kSlice;
  double acc = 0.0;
  for (int r = 0; r < rounds; ++r) {
    for (int c = gw; c < nslices; c += W) {
      const int base = c * kSlice;
      const int row = c * 32 + lane;
      const double e0 = __ldcg(ein + row), e1 = __ldcg(ein + row + 7), e2 = __ldg(ein + row + 13);
      double s = 0.0;
      int ci[kLoads];
      double cv[kLoads];
#pragma unroll
      for (int j = 0; j < kLoads; ++j) ci[j] = __ldg(idx + base + j * 32 + lane), cv[j] = __ldg(val + base + j * 32 + lane);
      for (int k0 = 0; k0 < kRowLen; k0 += kLoads) {
        int ni[kLoads];
        double nv[kLoads];
        const int kn = k0 + kLoads;
#pragma unroll
        for (int j = 0; j < kLoads; ++j) {
          const bool ok = kn + j < kRowLen;
          ni[j] = ok ? __ldg(idx + base + (kn + j) * 32 + lane) : 0;
          nv[j] = ok ? __ldg(val + base + (kn + j) * 32 + lane) : 0.0;
        }
        double g[kLoads];
#pragma unroll
        for (int j = 0; j < kLoads; ++j) g[j] = k0 + j < kRowLen ? __ldca(x + ci[j]) : 0.0;
#pragma unroll
        for (int j = 0; j < kLoads; ++j)
          if (k0 + j < kRowLen) s += cv[j] * g[j];
#pragma unroll
        for (int j = 0; j < kLoads; ++j) ci[j] = ni[j], cv[j] = nv[j];
      }
      const double v = e0 - 0.5 * (s + e2);
      eout[row] = v < 0 ? 0 : v;
      eout[row + 1000000] = e1 * v;
      acc += s;
    }
  }
  if (acc == 12345.678) out[0] = acc;
}

// ---- F / G: bulk-copy staging -------------------------------------------
constexpr int kStageIdx = kChunk * 4, kStageVal = kChunk * 8;
template <int S>
struct alignas(128) TmaWarp {
  double prod[kChunk];
  double val[S][kChunk];
  int idx[S][kChunk];
  unsigned long long bar[S];
};
__device__ __forceinline__ unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void bar_init(unsigned long long* b) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void bulk_issue(unsigned long long* b, void* dst_i, const int* src_i, void* dst_v,
                                           const double* src_v) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(kStageIdx + kStageVal)
               : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst_i)),
               "l"(src_i), "r"(kStageIdx), "r"(smem_u32(b))
               : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst_v)),
               "l"(src_v), "r"(kStageVal), "r"(smem_u32(b))
               : "memory");
}
__device__ __forceinline__ void bar_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}

template <int S>
__global__ void __launch_bounds__(kThreads, 1) engine_tma(const int* __restrict__ idx, const double* __restrict__ val,
                                                          const double* __restrict__ x, int nnz,
                                                          const double* __restrict__ ein, double* __restrict__ eout,
                                                          int rounds, double* out) {
  extern __shared__ __align__(128) unsigned char dsm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int W = gridDim.x * (kThreads / 32), gw = blockIdx.x * (kThreads / 32) + warp;
  const int nchunks = nnz / kChunk;
  TmaWarp<S>* tw = reinterpret_cast<TmaWarp<S>*>(dsm) + warp;
  if (lane == 0)
    for (int k = 0; k < S; ++k) bar_init(&tw->bar[k]);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  unsigned par[S];
  for (int k = 0; k < S; ++k) par[k] = 0;
  double acc = 0.0;
  const int rows = kChunk / kRowLen;
  auto issue = [&](int c, int k) {
    if (lane == 0 && c < nchunks)
      bulk_issue(&tw->bar[k], tw->idx[k], idx + static_cast<size_t>(c) * kChunk, tw->val[k],
                 val + static_cast<size_t>(c) * kChunk);
  };
  auto finish = [&](int c, int k, const double (&g)[kLoads]) {
    const int row = c * rows + lane;
    double e0 = 0, e1 = 0, e2 = 0;
    if (lane < rows) e0 = __ldcg(ein + row), e1 = __ldcg(ein + row + 7), e2 = __ldg(ein + row + 13);
#pragma unroll
    for (int j = 0; j < kLoads; ++j) tw->prod[j * 32 + lane] = tw->val[k][j * 32 + lane] * g[j];
    __syncwarp();
    if (lane < rows) {
      double s = 0.0;
      for (int q = lane * kRowLen; q < (lane + 1) * kRowLen; ++q) s += tw->prod[q];
      const double v = e0 - 0.5 * (s + e2);
      eout[row] = v < 0 ? 0 : v;
      eout[row + 1000000] = e1 * v;
      acc += s;
    }
    __syncwarp();
  };
  for (int r = 0; r < rounds; ++r) {
    if (S == 2) {
      int k = 0;
      issue(gw, 0);
      for (int c = gw; c < nchunks; c += W) {
        issue(c + W, k ^ 1);
        bar_wait(&tw->bar[k], par[k]);
        par[k] ^= 1;
        double g[kLoads];
#pragma unroll
        for (int j = 0; j < kLoads; ++j) g[j] = __ldca(x + tw->idx[k][j * 32 + lane]);
        finish(c, k, g);
        k ^= 1;
      }
      if (gw < nchunks && ((nchunks - 1 - gw) / W + 1) % 1 == 0) {
        // drain: the over-issued copy (c + W past the end) was never issued
      }
    } else {
      // three stages: chunk c in stage k, c + W in k1, c + 2W into k2
      int k = 0;
      issue(gw, 0);
      issue(gw + W, 1);
      double g[kLoads];
      if (gw < nchunks) {
        bar_wait(&tw->bar[0], par[0]);
        par[0] ^= 1;
#pragma unroll
        for (int j = 0; j < kLoads; ++j) g[j] = __ldca(x + tw->idx[0][j * 32 + lane]);
      }
      for (int c = gw; c < nchunks; c += W) {
        const int k1 = k == S - 1 ? 0 : k + 1, k2 = k1 == S - 1 ? 0 : k1 + 1;
        issue(c + 2 * W, k2);
        double gn[kLoads];
        if (c + W < nchunks) {
          bar_wait(&tw->bar[k1], par[k1]);
          par[k1] ^= 1;
#pragma unroll
          for (int j = 0; j < kLoads; ++j) gn[j] = __ldca(x + tw->idx[k1][j * 32 + lane]);
        }
        finish(c, k, g);
#pragma unroll
        for (int j = 0; j < kLoads; ++j) g[j] = gn[j];
        k = k1;
      }
    }
  }
  if (acc == 12345.678) out[0] = acc;
}

int main() {
  const int n = 430000, nnz = 2430000 / kChunk * kChunk;
  std::vector<int> hi(nnz);
  unsigned s = 12345;
  for (int i = 0; i < nnz; ++i) {
    s = s * 1664525u + 1013904223u;
    hi[i] = static_cast<int>((s >> 8) % n);
  }
  int* idx;
  double *val, *x, *ein, *eout, *out;
  cudaMalloc(&idx, nnz * sizeof(int));
  cudaMalloc(&val, nnz * sizeof(double));
  cudaMalloc(&x, n * sizeof(double));
  cudaMalloc(&ein, 2000000 * sizeof(double));
  cudaMalloc(&eout, 2000000 * sizeof(double));
  cudaMalloc(&out, 8);
  cudaMemcpy(idx, hi.data(), nnz * sizeof(int), cudaMemcpyHostToDevice);
  cudaMemset(val, 0, nnz * sizeof(double));
  cudaMemset(x, 0, n * sizeof(double));
  cudaMemset(ein, 0, 2000000 * sizeof(double));
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int rounds = 20;
  auto run = [&](auto kern, const char* name) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      kern<<<sms, kThreads>>>(idx, val, x, nnz, ein, eout, rounds, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep == 2)
        printf("%-62s %.3f ms per SpMV-sized pass, %.1f G gathers/s\n", name, ms / rounds,
               static_cast<double>(nnz) * rounds / ms / 1e6);
    }
  };
  run(engine<0>, "A gathers + idx/val streams, register sums");
  run(engine<1>, "B + shared product buffer, lane-per-row sums");
  run(engine<2>, "C + per-row epilogue loads/stores");
  run(engine<3>, "D = C with next chunk's idx/val preloaded");
  run(engine_sell, "E sliced-ELL: lane = row, register sums, epilogue");
  auto run_dyn = [&](auto kern, size_t smem, const char* name) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      kern<<<sms, kThreads, smem>>>(idx, val, x, nnz, ein, eout, rounds, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep == 2)
        printf("%-62s %.3f ms per SpMV-sized pass, %.1f G gathers/s (%s)\n", name, ms / rounds,
               static_cast<double>(nnz) * rounds / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
  };
  run_dyn(engine_tma<2>, sizeof(TmaWarp<2>) * (kThreads / 32), "F idx/val by bulk copy, 2 stages");
  run_dyn(engine_tma<3>, sizeof(TmaWarp<3>) * (kThreads / 32), "G 3 stages, next chunk's gathers before the sums");
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
