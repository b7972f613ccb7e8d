// Where does the SpMV engine lose against the random-gather ceiling?  Synthetic
// stream of 2.43M random column indices into a 430k fp64 vector (configs[1]
// sizes); every warp walks 256-nnz chunks w, w + W, ... like the engine's
// tasks, kLoads = 8 per lane, and adds one ingredient at a time:
//   A  idx/val coalesced loads + gathers, products summed in registers
//   B  A + products through the per-warp shared buffer, lane-per-row sums (rows of 20)
//   C  B + a per-row epilogue (3 coalesced loads, 2 stores per row, 2 rows per lane)
//   D  C with the next chunk's idx/val loaded before this chunk's gathers (the engine's pipeline)
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
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
