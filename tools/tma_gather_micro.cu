// Can the TMA unit gather faster than the L1TEX line-per-clock ceiling?
// Random fp64 gathers (configs[1] sizes: 2.43M indices into a 430k vector,
// 16 rounds) through
//   L  LDG: each lane gathers its own x[idx] (8 in flight per lane)
//   T  TMA tile::gather4: x viewed as [n/2][2] doubles (16-byte rows); each
//      lane issues G gather4 copies (4 rows each) into a per-warp shared
//      buffer, completion on a per-warp mbarrier, two stages; the lane then
//      reads its values back from shared memory and picks x[idx] = row[idx & 1]
// Both sum idx-weighted products so the work cannot be elided.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_gather_micro tools/tma_gather_micro.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess) {                                                          \
      std::printf("%s:%d %s -> %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      std::exit(1);                                                                   \
    }                                                                                 \
  } while (0)

constexpr int kThreads = 256, kWarps = kThreads / 32;

__global__ void __launch_bounds__(kThreads, 1) ldg_kernel(const int* __restrict__ idx, const double* __restrict__ x,
                                                          int nnz, int rounds, double* out) {
  const int lane = threadIdx.x & 31;
  const int W = gridDim.x * kWarps, gw = blockIdx.x * kWarps + (threadIdx.x >> 5);
  constexpr int kL = 8, kChunk = 32 * kL;
  const int nchunks = nnz / kChunk;
  double acc = 0.0;
  for (int r = 0; r < rounds; ++r)
    for (int c = gw; c < nchunks; c += W) {
      int ci[kL];
#pragma unroll
      for (int j = 0; j < kL; ++j) ci[j] = __ldg(idx + c * kChunk + j * 32 + lane);
#pragma unroll
      for (int j = 0; j < kL; ++j) acc += __ldca(x + ci[j]);
    }
  if (acc == 12345.678) out[0] = acc;
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}

// G gather4 copies per lane per stage; each lands in a 128-byte slot (64 bytes used)
template <int G, int SLOT>
__global__ void __launch_bounds__(kThreads, 1) tma_kernel(const __grid_constant__ CUtensorMap map,
                                                          const int* __restrict__ idx, int nnz, int rounds,
                                                          double* out) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int kPer = G * 4;           // gathers per lane per stage
  constexpr int kChunk = 32 * kPer;     // gathers per warp per stage
  constexpr int kStageBytes = 32 * G * SLOT;
  unsigned char* wbuf = smem + warp * 2 * kStageBytes;
  __shared__ unsigned long long bar[kWarps][2];
  if (lane == 0) {
    mbar_init(&bar[warp][0], 1);
    mbar_init(&bar[warp][1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const int W = gridDim.x * kWarps, gw = blockIdx.x * kWarps + warp;
  const int nchunks = nnz / kChunk;
  double acc = 0.0;
  unsigned phase[2] = {0, 0};
  auto issue = [&](int c, int s) {
    const int4* ip = reinterpret_cast<const int4*>(idx + c * kChunk + lane * kPer);
    if (lane == 0) mbar_expect(&bar[warp][s], 32 * G * 64);
    __syncwarp();
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int4 q = __ldg(ip + g);
      const unsigned dst = smem_u32(wbuf + s * kStageBytes + (lane * G + g) * SLOT);
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
          "l"(&map), "r"(0), "r"(q.x >> 1), "r"(q.y >> 1), "r"(q.z >> 1), "r"(q.w >> 1),
          "r"(smem_u32(&bar[warp][s]))
          : "memory");
    }
  };
  auto consume = [&](int c, int s) {
    mbar_wait(&bar[warp][s], phase[s]);
    phase[s] ^= 1;
    const int4* ip = reinterpret_cast<const int4*>(idx + c * kChunk + lane * kPer);
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int4 q = __ldg(ip + g);
      const double* row = reinterpret_cast<const double*>(wbuf + s * kStageBytes + (lane * G + g) * SLOT);
      acc += row[0 + (q.x & 1)] + row[2 + (q.y & 1)] + row[4 + (q.z & 1)] + row[6 + (q.w & 1)];
    }
    __syncwarp();
  };
  for (int r = 0; r < rounds; ++r) {
    int c = gw, s = 0;
    if (c < nchunks) issue(c, 0);
    for (; c < nchunks; c += W, s ^= 1) {
      if (c + W < nchunks) issue(c + W, s ^ 1);
      consume(c, s);
    }
  }
  if (acc == 12345.678) out[0] = acc;
}

int main() {
  const int n = 430000, nnz = 2430000 / 2048 * 2048, rounds = 16;
  std::vector<int> hidx(nnz);
  unsigned long long s = 88172645463325252ull;
  for (int i = 0; i < nnz; ++i) {
    s ^= s << 13, s ^= s >> 7, s ^= s << 17;
    hidx[i] = static_cast<int>(s % n);
  }
  std::vector<double> hx(n);
  for (int i = 0; i < n; ++i) hx[i] = 1.0 + i * 1e-6;
  int* idx;
  double *x, *out;
  CK(cudaMalloc(&idx, nnz * 4));
  CK(cudaMalloc(&x, n * 8));
  CK(cudaMalloc(&out, 8));
  CK(cudaMemcpy(idx, hidx.data(), nnz * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(x, hx.data(), n * 8, cudaMemcpyHostToDevice));

  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  using Enc = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                           const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                           CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  CUtensorMap map;
  cuuint64_t gdim[2] = {2, static_cast<cuuint64_t>(n / 2)};
  cuuint64_t gstride[1] = {16};
  cuuint32_t box[2] = {2, 1};
  cuuint32_t estr[2] = {1, 1};
  CUresult cr = reinterpret_cast<Enc>(fn)(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, x, gdim, gstride, box, estr,
                                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                          CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  std::printf("encode: %d\n", static_cast<int>(cr));

  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  auto report = [&](const char* name, float ms) {
    const double g = static_cast<double>(nnz) * rounds / (ms * 1e-3) / 1e9;
    std::printf("%-34s %.3f ms  %.1f G gathers/s\n", name, ms, g);
  };
  for (int rep = 0; rep < 2; ++rep) {
    ldg_kernel<<<148, kThreads>>>(idx, x, nnz, rounds, out);
    CK(cudaEventRecord(e0));
    ldg_kernel<<<148, kThreads>>>(idx, x, nnz, rounds, out);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    report("LDG 8/lane, 8 warps x 148", ms);
  }
  auto run_tma = [&](auto kern, int G, int slot, int ctas, const char* name) {
    const int sm = kWarps * 2 * 32 * G * slot;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
    kern<<<ctas, kThreads, sm>>>(map, idx, nnz, rounds, out);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0));
    kern<<<ctas, kThreads, sm>>>(map, idx, nnz, rounds, out);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    report(name, ms);
  };
  run_tma(tma_kernel<1, 128>, 1, 128, 148, "TMA gather4 G=1 slot128");
  run_tma(tma_kernel<2, 128>, 2, 128, 148, "TMA gather4 G=2 slot128");
  run_tma(tma_kernel<4, 64>, 4, 64, 148, "TMA gather4 G=4 slot64");
  run_tma(tma_kernel<2, 64>, 2, 64, 296, "TMA gather4 G=2 slot64 2 CTA/SM");
  // check: sum through TMA equals sum through LDG (single warp-ordered reduction not compared; rates only)
  return 0;
}
