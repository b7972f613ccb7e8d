// Grid-barrier latency on B200: one persistent cooperative kernel (1 CTA x
// 512 threads per SM) runs N barrier rounds; each round optionally stores a
// row of doubles per thread first (the phase epilogue's outstanding writes).
// Variants:
//   0 counter : red.release.gpu on one 64-bit counter, acquire spin (hx today)
//   1 flags   : per-CTA flag stores (st.release), CTA 0 polls all flags with a
//               warp, then releases a generation word everyone spins on
//   2 counter+fence split: __threadfence() then relaxed red, acquire spin
//   3 atom.add.acq_rel with return: the last arriver releases `go`
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/barrier_micro tools/barrier_micro.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ unsigned long long ld_acq(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_rlx(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

struct Bar {
  unsigned long long count;
  unsigned long long pad0[15];
  unsigned long long go;
  unsigned long long pad1[15];
  unsigned long long flags[1024 * 16];  // one 128-byte line per CTA
};

__global__ void __launch_bounds__(512, 1) bar_kernel(Bar* b, int variant, int rounds, int store_doubles, double* sink) {
  const int G = gridDim.x;
  unsigned long long target = 0;
  for (int r = 1; r <= rounds; ++r) {
    if (store_doubles) {
      double* row = sink + (static_cast<size_t>(blockIdx.x) * 512 + threadIdx.x) * store_doubles;
      for (int k = 0; k < store_doubles; ++k) row[k] = r + k;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      if (variant == 0) {
        target += G;
        asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(&b->count), "l"(1ull) : "memory");
        while (ld_acq(&b->count) < target) {
        }
      } else if (variant == 2) {
        target += G;
        __threadfence();
        asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(&b->count), "l"(1ull) : "memory");
        while (ld_rlx(&b->count) < target) {
        }
        __threadfence();
      } else if (variant == 3) {
        unsigned long long old;
        asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], %2;" : "=l"(old) : "l"(&b->count), "l"(1ull) : "memory");
        if (old == static_cast<unsigned long long>(r) * G - 1)
          asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(&b->go), "l"(static_cast<unsigned long long>(r)) : "memory");
        while (ld_acq(&b->go) < static_cast<unsigned long long>(r)) {
        }
      }
    }
    if (variant == 1) {
      if (threadIdx.x == 0)
        asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(&b->flags[blockIdx.x * 16]),
                     "l"(static_cast<unsigned long long>(r)) : "memory");
      if (blockIdx.x == 0 && threadIdx.x < 32) {
        for (int c = threadIdx.x; c < G; c += 32)
          while (ld_acq(&b->flags[c * 16]) < static_cast<unsigned long long>(r)) {
          }
        __syncwarp();
        if (threadIdx.x == 0)
          asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(&b->go), "l"(static_cast<unsigned long long>(r)) : "memory");
      } else if (threadIdx.x == 0) {
        while (ld_acq(&b->go) < static_cast<unsigned long long>(r)) {
        }
      }
    }
    __syncthreads();
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  Bar* b;
  cudaMalloc(&b, sizeof(Bar));
  double* sink;
  cudaMalloc(&sink, static_cast<size_t>(sms) * 512 * 16 * sizeof(double));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int rounds = 2000;
  for (int stores : {0, 4, 16}) {
    for (int v = 0; v < 4; ++v) {
      float best = 1e30f;
      for (int rep = 0; rep < 3; ++rep) {
        cudaMemset(b, 0, sizeof(Bar));
        int vv = v, rr = rounds, ss = stores;
        void* args[] = {&b, &vv, &rr, &ss, &sink};
        cudaEventRecord(e0);
        cudaLaunchCooperativeKernel((void*)bar_kernel, sms, 512, args, 0, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      cudaError_t err = cudaGetLastError();
      printf("stores/thread %2d variant %d: %.3f us per barrier round %s\n", stores, v, best * 1e3f / rounds,
             err == cudaSuccess ? "" : cudaGetErrorString(err));
    }
  }
  return 0;
}
