// LDS.64 rate per SM against the address pattern (does broadcast make a
// shared-memory load cheaper, or does every LDS.64 cost the return of
// 32 x 8 B?  Measured: it costs its wavefronts, 1 cycle per SM each -- a
// broadcast or <= 2-per-quad, <= 16-distinct LDS.64 is ONE cycle).  One CTA per SM, 16 warps, each issuing independent LDS.64 in a
// long unrolled loop from per-lane addresses:
//   pattern 0: all lanes one address                      (1 wavefront)
//   pattern 1: 16 distinct doubles, <= 2 per lane quad     (1 wavefront)
//   pattern 2: 32 distinct consecutive doubles             (2 wavefronts)
//   pattern 3: 4 distinct doubles on lane bits 0, 1        (2 wavefronts by the quad rule)
//   pattern 4: 32 distinct doubles, stride 2 (2-way bank conflict in each half)  (4 wavefronts)
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lds_rate tools/lds_rate.cu && ./lds_rate
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096, kUnroll = 16;

__global__ void __launch_bounds__(512, 1) k_lds(int pattern, double *sink, long long *cycles) {
  __shared__ double buf[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) buf[i] = (double)i;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  int off;
  switch (pattern) {
    case 0: off = 0; break;
    case 1: off = (lane >> 1); break;                 // lanes 2i, 2i+1 share a double: 16 distinct, 2 per quad
    case 2: off = lane; break;
    case 3: off = (lane & 1) + 6 * ((lane >> 1) & 1); break;
    default: off = 2 * lane; break;
  }
  const unsigned base = (unsigned)__cvta_generic_to_shared(buf + off);
  unsigned long long acc[kUnroll];
#pragma unroll
  for (int u = 0; u < kUnroll; ++u) acc[u] = 0ull;
  __syncthreads();
  const long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      unsigned long long v;
      // volatile: one LDS.64 per statement, not hoisted; the offset varies with u and it
      // 32 slots of 64 doubles: the "memory" clobber keeps nvcc from merging the identical
      // loads of its unrolled trips (it did: 4x fewer LDS than written)
      asm volatile("ld.shared.b64 %0, [%1];" : "=l"(v) : "r"(base + 512u * (unsigned)((it * kUnroll + u) & 31)) : "memory");
      acc[u] ^= v;  // integer pipe: the FP64 pipe stays out of the measurement
    }
  }
  const long long t1 = clock64();
  unsigned long long s = 0ull;
#pragma unroll
  for (int u = 0; u < kUnroll; ++u) s ^= acc[u];
  if (s == 0x123456789abcdefull) sink[0] = (double)s;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double *sink;
  long long *cyc;
  cudaMalloc(&sink, 8);
  cudaMallocManaged(&cyc, nsm * sizeof(long long));
  const char *names[] = {"1 address (broadcast)", "16 distinct, 2 per quad", "32 distinct consecutive", "4 distinct on lane bits 0,1",
                         "32 distinct, stride 2"};
  for (int pat = 0; pat < 5; ++pat) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_lds<<<nsm, 512>>>(pat, sink, cyc);
    cudaEventRecord(e0);
    k_lds<<<nsm, 512>>>(pat, sink, cyc);
    cudaEventRecord(e1);
    cudaDeviceSynchronize();
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    double mean = 0;
    for (int i = 0; i < nsm; ++i) mean += (double)cyc[i];
    mean /= nsm;
    const double lds = 16.0 * kIters * kUnroll;  // warp-level LDS.64 per SM (16 warps)
    printf("pattern %d (%s): %.0f clock64 cycles (%.1f us by events -> %.0f MHz), %.3f LDS.64 / clk / SM = %.2f cycles per LDS.64\n",
           pat, names[pat], mean, 1e3 * ms, mean / (1e3 * ms), lds / mean, mean / lds);
  }
  return 0;
}
