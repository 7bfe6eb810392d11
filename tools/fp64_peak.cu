#include <cstdlib>
// FP64 pipe microbenchmark for B200 (sm_100a): DFMA vs DMMA (mma.sync f64) throughput.
// Decides the moment-kernel MAC strategy.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int NACC>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += acc[i];
  if (s == 12345.678) out[0] = s;
}

template <int NACC>
__global__ void dmma884_kernel(double* out, int iters, double a, double b) {
  double c[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = 0; c[i][1] = 0; }
  double av = a + threadIdx.x, bv = b - threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(av), "d"(bv));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

template <int NACC>
__global__ void dmma16816_kernel(double* out, int iters, double a, double b) {
  double c[NACC][4];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0; }
  double av[8], bv[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) av[i] = a + i + threadIdx.x;
#pragma unroll
  for (int i = 0; i < 4; ++i) bv[i] = b - i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(av[0]), "d"(av[1]), "d"(av[2]), "d"(av[3]), "d"(av[4]), "d"(av[5]), "d"(av[6]), "d"(av[7]),
                     "d"(bv[0]), "d"(bv[1]), "d"(bv[2]), "d"(bv[3]));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.678) out[0] = s;
}

// DMMA with concurrent DMUL stream (KR-construction contention probe)
template <int NACC, int NMUL>
__global__ void dmma_dmul_kernel(double* out, int iters, double a, double b) {
  double c[NACC][2];
  double p[NMUL > 0 ? NMUL : 1];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = 0; c[i][1] = 0; }
#pragma unroll
  for (int i = 0; i < NMUL; ++i) p[i] = 1.0 + i * 1e-9;
  double av = a + threadIdx.x, bv = b - threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(av), "d"(bv));
#pragma unroll
    for (int i = 0; i < NMUL; ++i) p[i] = p[i] * a;
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
#pragma unroll
  for (int i = 0; i < NMUL; ++i) s += p[i];
  if (s == 12345.678) out[0] = s;
}

template <typename K>
float timeit(K kern, int grid, int block, int iters, double* d) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  kern<<<grid, block>>>(d, 10, 1.0000001, 1e-9);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    kern<<<grid, block>>>(d, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best;
}

int main(int argc, char **argv) {
  double* d; CK(cudaMalloc(&d, 64));
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs %d, max clock %d MHz\n", sms, clk / 1000);
  if (argc > 1) {  // sustained: the best DMMA configuration back to back for argv[1] seconds
    const double secs = atof(argv[1]);
    const int grid = sms * 2, threads = 256, it = 200000;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    dmma884_kernel<8><<<grid, threads>>>(d, 10, 1.0000001, 1e-9);
    cudaDeviceSynchronize();
    double total_ms = 0, fl = 0;
    int launches = 0;
    cudaEventRecord(e0);
    while (total_ms < secs * 1e3) {
      for (int k = 0; k < 8; ++k) dmma884_kernel<8><<<grid, threads>>>(d, it, 1.0000001, 1e-9);
      launches += 8;
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      total_ms = ms;
    }
    fl = 2.0 * 256 * 8 * (double)it * grid * (threads / 32) * launches;
    printf("DMMA884 sustained %d launches, %.1f ms: %.2f TFLOP/s\n", launches, total_ms, fl / total_ms / 1e9);
    CK(cudaGetLastError());
    return 0;
  }
  int iters = 20000;
  for (int bpsm : {1, 2, 4}) for (int threads : {128, 256, 512}) {
    int grid = sms * bpsm;
    float ms = timeit(dfma_kernel<8>, grid, threads, iters, d);
    double fl = 2.0 * 8 * iters * (double)grid * threads;
    printf("DFMA      nacc=8  grid=%d thr=%d: %.3f ms  %.2f TFLOP/s\n", grid, threads, ms, fl / ms / 1e9);
  }
  for (int bpsm : {1, 2, 4}) for (int threads : {128, 256, 512}) {
    int grid = sms * bpsm;
    float ms = timeit(dmma884_kernel<8>, grid, threads, iters, d);
    double fl = 2.0 * 256 * 8 * iters * (double)grid * (threads / 32);
    printf("DMMA884   nacc=8  grid=%d thr=%d: %.3f ms  %.2f TFLOP/s\n", grid, threads, ms, fl / ms / 1e9);
  }
  for (int bpsm : {1, 2}) for (int threads : {128, 256}) {
    int grid = sms * bpsm;
    float ms = timeit(dmma884_kernel<16>, grid, threads, iters, d);
    double fl = 2.0 * 256 * 16 * iters * (double)grid * (threads / 32);
    printf("DMMA884   nacc=16 grid=%d thr=%d: %.3f ms  %.2f TFLOP/s\n", grid, threads, ms, fl / ms / 1e9);
  }
  for (int bpsm : {1, 2}) for (int threads : {128, 256, 512}) {
    int grid = sms * bpsm;
    float ms = timeit(dmma16816_kernel<4>, grid, threads, iters / 4, d);
    double fl = 2.0 * 2048 * 4 * (iters / 4) * (double)grid * (threads / 32);
    printf("DMMA16816 nacc=4  grid=%d thr=%d: %.3f ms  %.2f TFLOP/s\n", grid, threads, ms, fl / ms / 1e9);
  }
  {
    int grid = sms * 2, threads = 256;
    float ms0 = timeit(dmma_dmul_kernel<8, 0>, grid, threads, iters, d);
    float ms1 = timeit(dmma_dmul_kernel<8, 2>, grid, threads, iters, d);
    float ms2 = timeit(dmma_dmul_kernel<8, 8>, grid, threads, iters, d);
    float ms3 = timeit(dmma_dmul_kernel<8, 32>, grid, threads, iters, d);
    double fl = 2.0 * 256 * 8 * iters * (double)grid * (threads / 32);
    printf("DMMA+DMUL 8 mma + {0,2,8,32} dmul/iter: %.3f %.3f %.3f %.3f ms (mma-only TF %.2f)\n", ms0, ms1, ms2, ms3, fl / ms0 / 1e9);
  }
  CK(cudaGetLastError());
  return 0;
}
