// FP64 throughput microbenchmark for B200 (sm_100a): DFMA (FP64 pipe) vs
// DMMA (mma.sync .f64 tensor path, shapes m8n8k4 / m16n8k4 / m16n8k8 /
// m16n8k16). Each thread runs independent accumulator chains so the number is
// a throughput ceiling, not a latency. Output: one line per variant,
// TFLOP/s = 2 * FMAs / time (CUDA events, best of 5).
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CHECK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

constexpr int ITERS = 4096;

__global__ void dfma_kernel(double* out, double a, double b) {
  double acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += acc[i];
  if (s == 1234.5) out[0] = s;
}

__global__ void dmma884_kernel(double* out, double a0, double b0) {
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = threadIdx.x; c[i][1] = i; }
  double a = a0 + threadIdx.x * 1e-12, b = b0;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 1234.5) out[0] = s;
}

__global__ void dmma1684_kernel(double* out, double a0, double b0) {
  double c[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i) for (int j = 0; j < 4; ++j) c[i][j] = threadIdx.x + j;
  double a = a0 + threadIdx.x * 1e-12, a1 = a0 * 0.5, b = b0;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a), "d"(a1), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 1234.5) out[0] = s;
}

__global__ void dmma1688_kernel(double* out, double a0, double b0) {
  double c[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i) for (int j = 0; j < 4; ++j) c[i][j] = threadIdx.x + j;
  double a[4] = {a0, a0 * 0.5, a0 * 0.25, a0 + threadIdx.x * 1e-12}, b[2] = {b0, b0 * 0.5};
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 1234.5) out[0] = s;
}

__global__ void dmma16816_kernel(double* out, double a0, double b0) {
  double c[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i) for (int j = 0; j < 4; ++j) c[i][j] = threadIdx.x + j;
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = a0 * (1.0 + i * 1e-3) + threadIdx.x * 1e-12;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = b0 * (1.0 + i * 1e-3);
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 1234.5) out[0] = s;
}

template <typename K>
static float time_kernel(K kern, int blocks, int threads, double* out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  kern<<<blocks, threads>>>(out, 0.999, 1e-3);  // warm-up
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    kern<<<blocks, threads>>>(out, 0.999, 1e-3);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int dev = 0, sms = 0;
  CHECK(cudaGetDevice(&dev));
  CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  double* out;
  CHECK(cudaMalloc(&out, 64));
  for (int bpsm : {1, 2, 4}) {
    const int blocks = sms * bpsm, threads = 256;
    const double nthreads = double(blocks) * threads;
    float ms = time_kernel(dfma_kernel, blocks, threads, out);
    printf("{\"variant\": \"dfma\", \"blocks_per_sm\": %d, \"tflops\": %.3f}\n", bpsm,
           2.0 * nthreads * ITERS * 16 / (ms * 1e-3) / 1e12);
    const double nwarps = nthreads / 32;
    ms = time_kernel(dmma884_kernel, blocks, threads, out);
    printf("{\"variant\": \"dmma_m8n8k4\", \"blocks_per_sm\": %d, \"tflops\": %.3f}\n", bpsm,
           2.0 * nwarps * ITERS * 8 * 256 / (ms * 1e-3) / 1e12);
    ms = time_kernel(dmma1684_kernel, blocks, threads, out);
    printf("{\"variant\": \"dmma_m16n8k4\", \"blocks_per_sm\": %d, \"tflops\": %.3f}\n", bpsm,
           2.0 * nwarps * ITERS * 8 * 512 / (ms * 1e-3) / 1e12);
    ms = time_kernel(dmma1688_kernel, blocks, threads, out);
    printf("{\"variant\": \"dmma_m16n8k8\", \"blocks_per_sm\": %d, \"tflops\": %.3f}\n", bpsm,
           2.0 * nwarps * ITERS * 8 * 1024 / (ms * 1e-3) / 1e12);
    ms = time_kernel(dmma16816_kernel, blocks, threads, out);
    printf("{\"variant\": \"dmma_m16n8k16\", \"blocks_per_sm\": %d, \"tflops\": %.3f}\n", bpsm,
           2.0 * nwarps * ITERS * 8 * 2048 / (ms * 1e-3) / 1e12);
  }
  cudaError_t e = cudaGetLastError();
  printf("{\"status\": \"%s\"}\n", cudaGetErrorString(e));
  return 0;
}
