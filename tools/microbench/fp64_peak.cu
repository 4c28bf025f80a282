// FP64 throughput microbenchmark for sm_100a: DFMA vs DMMA (mma.sync .f64 shapes).
// Used once to pick the K1 inner-product engine; numbers go to profiles/.
#include <cstdio>
#include <cuda_runtime.h>

#define ITERS 4096

__global__ void dfma_kernel(double* out, double a, double b) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 1234.5) out[threadIdx.x] = s;
}

__global__ void dmma_m8n8k4(double* out) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[4][2] = {};
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int j = 0; j < 4; ++j) s += c[j][0] + c[j][1];
  if (s == 1234.5) out[threadIdx.x] = s;
}

__global__ void dmma_m16n8k4(double* out) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, b = 1.0 + threadIdx.x * 1e-4;
  double c[4][4] = {};
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                   : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3]) : "d"(a0), "d"(a1), "d"(b));
  }
  double s = 0;
  for (int j = 0; j < 4; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  if (s == 1234.5) out[threadIdx.x] = s;
}

__global__ void dmma_m16n8k8(double* out) {
  double a[4], b[2];
  for (int i = 0; i < 4; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int i = 0; i < 2; ++i) b[i] = 1.0 + threadIdx.x * 1e-4 + i;
  double c[4][4] = {};
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
  }
  double s = 0;
  for (int j = 0; j < 4; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  if (s == 1234.5) out[threadIdx.x] = s;
}

__global__ void dmma_m16n8k16(double* out) {
  double a[8], b[4];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int i = 0; i < 4; ++i) b[i] = 1.0 + threadIdx.x * 1e-4 + i;
  double c[4][4] = {};
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
  for (int j = 0; j < 4; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  if (s == 1234.5) out[threadIdx.x] = s;
}

template <typename F>
float timeit(F f) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  f(); cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0); f(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  return best;
}

int main() {
  double* out; cudaMalloc(&out, 1024 * sizeof(double));
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int bpsm : {1, 2, 4}) {
    for (int threads : {256, 512}) {
      int grid = sms * bpsm;
      double tot_thr = (double)grid * threads;
      float ms = timeit([&] { dfma_kernel<<<grid, threads>>>(out, 1.0000001, 1e-9); });
      printf("DFMA   grid=%d thr=%d : %.2f TFLOP/s\n", grid, threads, tot_thr * ITERS * 8 * 2 / (ms * 1e-3) / 1e12);
      double warps = tot_thr / 32;
      ms = timeit([&] { dmma_m8n8k4<<<grid, threads>>>(out); });
      printf("m8n8k4  grid=%d thr=%d : %.2f TFLOP/s\n", grid, threads, warps * ITERS * 4 * (8 * 8 * 4) * 2 / (ms * 1e-3) / 1e12);
      ms = timeit([&] { dmma_m16n8k4<<<grid, threads>>>(out); });
      printf("m16n8k4 grid=%d thr=%d : %.2f TFLOP/s\n", grid, threads, warps * ITERS * 4 * (16 * 8 * 4) * 2 / (ms * 1e-3) / 1e12);
      ms = timeit([&] { dmma_m16n8k8<<<grid, threads>>>(out); });
      printf("m16n8k8 grid=%d thr=%d : %.2f TFLOP/s\n", grid, threads, warps * ITERS * 4 * (16 * 8 * 8) * 2 / (ms * 1e-3) / 1e12);
      ms = timeit([&] { dmma_m16n8k16<<<grid, threads>>>(out); });
      printf("m16n8k16 grid=%d thr=%d : %.2f TFLOP/s\n", grid, threads, warps * ITERS * 4 * (16 * 8 * 16) * 2 / (ms * 1e-3) / 1e12);
    }
  }
  cudaError_t e = cudaGetLastError();
  printf("err: %s\n", cudaGetErrorString(e));
  return 0;
}
