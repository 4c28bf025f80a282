// Launch cost of a mostly-early-exit kernel vs its dynamic shared-memory reservation (k_backsub shape)
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_exit(const int* phase, double* out, int smem_doubles) {
  extern __shared__ double sm[];
  const int slot = blockIdx.x;
  if (phase[slot] != 3) return;
  sm[threadIdx.x] = threadIdx.x;
  __syncthreads();
  out[slot] = sm[(threadIdx.x + 1) % blockDim.x] + smem_doubles;
}
__global__ void k_exit_gs(const int* phase, double* out, int nslot) {
  extern __shared__ double sm[];
  for (int slot = blockIdx.x; slot < nslot; slot += gridDim.x) {
    if (phase[slot] != 3) continue;
    sm[threadIdx.x] = threadIdx.x;
    __syncthreads();
    out[slot] = sm[(threadIdx.x + 1) % blockDim.x];
    __syncthreads();
  }
}
int main() {
  const int nslot = 512;
  int* ph; double* out;
  cudaMalloc(&ph, nslot * 4); cudaMalloc(&out, nslot * 8);
  cudaMemset(ph, 0, nslot * 4);
  cudaFuncSetAttribute(k_exit, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaFuncSetAttribute(k_exit_gs, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  size_t sizes[] = {0, 8 * 1024, 48 * 1024, 104 * 1024, 200 * 1024};
  for (size_t s : sizes) {
    for (int w = 0; w < 10; ++w) k_exit<<<nslot, 256, s>>>(ph, out, (int)s);
    cudaEventRecord(a);
    for (int w = 0; w < 100; ++w) k_exit<<<nslot, 256, s>>>(ph, out, (int)s);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("grid %d smem %6zu B: %.2f us/launch\n", nslot, s, ms * 10.f);
  }
  for (size_t s : sizes) {
    for (int w = 0; w < 10; ++w) k_exit_gs<<<148, 256, s>>>(ph, out, nslot);
    cudaEventRecord(a);
    for (int w = 0; w < 100; ++w) k_exit_gs<<<148, 256, s>>>(ph, out, nslot);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("grid 148 (grid-stride) smem %6zu B: %.2f us/launch\n", s, ms * 10.f);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
