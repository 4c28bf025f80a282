// Standalone check + timing of the tcgen05 3xTF32 K1 GEMM (paper_2312_08201_b200/csrc/umma.cuh)
// against an FP64 reference on sampled entries, and against three cuBLAS TF32 GEMMs.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo umma_tf32x3.cu -lcublas -o umma_tf32x3
// ./umma_tf32x3 [npad] [ncol] [Kd]
#include <cublas_v2.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include <cuda_fp16.h>

#include "../../paper_2312_08201_b200/csrc/umma.cuh"

#define CK(x)                                                                            \
  do {                                                                                   \
    cudaError_t e = (x);                                                                 \
    if (e != cudaSuccess) {                                                              \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);     \
      exit(1);                                                                           \
    }                                                                                    \
  } while (0)

static float tf32_host(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  u = (u + 0x1000u) & 0xFFFFE000u;
  float r;
  memcpy(&r, &u, 4);
  return r;
}

static CUtensorMap tmap_sw(const void* p, uint64_t inner, uint64_t outer, uint32_t bi, uint32_t bo,
                           CUtensorMapSwizzle sw, int eb = 4);
static CUtensorMap tmap(const float* p, uint64_t inner, uint64_t outer, uint32_t bi, uint32_t bo) {
  return tmap_sw(p, inner, outer, bi, bo, CU_TENSOR_MAP_SWIZZLE_128B);
}
static CUtensorMap tmap_sw(const void* p, uint64_t inner, uint64_t outer, uint32_t bi, uint32_t bo,
                           CUtensorMapSwizzle sw, int eb) {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q));
    fn = (PFN_cuTensorMapEncodeTiled_v12000)f;
  }
  CUtensorMap m;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {inner * (uint64_t)eb};
  cuuint32_t box[2] = {bi, bo};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(&m, eb == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, (void*)p, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    printf("cuTensorMapEncodeTiled failed %d\n", (int)r);
    exit(1);
  }
  return m;
}

int main(int argc, char** argv) {
  const int npad = argc > 1 ? atoi(argv[1]) : 4096;
  const int ncol = argc > 2 ? atoi(argv[2]) : 4864;
  const int Kd = argc > 3 ? atoi(argv[3]) : 4000;
  std::mt19937_64 rng(1);
  std::normal_distribution<double> nd;
  std::vector<double> A((size_t)npad * npad, 0.0), B((size_t)npad * ncol, 0.0);  // A[m][k], B[k][n]
  for (int m = 0; m < npad; ++m)
    for (int k = 0; k < Kd; ++k) A[(size_t)m * npad + k] = nd(rng) / (1.0 + std::abs(m - k));
  for (int k = 0; k < Kd; ++k)
    for (int n = 0; n < ncol; ++n) B[(size_t)k * ncol + n] = nd(rng) * std::pow(10.0, (n % 7) - 3);
  std::vector<float> A32((size_t)npad * 2 * npad), B32((size_t)2 * ncol * npad, 0.f);
  for (int m = 0; m < npad; ++m)
    for (int k = 0; k < npad; ++k) {
      const double x = A[(size_t)m * npad + k];
      const float hi = tf32_host((float)x);
      A32[(size_t)m * 2 * npad + k] = hi;
      A32[(size_t)m * 2 * npad + npad + k] = (float)(x - (double)hi);
    }
  for (int k = 0; k < npad; ++k)
    for (int n = 0; n < ncol; ++n) {
      const double x = B[(size_t)k * ncol + n];
      const float hi = tf32_host((float)x);
      B32[(size_t)(ncol + n) * npad + k] = hi;
      B32[(size_t)n * npad + k] = (float)(x - (double)hi);
    }
  float *dA, *dB, *dU, *dU2;
  CK(cudaMalloc(&dA, A32.size() * 4));
  CK(cudaMalloc(&dB, B32.size() * 4));
  CK(cudaMalloc(&dU, (size_t)ncol * npad * 4));
  CK(cudaMalloc(&dU2, (size_t)ncol * npad * 4));
  CK(cudaMemcpy(dA, A32.data(), A32.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B32.data(), B32.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemset(dU, 0, (size_t)ncol * npad * 4));
  const int Kr = (Kd + 31) / 32 * 32;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int R = 10;
  float ms;
  const double fl = 3.0 * 2.0 * npad * (double)ncol * Kr;
  std::vector<float> U((size_t)ncol * npad);
  CUtensorMap ta = tmap(dA, 2 * (uint64_t)npad, npad, lyap::UM_BK, lyap::UM_BM);
  auto variant = [&](auto kern, int BN, int smem, const char* name) {
    if (ncol % BN) return;
    CUtensorMap tb = tmap(dB, npad, 2 * (uint64_t)ncol, lyap::UM_BK, BN);
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    dim3 grid(ncol / BN, npad / lyap::UM_BM);
    CK(cudaMemset(dU, 0, (size_t)ncol * npad * 4));
    kern<<<grid, 128, smem>>>(ta, tb, dU, npad, ncol, Kr, nullptr, 1);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(U.data(), dU, U.size() * 4, cudaMemcpyDeviceToHost));
    double maxrel = 0;
    std::mt19937_64 r2(5);
    std::uniform_int_distribution<int> um(0, npad - 1), un(0, ncol - 1);
    for (int t = 0; t < 2000; ++t) {
      const int m = um(r2), n = un(r2);
      double ref = 0, mag = 0;
      for (int k = 0; k < Kd; ++k) {
        ref += A[(size_t)m * npad + k] * B[(size_t)k * ncol + n];
        mag += std::abs(A[(size_t)m * npad + k] * B[(size_t)k * ncol + n]);
      }
      maxrel = std::max(maxrel, std::abs(U[(size_t)n * npad + m] - ref) / mag);
    }
    cudaEventRecord(e0);
    for (int r = 0; r < R; ++r) kern<<<grid, 128, smem>>>(ta, tb, dU, npad, ncol, Kr, nullptr, 1);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= R;
    printf("umma %-10s: err/sum|ab| %.2e  %.3f ms  %.1f TFLOP/s (3 passes)\n", name, maxrel, ms, fl / ms * 1e-9);
  };
  variant(lyap::k1_umma_tf32x3<256, 2>, 256, lyap::UmCfg<256, 2>::SMEM, "256x2");
  variant(lyap::k1_umma_tf32x3<128, 3>, 128, lyap::UmCfg<128, 3>::SMEM, "128x3");
  variant(lyap::k1_umma_tf32x3<128, 2>, 128, lyap::UmCfg<128, 2>::SMEM, "128x2");
  variant(lyap::k1_umma_tf32x3<192, 2>, 192, lyap::UmCfg<192, 2>::SMEM, "192x2");
  variant(lyap::k1_umma_tf32x3<64, 4>, 64, lyap::UmCfg<64, 4>::SMEM, "64x4");
  variant(lyap::k1_umma_tf32x3<256, 2>, 256, lyap::UmCfg<256, 2>::SMEM, "256x2");
  auto pvariant = [&](auto kern, int BN, int smem, const char* name, int BK = 32) {
    if (ncol % BN) return;
    const CUtensorMapSwizzle sw = BK == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
    CUtensorMap tb = tmap_sw(dB, npad, 2 * (uint64_t)ncol, BK, BN, sw);
    CUtensorMap ta = tmap_sw(dA, 2 * (uint64_t)npad, npad, BK, lyap::UM_BM, sw);
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const int tiles = (ncol / BN) * (npad / lyap::UM_BM);
    dim3 grid(std::min(nsm, tiles));
    CK(cudaMemset(dU, 0, (size_t)ncol * npad * 4));
    lyap::K1EpiArgs ep{};
    int* tctr = nullptr;
    CK(cudaMalloc(&tctr, 8));
    CK(cudaMemset(tctr, 0, 8));
    kern<<<grid, 192, smem>>>(ta, tb, dU, npad, ncol, Kr, nullptr, 1, ep, tctr, nullptr);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(U.data(), dU, U.size() * 4, cudaMemcpyDeviceToHost));
    double maxrel = 0;
    std::mt19937_64 r2(5);
    std::uniform_int_distribution<int> um(0, npad - 1), un(0, ncol - 1);
    for (int t = 0; t < 2000; ++t) {
      const int m = um(r2), n = un(r2);
      double ref = 0, mag = 0;
      for (int k = 0; k < Kd; ++k) {
        ref += A[(size_t)m * npad + k] * B[(size_t)k * ncol + n];
        mag += std::abs(A[(size_t)m * npad + k] * B[(size_t)k * ncol + n]);
      }
      maxrel = std::max(maxrel, std::abs(U[(size_t)n * npad + m] - ref) / mag);
    }
    cudaEventRecord(e0);
    for (int r = 0; r < R; ++r) kern<<<grid, 192, smem>>>(ta, tb, dU, npad, ncol, Kr, nullptr, 1, ep, tctr, nullptr);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= R;
    printf("persistent %-10s: err/sum|ab| %.2e  %.3f ms  %.1f TFLOP/s (3 passes)\n", name, maxrel, ms, fl / ms * 1e-9);
  };
  pvariant(lyap::k1_umma_persistent<256, 2, 0>, 256, lyap::UmCfg<256, 2>::SMEM, "256x2");
  pvariant(lyap::k1_umma_persistent<128, 3, 0>, 128, lyap::UmCfg<128, 3>::SMEM, "128x3");
  pvariant(lyap::k1_umma_persistent<256, 4, 0, 16>, 256, lyap::UmCfg<256, 4, 16>::SMEM, "256x4 bk16", 16);
  pvariant(lyap::k1_umma_persistent<128, 6, 0, 16>, 128, lyap::UmCfg<128, 6, 16>::SMEM, "128x6 bk16", 16);
  pvariant(lyap::k1_umma_persistent<256, 3, 0, 16>, 256, lyap::UmCfg<256, 3, 16>::SMEM, "256x3 bk16", 16);
  {
    // 3xFP16 with power-of-two scales: A global (max -> 2^14), B per column (max -> 2^13)
    double amax = 0;
    for (double x : A) amax = std::max(amax, std::abs(x));
    const int eA = 14 - (int)std::ceil(std::log2(amax));
    std::vector<__half> A16((size_t)npad * 2 * npad), B16((size_t)2 * ncol * npad);
    std::vector<float> cs(ncol);
    for (int m = 0; m < npad; ++m)
      for (int k = 0; k < npad; ++k) {
        const double x = std::ldexp(A[(size_t)m * npad + k], eA);
        const __half hi = __float2half_rn((float)x);
        A16[(size_t)m * 2 * npad + k] = hi;
        A16[(size_t)m * 2 * npad + npad + k] = __float2half_rn((float)(x - (double)__half2float(hi)));
      }
    for (int n = 0; n < ncol; ++n) {
      double bmax = 1e-300;
      for (int k = 0; k < Kd; ++k) bmax = std::max(bmax, std::abs(B[(size_t)k * ncol + n]));
      const int en = 13 - (int)std::ceil(std::log2(bmax));
      cs[n] = std::ldexp(1.0f, -(eA + en));
      for (int k = 0; k < npad; ++k) {
        const double x = std::ldexp(B[(size_t)k * ncol + n], en);
        const __half hi = __float2half_rn((float)x);
        B16[(size_t)(ncol + n) * npad + k] = hi;
        B16[(size_t)n * npad + k] = __float2half_rn((float)(x - (double)__half2float(hi)));
      }
    }
    __half *dA16, *dB16;
    float* dcs;
    CK(cudaMalloc(&dA16, A16.size() * 2));
    CK(cudaMalloc(&dB16, B16.size() * 2));
    CK(cudaMalloc(&dcs, ncol * 4));
    CK(cudaMemcpy(dA16, A16.data(), A16.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB16, B16.data(), B16.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dcs, cs.data(), ncol * 4, cudaMemcpyHostToDevice));
    auto f16variant = [&](auto kern, int BN, int smem, const char* name) {
      if (ncol % BN) return;
      CUtensorMap ta16 = tmap_sw(dA16, 2 * (uint64_t)npad, npad, 32, lyap::UM_BM, CU_TENSOR_MAP_SWIZZLE_64B, 2);
      CUtensorMap tb16 = tmap_sw(dB16, npad, 2 * (uint64_t)ncol, 32, BN, CU_TENSOR_MAP_SWIZZLE_64B, 2);
      CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      int nsm = 0;
      cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
      dim3 grid(std::min(nsm, (ncol / BN) * (npad / lyap::UM_BM)));
      int* tctr = nullptr;
      CK(cudaMalloc(&tctr, 8));
      CK(cudaMemset(tctr, 0, 8));
      lyap::K1EpiArgs ep{};
      CK(cudaMemset(dU, 0, (size_t)ncol * npad * 4));
      kern<<<grid, 192, smem>>>(ta16, tb16, dU, npad, ncol, Kr, nullptr, 1, ep, tctr, dcs);
      CK(cudaGetLastError());
      CK(cudaDeviceSynchronize());
      CK(cudaMemcpy(U.data(), dU, U.size() * 4, cudaMemcpyDeviceToHost));
      double maxrel = 0;
      std::mt19937_64 r2(5);
      std::uniform_int_distribution<int> um(0, npad - 1), un(0, ncol - 1);
      for (int t = 0; t < 2000; ++t) {
        const int m = um(r2), n = un(r2);
        double ref = 0, mag = 0;
        for (int k = 0; k < Kd; ++k) {
          ref += A[(size_t)m * npad + k] * B[(size_t)k * ncol + n];
          mag += std::abs(A[(size_t)m * npad + k] * B[(size_t)k * ncol + n]);
        }
        maxrel = std::max(maxrel, std::abs(U[(size_t)n * npad + m] - ref) / mag);
      }
      cudaEventRecord(e0);
      for (int r = 0; r < R; ++r) kern<<<grid, 192, smem>>>(ta16, tb16, dU, npad, ncol, Kr, nullptr, 1, ep, tctr, dcs);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
      ms /= R;
      printf("persistent f16 %-10s: err/sum|ab| %.2e  %.3f ms  %.1f TFLOP/s (3 passes)\n", name, maxrel, ms, fl / ms * 1e-9);
    };
    f16variant(lyap::k1_umma_persistent<256, 4, 0, 32, 2>, 256, lyap::UmCfg<256, 4, 32, 2>::SMEM, "256x4 bk32");
    f16variant(lyap::k1_umma_persistent<128, 6, 0, 32, 2>, 128, lyap::UmCfg<128, 6, 32, 2>::SMEM, "128x6 bk32");
  }
  // cuBLAS: three TF32 GEMMs (column-major C (npad x ncol, ld npad) = A^T(op T) * Bt)
  cublasHandle_t h;
  cublasCreate(&h);
  const float one = 1.f, zero = 0.f;
  auto cub = [&]() {
    cublasGemmEx(h, CUBLAS_OP_T, CUBLAS_OP_N, npad, ncol, Kr, &one, dA, CUDA_R_32F, 2 * npad, dB, CUDA_R_32F, npad, &zero,
                 dU2, CUDA_R_32F, npad, CUBLAS_COMPUTE_32F_FAST_TF32, CUBLAS_GEMM_DEFAULT);
    cublasGemmEx(h, CUBLAS_OP_T, CUBLAS_OP_N, npad, ncol, Kr, &one, dA + npad, CUDA_R_32F, 2 * npad,
                 dB + (size_t)ncol * npad, CUDA_R_32F, npad, &one, dU2, CUDA_R_32F, npad, CUBLAS_COMPUTE_32F_FAST_TF32,
                 CUBLAS_GEMM_DEFAULT);
    cublasGemmEx(h, CUBLAS_OP_T, CUBLAS_OP_N, npad, ncol, Kr, &one, dA, CUDA_R_32F, 2 * npad, dB + (size_t)ncol * npad,
                 CUDA_R_32F, npad, &one, dU2, CUDA_R_32F, npad, CUBLAS_COMPUTE_32F_FAST_TF32, CUBLAS_GEMM_DEFAULT);
  };
  cub();
  CK(cudaDeviceSynchronize());
  cudaEventRecord(e0);
  for (int r = 0; r < R; ++r) cub();
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= R;
  printf("cublas 3 x tf32: %.3f ms  %.1f TFLOP/s (3 passes)\n", ms, fl / ms * 1e-9);
  std::vector<float> U2((size_t)ncol * npad);
  CK(cudaMemcpy(U2.data(), dU2, U2.size() * 4, cudaMemcpyDeviceToHost));
  double d = 0, nrm = 0;
  for (size_t i = 0; i < U.size(); ++i) {
    d = std::max(d, (double)std::abs(U[i] - U2[i]));
    nrm = std::max(nrm, (double)std::abs(U2[i]));
  }
  printf("last umma vs cublas: max diff %.3e (max |U| %.3e)\n", d, nrm);
  return 0;
}
