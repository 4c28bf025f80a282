// lyapgpu — C-ABI implementation (include/lyapgpu.h).  One translation unit: the kernels live in
// the .cuh files next to this one; this file holds the host control (setup flow, engine loop).
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cusolverDn.h>

#include <algorithm>
#include <cmath>
#include <limits>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/lyapgpu.h"
#include "common.cuh"
#include "ctx.h"
#include "engine.cuh"
#include "k1.cuh"
#include "umma.cuh"
#include "sched.cuh"
#include "stab.cuh"
#include "setup.cuh"

using namespace lyap;

namespace {

thread_local std::string g_last_error = "no error";

struct Fail {
  int code;
};

void set_err(lyap_ctx* c, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
  if (c) c->err = buf;
}

#define CK(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess) {                                                              \
      set_err(ctx, "%s:%d %s: %s", __FILE__, __LINE__, #call, cudaGetErrorString(e_));    \
      throw Fail{e_ == cudaErrorMemoryAllocation ? LYAP_ENOMEM : LYAP_ECUDA};             \
    }                                                                                     \
  } while (0)
#define CKB(call)                                                                         \
  do {                                                                                    \
    cublasStatus_t e_ = (call);                                                           \
    if (e_ != CUBLAS_STATUS_SUCCESS) {                                                    \
      set_err(ctx, "%s:%d %s: cublas status %d", __FILE__, __LINE__, #call, (int)e_);     \
      throw Fail{LYAP_ECUDA};                                                             \
    }                                                                                     \
  } while (0)
#define CKS(call)                                                                         \
  do {                                                                                    \
    cusolverStatus_t e_ = (call);                                                         \
    if (e_ != CUSOLVER_STATUS_SUCCESS) {                                                  \
      set_err(ctx, "%s:%d %s: cusolver status %d", __FILE__, __LINE__, #call, (int)e_);   \
      throw Fail{LYAP_ECUDA};                                                             \
    }                                                                                     \
  } while (0)
#define LAUNCHED()                      \
  do {                                  \
    CK(cudaGetLastError());             \
    ctx->stats.kernel_launches++;       \
  } while (0)

template <typename T>
T* dalloc(lyap_ctx* ctx, size_t count, bool zero = true) {
  void* p = nullptr;
  CK(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)));
  if (zero) CK(cudaMemset(p, 0, std::max<size_t>(count, 1) * sizeof(T)));
  return static_cast<T*>(p);
}
void dfree(void* p) {
  if (p) cudaFree(p);
}

int64_t roundup(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

// K1 GEMM configuration
#ifndef SMALL_BK
#define SMALL_BK 16
#endif
// large n: 128 x 128 CTA tiles (8 warps of 64 x 32), one CTA per SM
constexpr int G_BM = 128, G_BN = 128, G_WM = 64, G_WN = 32, G_ST = 3, G_BK = 32;
using GCfg = DgemmCfg<G_BM, G_BN, G_WM, G_WN, G_ST, G_BK>;
// small n (<= SMALL_N): 64 x 64 tiles (4 warps of 32 x 32), several CTAs per SM -> less padding
// and finer wave quantisation
constexpr int S_BM = 64, S_BN = 64, S_WM = 32, S_WN = 32, S_ST = 3, S_BK = SMALL_BK;
using SCfg = DgemmCfg<S_BM, S_BN, S_WM, S_WN, S_ST, S_BK>;
constexpr int64_t SMALL_N = 1536;
// VERIFY-only DMMA GEMM of the mixed-precision path (few columns): 64 x 32 tiles, 4 warps of 32 x 16
constexpr int V_BM = 64, V_BN = 32, V_WM = 32, V_WN = 16, V_ST = 3, V_BK = 16;
inline int tile_m(const Seed& s) { return s.n <= SMALL_N ? S_BM : G_BM; }
inline int tile_n(const Seed& s) { return s.n <= SMALL_N ? S_BN : G_BN; }

#define K_DISPATCH(KV, ...)     \
  switch (KV) {                  \
    case 1: { constexpr int KK = 1; __VA_ARGS__; } break; \
    case 2: { constexpr int KK = 2; __VA_ARGS__; } break; \
    case 3: { constexpr int KK = 3; __VA_ARGS__; } break; \
    case 4: { constexpr int KK = 4; __VA_ARGS__; } break; \
    case 5: { constexpr int KK = 5; __VA_ARGS__; } break; \
    case 6: { constexpr int KK = 6; __VA_ARGS__; } break; \
    case 7: { constexpr int KK = 7; __VA_ARGS__; } break; \
    case 8: { constexpr int KK = 8; __VA_ARGS__; } break; \
    default: break;              \
  }

// device scratch of the scheduler: [0, k) cost weights, [8, 8 + 2k) bounding box, [32, ...) the log
// seeds of the recycle regimes (nreg x k <= 2^KMAX x KMAX)
constexpr size_t DWORK_SEEDS = 32;
void ensure_dwork(lyap_ctx* ctx) {
  Seed& sd = ctx->seed;
  if (sd.dwork) return;
  sd.dwork = dalloc<double>(ctx, DWORK_SEEDS + ((size_t)1 << LYAP_KMAX) * LYAP_KMAX);
  CK(cudaMemcpy(sd.dwork, sd.wcost, sizeof(double) * sd.k, cudaMemcpyHostToDevice));
}
void upload_seeds(lyap_ctx* ctx) {
  ensure_dwork(ctx);
  if (!ctx->reg_seeds.empty())
    CK(cudaMemcpy(ctx->seed.dwork + DWORK_SEEDS, ctx->reg_seeds.data(), ctx->reg_seeds.size(), cudaMemcpyHostToDevice));
}

// ------------------------------------------------------------------ engine allocation
void free_engine(Engine& g, bool keep_order = true) {
  void* ps[] = {g.Bop, g.U, g.Bop32, g.U32, g.umctr, g.xmax, g.bmax, g.colscale, g.Xin, g.X, g.Qb, g.Qf, g.Minv, g.sigma, g.mask, g.eta, g.H, g.e, g.y,
                g.bnorm, g.part, g.part3, g.phase, g.m, g.vidx, g.applies, g.restarts, g.ctrl,
                g.part2, g.Gq, g.cf, g.Hraw, g.rhs, g.t0s, g.Zb, g.Rbuf, g.Yz, g.Cc, g.Wc, g.Einv};
  for (void* p : ps) dfree(p);
  if (g.h_ctrl) cudaFreeHost(g.h_ctrl);
  int* order = g.order;
  int* regq = g.regq;
  const int64_t cap = g.order_cap, rcap = g.regq_cap;
  double *skey = g.skey, *skey2 = g.skey2;
  int* sidx = g.sidx;
  void* cub_tmp = g.cub_tmp;
  const size_t cub_bytes = g.cub_bytes;
  const int64_t scap = g.sched_cap;
  if (!keep_order) {
    dfree(order);
    dfree(regq);
    dfree(skey);
    dfree(skey2);
    dfree(sidx);
    dfree(cub_tmp);
  }
  g = Engine{};
  if (keep_order) {
    g.order = order;
    g.regq = regq;
    g.order_cap = cap;
    g.regq_cap = rcap;
    g.skey = skey;
    g.skey2 = skey2;
    g.sidx = sidx;
    g.cub_tmp = cub_tmp;
    g.cub_bytes = cub_bytes;
    g.sched_cap = scap;
  }
}

int mp_mode(const lyap_ctx* ctx);
int auto_mmax(const lyap_ctx* ctx);
int auto_batch(const lyap_ctx* ctx, int64_t nv) {
  const Seed& s = ctx->seed;
  int b = ctx->opts.batch;
  if (b <= 0) {
    // two slot groups, each aiming for ~8 waves of K1 tiles (16 for the small-tile config) on 148
    // SMs, but at least ~4 v per slot so the cost-ordered queue can balance the slots
    // Mixed precision (one slot group, every kernel of an iteration fills the GPU): wider batches amortise
    // the per-iteration latency and the tile tails of both GEMMs; measured on c5 (tools/gpu_smallshard.sh):
    // 4096 v: b = 448 / 592 / 768 / 1024 -> 1108 / 1082 / 1049 / 1037 ms; a 512-v shard: b = 128 / 256 / 384 ->
    // 208 / 196 / 204 ms.  Hence up to 1024 slots and at least 256 (or all v).
    const bool mp = mp_mode(ctx) != 0;
    const int64_t mt = s.npad / tile_m(s);
    const int64_t waves = (s.n <= SMALL_N || mp) ? 16 * 148 : 8 * 148;
    const int64_t target_cols = (waves + mt - 1) / mt * tile_n(s);
    const int64_t per_group = std::max<int64_t>(32, std::min<int64_t>(1024, target_cols / (s.k * s.k)));
    b = (int)std::min<int64_t>(2 * per_group, std::max<int64_t>(mp ? 256 : 64, nv / 4));
    // HBM budget: the Krylov basis ((mmax + 1) vectors of L elements per slot, FP32 under mixed precision)
    // dominates; with the per-slot operands, iterates and preconditioner blocks (~80 L bytes) the engine
    // takes at most 70 % of the memory that is free now or already held by this context's engine
    // (queried only when the estimate exceeds 16 GB: small problems never pay for the query)
    size_t fr = 0, tot = 0;
    const double L = (double)s.npad * s.k;
    const double per_slot = (auto_mmax(ctx) + 1) * L * (mp ? 4.0 : 8.0) + 80.0 * L;
    if (b * per_slot > 16e9 && b > ctx->eng.bcap && cudaMemGetInfo(&fr, &tot) == cudaSuccess) {
      const double held = (double)ctx->eng.bcap * per_slot;
      const int64_t cap = (int64_t)(0.7 * ((double)fr + held) / per_slot);
      if (cap >= 1 && b > cap) b = (int)cap;
    }
  }
  b = (int)std::min<int64_t>(b, std::max<int64_t>(nv, 1));
  b = std::max(1, std::min(b, 2048));  // <= 1024 per slot group (k_assign is one block)
  return b;
}

int auto_mmax(const lyap_ctx* ctx) {
  if (ctx->opts.max_dim > 0) return std::min(ctx->opts.max_dim, 32 * CTRL_RMAX);
  // long cycles where the T-apply dominates (restarts cost iterations: c5 224 vs 160 -> +20 % v/s),
  // shorter where the HBM-bound orthogonalisation does
  return ctx->seed.n * ctx->seed.k >= 12000 ? 384 : 160;
}

int engine_groups(int b, int mp = 0) {
  // FP64: two slot groups, so one group's DMMA GEMM overlaps the other's HBM-bound Krylov kernels.
  // Mixed precision: the tcgen05 GEMM is short and every kernel fills the GPU, so the groups only
  // interleave; one group (up to 1024 slots, k_assign is one block) measured 2375 -> 2420 v/s on c5.
  int G = mp ? (b + 1023) / 1024 : (b >= 64 ? 2 : 1);
  if (const char* ev = std::getenv("LYAP_GROUPS")) G = std::max(1, std::min(4, std::atoi(ev)));  // experiments
  return std::max(1, std::min(G, b / 32));  // every group keeps >= 32 slots
}

// Sets the run shape (slots b, slot groups, K1 columns per group) of an allocated engine.
// K1 GEMM column tile: the tcgen05 mixed-precision GEMM takes 256 columns per CTA
int64_t col_tile(const Seed& s, int mp) { return mp ? 256 : (s.n <= SMALL_N ? S_BN : G_BN); }
void configure_run(const Seed& s, Engine& g, int b) {
  g.b = b;
  g.groups = engine_groups(b, g.mp);
  g.ncol = roundup((int64_t)((b + g.groups - 1) / g.groups) * s.k * s.k, col_tile(s, g.mp));
}

// The engine is allocated for a capacity of bcap slots and reused by any later call that needs
// b <= bcap slots with the same restart length (NEXT row f3: optimizer-style callers change nv on
// every call; reallocating the multi-GB Krylov basis each time dominated their run time).
int coarse_size(const lyap_ctx* ctx);
void ensure_coarse(lyap_ctx* ctx);

// Mixed-precision iterative refinement (opts.mixed): 0 off, 1 3xTF32 (operands split
// hi + lo, two cuBLAS TF32 GEMMs), 2 one float plane with the cuBLAS compute type LYAP_MP_GEMM names
// (bf16x9 | tf32 | fp32: measurement alternatives).
int mp_mode(const lyap_ctx* ctx) {
  const int o = ctx->opts.mixed;
  if (!(o > 0 || (o < 0 && ctx->seed.n > SMALL_N))) return 0;
  const char* ev = std::getenv("LYAP_MP_GEMM");
  const bool plane = ev && (!std::strcmp(ev, "bf16x9") || !std::strcmp(ev, "tf32") || !std::strcmp(ev, "fp32"));
  if (plane) return 2;
  // 3xFP16 on the tcgen05 kernel (mode 3) needs npad % 128 == 0; LYAP_MP_GEMM=tf32x3 / cublas: 3xTF32
  const bool f16 = !(ev && (!std::strcmp(ev, "tf32x3") || !std::strcmp(ev, "cublas")));
  return (f16 && ctx->seed.npad % 128 == 0) ? 3 : 1;
}
// the 3xTF32 product runs on the repo's tcgen05 kernel (umma.cuh); LYAP_MP_GEMM=cublas: three cuBLAS
// TF32 GEMMs instead (measurement alternative)
bool mp_umma() {
  const char* ev = std::getenv("LYAP_MP_GEMM");
  return !(ev && std::strcmp(ev, "cublas") == 0);
}
// UMMA column tile (LYAP_UM_BN=128: the 128 x 128, 3-stage configuration; measurement alternative)
int um_bn() {
  static const int bn = [] {
    const char* ev = std::getenv("LYAP_UM_BN");
    return (ev && std::atoi(ev) == 128) ? 128 : UM_BN;
  }();
  return bn;
}
CUtensorMap make_tmap_f32(lyap_ctx* ctx, const void* p, uint64_t inner, uint64_t outer, uint32_t box_inner,
                          uint32_t box_outer, int eb = 4) {
  // the swizzle spans one box row: 128 B or 64 B (must match the UMMA descriptors); eb = element bytes
  const CUtensorMapSwizzle sw = box_inner * eb == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q));
    if (!f || q != cudaDriverEntryPointSuccess) {
      set_err(ctx, "cuTensorMapEncodeTiled unavailable");
      throw Fail{LYAP_ECUDA};
    }
    encode = (PFN_cuTensorMapEncodeTiled_v12000)f;
  }
  CUtensorMap m;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {inner * (uint64_t)eb};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t es[2] = {1, 1};
  if (encode(&m, eb == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, (void*)p, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
      CUDA_SUCCESS) {
    set_err(ctx, "cuTensorMapEncodeTiled failed");
    throw Fail{LYAP_ECUDA};
  }
  return m;
}
cublasComputeType_t mp_compute(int mode) {
  if (mode == 1) return CUBLAS_COMPUTE_32F_FAST_TF32;
  const char* ev = std::getenv("LYAP_MP_GEMM");
  if (ev && std::strcmp(ev, "bf16x9") == 0) return CUBLAS_COMPUTE_32F_EMULATED_16BFX9;
  if (ev && std::strcmp(ev, "tf32") == 0) return CUBLAS_COMPUTE_32F_FAST_TF32;
  return CUBLAS_COMPUTE_32F;
}
// float planes of the folded Cauchy matrix for the mixed-precision GEMM (once per seed basis)
void ensure_lf32(lyap_ctx* ctx, int mode) {
  Basis& B = *ctx->basis;
  if (B.Lf32 && B.lf32_mode == mode) return;
  if (B.Lf32) cudaFree(B.Lf32);
  B.Lf32 = nullptr;
  const int64_t np = ctx->seed.npad;
  B.Lf32 = dalloc<float>(ctx, (size_t)np * 2 * np, false);
  B.lf32_mode = mode;
  if (mode == 3) {  // 3xFP16: one power-of-two scale for all of Lf (max |Lf| -> 2^14)
    float* dmax = dalloc<float>(ctx, 1);
    k_absmax<<<1, 1024, 0, ctx->stream>>>(B.Lf, np * np, dmax);
    LAUNCHED();
    float hmax = 0.f;
    CK(cudaMemcpyAsync(&hmax, dmax, sizeof(float), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    dfree(dmax);
    B.lf_eA = hmax > 0.f ? 14 - (int)std::ceil(std::log2((double)hmax)) : 0;
    k_split_Lf16<<<1184, 256, 0, ctx->stream>>>(B.Lf, np, B.lf_eA, reinterpret_cast<__half*>(B.Lf32));
  } else if (mode == 1) {
    k_split_Lf<1><<<1184, 256, 0, ctx->stream>>>(B.Lf, np, B.Lf32);
  } else {
    k_split_Lf<2><<<1184, 256, 0, ctx->stream>>>(B.Lf, np, B.Lf32);
  }
  LAUNCHED();
}

void ensure_engine(lyap_ctx* ctx, int b, int mmax) {
  Engine& g = ctx->eng;
  const Seed& s = ctx->seed;
  const int pc = ctx->coarse.p;
  const int mp = mp_mode(ctx);
  if ((g.Qb || g.Qf) && g.mmax == mmax && g.bcap >= b && g.pc == pc && g.mp == mp) {
    configure_run(s, g, b);
    return;
  }
  free_engine(g);
  g.bcap = b;
  g.mmax = mmax;
  g.mp = mp;
  g.L = s.k * s.npad;
  // K1 operand columns for any run b' <= b and any group count (sum over groups of the rounded
  // per-group widths)
  int64_t colcap = 0;
  for (int G = 1; G <= 4; ++G)
    colcap = std::max<int64_t>(colcap, G * roundup((int64_t)((b + G - 1) / G) * s.k * s.k, col_tile(s, mp)));
  configure_run(s, g, b);
  g.nchunk = (int)((g.L + RED_CE - 1) / RED_CE);
  g.Bop = dalloc<double>(ctx, (size_t)s.npad * colcap);
  g.U = dalloc<double>(ctx, (size_t)s.npad * colcap);
  if (mp) {
    g.Bop32 = dalloc<float>(ctx, (size_t)2 * s.npad * colcap);
    g.U32 = dalloc<float>(ctx, (size_t)s.npad * colcap);
    g.umctr = dalloc<int>(ctx, 8);  // tile counters of the persistent tcgen05 GEMM (2 per slot group), zeroed
    if (mp == 3) {
      g.xmax = dalloc<float>(ctx, (size_t)b * s.k);
      g.bmax = dalloc<float>(ctx, s.k);
      g.colscale = dalloc<float>(ctx, (size_t)colcap);
      k_bmax<<<(unsigned)s.k, 256, 0, ctx->stream>>>(s.bhr, s.npad, (int)s.k, (int)(2 * s.npairs), g.bmax);
      LAUNCHED();
    }
  }
  g.Xin = dalloc<double>(ctx, (size_t)b * g.L);
  g.X = dalloc<double>(ctx, (size_t)b * g.L);
  if (mp)  // mixed precision: FP32 Krylov basis
    g.Qf = dalloc<float>(ctx, (size_t)b * (mmax + 1) * g.L);
  else
    g.Qb = dalloc<double>(ctx, (size_t)b * (mmax + 1) * g.L);
  g.Minv = dalloc<float>(ctx, (size_t)b * s.nrep * s.k * s.k * 4);
  g.sigma = dalloc<double>(ctx, (size_t)b * s.k);
  g.mask = dalloc<double>(ctx, (size_t)b * s.k);
  g.eta = dalloc<double>(ctx, (size_t)b * (mmax + 1));
  g.H = dalloc<double>(ctx, (size_t)b * (mmax + 1) * mmax);
  g.e = dalloc<double>(ctx, (size_t)b * (mmax + 1) + 2 * (size_t)b * mmax);  // e | cs | sn (b x mmax each)
  g.y = dalloc<double>(ctx, (size_t)b * mmax);
  g.bnorm = dalloc<double>(ctx, b);
  g.part = dalloc<double>(ctx, (size_t)b * (mmax + 2) * g.nchunk);
  g.part3 = dalloc<double>(ctx, (size_t)b * g.nchunk * 3);
  g.part2 = dalloc<double>(ctx, (size_t)b * (mmax + 2) * g.nchunk);
  g.Gq = dalloc<double>(ctx, (size_t)b * (mmax + 1) * (mmax + 1));
  g.cf = dalloc<double>(ctx, (size_t)b * (mmax + 1));
  g.Hraw = dalloc<double>(ctx, (size_t)b * (mmax + 1) * mmax);
  if (s.qlin) {  // per-slot right-hand side G0(v) and t0(v) of a v-linear Q
    g.rhs = dalloc<double>(ctx, (size_t)b * g.L);
    g.t0s = dalloc<double>(ctx, b);
  }
  g.pc = pc;
  if (pc > 0) {  // two-level preconditioner: flexible basis and coarse scratch
    g.Zb = dalloc<double>(ctx, (size_t)b * (mmax + 1) * g.L, false);
    g.Rbuf = dalloc<double>(ctx, (size_t)b * g.L);
    g.Yz = dalloc<double>(ctx, (size_t)b * 2 * g.L);  // per slot [Z w; T Z w]
    g.Cc = dalloc<double>(ctx, (size_t)b * pc);
    g.Wc = dalloc<double>(ctx, (size_t)b * pc);
    g.Einv = dalloc<double>(ctx, (size_t)b * pc * pc);
  }
  g.phase = dalloc<int>(ctx, b);
  g.m = dalloc<int>(ctx, b);
  g.vidx = dalloc<int>(ctx, b);
  g.applies = dalloc<int>(ctx, b);
  g.restarts = dalloc<int>(ctx, 5 * (size_t)b);  // restarts | newv | alist | su | reg
  g.ctrl = dalloc<int>(ctx, 8 * 5);               // up to 4 groups + the shared block
  CK(cudaMallocHost(&g.h_ctrl, 8 * 5 * sizeof(int)));
  ctx->info.max_dim = mmax;
}

// ------------------------------------------------------------------ K1 launch (prologue, GEMM, epilogue)

// K1 with the epilogue fused into the GEMM (k = 1, 2, 4: a slot's k^2 columns never straddle a CTA
// tile) for the small-tile configuration (n <= SMALL_N): prologue + one GEMM launch.  Otherwise
// prologue, GEMM, k1_epi.  Measured (bench, B200): c2 94.5k -> 96.0k v/s fused; c5 907.9 -> 898.9
// fused -- with 1 CTA per SM the large-tile GEMM runs the epilogue at 8 warps per SM, slower than
// the separate, fully occupied k1_epi, so the large configuration keeps it separate.
inline bool k1_fused(int64_t k, int64_t n, int mp = 0) { return (k == 1 || k == 2 || k == 4) && n <= SMALL_N && !mp; }

template <int BM, int BN, int WM, int WN, int ST, int BK>
void set_smem_attrs(lyap_ctx* ctx) {
  using Cfg = DgemmCfg<BM, BN, WM, WN, ST, BK>;
  CK(cudaFuncSetAttribute(k1_dgemm<BM, BN, WM, WN, ST, BK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::SMEM));
  CK(cudaFuncSetAttribute(k1_dgemm<BM, BN, WM, WN, ST, BK, 0, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)Cfg::SMEM));
  CK(cudaFuncSetAttribute(k1_dgemm<BM, BN, WM, WN, ST, BK, 0, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)Cfg::SMEM));
  CK(cudaFuncSetAttribute(k1_dgemm<BM, BN, WM, WN, ST, BK, 0, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)Cfg::SMEM));
}

template <int BM, int BN, int WM, int WN, int ST, int BK>
void launch_gemm(lyap_ctx* ctx, const Seed& s, const double* Bop, double* U, int64_t ncol, const K1Args& a,
                 cudaStream_t st, bool fuse) {
  using Cfg = DgemmCfg<BM, BN, WM, WN, ST, BK>;
  const int kpad = (int)std::min<int64_t>(roundup(s.n, BK), s.npad);  // skip zero rows
  dim3 grid((unsigned)((ncol / BN) * (s.npad / BM)));
  K1EpiArgs ep{a, s.btl, s.F, s.g0, (int)s.npad, (int)(2 * s.npairs), (int)s.npairs, (int)s.n};
  const int cpa = (int)(s.k * s.k);
  switch (fuse ? (int)s.k : 0) {
    case 1:
      k1_dgemm<BM, BN, WM, WN, ST, BK, 0, 1><<<grid, Cfg::THREADS, Cfg::SMEM, st>>>(
          s.Lf, Bop, nullptr, (int)s.npad, (int)ncol, kpad, (int)s.npad, a.nactive, cpa, DgemmOut{}, ep);
      break;
    case 2:
      k1_dgemm<BM, BN, WM, WN, ST, BK, 0, 2><<<grid, Cfg::THREADS, Cfg::SMEM, st>>>(
          s.Lf, Bop, nullptr, (int)s.npad, (int)ncol, kpad, (int)s.npad, a.nactive, cpa, DgemmOut{}, ep);
      break;
    case 4:
      k1_dgemm<BM, BN, WM, WN, ST, BK, 0, 4><<<grid, Cfg::THREADS, Cfg::SMEM, st>>>(
          s.Lf, Bop, nullptr, (int)s.npad, (int)ncol, kpad, (int)s.npad, a.nactive, cpa, DgemmOut{}, ep);
      break;
    default:
      k1_dgemm<BM, BN, WM, WN, ST, BK><<<grid, Cfg::THREADS, Cfg::SMEM, st>>>(s.Lf, Bop, U, (int)s.npad, (int)ncol,
                                                                         kpad, (int)s.npad, a.nactive, cpa);
  }
}

// persistent tcgen05 3xTF32 GEMM (umma.cuh), one CTA per SM over the active tiles; epi = k fuses the K1
// epilogue (k = 1, 2, 4), epi = 0 writes U32t for k1_epi
// stream priorities: the engine's main streams run at the greatest priority, the VERIFY side stream at the
// least, so the block scheduler places the tcgen05 kernel's CTAs before the DMMA blocks beside them
int stream_prio(bool high) {
  static int lo = 0, hi = 0, init = 0;
  if (!init) {
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    init = 1;
  }
  return high ? hi : lo;
}
int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}
template <int BN, int ST, int BK, int EB = 4>
void launch_umma(lyap_ctx* ctx, int epi, const CUtensorMap& ta, const CUtensorMap& tb, float* U32, int npad, int Nc,
                 int Kd, const int* nactive, int cpa, const K1EpiArgs& ep, cudaStream_t st, int* tctr,
                 const float* colscale = nullptr) {
  const int tiles = (Nc / BN) * (npad / UM_BM);
  const dim3 grid((unsigned)std::max(1, std::min(num_sms(), tiles)));
  constexpr int SM = UmCfg<BN, ST, BK, EB>::SMEM;
  switch (epi) {
    case 1:
      k1_umma_persistent<BN, ST, 1, BK, EB><<<grid, 192, SM, st>>>(ta, tb, U32, npad, Nc, Kd, nactive, cpa, ep, tctr,
                                                                   colscale);
      break;
    case 2:
      k1_umma_persistent<BN, ST, 2, BK, EB><<<grid, 192, SM, st>>>(ta, tb, U32, npad, Nc, Kd, nactive, cpa, ep, tctr,
                                                                   colscale);
      break;
    case 4:
      k1_umma_persistent<BN, ST, 4, BK, EB><<<grid, 192, SM, st>>>(ta, tb, U32, npad, Nc, Kd, nactive, cpa, ep, tctr,
                                                                   colscale);
      break;
    default:
      k1_umma_persistent<BN, ST, 0, BK, EB><<<grid, 192, SM, st>>>(ta, tb, U32, npad, Nc, Kd, nactive, cpa, ep, tctr,
                                                                   colscale);
  }
  LAUNCHED();
}
template <int BN, int ST, int BK, int EB = 4>
void set_umma_attrs(lyap_ctx* ctx) {
  constexpr int SM = UmCfg<BN, ST, BK, EB>::SMEM;
  CK(cudaFuncSetAttribute(k1_umma_persistent<BN, ST, 0, BK, EB>, cudaFuncAttributeMaxDynamicSharedMemorySize, SM));
  CK(cudaFuncSetAttribute(k1_umma_persistent<BN, ST, 1, BK, EB>, cudaFuncAttributeMaxDynamicSharedMemorySize, SM));
  CK(cudaFuncSetAttribute(k1_umma_persistent<BN, ST, 2, BK, EB>, cudaFuncAttributeMaxDynamicSharedMemorySize, SM));
  CK(cudaFuncSetAttribute(k1_umma_persistent<BN, ST, 4, BK, EB>, cudaFuncAttributeMaxDynamicSharedMemorySize, SM));
}

void launch_k1(lyap_ctx* ctx, const K1Args& a, cudaStream_t st, cudaEvent_t evb = nullptr, cudaEvent_t eve = nullptr,
               unsigned evflags = 0, int group = 0, int mp = 0) {
  const Seed& s = ctx->seed;
  Engine g = ctx->eng;  // copy: operand buffers of this slot group
  g.Bop += (size_t)group * s.npad * g.ncol;
  g.U += (size_t)group * s.npad * g.ncol;
  const int two_np = (int)(2 * s.npairs);
  const bool fuse = k1_fused(s.k, s.n, mp);
  // mixed precision with the tcgen05 kernel and k = 1, 2, 4: both GEMMs carry the K1 epilogue (the
  // DMMA one for the VERIFY positions, the tcgen05 one for the ITER positions), k1_epi is not launched
  const bool fuse_mp =
      (mp == 1 || mp == 3) && a.mode == 1 && mp_umma() && s.npad % UM_BM == 0 &&
      (s.k == 1 || s.k == 2 || s.k == 4);
  static const int fmask = [] {  // LYAP_MP_FUSE (diagnostics): bit 0 tcgen05 epilogue, bit 1 DMMA epilogue
    const char* ev = std::getenv("LYAP_MP_FUSE");
    return ev ? std::atoi(ev) : 3;
  }();
  const bool fuse_um = fuse_mp && (fmask & 1), fuse_dm = fuse_mp && (fmask & 2);
  float* B32 = mp ? g.Bop32 + (size_t)group * 2 * s.npad * g.ncol : nullptr;
  float* U32 = mp ? g.U32 + (size_t)group * s.npad * g.ncol : nullptr;
  K_DISPATCH(s.k, {
    dim3 grid((unsigned)(s.npad / K1_TILE_C), (unsigned)((a.nslot + K1Tile<KK>::TS - 1) / K1Tile<KK>::TS));
    if (mp == 3) {
      // per-position max |X_t| first: the FP16 column scales (k1_gen) need it
      // (slot indices are local to the slot group: each group has its own xmax rows)
      float* xm = g.xmax + (size_t)group * ((g.b + g.groups - 1) / g.groups) * s.k;
      // (engine mode: k_prec has already accumulated them while writing Xin)
      if (a.mode != 1) k_xmax<KK><<<(unsigned)a.nslot, 256, 0, st>>>(a, (int)s.npad, xm);
      K1Args a3 = a;
      a3.xmax = xm;
      a3.bmax = g.bmax;
      a3.eA = ctx->basis->lf_eA;
      a3.colscale = g.colscale + (size_t)group * g.ncol;
      dim3 g16((unsigned)((s.npad + 2 * K1G16_THREADS - 1) / (2 * K1G16_THREADS)), (unsigned)a.nslot);
      k1_gen16<KK><<<g16, K1G16_THREADS, 0, st>>>(a3, s.bhr, (int)s.npad, two_np, g.Bop, g.ncol,
                                                  reinterpret_cast<__half*>(B32));
    } else if (mp == 1)
      k1_gen<KK, 1><<<grid, K1_THREADS, 0, st>>>(a, s.bhr, (int)s.npad, two_np, g.Bop, g.ncol, B32);
    else if (mp == 2)
      k1_gen<KK, 2><<<grid, K1_THREADS, 0, st>>>(a, s.bhr, (int)s.npad, two_np, g.Bop, g.ncol, B32);
    else
      k1_gen<KK><<<grid, K1_THREADS, 0, st>>>(a, s.bhr, (int)s.npad, two_np, g.Bop, g.ncol);
  });
  LAUNCHED();
  if (evb) CK(cudaEventRecordWithFlags(evb, st, evflags));
  if (!mp) {
    if (s.n <= SMALL_N)
      launch_gemm<S_BM, S_BN, S_WM, S_WN, S_ST, S_BK>(ctx, s, g.Bop, g.U, g.ncol, a, st, fuse);
    else
      launch_gemm<G_BM, G_BN, G_WM, G_WN, G_ST, G_BK>(ctx, s, g.Bop, g.U, g.ncol, a, st, fuse);
    LAUNCHED();
  } else {
    // mixed precision: the exact FP64 GEMM of the VERIFY positions [0, nver) (few
    // columns: the small-tile DMMA configuration) on the group's side stream, beside the float GEMM
    // of all positions on the tensor cores; k1_epi picks U or U32 per position
    if (!ctx->mpstream[group]) {
      CK(cudaStreamCreateWithPriority(&ctx->mpstream[group], cudaStreamNonBlocking, stream_prio(false)));
      CK(cudaEventCreateWithFlags(&ctx->mpfork[group], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&ctx->mpjoin[group], cudaEventDisableTiming));
    }
    static const bool serial = std::getenv("LYAP_MP_SERIAL") != nullptr;  // diagnostics: no side stream
    // Order (LYAP_MP_ORDER, default 1): the persistent tcgen05 kernel is launched FIRST, from the
    // higher-priority stream, so its one CTA per SM owns the SMs for its whole run; the VERIFY GEMM
    // follows on the low-priority side stream and fills the tcgen05 kernel's tail.  0: DMMA first (its
    // blocks then hold the SMs and the tcgen05 CTAs wait for them).  Measured on c5 (tools/gpu_order.sh):
    // same step time within 2 % either way (the board is at its power cap), but the tcgen05 launch takes
    // 0.72 ms instead of 1.15 ms, i.e. the events around it time the kernel, not the queue behind DMMA.
    // Co-residency (LYAP_VER_CFG=2: a 2-stage 29.7 KB DMMA CTA beside the 193 KB tcgen05 CTA, or
    // LYAP_UM_ST=3) was measured too and gains nothing under the power cap.
    static const int order = [] {
      const char* ev = std::getenv("LYAP_MP_ORDER");
      return ev ? std::atoi(ev) : 1;
    }();
    const bool um_first = order == 1 && !serial && (mp == 1 || mp == 3) && mp_umma() && s.npad % UM_BM == 0;
    cudaStream_t ss = serial ? st : ctx->mpstream[group];
    CK(cudaEventRecord(ctx->mpfork[group], st));
    auto launch_verify = [&] {
      CK(cudaStreamWaitEvent(ss, ctx->mpfork[group], 0));
      K1Args av = a;
      av.nactive = a.nver;
      static const int vcfg = [] {  // LYAP_VER_CFG: 0 = 64 x 32 x 16 in 3 stages, 1 = 64 x 64, 2 = 64 x 32 x 16 in 2 stages
        const char* ev = std::getenv("LYAP_VER_CFG");
        return ev ? std::atoi(ev) : -1;
      }();
      const int cfg = vcfg >= 0 ? vcfg : 0;
      if (cfg == 2)
        launch_gemm<V_BM, V_BN, V_WM, V_WN, 2, V_BK>(ctx, s, g.Bop, g.U, g.ncol, av, ss, fuse_dm);
      else if (cfg == 0)
        launch_gemm<V_BM, V_BN, V_WM, V_WN, V_ST, V_BK>(ctx, s, g.Bop, g.U, g.ncol, av, ss, fuse_dm);
      else
        launch_gemm<S_BM, S_BN, S_WM, S_WN, S_ST, S_BK>(ctx, s, g.Bop, g.U, g.ncol, av, ss, fuse_dm);
      LAUNCHED();
      CK(cudaEventRecord(ctx->mpjoin[group], ss));
    };
    if (!um_first) launch_verify();
    const int Nc = (int)g.ncol, M = (int)s.npad;
    const float* A32 = ctx->basis->Lf32;  // row-major npad x 2 npad: [hi | lo]
    if ((mp == 1 || mp == 3) && mp_umma() && s.npad % UM_BM == 0) {
      // tcgen05 3xTF32 GEMM (umma.cuh): U32t = A_hi B_lo + A_lo B_hi + A_hi B_hi in one TMEM accumulator
      // 3xFP16: 32 half per 64-byte row; 3xTF32: 16 (or 32 for the 128-wide alternative) floats
      const int eb = mp == 3 ? 2 : 4;
      const uint32_t bk = mp == 3 ? 32u : (um_bn() == 128 ? 32u : (uint32_t)UM_BKE);
      const uint32_t bn = mp == 3 ? (uint32_t)UM_BN : (uint32_t)um_bn();
      if (ctx->um_ta_ptr != A32 || ctx->um_ta_mode != mp) {
        ctx->um_ta = make_tmap_f32(ctx, A32, 2 * (uint64_t)s.npad, (uint64_t)s.npad, bk, UM_BM, eb);
        ctx->um_ta_ptr = A32;
        ctx->um_ta_mode = mp;
      }
      if (ctx->um_tb_ptr[group] != B32 || ctx->um_tb_ncol[group] != g.ncol || ctx->um_tb_mode[group] != mp) {
        ctx->um_tb[group] = make_tmap_f32(ctx, B32, (uint64_t)s.npad, 2 * (uint64_t)g.ncol, bk, bn, eb);
        ctx->um_tb_mode[group] = mp;
        ctx->um_tb_ptr[group] = B32;
        ctx->um_tb_ncol[group] = g.ncol;
      }
      const int Kd = (int)std::min<int64_t>(roundup(s.n, 32), s.npad);  // zero rows skipped (multiple of both BKs)
      K1EpiArgs ep{a, s.btl, s.F, s.g0, (int)s.npad, two_np, (int)s.npairs, (int)s.n};
      const int cpa = (int)(s.k * s.k), epi = fuse_um ? (int)s.k : 0;
      static const bool um3 = [] {  // LYAP_UM_ST=3: 3-stage ring (145 KB; leaves room for a 3-stage DMMA CTA)
        const char* ev = std::getenv("LYAP_UM_ST");
        return ev && std::atoi(ev) == 3;
      }();
      if (mp == 3 && um3)
        launch_umma<UM_BN, 3, 32, 2>(ctx, epi, ctx->um_ta, ctx->um_tb[group], U32, (int)s.npad, Nc, Kd, a.nactive, cpa, ep,
                                     st, g.umctr + 2 * group, g.colscale + (size_t)group * g.ncol);
      else if (mp == 3)
        launch_umma<UM_BN, UM_STAGES, 32, 2>(ctx, epi, ctx->um_ta, ctx->um_tb[group], U32, (int)s.npad, Nc, Kd, a.nactive,
                                             cpa, ep, st, g.umctr + 2 * group, g.colscale + (size_t)group * g.ncol);
      else if (um_bn() == 128)
        launch_umma<128, 3, 32>(ctx, epi, ctx->um_ta, ctx->um_tb[group], U32, (int)s.npad, Nc, Kd, a.nactive, cpa, ep, st,
                            g.umctr + 2 * group);
      else
        launch_umma<UM_BN, UM_STAGES, UM_BKE>(ctx, epi, ctx->um_ta, ctx->um_tb[group], U32, (int)s.npad, Nc, Kd, a.nactive, cpa,
                                      ep, st, g.umctr + 2 * group);
    } else {
      if (!ctx->cublas_eng[group]) {  // (the engine creates it; a standalone apply may come first)
        CKB(cublasCreate(&ctx->cublas_eng[group]));
        ctx->cublas_ws[group] = dalloc<double>(ctx, (32u << 20) / 8, false);
        CKB(cublasSetWorkspace(ctx->cublas_eng[group], ctx->cublas_ws[group], 32u << 20));
      }
      cublasHandle_t hb = ctx->cublas_eng[group];
      CKB(cublasSetStream(hb, st));
      const int Kd = (int)std::min<int64_t>(roundup(s.n, 16), s.npad);  // zero rows skipped
      const float one = 1.f, zero = 0.f;
      const float* Bhi = B32 + (size_t)s.npad * g.ncol;
      // column-major U32t (M x Nc, ld npad) = op(A32^T) B32t, B32t K-major (ld npad)
      if (mp == 1) {
        CKB(cublasGemmEx(hb, CUBLAS_OP_T, CUBLAS_OP_N, M, Nc, Kd, &one, A32, CUDA_R_32F, (int)(2 * s.npad), B32,
                         CUDA_R_32F, (int)s.npad, &zero, U32, CUDA_R_32F, M, CUBLAS_COMPUTE_32F_FAST_TF32,
                         CUBLAS_GEMM_DEFAULT));
        CKB(cublasGemmEx(hb, CUBLAS_OP_T, CUBLAS_OP_N, M, Nc, Kd, &one, A32 + s.npad, CUDA_R_32F, (int)(2 * s.npad), Bhi,
                         CUDA_R_32F, (int)s.npad, &one, U32, CUDA_R_32F, M, CUBLAS_COMPUTE_32F_FAST_TF32,
                         CUBLAS_GEMM_DEFAULT));
        CKB(cublasGemmEx(hb, CUBLAS_OP_T, CUBLAS_OP_N, M, Nc, Kd, &one, A32, CUDA_R_32F, (int)(2 * s.npad), Bhi,
                         CUDA_R_32F, (int)s.npad, &one, U32, CUDA_R_32F, M, CUBLAS_COMPUTE_32F_FAST_TF32,
                         CUBLAS_GEMM_DEFAULT));
      } else {
        CKB(cublasGemmEx(hb, CUBLAS_OP_T, CUBLAS_OP_N, M, Nc, Kd, &one, A32, CUDA_R_32F, (int)(2 * s.npad), Bhi,
                         CUDA_R_32F, (int)s.npad, &zero, U32, CUDA_R_32F, M, mp_compute(mp), CUBLAS_GEMM_DEFAULT));
      }
    }
    // profile events bracket the tensor-core GEMM (the side-stream DMMA overlaps it)
    if (eve) CK(cudaEventRecordWithFlags(eve, st, evflags));
    if (um_first) launch_verify();
    CK(cudaStreamWaitEvent(st, ctx->mpjoin[group], 0));
  }
  if (eve && !mp) CK(cudaEventRecordWithFlags(eve, st, evflags));
  if (mp && !(fuse_um && fuse_dm)) {
    const int which = fuse_um ? 1 : (fuse_dm ? 2 : 0);
    K_DISPATCH(s.k, {
      dim3 grid((unsigned)(s.npad / K1_TILE_C), (unsigned)((a.nslot + K1Tile<KK>::TS - 1) / K1Tile<KK>::TS));
      k1_epi<KK, true><<<grid, K1_THREADS, 0, st>>>(a, g.U, g.ncol, s.btl, s.F, s.g0, (int)s.npad, two_np,
                                                    (int)s.npairs, (int)s.n, U32, which);
    });
    LAUNCHED();
  } else if (!mp && !fuse) {
    K_DISPATCH(s.k, {
      dim3 grid((unsigned)(s.npad / K1_TILE_C), (unsigned)((a.nslot + K1Tile<KK>::TS - 1) / K1Tile<KK>::TS));
      k1_epi<KK><<<grid, K1_THREADS, 0, st>>>(a, g.U, g.ncol, s.btl, s.F, s.g0, (int)s.npad, two_np, (int)s.npairs,
                                              (int)s.n);
    });
    LAUNCHED();
  }
}


// ------------------------------------------------------------------ the batched engine
int run_batch(lyap_ctx* ctx, int64_t nv, const double* dV, const int* dorder, double* dtr, int32_t* dst,
              int32_t* dap, double* dres, cudaStream_t user_st, double* gout = nullptr, const int* dregq = nullptr,
              int record = 0, const double* x0 = nullptr) {
  // the engine runs on the library's own streams (graph capture is illegal on the legacy default
  // stream a caller may pass); it is ordered after, and the caller's stream after it, by events
  cudaStream_t st = ctx->stream;
  if (!ctx->evfork) CK(cudaEventCreateWithFlags(&ctx->evfork, cudaEventDisableTiming));
  if (!ctx->evjoin) CK(cudaEventCreateWithFlags(&ctx->evjoin, cudaEventDisableTiming));
  if (user_st != st) {
    CK(cudaEventRecord(ctx->evfork, user_st));
    CK(cudaStreamWaitEvent(st, ctx->evfork, 0));
  }
  const Seed& s = ctx->seed;
  const int b = auto_batch(ctx, nv), mmax = auto_mmax(ctx);
  if (coarse_size(ctx) > 0 && !record) ensure_coarse(ctx);
  const bool two_level = ctx->coarse.p > 0 && !record;
  ensure_engine(ctx, b, mmax);
  ctx->info.batch = b;
  Engine& g = ctx->eng;
  const int G = g.groups;
  CK(cudaMemsetAsync(g.phase, 0, sizeof(int) * b, st));  // PH_FREE
  CK(cudaMemsetAsync(g.ctrl, 0, sizeof(int) * 8 * (G + 1), st));
  CK(cudaMemsetAsync(g.X, 0, sizeof(double) * (size_t)b * g.L, st));
  CK(cudaMemsetAsync(g.restarts, 0, sizeof(int) * 5 * (size_t)b, st));
  if (record) CK(cudaMemsetAsync(g.Hraw, 0, sizeof(double) * (size_t)b * (mmax + 1) * mmax, st));

  EngArgs a{};
  a.b = b;
  a.mmax = mmax;
  a.K = (int)s.k;
  a.nv = (int)nv;
  a.L = g.L;
  a.npad = s.npad;
  a.nrep = s.nrep;
  a.npairs = s.npairs;
  a.two_np = 2 * s.npairs;
  a.n = s.n;
  a.nchunk = g.nchunk;
  a.tol = ctx->opts.tol;
  a.tol_inner = 0.5 * ctx->opts.tol;
  const int mp = record ? 0 : mp_mode(ctx);
  a.eta_rel = mp ? ctx->opts.mixed_eta : 0.0;
  if (mp) ensure_lf32(ctx, mp);  // (3xFP16: the half planes, in the same buffer)
  a.t0 = s.t0;
  a.nterms = s.qlin ? s.nterms : 0;
  a.t0t = s.t0t;
  a.rhs = s.qlin ? g.rhs : nullptr;
  a.t0s = s.qlin ? g.t0s : nullptr;
  a.pc = two_level ? g.pc : 0;
  a.Zc = ctx->coarse.Z;
  a.Phi = ctx->coarse.Phi;
  a.Psi = ctx->coarse.Psi;
  a.max_restarts = ctx->opts.max_restarts;
  a.warm = ctx->opts.warm_start;
  a.V = dV;
  a.order = dorder;
  a.g0 = s.g0;
  a.hf = s.hf;
  a.Pb = s.Pb;
  a.traces = dtr;
  a.status = dst;
  a.out_applies = dap;
  a.out_resid = dres;
  a.gout = gout;
  a.x0 = x0;
  a.record = record;
  a.s_rec = (ctx->nreg > 0 && !mp) ? ctx->s_rec : 0;  // recycle spaces: FP64 engine only
  a.Ureg = ctx->Ureg;
  a.sreg = ctx->sreg;
  a.TUreg = ctx->TUreg;
  a.regq = ctx->nreg > 0 ? dregq : nullptr;
  a.qctr = g.ctrl + 8 * G;

  // slot group gi owns slots [s0, s0 + bg): every per-slot array is offset, so the kernels see a
  // self-contained engine of bg slots; only the v queue and the done counter are shared
  const int bg0 = (b + G - 1) / G;
  std::vector<EngArgs> ga(G);
  std::vector<K1Args> gk(G);
  std::vector<int> gb(G);
  for (int gi = 0; gi < G; ++gi) {
    const int64_t s0 = (int64_t)gi * bg0;
    const int bg = (int)std::min<int64_t>(bg0, b - s0);
    gb[gi] = bg;
    EngArgs x = a;
    x.b = bg;
    const int64_t ld = mmax + 1;
    x.X = g.X + s0 * g.L;
    x.Xin = g.Xin + s0 * g.L;
    x.Qb = g.Qb ? g.Qb + s0 * ld * g.L : nullptr;
    x.Qf = g.Qf ? g.Qf + s0 * ld * g.L : nullptr;
    x.Minv = g.Minv + s0 * s.nrep * s.k * s.k * 4;
    // (the same rows launch_k1 hands to k1_gen16: group * bg0 * k)
    x.xmaxu = mp == 3 ? reinterpret_cast<unsigned int*>(g.xmax + s0 * s.k) : nullptr;
    x.sigma = g.sigma + s0 * s.k;
    x.mask = g.mask + s0 * s.k;
    x.eta = g.eta + s0 * ld;
    x.H = g.H + s0 * ld * mmax;
    x.e = g.e + s0 * ld;
    x.cs = g.e + (int64_t)b * ld + s0 * mmax;
    x.sn = g.e + (int64_t)b * ld + (int64_t)b * mmax + s0 * mmax;
    x.y = g.y + s0 * mmax;
    x.bnorm = g.bnorm + s0;
    x.part = g.part + s0 * (mmax + 2) * g.nchunk;
    x.part2 = g.part2 + s0 * (mmax + 2) * g.nchunk;
    x.part3 = g.part3 + s0 * g.nchunk * 3;
    x.Gq = g.Gq + s0 * ld * ld;
    x.cf = g.cf + s0 * ld;
    x.phase = g.phase + s0;
    x.m = g.m + s0;
    x.vidx = g.vidx + s0;
    x.applies = g.applies + s0;
    x.restarts = g.restarts + s0;
    x.newv = g.restarts + b + s0;
    x.alist = g.restarts + 2 * b + s0;
    x.su = g.restarts + 3 * b + s0;
    x.reg = g.restarts + 4 * b + s0;
    if (x.rhs) {
      x.rhs = g.rhs + s0 * g.L;
      x.t0s = g.t0s + s0;
    }
    if (x.pc > 0) {
      x.Zb = g.Zb + s0 * ld * g.L;
      x.Rbuf = g.Rbuf + s0 * g.L;
      x.Yz = g.Yz + s0 * 2 * g.L;
      x.Cc = g.Cc + s0 * x.pc;
      x.Wc = g.Wc + s0 * x.pc;
      x.Einv = g.Einv + s0 * (int64_t)x.pc * x.pc;
    }
    x.Hraw = g.Hraw + s0 * ld * mmax;
    x.ctrl = g.ctrl + 8 * gi;
    ga[gi] = x;
    K1Args k1{};
    k1.Xin = x.Xin;
    k1.L = g.L;
    k1.nslot = bg;
    k1.mode = 1;
    k1.mask = x.mask;
    k1.sigma = x.sigma;
    k1.phase = x.phase;
    k1.m = x.m;
    k1.Qb = x.Qb;
    k1.Qf = x.Qf;
    k1.qstride = ld * g.L;
    k1.nactive = x.ctrl + 2;
    k1.alist = x.alist;
    k1.rhs = x.rhs;
    k1.nver = mp ? x.ctrl + 3 : nullptr;
    gk[gi] = k1;
  }

  const size_t upd_smem = sizeof(double) * (mmax + 1);
  const size_t cf_smem = sizeof(double) * (size_t)a.pc * a.pc + sizeof(int) * (size_t)a.pc + 16;
  if (a.pc > 0) CK(cudaFuncSetAttribute(k_cfactor, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cf_smem));
  if (a.pc > 0 || mp) {
    for (int gi = 0; gi < G; ++gi)
      if (!ctx->cublas_eng[gi]) {  // a handle per slot group with its own workspace (graph capture)
        CKB(cublasCreate(&ctx->cublas_eng[gi]));
        ctx->cublas_ws[gi] = dalloc<double>(ctx, (32u << 20) / 8, false);
        CKB(cublasSetWorkspace(ctx->cublas_eng[gi], ctx->cublas_ws[gi], 32u << 20));
      }
  }
  const size_t ctrl_smem = sizeof(double) * 16 * (size_t)(mmax + 2);
  const size_t gram_smem = sizeof(double) * (size_t)(mmax + 1);
  if (gram_smem > 48 * 1024) CK(cudaFuncSetAttribute(k_gram, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gram_smem));
  if (ctrl_smem > 48 * 1024) CK(cudaFuncSetAttribute(k_ctrl, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ctrl_smem));
  if (upd_smem > 48 * 1024) {
    CK(cudaFuncSetAttribute(k_upd<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)upd_smem));
    CK(cudaFuncSetAttribute(k_upd<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)upd_smem));
  }
  const int64_t per_v = (int64_t)(ctx->opts.max_restarts + 1) * (mmax + 2);
  const int64_t max_iter = ((nv + bg0 - 1) / bg0) * per_v + 64;
  const int poll = 8;
  std::vector<cudaStream_t> sts(G);
  sts[0] = st;
  CK(cudaEventRecord(ctx->ev0, st));
  if (G > 1) {
    CK(cudaEventRecord(ctx->evfork, st));
    for (int gi = 1; gi < G; ++gi) {
      if (!ctx->xstream[gi]) CK(cudaStreamCreateWithPriority(&ctx->xstream[gi], cudaStreamNonBlocking, stream_prio(true)));
      sts[gi] = ctx->xstream[gi];
      CK(cudaStreamWaitEvent(sts[gi], ctx->evfork, 0));
    }
  }
  // one engine iteration of slot group gi on stream sg (optionally with events around the GEMM)
  auto issue = [&](int gi, cudaStream_t sg, cudaEvent_t evb, cudaEvent_t eve, unsigned evflags) -> int64_t {
    const int64_t l0 = ctx->stats.kernel_launches;
    const EngArgs& x = ga[gi];
    const int bg = gb[gi];
    const dim3 grep((unsigned)((s.nrep + 127) / 128), (unsigned)bg);
    const dim3 gred((unsigned)g.nchunk, (unsigned)bg);
    const int xw = g.Qf ? 128 : 64;  // k_xcomb's coordinate window
    const dim3 gxc((unsigned)std::min<int64_t>((s.npad + xw - 1) / xw, 128), (unsigned)bg);
    k_assign<<<1, (int)roundup(bg, 32), 0, sg>>>(x);
    LAUNCHED();
    K_DISPATCH(s.k, (k_pfactor<KK><<<grep, 128, 0, sg>>>(x)));
    LAUNCHED();
    if (x.pc > 0) {  // two-level preconditioner: coarse factor, Z^T r, E^{-1}, Z w and T Z w (cuBLAS)
      const int p = x.pc, Li = (int)g.L;
      const double one = 1.0, zero = 0.0;
      cublasHandle_t hb = ctx->cublas_eng[gi];
      CKB(cublasSetStream(hb, sg));
      if (p <= 32)
        k_cfactor32<<<(unsigned)((bg + 3) / 4), 128, 0, sg>>>(x);
      else
        k_cfactor<<<bg, 256, cf_smem, sg>>>(x, 0);
      LAUNCHED();
      k_cpre<<<dim3((unsigned)std::min<int64_t>((g.L + 255) / 256, 64), (unsigned)bg), 256, 0, sg>>>(x);
      LAUNCHED();
      CKB(cublasDgemm(hb, CUBLAS_OP_T, CUBLAS_OP_N, p, bg, Li, &one, x.Zc, 2 * Li, x.Rbuf, Li, &zero, x.Cc, p));
      k_cw<<<bg, 128, 0, sg>>>(x);
      LAUNCHED();
      CKB(cublasDgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, 2 * Li, bg, p, &one, x.Zc, 2 * Li, x.Wc, p, &zero, x.Yz, 2 * Li));
    }
    if (g.Qf) {
      K_DISPATCH(s.k, (k_prec<KK, float><<<grep, 128, 0, sg>>>(x)));
    } else {
      K_DISPATCH(s.k, (k_prec<KK><<<grep, 128, 0, sg>>>(x)));
    }
    LAUNCHED();
    if (x.s_rec > 0) {
      k_uapply<<<dim3((unsigned)std::min<int64_t>((g.L + 255) / 256, 64), (unsigned)bg), 256, 0, sg>>>(x);
      LAUNCHED();
    }
    launch_k1(ctx, gk[gi], sg, evb, eve, evflags, gi, mp);
    const int zfull = (mmax + DOT_IG) / DOT_IG;  // short vectors (few chunks) keep one block per DOT_IG basis vectors
    const dim3 gdot((unsigned)g.nchunk, (unsigned)bg, (unsigned)(g.nchunk >= 16 ? std::min(zfull, DOT_Z) : zfull));
    if (g.Qf)
      k_dots<float><<<gdot, 256, 0, sg>>>(x);
    else
      k_dots<<<gdot, 256, 0, sg>>>(x);
    LAUNCHED();
    k_gram<<<bg, 256, gram_smem, sg>>>(x);
    LAUNCHED();
    if (g.Qf)
      k_upd<float><<<gred, 256, upd_smem, sg>>>(x);
    else
      k_upd<<<gred, 256, upd_smem, sg>>>(x);
    LAUNCHED();
    k_ctrl<<<(bg + 3) / 4, 128, ctrl_smem, sg>>>(x);
    LAUNCHED();
    if (x.gout) {
      k_gout<<<dim3((unsigned)std::min<int64_t>((g.L + 255) / 256, 64), (unsigned)bg), 256, 0, sg>>>(x);
      LAUNCHED();
    }
    if (g.Qf) {
      K_DISPATCH(s.k, (k_xcomb<KK, float><<<gxc, 256, 0, sg>>>(x)));
    } else {
      K_DISPATCH(s.k, (k_xcomb<KK><<<gxc, 256, 0, sg>>>(x)));
    }
    LAUNCHED();
    return ctx->stats.kernel_launches - l0;
  };
  // CUDA graphs: `poll` iterations per group are captured once (each with its own GEMM event pair
  // when profiling) and replayed; the host only polls the done counter between replays.
  const bool prof = ctx->opts.profile != 0;
  std::vector<cudaEvent_t>& evs = ctx->prof_evs;
  if (prof && evs.size() < (size_t)2 * G * poll) {
    for (auto& e : evs) cudaEventDestroy(e);
    evs.assign((size_t)2 * G * poll, nullptr);
    for (auto& e : evs) CK(cudaEventCreate(&e));
  }
  // the instantiated graphs are kept in the ctx: a later call re-captures (cheap) and updates the
  // executable in place when the topology matches (cudaGraphExecUpdate), instead of re-instantiating
  cudaGraphExec_t* gexec = ctx->gexec;
  int64_t launches_per_replay = 0;
  for (int gi = 0; gi < G; ++gi) {
    cudaGraph_t graph;
    CK(cudaStreamBeginCapture(sts[gi], cudaStreamCaptureModeThreadLocal));
    for (int p = 0; p < poll; ++p) {
      cudaEvent_t eb = prof ? evs[(size_t)2 * (gi * poll + p)] : nullptr;
      cudaEvent_t ee = prof ? evs[(size_t)2 * (gi * poll + p) + 1] : nullptr;
      launches_per_replay += issue(gi, sts[gi], eb, ee, cudaEventRecordExternal);
    }
    CK(cudaStreamEndCapture(sts[gi], &graph));
    if (gexec[gi]) {
      cudaGraphExecUpdateResultInfo info;
      if (cudaGraphExecUpdate(gexec[gi], graph, &info) != cudaSuccess) {
        cudaGetLastError();
        cudaGraphExecDestroy(gexec[gi]);
        gexec[gi] = nullptr;
      } else {
        ctx->stats.graph_updates++;
      }
    }
    if (!gexec[gi]) {
      CK(cudaGraphInstantiate(&gexec[gi], graph, 0));
      ctx->stats.graph_instantiations++;
    }
    CK(cudaGraphDestroy(graph));
  }
  ctx->stats.kernel_launches -= launches_per_replay;  // counted per replay below
  int64_t it = 0;
  int rc = LYAP_OK;
  for (;;) {
    for (int gi = 0; gi < G; ++gi) CK(cudaGraphLaunch(gexec[gi], sts[gi]));
    it += poll;
    ctx->stats.kernel_launches += launches_per_replay;
    ctx->stats.k1_launches += (int64_t)G * poll;
    for (int gi = 1; gi < G; ++gi) CK(cudaStreamSynchronize(sts[gi]));
    CK(cudaMemcpyAsync(g.h_ctrl, g.ctrl, 8 * (G + 1) * sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (prof) {
      for (size_t i = 0; i < (size_t)2 * G * poll; i += 2) {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, evs[i], evs[i + 1]));
        ctx->stats.k1_ms += ms;
      }
    }
    const int done = g.h_ctrl[8 * G + 1];
    if (done >= nv) break;
    if (it > max_iter) {
      set_err(ctx, "engine did not finish after %lld iterations (%d of %lld done)", (long long)it, done,
              (long long)nv);
      rc = LYAP_ECUDA;
      break;
    }
  }
  for (int gi = 1; gi < G; ++gi) {
    if (!ctx->xjoin[gi]) CK(cudaEventCreateWithFlags(&ctx->xjoin[gi], cudaEventDisableTiming));
    CK(cudaEventRecord(ctx->xjoin[gi], sts[gi]));
    CK(cudaStreamWaitEvent(st, ctx->xjoin[gi], 0));
  }
  CK(cudaMemcpyAsync(g.h_ctrl, g.ctrl, 8 * (G + 1) * sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaEventRecord(ctx->ev1, st));
  CK(cudaEventSynchronize(ctx->ev1));
  if (user_st != st) {
    CK(cudaEventRecord(ctx->evjoin, st));
    CK(cudaStreamWaitEvent(user_st, ctx->evjoin, 0));
  }
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
  ctx->stats.batch_ms = ms;
  ctx->stats.iterations += it;
  for (int gi = 0; gi < G; ++gi) {
    unsigned long long nvec = 0;
    std::memcpy(&nvec, g.h_ctrl + 8 * gi + 4, 8);
    ctx->stats.k1_vectors += (int64_t)nvec;
    unsigned long long nexact = nvec;
    if (mp) std::memcpy(&nexact, g.h_ctrl + 8 * gi + 6, 8);
    ctx->stats.k1_exact_vectors += (int64_t)nexact;
    ctx->stats.k1_flops += 2.0 * (double)s.n * s.n * s.k * s.k * (double)nvec;
  }
  return rc;
}

// (Bl, Br)-dependent seed state on top of ctx->basis (NEXT row f4): B~l = S_r^{-1} Bl,
// B^r = S_r^T Br (DGEMM), then G0, H, F, t0 per representative (k_seed_rep), folding, scheduling
// weights.  Blc, Brc: device column-major n x k.  Throws Fail.
void build_config(lyap_ctx* ctx, const double* Blc, const double* Brc) {
  Seed& s = ctx->seed;
  const Basis& B = *ctx->basis;
  cudaStream_t st = ctx->stream;
  const int64_t n = s.n, k = s.k, two_np = 2 * s.npairs;
  const int ni = (int)n, ki = (int)k;
  const double one = 1.0, zero = 0.0;
  double *Blr = nullptr, *Brr = nullptr, *t0part = nullptr, *t0d = nullptr;
  try {
    Blr = dalloc<double>(ctx, (size_t)n * k, false);
    Brr = dalloc<double>(ctx, (size_t)n * k, false);
    t0part = dalloc<double>(ctx, s.nrep);
    t0d = dalloc<double>(ctx, 1);
    CKB(cublasDgemm(ctx->cublas, CUBLAS_OP_N, CUBLAS_OP_N, ni, ki, ni, &one, B.Sinv, ni, Blc, ni, &zero, Blr, ni));
    CKB(cublasDgemm(ctx->cublas, CUBLAS_OP_T, CUBLAS_OP_N, ni, ki, ni, &one, B.Sr, ni, Brc, ni, &zero, Brr, ni));
    const int nterms = s.nterms;
    s.g0 = dalloc<double>(ctx, (size_t)nterms * k * s.npad);
    s.hf = dalloc<double>(ctx, (size_t)k * s.npad);
    s.F = dalloc<double>(ctx, (size_t)s.nrep * k * k * 2);
    s.bhr = dalloc<double>(ctx, (size_t)s.npad * k);
    s.btl = dalloc<double>(ctx, (size_t)s.npad * k);
    s.t0t = dalloc<double>(ctx, nterms);
    s.t0h.assign(nterms, 0.0);
    // one right-hand side per Q term (Q(v) = sum_i v_i Q_i: G0(v), t0(v) linear in v)
    for (int q = nterms - 1; q >= 0; --q) {
      K_DISPATCH(k, (k_seed_rep<KK><<<(unsigned)s.nrep, 128, 0, st>>>(B.lam, B.Qr + (size_t)q * n * n, B.Er, Blr, Brr, n,
                                                                         s.npad, two_np, s.npairs,
                                                                         s.g0 + (size_t)q * k * s.npad, s.hf, s.F,
                                                                         t0part)));
      LAUNCHED();
      k_sum<<<1, 1024, 0, st>>>(t0part, s.nrep, s.t0t + q);
      LAUNCHED();
    }
    k_fold_b<<<(unsigned)((s.npad * k + 255) / 256), 256, 0, st>>>(Blr, Brr, n, s.npad, k, two_np, s.btl, s.bhr);
    LAUNCHED();
    s.Pb = dalloc<double>(ctx, (size_t)s.nrep * k * k * 4);
    K_DISPATCH(k, (k_pblock<KK><<<(unsigned)((s.nrep + 127) / 128), 128, 0, st>>>(B.Lf, s.npad, s.bhr, s.btl, s.F,
                                                                                     s.npairs, s.nrep, s.Pb)));
    LAUNCHED();
    CK(cudaMemcpyAsync(s.t0h.data(), s.t0t, 8 * nterms, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    s.t0 = s.t0h[0];
    // scheduling weights ||B~l_t|| ||B^r_t|| (folded coordinates)
    std::vector<double> hb((size_t)s.npad * k), hr((size_t)s.npad * k);
    CK(cudaMemcpy(hb.data(), s.btl, hb.size() * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hr.data(), s.bhr, hr.size() * 8, cudaMemcpyDeviceToHost));
    for (int64_t t = 0; t < k; ++t) {
      double nb = 0.0, nr = 0.0;
      for (int64_t c = 0; c < s.npad; ++c) {
        nb += hb[c * k + t] * hb[c * k + t];
        nr += hr[c * k + t] * hr[c * k + t];
      }
      s.wcost[t] = std::sqrt(nb * nr);
      ctx->info.wcost[t] = s.wcost[t];
    }
    ctx->info.t0 = s.t0;
    bool fin = true;
    for (double t : s.t0h) fin = fin && std::isfinite(t);
    if (!fin) {
      set_err(ctx, "seed trace t0 is not finite");
      throw Fail{LYAP_EEIG};
    }
  } catch (Fail) {
    for (void* p : {(void*)Blr, (void*)Brr, (void*)t0part, (void*)t0d}) dfree(p);
    throw;
  }
  for (void* p : {(void*)Blr, (void*)Brr, (void*)t0part, (void*)t0d}) dfree(p);
}

// Stability-filter tables (stab.cuh): the pole-resolving frequency grid, G(i w) on it, the moments
// for the tail.  Throws Fail.
void ensure_stab(lyap_ctx* ctx) {
  StabTables& T = ctx->stab;
  if (T.Gf) return;
  const Seed& s = ctx->seed;
  cudaStream_t st = ctx->stream;
  std::vector<double> hl(2 * (size_t)s.npad), hb((size_t)s.npad * s.k), ht((size_t)s.npad * s.k);
  CK(cudaMemcpy(hl.data(), s.lam, hl.size() * 8, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(hb.data(), s.bhr, hb.size() * 8, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(ht.data(), s.btl, ht.size() * 8, cudaMemcpyDeviceToHost));
  double maxabs = 0.0, minabs = 1e300, rho = 0.0;
  int PR = 0;
  std::vector<double> w{0.0};
  const double ms[] = {-8, -4, -2, -1.5, -1, -0.6, -0.3, 0, 0.3, 0.6, 1, 1.5, 2, 4, 8};
  for (int64_t rep = 0; rep < s.nrep; ++rep) {
    const bool pair = rep < s.npairs;
    const int64_t c = pair ? 2 * rep : rep + s.npairs;
    const double re = hl[2 * c], im = hl[2 * c + 1];
    const double a = std::hypot(re, im);
    maxabs = std::max(maxabs, a);
    minabs = std::min(minabs, a);
    if (re > 0.0) PR += pair ? 2 : 1;
    double nb = 0.0, nt = 0.0;
    for (int64_t t = 0; t < s.k; ++t) {
      nb += hb[c * s.k + t] * hb[c * s.k + t] + (pair ? hb[(c + 1) * s.k + t] * hb[(c + 1) * s.k + t] : 0.0);
      nt += ht[c * s.k + t] * ht[c * s.k + t] + (pair ? ht[(c + 1) * s.k + t] * ht[(c + 1) * s.k + t] : 0.0);
    }
    rho += (pair ? 2.0 : 1.0) * std::sqrt(nb * nt);
    const double ctr = pair ? im : 0.0, wid = pair ? std::fabs(re) : std::fabs(re);
    for (double m : ms) {
      const double x = ctr + m * wid;
      if (x > 0.0) w.push_back(x);
    }
  }
  const double wtail0 = 4.0 * maxabs;
  const double lo = 1e-4 * std::max(minabs, 1e-300);
  const int nbg = 512;
  for (int q = 0; q <= nbg; ++q) w.push_back(lo * std::pow(wtail0 / lo, (double)q / nbg));
  std::sort(w.begin(), w.end());
  std::vector<double> wg;
  for (double x : w)
    if (x <= wtail0 && (wg.empty() || x > wg.back() * (1.0 + 1e-13) + 1e-300)) wg.push_back(x);
  T.F = (int)wg.size();
  T.PR = PR;
  T.scale = std::max(maxabs, 1e-300);
  T.wtail0 = wtail0;
  T.rho = rho;
  T.wgrid = dalloc<double>(ctx, wg.size(), false);
  CK(cudaMemcpy(T.wgrid, wg.data(), wg.size() * 8, cudaMemcpyHostToDevice));
  T.Gf = dalloc<double>(ctx, (size_t)T.F * s.k * s.k * 2, false);
  T.Mm = dalloc<double>(ctx, (size_t)STAB_MOMENTS * s.k * s.k * 2, false);
  K_DISPATCH(s.k, (k_stab_G<KK><<<(unsigned)T.F, 128, 0, st>>>(s.lam, s.bhr, s.btl, s.nrep, s.npairs, T.wgrid, T.Gf)));
  LAUNCHED();
  K_DISPATCH(s.k, (k_stab_moments<KK><<<STAB_MOMENTS, 128, 0, st>>>(s.lam, s.bhr, s.btl, s.nrep, s.npairs, T.scale,
                                                                     T.Mm)));
  LAUNCHED();
  CK(cudaStreamSynchronize(st));
}

// nunstable[i] = eigenvalues of A(V[i]) in the open right half-plane (-1: marginal / unresolved).
// Device pointers, ordered on st.
void stab_count(lyap_ctx* ctx, int64_t nv, const double* dV, int32_t* dnu, cudaStream_t st) {
  ensure_stab(ctx);
  const Seed& s = ctx->seed;
  const StabTables& T = ctx->stab;
  StabArgs a{};
  a.lam = s.lam;
  a.bhr = s.bhr;
  a.btl = s.btl;
  a.wgrid = T.wgrid;
  a.Gf = T.Gf;
  a.Mm = T.Mm;
  a.nrep = s.nrep;
  a.npairs = s.npairs;
  a.F = T.F;
  a.scale = T.scale;
  a.wtail0 = T.wtail0;
  a.rho = T.rho;
  a.PR = T.PR;
  a.V = dV;
  a.nv = (int)nv;
  a.nunstable = dnu;
  const unsigned blocks = (unsigned)((nv * 32 + 127) / 128);
  K_DISPATCH(s.k, (k_stab_count<KK><<<blocks, 128, 0, st>>>(a)));
  LAUNCHED();
}

// size of the coarse space (opts.coarse): auto = 32 when n k >= 2000 (measured, B200, v/s with p =
// 0 / 32 / 48 / 64 / 96: c5 922 / 961 / 967 / 967 / 955; c4 11.67k / 12.4-12.6k / 12.0-12.6k / 12.48k /
// 12.11k; c3 113.7k / 203-206k / 154-175k; c2 100.2k / 85-86k / - / 67.3k: the coarse products cost
// more than they save when a T-apply is cheap and the off-block coupling is not low-rank)
int coarse_size(const lyap_ctx* ctx) {
  const Seed& s = ctx->seed;
  // auto: 32 when n k >= 2000 -- except under mixed precision, where the coarse products cost what they
  // save (c5 2280 with / 2315 v/s without)
  if (mp_mode(ctx)) return 0;  // the coarse space is an FP64-engine option (the FP32 basis has no Zb)
  int p = ctx->opts.coarse < 0 ? (s.n * s.k >= 2000 ? 32 : 0) : ctx->opts.coarse;
  p = std::min<int>(p, 256);
  p = std::min<int64_t>(p, (s.n * s.k) / 2);
  return p < 8 ? 0 : p / 8 * 8;
}

// In-place orthonormal basis of the columns of A (m x l, column-major): Householder QR (cuSOLVER).
void qr_inplace(lyap_ctx* ctx, double* A, int m, int l) {
  cudaStream_t st = ctx->stream;
  double* tau = dalloc<double>(ctx, l, false);
  int* dinfo = dalloc<int>(ctx, 1);
  int lw1 = 0, lw2 = 0;
  CKS(cusolverDnDgeqrf_bufferSize(ctx->cusolver, m, l, A, m, &lw1));
  CKS(cusolverDnDorgqr_bufferSize(ctx->cusolver, m, l, l, A, m, tau, &lw2));
  double* work = dalloc<double>(ctx, std::max(lw1, lw2), false);
  CKS(cusolverDnDgeqrf(ctx->cusolver, m, l, A, m, tau, work, std::max(lw1, lw2), dinfo));
  CKS(cusolverDnDorgqr(ctx->cusolver, m, l, l, A, m, tau, work, std::max(lw1, lw2), dinfo));
  CK(cudaStreamSynchronize(st));
  dfree(tau);
  dfree(dinfo);
  dfree(work);
}

// Coarse space of the two-level preconditioner, built once per ctx: the explicit
// folded T (K1 on unit vectors), minus its pair blocks (the part P(v) already inverts exactly) = T_o';
// Z = the p dominant right singular vectors of T_o' (randomized range finder, two power iterations,
// cuSOLVER QR/SVD of the tall sketches); T Z (K1); the Gram blocks Phi_t = Z_t^T Z_t and
// Psi_t = Z_t^T (T Z)_t from which every v's coarse matrix E(v) = sum_t sigma_t Phi_t - Psi_t is formed.
void ensure_coarse(lyap_ctx* ctx) {
  CoarseSpace& C = ctx->coarse;
  const int p = coarse_size(ctx);
  if (p == 0 || (C.Z && C.p == p)) return;
  const Seed& s = ctx->seed;
  const int64_t L = s.k * s.npad, k = s.k;
  const int l = p + 16, Li = (int)L;
  cudaStream_t st = ctx->stream;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, st));
  double *Tm = nullptr, *X = nullptr, *Y = nullptr, *Om = nullptr, *Ys = nullptr, *Bt = nullptr, *Sv = nullptr,
         *U = nullptr, *work = nullptr, *rwork = nullptr;
  int* dinfo = nullptr;
  try {
    for (double* q : {C.Z, C.Phi, C.Psi}) dfree(q);  // TZ lives inside Z
    C = CoarseSpace{};
    // 1. explicit folded T, column-major L x L
    Tm = dalloc<double>(ctx, (size_t)L * L, false);
    const int64_t cb = 512;
    X = dalloc<double>(ctx, (size_t)cb * L, false);
    Y = dalloc<double>(ctx, (size_t)cb * L, false);
    for (int64_t c0 = 0; c0 < L; c0 += cb) {
      const int64_t nb = std::min(cb, L - c0);
      k_unit_vectors<<<1024, 256, 0, st>>>(X, c0, nb, L);
      LAUNCHED();
      const int rc = lyap_apply_C(ctx, nb, X, nullptr, Y, st);
      if (rc != LYAP_OK) throw Fail{rc};
      k_neg_copy<<<1024, 256, 0, st>>>(Y, Tm + c0 * L, nb * L);
      LAUNCHED();
    }
    // 2. minus the pair blocks
    K_DISPATCH(k, (k_sub_pblocks<KK><<<(unsigned)((s.nrep + 127) / 128), 128, 0, st>>>(Tm, L, s.npad, s.Pb, s.npairs,
                                                                                          s.nrep)));
    LAUNCHED();
    // 3. randomized SVD: right singular vectors of T_o'
    {
      std::vector<double> h((size_t)L * l);
      uint64_t x = 0x2545f4914f6cdd1dULL;
      for (double& e : h) {
        x += 0x9e3779b97f4a7c15ULL;
        uint64_t z = x;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        z ^= z >> 31;
        e = (double)(z >> 11) * (2.0 / 9007199254740992.0) - 1.0;
      }
      Om = dalloc<double>(ctx, h.size(), false);
      CK(cudaMemcpy(Om, h.data(), h.size() * 8, cudaMemcpyHostToDevice));
    }
    Ys = dalloc<double>(ctx, (size_t)L * l, false);
    const double one = 1.0, zero = 0.0;
    CKB(cublasDgemm(ctx->cublas, CUBLAS_OP_N, CUBLAS_OP_N, Li, l, Li, &one, Tm, Li, Om, Li, &zero, Ys, Li));
    for (int q = 0; q < 2; ++q) {  // power iterations: (T T^T)^q T Omega, re-orthonormalised
      qr_inplace(ctx, Ys, Li, l);
      CKB(cublasDgemm(ctx->cublas, CUBLAS_OP_T, CUBLAS_OP_N, Li, l, Li, &one, Tm, Li, Ys, Li, &zero, Om, Li));
      qr_inplace(ctx, Om, Li, l);
      CKB(cublasDgemm(ctx->cublas, CUBLAS_OP_N, CUBLAS_OP_N, Li, l, Li, &one, Tm, Li, Om, Li, &zero, Ys, Li));
    }
    qr_inplace(ctx, Ys, Li, l);  // Q: range of T_o'
    Bt = Om;                     // B^T = T_o'^T Q  (L x l); B = Q^T T_o' = V S U^T, so the left singular
    CKB(cublasDgemm(ctx->cublas, CUBLAS_OP_T, CUBLAS_OP_N, Li, l, Li, &one, Tm, Li, Ys, Li, &zero, Bt, Li));
    Sv = dalloc<double>(ctx, l, false);  // vectors of B^T are T_o''s right singular vectors
    U = dalloc<double>(ctx, (size_t)L * l, false);
    dinfo = dalloc<int>(ctx, 1);
    int lwork = 0;
    CKS(cusolverDnDgesvd_bufferSize(ctx->cusolver, Li, l, &lwork));
    work = dalloc<double>(ctx, std::max(lwork, 1), false);
    rwork = dalloc<double>(ctx, l, false);
    signed char ju = 'S', jv = 'N';
    CKS(cusolverDnDgesvd(ctx->cusolver, ju, jv, Li, l, Bt, Li, Sv, U, Li, nullptr, 1, work, lwork, rwork, dinfo));
    int hinfo = 0;
    CK(cudaMemcpyAsync(&hinfo, dinfo, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (hinfo != 0) {
      set_err(ctx, "coarse space: gesvd info = %d", hinfo);
      throw Fail{LYAP_ECUDA};
    }
    dfree(Tm);
    Tm = nullptr;
    // 4. Z = the first p columns; T Z through K1.  Stored interleaved as one 2L x p column-major
    //    matrix [Z; T Z] (column i = [z_i; T z_i]): the engine forms Z w and T Z w with ONE GEMM
    double* TZt = dalloc<double>(ctx, (size_t)L * p, false);
    {
      const int rc = lyap_apply_C(ctx, p, U, nullptr, TZt, st);
      if (rc != LYAP_OK) {
        dfree(TZt);
        throw Fail{rc};
      }
      k_negate<<<(unsigned)std::min<int64_t>((L * p + 255) / 256, 65535), 256, 0, st>>>(TZt, L * p);
      LAUNCHED();
    }
    C.Z = dalloc<double>(ctx, (size_t)2 * L * p, false);
    C.TZ = C.Z + L;  // rows L..2L of every column (leading dimension 2L)
    CK(cudaMemcpy2DAsync(C.Z, 2 * L * 8, U, L * 8, L * 8, p, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpy2DAsync(C.Z + L, 2 * L * 8, TZt, L * 8, L * 8, p, cudaMemcpyDeviceToDevice, st));
    CK(cudaStreamSynchronize(st));
    dfree(TZt);
    // 5. Gram blocks per parameter t (row block t of Z / T Z)
    C.Phi = dalloc<double>(ctx, (size_t)k * p * p, false);
    C.Psi = dalloc<double>(ctx, (size_t)k * p * p, false);
    const int np = (int)s.npad;
    const int ld2 = 2 * Li;
    for (int64_t t = 0; t < k; ++t) {
      CKB(cublasDgemm(ctx->cublas, CUBLAS_OP_T, CUBLAS_OP_N, p, p, np, &one, C.Z + t * np, ld2, C.Z + t * np, ld2, &zero,
                      C.Phi + t * p * p, p));
      CKB(cublasDgemm(ctx->cublas, CUBLAS_OP_T, CUBLAS_OP_N, p, p, np, &one, C.Z + t * np, ld2, C.TZ + t * np, ld2,
                      &zero, C.Psi + t * p * p, p));
    }
    C.p = p;
    CK(cudaEventRecord(e1, st));
    CK(cudaEventSynchronize(e1));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    C.build_ms = ms;
    ctx->info.coarse = p;
    ctx->info.coarse_build_ms = ms;
  } catch (Fail f) {
    for (void* q : {(void*)Tm, (void*)X, (void*)Y, (void*)Om, (void*)Ys, (void*)Sv, (void*)U, (void*)work,
                    (void*)rwork, (void*)dinfo})
      dfree(q);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    throw;
  }
  for (void* q : {(void*)Tm, (void*)X, (void*)Y, (void*)Om, (void*)Ys, (void*)Sv, (void*)U, (void*)work, (void*)rwork,
                  (void*)dinfo})
    dfree(q);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
}

}  // namespace

// ====================================================================== C-ABI
extern "C" {

void lyap_default_opts(lyap_opts* o) {
  if (!o) return;
  std::memset(o, 0, sizeof *o);
  o->tol = 1e-12;
  o->max_dim = 0;
  o->max_restarts = 30;
  o->batch = 0;
  o->warm_start = 0;
  o->max_cond_S = 1e8;
  o->device = -1;
  o->profile = 0;
  o->schedule = 1;
  o->recycle = -1;
  o->check_stable = 0;
  o->coarse = -1;
  o->mixed = -1;
  o->mixed_eta = 1e-4;
}

const char* lyap_last_error(const lyap_ctx* c) { return c ? c->err.c_str() : g_last_error.c_str(); }

static void destroy_impl(lyap_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  free_engine(c->eng, false);
  Seed& s = c->seed;
  void* ps[] = {s.bhr, s.btl, s.F, s.Pb, s.g0, s.hf, s.dwork, s.t0t};  // lam, Lf, Sr, Qr belong to the shared Basis
  if (!c->basis) {  // setup failed before the Basis took ownership
    dfree(s.lam);
    dfree(s.Lf);
  }
  for (void* p : ps) dfree(p);
  if (c->cublas) cublasDestroy(c->cublas);
  if (c->cusolver) cusolverDnDestroy(c->cusolver);
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  dfree(c->Ureg);
  dfree(c->TUreg);
  dfree(c->sreg);
  c->basis.reset();
  if (c->stream) cudaStreamDestroy(c->stream);
  for (int gi = 1; gi < 4; ++gi) {
    if (c->xstream[gi]) cudaStreamDestroy(c->xstream[gi]);
    if (c->xjoin[gi]) cudaEventDestroy(c->xjoin[gi]);
  }
  dfree(c->Spad);
  for (double* q : {c->coarse.Z, c->coarse.Phi, c->coarse.Psi}) dfree(q);  // TZ lives inside Z
  for (int gi = 0; gi < 4; ++gi) {
    if (c->cublas_eng[gi]) cublasDestroy(c->cublas_eng[gi]);
    dfree(c->cublas_ws[gi]);
  }
  dfree(c->stab.wgrid);
  dfree(c->stab.Gf);
  dfree(c->stab.Mm);
  for (auto& ge : c->gexec)
    if (ge) cudaGraphExecDestroy(ge);
  for (auto& e : c->prof_evs) cudaEventDestroy(e);
  if (c->evfork) cudaEventDestroy(c->evfork);
  if (c->evjoin) cudaEventDestroy(c->evjoin);
  delete c;
}

void lyap_destroy(lyap_ctx* c) { destroy_impl(c); }

// nq = 0: one fixed Q (lyap_setup); nq = k: Q(v) = sum_i v_i Q_i (lyap_setup_qlin), Q holds nq matrices
static int setup_core(int64_t n, int64_t k, const double* A0, const double* Bl, const double* Br, const double* Q,
                      int nq, const double* E, const lyap_opts* opts, lyap_ctx** out) {
  lyap_ctx* ctx = nullptr;
  if (!out) {
    set_err(nullptr, "lyap_setup: out is NULL");
    return LYAP_EINVAL;
  }
  *out = nullptr;
  if (n < 1 || k < 1 || k > LYAP_KMAX || !A0 || !Bl || !Br || !Q || !E) {
    set_err(nullptr, "lyap_setup: invalid arguments (n=%lld, k=%lld, k must be 1..%d, no NULL inputs)",
            (long long)n, (long long)k, LYAP_KMAX);
    return LYAP_EINVAL;
  }
  const int nterms = nq > 0 ? nq : 1;
  for (int q = 0; q < nterms; ++q) {  // Q symmetric (the nk reduction needs Q = Q^T)
    const double* Qq = Q + (size_t)q * n * n;
    double mx = 0.0, asym = 0.0;
    for (int64_t i = 0; i < n; ++i)
      for (int64_t j = 0; j < n; ++j) {
        mx = std::max(mx, std::fabs(Qq[i * n + j]));
        asym = std::max(asym, std::fabs(Qq[i * n + j] - Qq[j * n + i]));
      }
    if (asym > 1e-13 * mx) {
      set_err(nullptr, "lyap_setup: Q is not symmetric (max |Q - Q^T| = %.3e, max |Q| = %.3e)", asym, mx);
      return LYAP_EINVAL;
    }
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    set_err(nullptr, "lyap_setup: no CUDA device (this library has no CPU path)");
    return LYAP_ENODEV;
  }
  ctx = new lyap_ctx();
  lyap_default_opts(&ctx->opts);
  if (opts) ctx->opts = *opts;
  if (!(ctx->opts.tol > 0)) ctx->opts.tol = 1e-12;
  if (ctx->opts.max_restarts <= 0) ctx->opts.max_restarts = 30;
  if (!(ctx->opts.max_cond_S > 0)) ctx->opts.max_cond_S = 1e8;
  if (!(ctx->opts.mixed_eta > 0 && ctx->opts.mixed_eta < 1)) ctx->opts.mixed_eta = 1e-4;
  // scratch
  double *dA = nullptr, *dBl = nullptr, *dBr = nullptr, *dQ = nullptr, *dE = nullptr, *Acm = nullptr, *Qs = nullptr,
         *Es = nullptr, *Blc = nullptr, *Brc = nullptr, *VR = nullptr, *Sr = nullptr, *Sinv = nullptr, *LU = nullptr,
         *T1 = nullptr, *Qr = nullptr, *Er = nullptr, *Blr = nullptr, *Brr = nullptr, *W = nullptr, *work = nullptr,
         *t0part = nullptr, *t0d = nullptr;
  int *perm = nullptr, *ipiv = nullptr, *dinfo = nullptr;
  unsigned long long* ext = nullptr;
  void* hwork = nullptr;
  int rc = LYAP_OK;
  try {
    int dev = ctx->opts.device;
    if (dev < 0) CK(cudaGetDevice(&dev));
    ctx->device = dev;
    CK(cudaSetDevice(dev));
    CK(cudaStreamCreateWithPriority(&ctx->stream, cudaStreamNonBlocking, stream_prio(true)));
    CK(cudaEventCreate(&ctx->ev0));
    CK(cudaEventCreate(&ctx->ev1));
    CKB(cublasCreate(&ctx->cublas));
    CKB(cublasSetStream(ctx->cublas, ctx->stream));
    CKS(cusolverDnCreate(&ctx->cusolver));
    CKS(cusolverDnSetStream(ctx->cusolver, ctx->stream));
    set_smem_attrs<G_BM, G_BN, G_WM, G_WN, G_ST, G_BK>(ctx);
    set_smem_attrs<S_BM, S_BN, S_WM, S_WN, S_ST, S_BK>(ctx);
    set_smem_attrs<V_BM, V_BN, V_WM, V_WN, V_ST, V_BK>(ctx);
    set_smem_attrs<V_BM, V_BN, V_WM, V_WN, 2, V_BK>(ctx);
    set_umma_attrs<UM_BN, UM_STAGES, UM_BKE>(ctx);
    set_umma_attrs<128, 3, 32>(ctx);
    set_umma_attrs<UM_BN, UM_STAGES, 32, 2>(ctx);
    set_umma_attrs<UM_BN, 3, 32, 2>(ctx);
    cudaStream_t st = ctx->stream;
    CK(cudaEventRecord(ctx->ev0, st));
    Seed& s = ctx->seed;
    s.n = n;
    s.k = k;
    s.nterms = nterms;
    s.qlin = nq > 0;
    s.npad = roundup(n, n <= SMALL_N ? S_BM : G_BM);
    const size_t nn = (size_t)n * n;
    dA = dalloc<double>(ctx, nn, false);
    dQ = dalloc<double>(ctx, nn * nterms, false);
    dE = dalloc<double>(ctx, nn, false);
    dBl = dalloc<double>(ctx, (size_t)n * k, false);
    dBr = dalloc<double>(ctx, (size_t)n * k, false);
    CK(cudaMemcpyAsync(dA, A0, nn * 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(dQ, Q, nn * nterms * 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(dE, E, nn * 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(dBl, Bl, (size_t)n * k * 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(dBr, Br, (size_t)n * k * 8, cudaMemcpyHostToDevice, st));
    Acm = dalloc<double>(ctx, nn, false);
    Qs = dalloc<double>(ctx, nn * nterms, false);
    Es = dalloc<double>(ctx, nn, false);
    Blc = dalloc<double>(ctx, (size_t)n * k, false);
    Brc = dalloc<double>(ctx, (size_t)n * k, false);
    const dim3 tb(32, 8);
    k_transpose<<<dim3((unsigned)((n + 31) / 32), (unsigned)((n + 31) / 32)), tb, 0, st>>>(dA, Acm, n, n);
    LAUNCHED();
    k_transpose<<<dim3((unsigned)((k + 31) / 32), (unsigned)((n + 31) / 32)), tb, 0, st>>>(dBl, Blc, n, k);
    LAUNCHED();
    k_transpose<<<dim3((unsigned)((k + 31) / 32), (unsigned)((n + 31) / 32)), tb, 0, st>>>(dBr, Brc, n, k);
    LAUNCHED();
    for (int q = 0; q < nterms; ++q) {
      k_symmetrize<<<(unsigned)((nn + 255) / 256), 256, 0, st>>>(dQ + q * nn, Qs + q * nn, n);
      LAUNCHED();
    }
    k_symmetrize<<<(unsigned)((nn + 255) / 256), 256, 0, st>>>(dE, Es, n);
    LAUNCHED();

    // ---- S1: eig(A0) on the device (real input, LAPACK-style real eigenvector packing)
    VR = dalloc<double>(ctx, nn, false);
    W = dalloc<double>(ctx, 2 * (size_t)n, false);
    dinfo = dalloc<int>(ctx, 1);
    cusolverDnParams_t params;
    CKS(cusolverDnCreateParams(&params));
    size_t dws = 0, hws = 0;
    CKS(cusolverDnXgeev_bufferSize(ctx->cusolver, params, CUSOLVER_EIG_MODE_NOVECTOR, CUSOLVER_EIG_MODE_VECTOR, n,
                                   CUDA_R_64F, Acm, n, CUDA_C_64F, W, CUDA_R_64F, nullptr, n, CUDA_R_64F, VR, n,
                                   CUDA_R_64F, &dws, &hws));
    void* dwork = nullptr;
    CK(cudaMalloc(&dwork, std::max<size_t>(dws, 8)));
    hwork = std::malloc(std::max<size_t>(hws, 8));
    cusolverStatus_t gs =
        cusolverDnXgeev(ctx->cusolver, params, CUSOLVER_EIG_MODE_NOVECTOR, CUSOLVER_EIG_MODE_VECTOR, n, CUDA_R_64F,
                        Acm, n, CUDA_C_64F, W, CUDA_R_64F, nullptr, n, CUDA_R_64F, VR, n, CUDA_R_64F, dwork, dws,
                        hwork, hws, dinfo);
    cudaStreamSynchronize(st);
    cudaFree(dwork);
    cusolverDnDestroyParams(params);
    if (gs != CUSOLVER_STATUS_SUCCESS) {
      set_err(ctx, "cusolverDnXgeev failed with status %d", (int)gs);
      throw Fail{LYAP_EEIG};
    }
    int hinfo = 0;
    CK(cudaMemcpy(&hinfo, dinfo, sizeof(int), cudaMemcpyDeviceToHost));
    if (hinfo != 0) {
      set_err(ctx, "cusolverDnXgeev info = %d", hinfo);
      throw Fail{LYAP_EEIG};
    }
    // ---- pairing map (host logic): conjugate pairs first (Re, Im coordinates), then reals
    std::vector<double> hW(2 * (size_t)n);
    CK(cudaMemcpy(hW.data(), W, 2 * (size_t)n * 8, cudaMemcpyDeviceToHost));
    std::vector<int> pairs, reals;
    for (int64_t i = 0; i < n;) {
      const double re = hW[2 * i], im = hW[2 * i + 1];
      if (im > 0.0 && i + 1 < n && hW[2 * (i + 1)] == re && hW[2 * (i + 1) + 1] == -im) {
        pairs.push_back((int)i);
        i += 2;
      } else if (im == 0.0) {
        reals.push_back((int)i);
        i += 1;
      } else {
        set_err(ctx, "eig(A0): eigenvalue %lld (%.17g, %.17g) is not part of a conjugate pair in LAPACK order",
                (long long)i, re, im);
        throw Fail{LYAP_EEIG};
      }
    }
    s.npairs = (int64_t)pairs.size();
    s.nrep = s.npairs + (int64_t)reals.size();
    const int64_t two_np = 2 * s.npairs;
    std::vector<int> hperm(n);
    std::vector<double> hlam(2 * (size_t)s.npad, 0.0);
    for (int64_t r = 0; r < s.npairs; ++r) {
      const int i = pairs[r];
      hperm[2 * r] = i;
      hperm[2 * r + 1] = i + 1;
      for (int q = 0; q < 2; ++q) {
        hlam[2 * (2 * r + q)] = hW[2 * i];
        hlam[2 * (2 * r + q) + 1] = hW[2 * i + 1];
      }
    }
    for (size_t r = 0; r < reals.size(); ++r) {
      const int i = reals[r];
      hperm[two_np + r] = i;
      hlam[2 * (two_np + r)] = hW[2 * i];
      hlam[2 * (two_np + r) + 1] = 0.0;
    }
    perm = dalloc<int>(ctx, n, false);
    CK(cudaMemcpy(perm, hperm.data(), n * sizeof(int), cudaMemcpyHostToDevice));
    s.lam = dalloc<double>(ctx, 2 * (size_t)s.npad);
    CK(cudaMemcpy(s.lam, hlam.data(), 2 * (size_t)s.npad * 8, cudaMemcpyHostToDevice));
    Sr = dalloc<double>(ctx, nn, false);
    k_gather_cols<<<dim3((unsigned)((n + 255) / 256), (unsigned)n), 256, 0, st>>>(VR, perm, Sr, n);
    LAUNCHED();

    // ---- S2: S_r^{-1} (LU)
    LU = dalloc<double>(ctx, nn, false);
    Sinv = dalloc<double>(ctx, nn, false);
    ipiv = dalloc<int>(ctx, n, false);
    CK(cudaMemcpyAsync(LU, Sr, nn * 8, cudaMemcpyDeviceToDevice, st));
    int lwork = 0;
    CKS(cusolverDnDgetrf_bufferSize(ctx->cusolver, (int)n, (int)n, LU, (int)n, &lwork));
    work = dalloc<double>(ctx, std::max(lwork, 1), false);
    CKS(cusolverDnDgetrf(ctx->cusolver, (int)n, (int)n, LU, (int)n, work, ipiv, dinfo));
    k_set_identity<<<(unsigned)((nn + 255) / 256), 256, 0, st>>>(Sinv, n);
    LAUNCHED();
    CKS(cusolverDnDgetrs(ctx->cusolver, CUBLAS_OP_N, (int)n, (int)n, LU, (int)n, ipiv, Sinv, (int)n, dinfo));
    CK(cudaMemcpyAsync(&hinfo, dinfo, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (hinfo != 0) {
      set_err(ctx, "eigenvector matrix S is singular (getrf/getrs info = %d)", hinfo);
      throw Fail{LYAP_EEIG};
    }
    ext = dalloc<unsigned long long>(ctx, 4);
    k_norm1<<<(unsigned)n, 256, 0, st>>>(Sr, n, ext);
    LAUNCHED();
    k_norm1<<<(unsigned)n, 256, 0, st>>>(Sinv, n, ext + 1);
    LAUNCHED();
    // ---- S3-S5: real n^3 products (cuBLAS DGEMM, column-major)
    T1 = dalloc<double>(ctx, nn, false);
    Qr = dalloc<double>(ctx, nn * nterms, false);
    Er = dalloc<double>(ctx, nn, false);
    Blr = dalloc<double>(ctx, (size_t)n * k, false);
    Brr = dalloc<double>(ctx, (size_t)n * k, false);
    const double one = 1.0, zero = 0.0;
    const int ni = (int)n, ki = (int)k;
    for (int q = 0; q < nterms; ++q) {
      CKB(cublasDgemm(ctx->cublas, CUBLAS_OP_N, CUBLAS_OP_N, ni, ni, ni, &one, Sinv, ni, Qs + q * nn, ni, &zero, T1, ni));
      CKB(cublasDgemm(ctx->cublas, CUBLAS_OP_N, CUBLAS_OP_T, ni, ni, ni, &one, T1, ni, Sinv, ni, &zero, Qr + q * nn,
                      ni));
    }
    CKB(cublasDgemm(ctx->cublas, CUBLAS_OP_T, CUBLAS_OP_N, ni, ni, ni, &one, Sr, ni, Es, ni, &zero, T1, ni));
    CKB(cublasDgemm(ctx->cublas, CUBLAS_OP_N, CUBLAS_OP_N, ni, ni, ni, &one, T1, ni, Sr, ni, &zero, Er, ni));
    // ---- eigenvalue extremes
    {
      unsigned long long big = 0x7fefffffffffffffULL;  // DBL_MAX bits
      CK(cudaMemcpyAsync(ext + 2, &big, 8, cudaMemcpyHostToDevice, st));
      k_lam_extremes<<<dim3((unsigned)std::min<int64_t>((n + 255) / 256, 64), (unsigned)n), 256, 0, st>>>(
          s.lam, n, two_np, ext + 2, ext + 3);
      LAUNCHED();
    }
    s.Lf = dalloc<double>(ctx, (size_t)s.npad * s.npad, false);
    k_build_Lf<<<dim3((unsigned)((s.npad + 255) / 256), (unsigned)s.npad), 256, 0, st>>>(s.lam, n, s.npad, two_np,
                                                                                        s.Lf);
    LAUNCHED();
    // the A0-only state becomes a shared Basis (lyap_setup_like reuses it)
    ctx->basis = std::make_shared<Basis>();
    ctx->basis->device = ctx->device;
    ctx->basis->lam = s.lam;
    ctx->basis->Lf = s.Lf;
    ctx->basis->Sr = Sr;
    ctx->basis->Sinv = Sinv;
    ctx->basis->Qr = Qr;
    ctx->basis->Er = Er;
    s.Sr = Sr;
    s.Qr = Qr;
    Sr = Sinv = Qr = Er = nullptr;
    (void)ki;
    unsigned long long hext[4];
    CK(cudaMemcpyAsync(hext, ext, sizeof hext, cudaMemcpyDeviceToHost, st));
    CK(cudaEventRecord(ctx->ev1, st));
    CK(cudaStreamSynchronize(st));
    double n1S, n1Si, mins, maxl;
    std::memcpy(&n1S, &hext[0], 8);
    std::memcpy(&n1Si, &hext[1], 8);
    std::memcpy(&mins, &hext[2], 8);
    std::memcpy(&maxl, &hext[3], 8);
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
    lyap_info& in = ctx->info;
    in.n = n;
    in.k = k;
    in.npad = s.npad;
    in.n_pairs = s.npairs;
    in.t0 = s.t0;
    in.cond_S = n1S * n1Si;
    in.min_lam_sum = mins;
    in.max_abs_lam = maxl;
    in.setup_ms = ms;
    if (!(in.cond_S <= ctx->opts.max_cond_S)) {
      set_err(ctx, "eigenvector basis too ill-conditioned: cond_1(S_r) = %.3e > %.3e", in.cond_S,
              ctx->opts.max_cond_S);
      throw Fail{LYAP_EEIG};
    }
    if (!(mins > 1e-12 * maxl)) {
      set_err(ctx, "seed Lyapunov operator singular: min |lambda_i + lambda_j| = %.3e (max |lambda| = %.3e)", mins,
              maxl);
      throw Fail{LYAP_ESINGULAR};
    }
    build_config(ctx, Blc, Brc);  // (Bl, Br)-dependent part
    CK(cudaEventRecord(ctx->ev1, st));
    CK(cudaEventSynchronize(ctx->ev1));
    CK(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
    in.setup_ms = ms;
  } catch (Fail f) {
    rc = f.code;
  }
  void* tmp[] = {dA, dBl, dBr, dQ, dE, Acm, Qs, Es, Blc, Brc, VR, Sr, Sinv, LU, T1, Qr, Er, Blr, Brr, W, work,
                 t0part, t0d, perm, ipiv, dinfo, ext};
  for (void* p : tmp) dfree(p);
  std::free(hwork);
  if (rc != LYAP_OK) {
    g_last_error = ctx->err;
    destroy_impl(ctx);
    return rc;
  }
  *out = ctx;
  return LYAP_OK;
}

int lyap_setup(int64_t n, int64_t k, const double* A0, const double* Bl, const double* Br, const double* Q,
               const double* E, const lyap_opts* opts, lyap_ctx** out) {
  return setup_core(n, k, A0, Bl, Br, Q, 0, E, opts, out);
}

int lyap_setup_qlin(int64_t n, int64_t k, const double* A0, const double* Bl, const double* Br, const double* Qk,
                    const double* E, const lyap_opts* opts, lyap_ctx** out) {
  return setup_core(n, k, A0, Bl, Br, Qk, (int)k, E, opts, out);
}

int lyap_setup_like(const lyap_ctx* base, int64_t k, const double* Bl, const double* Br, const lyap_opts* opts,
                    lyap_ctx** out) {
  lyap_ctx* ctx = nullptr;
  if (!out || !base || !base->basis || k < 1 || k > LYAP_KMAX || !Bl || !Br || base->seed.qlin) {
    set_err(nullptr, "lyap_setup_like: invalid arguments (base with a basis, k = 1..%d, non-NULL Bl, Br)", LYAP_KMAX);
    return LYAP_EINVAL;
  }
  *out = nullptr;
  ctx = new lyap_ctx();
  ctx->opts = opts ? *opts : base->opts;
  if (!(ctx->opts.tol > 0)) ctx->opts.tol = 1e-12;
  if (ctx->opts.max_restarts <= 0) ctx->opts.max_restarts = 30;
  ctx->device = base->device;
  ctx->basis = base->basis;
  double *dBl = nullptr, *dBr = nullptr, *Blc = nullptr, *Brc = nullptr;
  int rc = LYAP_OK;
  try {
    CK(cudaSetDevice(ctx->device));
    CK(cudaStreamCreateWithPriority(&ctx->stream, cudaStreamNonBlocking, stream_prio(true)));
    CK(cudaEventCreate(&ctx->ev0));
    CK(cudaEventCreate(&ctx->ev1));
    CKB(cublasCreate(&ctx->cublas));
    CKB(cublasSetStream(ctx->cublas, ctx->stream));
    CKS(cusolverDnCreate(&ctx->cusolver));
    CKS(cusolverDnSetStream(ctx->cusolver, ctx->stream));
    cudaStream_t st = ctx->stream;
    CK(cudaEventRecord(ctx->ev0, st));
    Seed& s = ctx->seed;
    const Seed& b = base->seed;
    s.n = b.n;
    s.k = k;
    s.npad = b.npad;
    s.npairs = b.npairs;
    s.nrep = b.nrep;
    s.lam = ctx->basis->lam;
    s.Lf = ctx->basis->Lf;
    s.Sr = ctx->basis->Sr;
    s.Qr = ctx->basis->Qr;
    const int64_t n = s.n;
    dBl = dalloc<double>(ctx, (size_t)n * k, false);
    dBr = dalloc<double>(ctx, (size_t)n * k, false);
    Blc = dalloc<double>(ctx, (size_t)n * k, false);
    Brc = dalloc<double>(ctx, (size_t)n * k, false);
    CK(cudaMemcpyAsync(dBl, Bl, (size_t)n * k * 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(dBr, Br, (size_t)n * k * 8, cudaMemcpyHostToDevice, st));
    const dim3 tb(32, 8);
    k_transpose<<<dim3((unsigned)((k + 31) / 32), (unsigned)((n + 31) / 32)), tb, 0, st>>>(dBl, Blc, n, k);
    LAUNCHED();
    k_transpose<<<dim3((unsigned)((k + 31) / 32), (unsigned)((n + 31) / 32)), tb, 0, st>>>(dBr, Brc, n, k);
    LAUNCHED();
    ctx->info = base->info;
    ctx->info.k = k;
    ctx->info.coarse = 0;  // this configuration builds its own coarse space on first use
    ctx->info.coarse_build_ms = 0.0;
    build_config(ctx, Blc, Brc);
    CK(cudaEventRecord(ctx->ev1, st));
    CK(cudaEventSynchronize(ctx->ev1));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
    ctx->info.setup_ms = ms;
  } catch (Fail f) {
    rc = f.code;
  }
  for (void* p : {(void*)dBl, (void*)dBr, (void*)Blc, (void*)Brc}) dfree(p);
  if (rc != LYAP_OK) {
    g_last_error = ctx->err;
    destroy_impl(ctx);
    return rc;
  }
  *out = ctx;
  return LYAP_OK;
}

static int trace_batch_impl(lyap_ctx* ctx, int64_t nv, const double* V, double* traces, int32_t* status,
                            int32_t* applies, double* resid, int v_on_device, void* cuda_stream, const double* x0,
                            double* xout) {
  if (!ctx) {
    set_err(nullptr, "lyap_trace_batch: ctx is NULL");
    return LYAP_EINVAL;
  }
  if (nv < 0 || (nv > 0 && (!V || !traces)) || nv > (int64_t)INT32_MAX) {
    set_err(ctx, "lyap_trace_batch: invalid arguments (nv=%lld)", (long long)nv);
    return LYAP_EINVAL;
  }
  if (nv == 0) return LYAP_OK;
  double *dV = nullptr, *dtr = nullptr, *dres = nullptr;
  int32_t *dst = nullptr, *dap = nullptr, *own_nu = nullptr;
  bool own = !v_on_device;
  int rc = LYAP_OK;
  try {
    CK(cudaSetDevice(ctx->device));
    cudaStream_t st = v_on_device ? (cudaStream_t)cuda_stream : ctx->stream;
    const int64_t k = ctx->seed.k;
    if (own) {
      dV = dalloc<double>(ctx, (size_t)nv * k, false);
      dtr = dalloc<double>(ctx, nv, false);
      dst = dalloc<int32_t>(ctx, nv, false);
      if (applies) dap = dalloc<int32_t>(ctx, nv, false);
      if (resid) dres = dalloc<double>(ctx, nv, false);
      CK(cudaMemcpyAsync(dV, V, (size_t)nv * k * 8, cudaMemcpyHostToDevice, st));
    } else {
      dV = const_cast<double*>(V);
      dtr = traces;
      dst = status;
      dap = applies;
      dres = resid;
    }
    // schedule (device-side, on the call's stream; V never visits the host): expensive
    // (large-perturbation) v first, so slow systems do not form a tail (sched.cuh)
    const int* dorder = nullptr;
    const int s_auto = ctx->opts.recycle < 0 ? 0 : ctx->opts.recycle;
    Seed& sd = ctx->seed;
    ensure_dwork(ctx);
    if (s_auto > 0 && !ctx->recycle_manual && !mp_mode(ctx)) {
      // automatic recycle spaces from the corners of the batch's bounding box: the 2k box bounds are
      // the only host read of the call before the engine runs
      k_box<<<(unsigned)k, 256, 0, st>>>(dV, (int)nv, (int)k, sd.dwork + 8);
      LAUNCHED();
      std::vector<double> box(2 * k);
      CK(cudaMemcpyAsync(box.data(), sd.dwork + 8, sizeof(double) * 2 * k, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      bool positive = true, inside = !ctx->auto_box.empty();
      for (int64_t t = 0; t < k; ++t) {
        positive = positive && box[2 * t] > 0.0;
        if (inside) inside = box[2 * t] >= ctx->auto_box[2 * t] && box[2 * t + 1] <= ctx->auto_box[2 * t + 1];
      }
      // rebuild only for a box the current spaces do not cover (optimizer-style callers pass a new,
      // usually nested, box on every call)
      if (positive && !inside) {
        std::vector<double> seeds;
        for (int64_t c = 0; c < (int64_t(1) << k); ++c) {
          std::vector<double> v(k);
          for (int64_t t = 0; t < k; ++t) v[t] = box[2 * t + ((c >> (k - 1 - t)) & 1)];
          bool dup = false;  // a degenerate box (lo == hi on an axis) repeats corners
          for (size_t q = 0; q + k <= seeds.size() && !dup; q += k)
            dup = std::equal(v.begin(), v.end(), seeds.begin() + q);
          if (!dup) seeds.insert(seeds.end(), v.begin(), v.end());
        }
        const int brc = lyap_build_recycle(ctx, (int32_t)(seeds.size() / k), seeds.data(), s_auto);
        if (brc != LYAP_OK) throw Fail{brc};
        ctx->recycle_manual = false;  // automatic: rebuilt when a batch leaves the box
        ctx->auto_box = box;
      }
    }
    // stability filter (opts.check_stable): unstable v are marked and not solved
    int32_t* dnu = nullptr;
    int64_t nv_run = nv;
    if (ctx->opts.check_stable) {
      dnu = dalloc<int32_t>(ctx, nv, false);
      own_nu = dnu;
      stab_count(ctx, nv, dV, dnu, st);
      int* dcount = reinterpret_cast<int*>(sd.dwork + 16);  // scratch slot
      k_mark_unstable<<<1, 1024, 0, st>>>(dnu, (int)nv, dtr, dst, dap, dres, dcount);
      LAUNCHED();
      int hc = 0;
      CK(cudaMemcpyAsync(&hc, dcount, sizeof(int), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      nv_run = hc;
    }
    if (ctx->opts.schedule || dnu) {
      Engine& g = ctx->eng;
      if (g.sched_cap < nv || !g.order || !g.regq) {
        for (void* p : {(void*)g.order, (void*)g.regq, (void*)g.skey, (void*)g.skey2, (void*)g.sidx, g.cub_tmp}) dfree(p);
        g.order = g.regq = g.sidx = nullptr;
        g.skey = g.skey2 = nullptr;
        g.cub_tmp = nullptr;
        g.sched_cap = g.order_cap = g.regq_cap = 0;
        g.order = dalloc<int>(ctx, nv, false);
        g.regq = dalloc<int>(ctx, nv, false);
        g.sidx = dalloc<int>(ctx, nv, false);
        g.skey = dalloc<double>(ctx, nv, false);
        g.skey2 = dalloc<double>(ctx, nv, false);
        g.cub_bytes = 0;
        CK(cub::DeviceRadixSort::SortPairsDescending(nullptr, g.cub_bytes, g.skey, g.skey2, g.sidx, g.order, (int)nv,
                                                     0, 64, st));
        g.cub_tmp = dalloc<char>(ctx, g.cub_bytes, false);
        g.sched_cap = g.order_cap = g.regq_cap = nv;
      }
      const unsigned nb = (unsigned)std::min<int64_t>((nv + 255) / 256, 4096);
      k_cost<<<nb, 256, 0, st>>>(dV, (int)nv, (int)k, sd.dwork, dnu, g.skey, g.sidx);
      LAUNCHED();
      // stable descending radix sort: equal costs keep row order (the host std::stable_sort order)
      size_t bytes = g.cub_bytes;
      CK(cub::DeviceRadixSort::SortPairsDescending(g.cub_tmp, bytes, g.skey, g.skey2, g.sidx, g.order, (int)nv, 0, 64,
                                                   st));
      dorder = g.order;
      if (ctx->nreg > 0) {  // nearest regime seed in log|v|
        k_regime<<<nb, 256, 0, st>>>(dV, g.order, (int)nv, (int)k, sd.dwork + 32, ctx->nreg, g.regq);
        LAUNCHED();
      }
    }
    rc = nv_run > 0 ? run_batch(ctx, nv_run, dV, dorder, dtr, dst, dap, dres, st, xout,
                                (ctx->nreg > 0 && dorder) ? ctx->eng.regq : nullptr, 0, x0)
                    : LYAP_OK;
    if (rc == LYAP_OK) {
      // any per-v failure -> LYAP_EPARTIAL
      std::vector<int32_t> hs;
      const int32_t* sp = nullptr;
      if (own) {
        CK(cudaMemcpyAsync(traces, dtr, nv * 8, cudaMemcpyDeviceToHost, st));
        if (applies) CK(cudaMemcpyAsync(applies, dap, nv * 4, cudaMemcpyDeviceToHost, st));
        if (resid) CK(cudaMemcpyAsync(resid, dres, nv * 8, cudaMemcpyDeviceToHost, st));
        hs.resize(nv);
        CK(cudaMemcpyAsync(hs.data(), dst, nv * 4, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (status) std::memcpy(status, hs.data(), nv * 4);
        sp = hs.data();
      } else if (status) {
        hs.resize(nv);
        CK(cudaMemcpyAsync(hs.data(), status, nv * 4, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        sp = hs.data();
      }
      if (sp)
        for (int64_t i = 0; i < nv; ++i)
          if (sp[i] != 0 && sp[i] != LYAP_V_UNSTABLE) {  // a filtered v is not a failure
            rc = LYAP_EPARTIAL;
            set_err(ctx, "v %lld: status %d", (long long)i, (int)sp[i]);
            break;
          }
    }
  } catch (Fail f) {
    rc = f.code;
  }
  if (own) {
    dfree(dV);
    dfree(dtr);
    dfree(dst);
    dfree(dap);
    dfree(dres);
  }
  dfree(own_nu);
  return rc;
}

int lyap_trace_batch_ex(lyap_ctx* ctx, int64_t nv, const double* V, double* traces, int32_t* status,
                        int32_t* applies, double* resid, int v_on_device, void* cuda_stream) {
  return trace_batch_impl(ctx, nv, V, traces, status, applies, resid, v_on_device, cuda_stream, nullptr, nullptr);
}

int lyap_trace_batch_x(lyap_ctx* ctx, int64_t nv, const double* V, const double* X0, double* Xout, double* traces,
                       int32_t* status, int32_t* applies, double* resid, void* cuda_stream) {
  return trace_batch_impl(ctx, nv, V, traces, status, applies, resid, 1, cuda_stream, X0, Xout);
}

int lyap_stable_batch(lyap_ctx* ctx, int64_t nv, const double* V, int32_t* nunstable, int v_on_device,
                      void* cuda_stream) {
  if (!ctx || nv < 0 || (nv > 0 && (!V || !nunstable))) {
    set_err(ctx, "lyap_stable_batch: invalid arguments");
    return LYAP_EINVAL;
  }
  if (nv == 0) return LYAP_OK;
  double* dV = nullptr;
  int32_t* dnu = nullptr;
  int rc = LYAP_OK;
  try {
    CK(cudaSetDevice(ctx->device));
    cudaStream_t st = v_on_device ? (cudaStream_t)cuda_stream : ctx->stream;
    if (v_on_device) {
      stab_count(ctx, nv, V, nunstable, st);
    } else {
      dV = dalloc<double>(ctx, (size_t)nv * ctx->seed.k, false);
      dnu = dalloc<int32_t>(ctx, nv, false);
      CK(cudaMemcpyAsync(dV, V, (size_t)nv * ctx->seed.k * 8, cudaMemcpyHostToDevice, st));
      stab_count(ctx, nv, dV, dnu, st);
      CK(cudaMemcpyAsync(nunstable, dnu, nv * 4, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
    }
  } catch (Fail f) {
    rc = f.code;
  }
  dfree(dV);
  dfree(dnu);
  return rc;
}

int lyap_trace_batch(lyap_ctx* ctx, int64_t nv, const double* V, double* traces, int32_t* status,
                     int v_on_device, void* cuda_stream) {
  return lyap_trace_batch_ex(ctx, nv, V, traces, status, nullptr, nullptr, v_on_device, cuda_stream);
}

}  // extern "C"

namespace {
// Full solutions X(v) (n x n, row-major) of the nv rows of the DEVICE array dV, chunk by chunk
// (DESIGN.md §2.5): the engine solves every v (gout: the folded g), then per chunk Y_v is generated
// entrywise and X_v = S_r Y_v S_r^T comes from two batched DMMA GEMMs (k1_dgemm): T1 = [Y_1; ...] S_r^T
// written horizontally, X = S_r [T1_1 | ...] written compactly.  sink(v0, count, Xc) consumes each
// chunk (device, count x n x n) on ctx->stream.  Returns the engine status; hs gets the per-v codes,
// dtr (device, nullable) the traces.  Throws Fail.
template <class Sink>
int solution_chunks(lyap_ctx* ctx, int64_t nv, const double* dV, double* dtr, std::vector<int32_t>& hs, Sink sink) {
  const Seed& s = ctx->seed;
  cudaStream_t st = ctx->stream;
  const int64_t n = s.n, L = s.k * s.npad, np = roundup(n, G_BM);
  double *gout = nullptr, *Yst = nullptr, *T1 = nullptr, *Xc = nullptr, *dtr_own = nullptr;
  int32_t* dst = nullptr;
  int rc = LYAP_OK;
  try {
    gout = dalloc<double>(ctx, (size_t)nv * L);
    dst = dalloc<int32_t>(ctx, nv, false);
    if (!dtr) dtr = dtr_own = dalloc<double>(ctx, nv, false);
    rc = run_batch(ctx, nv, dV, nullptr, dtr, dst, nullptr, nullptr, st, gout);
    if (rc == LYAP_OK) {
      hs.resize(nv);
      CK(cudaMemcpyAsync(hs.data(), dst, nv * 4, cudaMemcpyDeviceToHost, st));
      if (!ctx->Spad) {
        ctx->Spad = dalloc<double>(ctx, 2 * (size_t)np * np, false);
        k_pad_basis<<<dim3((unsigned)((np + 255) / 256), (unsigned)np), 256, 0, st>>>(s.Sr, n, np, ctx->Spad,
                                                                                      ctx->Spad + np * np);
        LAUNCHED();
        CK(cudaFuncSetAttribute(k1_dgemm<G_BM, G_BN, G_WM, G_WN, G_ST, G_BK, 1>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GCfg::SMEM));
        CK(cudaFuncSetAttribute(k1_dgemm<G_BM, G_BN, G_WM, G_WN, G_ST, G_BK, 2>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GCfg::SMEM));
      }
      const double* Sc = ctx->Spad;              // S_r^T (row-major)
      const double* Srow = ctx->Spad + np * np;  // S_r (row-major)
      const int64_t per_v = np * np * 8;
      const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(nv, ((int64_t)1 << 30) / per_v));
      Yst = dalloc<double>(ctx, (size_t)chunk * np * np);  // zero padding stays zero
      T1 = dalloc<double>(ctx, (size_t)chunk * np * np, false);
      Xc = dalloc<double>(ctx, (size_t)chunk * n * n, false);
      for (int64_t v0 = 0; v0 < nv; v0 += chunk) {
        const int64_t bc = std::min(chunk, nv - v0);
        k_solution_Ystack<<<dim3((unsigned)((n + 127) / 128), (unsigned)n, (unsigned)bc), 128, 0, st>>>(
            s.lam, s.Qr, s.btl, gout + v0 * L, n, s.npad, s.k, 2 * s.npairs, np, Yst, dV, v0, s.qlin ? s.nterms : 0);
        LAUNCHED();
        DgemmOut o1{(int)np, (int)bc, (int)n};
        k1_dgemm<G_BM, G_BN, G_WM, G_WN, G_ST, G_BK, 1>
            <<<(unsigned)((np / G_BN) * (bc * np / G_BM)), GCfg::THREADS, GCfg::SMEM, st>>>(
                Yst, Sc, T1, (int)(bc * np), (int)np, (int)np, (int)np, nullptr, 1, o1);
        LAUNCHED();
        DgemmOut o2{(int)np, (int)bc, (int)n};
        k1_dgemm<G_BM, G_BN, G_WM, G_WN, G_ST, G_BK, 2>
            <<<(unsigned)((bc * np / G_BN) * (np / G_BM)), GCfg::THREADS, GCfg::SMEM, st>>>(
                Srow, T1, Xc, (int)np, (int)(bc * np), (int)np, (int)np, nullptr, 1, o2);
        LAUNCHED();
        sink(v0, bc, Xc);
      }
      CK(cudaStreamSynchronize(st));
    }
  } catch (Fail f) {
    rc = f.code;
  }
  for (void* p : {(void*)gout, (void*)Yst, (void*)T1, (void*)Xc, (void*)dst, (void*)dtr_own}) dfree(p);
  return rc;
}
}  // namespace

extern "C" {

int lyap_solution(lyap_ctx* ctx, int64_t nv, const double* V, double* X, double* traces) {
  if (!ctx || nv < 0 || (nv > 0 && (!V || !X))) {
    set_err(ctx, "lyap_solution: invalid arguments");
    return LYAP_EINVAL;
  }
  if (nv == 0) return LYAP_OK;
  const Seed& s = ctx->seed;
  double *dV = nullptr, *dtr = nullptr;
  int rc = LYAP_OK;
  try {
    CK(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    const int64_t n = s.n;
    dV = dalloc<double>(ctx, (size_t)nv * s.k, false);
    dtr = dalloc<double>(ctx, nv, false);
    CK(cudaMemcpyAsync(dV, V, (size_t)nv * s.k * 8, cudaMemcpyHostToDevice, st));
    std::vector<int32_t> hs;
    rc = solution_chunks(ctx, nv, dV, dtr, hs, [&](int64_t v0, int64_t bc, const double* Xc) {
      CK(cudaMemcpyAsync(X + v0 * n * n, Xc, (size_t)bc * n * n * 8, cudaMemcpyDeviceToHost, st));
    });
    if (rc == LYAP_OK) {
      if (traces) CK(cudaMemcpyAsync(traces, dtr, nv * 8, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      for (int64_t v = 0; v < nv; ++v)
        if (hs[v] != 0) {
          rc = LYAP_EPARTIAL;
          set_err(ctx, "v %lld: status %d", (long long)v, (int)hs[v]);
          break;
        }
    }
  } catch (Fail f) {
    rc = f.code;
  }
  dfree(dV);
  dfree(dtr);
  return rc;
}

int lyap_set_recycle(lyap_ctx* ctx, int32_t nreg, int32_t s, const double* U, const double* seeds) {
  if (ctx && nreg > 0 && mp_mode(ctx)) {
    set_err(ctx, "lyap_set_recycle: recycle spaces need the FP64 engine (opts.mixed = 0)");
    return LYAP_EINVAL;
  }
  if (ctx) ctx->recycle_manual = nreg > 0;  // user-managed spaces: no automatic rebuild
  if (!ctx || nreg < 0 || (nreg > 0 && (s < 1 || !U || !seeds))) {
    set_err(ctx, "lyap_set_recycle: invalid arguments");
    return LYAP_EINVAL;
  }
  try {
    CK(cudaSetDevice(ctx->device));
    dfree(ctx->Ureg);
    dfree(ctx->TUreg);
    ctx->Ureg = ctx->TUreg = nullptr;
    ctx->nreg = ctx->s_rec = 0;
    if (nreg == 0) return LYAP_OK;
    const Seed& sd = ctx->seed;
    const int mmax = auto_mmax(ctx);
    if (s > mmax - 8) {
      set_err(ctx, "lyap_set_recycle: s = %d must leave room in the restart length %d", s, mmax);
      return LYAP_EINVAL;
    }
    const int64_t L = sd.k * sd.npad, tot = (int64_t)nreg * s;
    cudaStream_t st = ctx->stream;
    ctx->Ureg = dalloc<double>(ctx, (size_t)tot * L, false);
    ctx->TUreg = dalloc<double>(ctx, (size_t)tot * L, false);
    CK(cudaMemcpyAsync(ctx->Ureg, U, (size_t)tot * L * 8, cudaMemcpyHostToDevice, st));
    // T U once (K1 with sigma = 0 gives -T U)
    CK(lyap_apply_C(ctx, tot, ctx->Ureg, nullptr, ctx->TUreg, st) == LYAP_OK ? cudaSuccess : cudaErrorUnknown);
    k_negate<<<(unsigned)std::min<int64_t>((tot * L + 255) / 256, 65535), 256, 0, st>>>(ctx->TUreg, tot * L);
    LAUNCHED();
    CK(cudaStreamSynchronize(st));
    std::vector<double> ls((size_t)nreg * sd.k);
    for (size_t i = 0; i < ls.size(); ++i) ls[i] = std::log(std::fabs(seeds[i]) + 1e-300);
    ctx->reg_seeds.assign(reinterpret_cast<const char*>(ls.data()), ls.size() * sizeof(double));
    upload_seeds(ctx);
    dfree(ctx->sreg);
    ctx->sreg = dalloc<int>(ctx, nreg, false);
    std::vector<int> hsz(nreg, s);
    CK(cudaMemcpy(ctx->sreg, hsz.data(), nreg * sizeof(int), cudaMemcpyHostToDevice));
    ctx->nreg = nreg;
    ctx->s_rec = s;
  } catch (Fail f) {
    return f.code;
  }
  return LYAP_OK;
}

static int build_recycle_impl(lyap_ctx* ctx, int32_t nseeds, const double* seeds, int32_t s);

int lyap_build_recycle(lyap_ctx* ctx, int32_t nseeds, const double* seeds, int32_t s) {
  if (ctx && mp_mode(ctx)) {
    set_err(ctx, "lyap_build_recycle: recycle spaces need the FP64 engine (opts.mixed = 0)");
    return LYAP_EINVAL;
  }
  if (!ctx || nseeds < 1 || !seeds || s < 1) {
    set_err(ctx, "lyap_build_recycle: invalid arguments");
    return LYAP_EINVAL;
  }
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, ctx->stream);
  const int rc = build_recycle_impl(ctx, nseeds, seeds, s);
  ctx->recycle_manual = rc == LYAP_OK;
  cudaEventRecord(e1, ctx->stream);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  ctx->stats.recycle_build_ms += ms;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (rc != LYAP_OK) ctx->auto_box.clear();
  return rc;
}

// 1 = select from plain GMRES cycles; 2 = plus one refinement pass.  The environment
// variable LYAP_RECYCLE_ROUNDS (1..4) overrides it, for measurements.
static int recycle_rounds() {
  const char* e = std::getenv("LYAP_RECYCLE_ROUNDS");
  const int r = e ? std::atoi(e) : 2;
  return r < 1 ? 1 : (r > 4 ? 4 : r);
}

static int build_recycle_impl(lyap_ctx* ctx, int32_t nseeds, const double* seeds, int32_t s) {
  const Seed& sd = ctx->seed;
  const int64_t k = sd.k, L = sd.k * sd.npad;
  for (int64_t i = 0; i < (int64_t)nseeds * k; ++i)
    if (!(seeds[i] != 0.0) || !std::isfinite(seeds[i])) {
      set_err(ctx, "lyap_build_recycle: seed parameters must be finite and non-zero");
      return LYAP_EINVAL;
    }
  const int mmax = auto_mmax(ctx);
  if (s > mmax - 8) {
    set_err(ctx, "lyap_build_recycle: s = %d must leave room in the restart length %d", s, mmax);
    return LYAP_EINVAL;
  }
  double *dV = nullptr, *dtr = nullptr, *Z = nullptr, *Qn = nullptr, *Am = nullptr, *Bm = nullptr, *Wv = nullptr,
         *work = nullptr, *HP = nullptr, *CU = nullptr, *sig = nullptr, *Unew = nullptr, *TUnew = nullptr;
  int32_t* dst = nullptr;
  int *dinfo = nullptr, *dreg = nullptr;
  int rc = LYAP_OK;
  try {
    CK(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    dfree(ctx->Ureg);
    dfree(ctx->TUreg);
    dfree(ctx->sreg);
    ctx->Ureg = ctx->TUreg = nullptr;
    ctx->sreg = nullptr;
    ctx->nreg = ctx->s_rec = 0;
    dV = dalloc<double>(ctx, (size_t)nseeds * k, false);
    dtr = dalloc<double>(ctx, nseeds, false);
    dst = dalloc<int32_t>(ctx, nseeds, false);
    dreg = dalloc<int>(ctx, nseeds, false);
    const int ld = mmax + 1;
    Z = dalloc<double>(ctx, (size_t)mmax * L);
    Qn = dalloc<double>(ctx, (size_t)(mmax + 1) * L, false);
    Am = dalloc<double>(ctx, (size_t)mmax * mmax, false);
    Bm = dalloc<double>(ctx, (size_t)mmax * mmax, false);
    Wv = dalloc<double>(ctx, mmax, false);
    HP = dalloc<double>(ctx, (size_t)(mmax + 1) * s, false);
    CU = dalloc<double>(ctx, (size_t)s * L, false);
    sig = dalloc<double>(ctx, k, false);
    dinfo = dalloc<int>(ctx, 1);
    {
      std::vector<int> ident(nseeds);
      for (int i = 0; i < nseeds; ++i) ident[i] = i;
      CK(cudaMemcpy(dreg, ident.data(), nseeds * sizeof(int), cudaMemcpyHostToDevice));
    }
    const double one = 1.0, zero = 0.0;
    std::vector<int> used;        // seeds that own a regime (round 1 decides)
    std::vector<int> sizes;       // per-regime space size
    std::vector<double> run_v;    // the parameter rows recorded this round
    const int rounds = recycle_rounds();
    for (int round = 0; round < rounds; ++round) {
      // round 0: one plain GMRES cycle per seed (no spaces yet).  round >= 1: every regime's seed
      // again, as an FGMRES cycle whose first search directions are the current space; the new space
      // is selected from span([U, Z]) -- a GCRO-DR-style refinement
      const int nrun = round == 0 ? nseeds : (int)used.size();
      if (round == 0) run_v.assign(seeds, seeds + (int64_t)nseeds * k);
      else {
        run_v.clear();
        for (int r : used) run_v.insert(run_v.end(), seeds + (int64_t)r * k, seeds + (int64_t)(r + 1) * k);
      }
      CK(cudaMemcpyAsync(dV, run_v.data(), (size_t)nrun * k * 8, cudaMemcpyHostToDevice, st));
      rc = run_batch(ctx, nrun, dV, nullptr, dtr, dst, nullptr, nullptr, st, nullptr, round ? dreg : nullptr, 1);
      if (rc != LYAP_OK) throw Fail{rc};
      const Engine& g = ctx->eng;
      std::vector<int> hph(g.b), hm(g.b), hv(g.b);
      CK(cudaMemcpy(hph.data(), g.phase, g.b * sizeof(int), cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(hm.data(), g.m, g.b * sizeof(int), cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(hv.data(), g.vidx, g.b * sizeof(int), cudaMemcpyDeviceToHost));
      std::vector<int> slot_of(nrun, -1);
      for (int sl = 0; sl < g.b; ++sl)
        if (hph[sl] == PH_IDLE && hm[sl] >= 1 && hv[sl] >= 0 && hv[sl] < nrun && slot_of[hv[sl]] < 0)
          slot_of[hv[sl]] = sl;
      if (round == 0) {
        for (int r = 0; r < nseeds; ++r)
          if (slot_of[r] >= 0) used.push_back(r);
        if (used.empty()) {
          set_err(ctx, "lyap_build_recycle: no seed produced a Krylov cycle (all converged immediately)");
          throw Fail{LYAP_EINVAL};
        }
      }
      const int nreg = (int)used.size();
      // a regime is re-selected when its cycle is at least as long as its current space (a seed the
      // space already solves within fewer steps keeps the space it has)
      std::vector<int> take(nreg), nsz(nreg);
      int stride = 1;
      for (int ri = 0; ri < nreg; ++ri) {
        const int sl = slot_of[round == 0 ? used[ri] : ri];
        const int cur = round == 0 ? 0 : sizes[ri];
        take[ri] = sl >= 0 && std::min(s, hm[sl]) >= std::max(cur, 1);
        nsz[ri] = take[ri] ? std::min(s, hm[sl]) : cur;
        stride = std::max(stride, nsz[ri]);
      }
      Unew = dalloc<double>(ctx, (size_t)nreg * stride * L);
      TUnew = dalloc<double>(ctx, (size_t)nreg * stride * L);
      // engine args for the helper kernels: slot-indexed arrays of the whole engine
      EngArgs ea{};
      ea.mmax = mmax;
      ea.L = L;
      ea.npad = sd.npad;
      ea.nrep = sd.nrep;
      ea.npairs = sd.npairs;
      ea.Qb = g.Qb;
      ea.eta = g.eta;
      ea.Minv = g.Minv;
      ea.su = g.restarts + 3 * g.b;
      ea.reg = g.restarts + 4 * g.b;
      ea.Ureg = ctx->Ureg;
      ea.s_rec = ctx->s_rec;
      for (int ri = 0; ri < nreg; ++ri) {
        const int r = used[ri];
        double* Ur = Unew + (int64_t)ri * stride * L;
        double* TUr = TUnew + (int64_t)ri * stride * L;
        if (!take[ri]) {  // keep the current space
          CK(cudaMemcpyAsync(Ur, ctx->Ureg + (int64_t)ri * ctx->s_rec * L, (size_t)nsz[ri] * L * 8,
                             cudaMemcpyDeviceToDevice, st));
          CK(cudaMemcpyAsync(TUr, ctx->TUreg + (int64_t)ri * ctx->s_rec * L, (size_t)nsz[ri] * L * 8,
                             cudaMemcpyDeviceToDevice, st));
          continue;
        }
        const int sl = slot_of[round == 0 ? r : ri], m1 = hm[sl], sr = nsz[ri];
        // Z = the cycle's search directions (u_j for j < su, else P^{-1} q_j) and normalised Q (j <= m1)
        const dim3 gz((unsigned)((sd.nrep + 127) / 128), (unsigned)m1);
        CK(cudaMemsetAsync(Z, 0, (size_t)m1 * L * 8, st));
        K_DISPATCH(k, (k_rec_z<KK><<<gz, 128, 0, st>>>(ea, sl, m1, Z)));
        LAUNCHED();
        std::vector<double> heta(m1 + 1);
        CK(cudaMemcpy(heta.data(), g.eta + (int64_t)sl * ld, (m1 + 1) * 8, cudaMemcpyDeviceToHost));
        for (int j = 0; j <= m1; ++j) {
          const double inv = 1.0 / heta[j];
          CKB(cublasDcopy(ctx->cublas, (int)L, g.Qb + ((int64_t)sl * ld + j) * L, 1, Qn + (int64_t)j * L, 1));
          CKB(cublasDscal(ctx->cublas, (int)L, &inv, Qn + (int64_t)j * L, 1));
        }
        const double* Hb = g.Hraw + (int64_t)sl * ld * mmax;  // column-major (m1+1) x m1, ld = mmax + 1
        // A = Hbar^T Hbar, B = Z^T Z (+ tiny ridge), generalised symmetric eigenproblem A p = theta B p
        CKB(cublasDgemm(ctx->cublas, CUBLAS_OP_T, CUBLAS_OP_N, m1, m1, m1 + 1, &one, Hb, ld, Hb, ld, &zero, Am, m1));
        CKB(cublasDgemm(ctx->cublas, CUBLAS_OP_T, CUBLAS_OP_N, m1, m1, (int)L, &one, Z, (int)L, Z, (int)L, &zero, Bm,
                        m1));
        {
          std::vector<double> hb((size_t)m1 * m1);
          CK(cudaMemcpy(hb.data(), Bm, hb.size() * 8, cudaMemcpyDeviceToHost));
          double tr = 0.0;
          for (int j = 0; j < m1; ++j) tr += hb[(size_t)j * m1 + j];
          const double ridge = 1e-10 * tr / m1;
          for (int j = 0; j < m1; ++j) hb[(size_t)j * m1 + j] += ridge;
          CK(cudaMemcpy(Bm, hb.data(), hb.size() * 8, cudaMemcpyHostToDevice));
        }
        int lwork = 0;
        CKS(cusolverDnDsygvd_bufferSize(ctx->cusolver, CUSOLVER_EIG_TYPE_1, CUSOLVER_EIG_MODE_VECTOR,
                                        CUBLAS_FILL_MODE_UPPER, m1, Am, m1, Bm, m1, Wv, &lwork));
        dfree(work);
        work = dalloc<double>(ctx, std::max(lwork, 1), false);
        CKS(cusolverDnDsygvd(ctx->cusolver, CUSOLVER_EIG_TYPE_1, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_UPPER, m1,
                             Am, m1, Bm, m1, Wv, work, lwork, dinfo));
        int hinfo = 0;
        CK(cudaMemcpy(&hinfo, dinfo, sizeof(int), cudaMemcpyDeviceToHost));
        if (hinfo != 0) {
          // Z^T Z numerically singular: select in the Euclidean metric of the coefficients instead
          // (smallest right singular vectors of Hbar; measured nearly as effective)
          CKB(cublasDgemm(ctx->cublas, CUBLAS_OP_T, CUBLAS_OP_N, m1, m1, m1 + 1, &one, Hb, ld, Hb, ld, &zero, Am,
                          m1));
          int lw2 = 0;
          CKS(cusolverDnDsyevd_bufferSize(ctx->cusolver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_UPPER, m1, Am,
                                          m1, Wv, &lw2));
          dfree(work);
          work = dalloc<double>(ctx, std::max(lw2, 1), false);
          CKS(cusolverDnDsyevd(ctx->cusolver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_UPPER, m1, Am, m1, Wv, work,
                               lw2, dinfo));
          CK(cudaMemcpy(&hinfo, dinfo, sizeof(int), cudaMemcpyDeviceToHost));
          if (hinfo != 0) {
            set_err(ctx, "lyap_build_recycle: syevd info = %d for seed %d", hinfo, r);
            throw Fail{LYAP_ECUDA};
          }
        }
        // P = eigenvectors of the sr smallest eigenvalues (ascending: first columns of Am);
        // U = Z P, C(v)U = Qn Hbar P, TU = Delta(v) U - C(v) U
        CKB(cublasDgemm(ctx->cublas, CUBLAS_OP_N, CUBLAS_OP_N, (int)L, sr, m1, &one, Z, (int)L, Am, m1, &zero, Ur,
                        (int)L));
        CKB(cublasDgemm(ctx->cublas, CUBLAS_OP_N, CUBLAS_OP_N, m1 + 1, sr, m1, &one, Hb, ld, Am, m1, &zero, HP,
                        m1 + 1));
        CKB(cublasDgemm(ctx->cublas, CUBLAS_OP_N, CUBLAS_OP_N, (int)L, sr, m1 + 1, &one, Qn, (int)L, HP, m1 + 1,
                        &zero, CU, (int)L));
        std::vector<double> hs(k);
        for (int64_t t = 0; t < k; ++t) hs[t] = 1.0 / seeds[(int64_t)r * k + t];
        CK(cudaMemcpy(sig, hs.data(), k * 8, cudaMemcpyHostToDevice));
        k_rec_tu<<<(unsigned)std::min<int64_t>(((int64_t)sr * L + 255) / 256, 65535), 256, 0, st>>>(
            Ur, CU, sig, L, sd.npad, sr, TUr);
        LAUNCHED();
      }
      CK(cudaStreamSynchronize(st));
      dfree(ctx->Ureg);
      dfree(ctx->TUreg);
      ctx->Ureg = Unew;
      ctx->TUreg = TUnew;
      Unew = TUnew = nullptr;
      sizes = nsz;
      dfree(ctx->sreg);
      ctx->sreg = dalloc<int>(ctx, nreg, false);
      CK(cudaMemcpy(ctx->sreg, sizes.data(), nreg * sizeof(int), cudaMemcpyHostToDevice));
      ctx->nreg = nreg;
      ctx->s_rec = stride;
    }
    std::vector<double> seeds_used;
    for (int r : used)
      for (int64_t t = 0; t < k; ++t) seeds_used.push_back(std::log(std::fabs(seeds[(int64_t)r * k + t])));
    ctx->reg_seeds.assign(reinterpret_cast<const char*>(seeds_used.data()), seeds_used.size() * sizeof(double));
    upload_seeds(ctx);
  } catch (Fail f) {
    rc = f.code;
    dfree(ctx->Ureg);
    dfree(ctx->TUreg);
    dfree(ctx->sreg);
    ctx->Ureg = ctx->TUreg = nullptr;
    ctx->sreg = nullptr;
    ctx->nreg = ctx->s_rec = 0;
  }
  for (void* p : {(void*)dV, (void*)dtr, (void*)dst, (void*)Z, (void*)Qn, (void*)Am, (void*)Bm, (void*)Wv, (void*)work,
                  (void*)HP, (void*)CU, (void*)sig, (void*)Unew, (void*)TUnew, (void*)dinfo, (void*)dreg})
    dfree(p);
  return rc;
}

static int apply_C_impl(lyap_ctx* ctx, int64_t nvec, const double* X, const double* sigma, double* Y, void* cuda_stream,
                        bool mixed) {
  if (!ctx || nvec < 0 || (nvec > 0 && (!X || !Y))) {
    set_err(ctx, "lyap_apply_C: invalid arguments");
    return LYAP_EINVAL;
  }
  if (mixed && mp_mode(ctx) != 1 && mp_mode(ctx) != 3) {
    set_err(ctx, "lyap_apply_C_mixed: mixed precision is off for this context (opts.mixed)");
    return LYAP_EINVAL;
  }
  try {
    CK(cudaSetDevice(ctx->device));
    cudaStream_t st = (cudaStream_t)cuda_stream;
    const int b = auto_batch(ctx, std::max<int64_t>(nvec, 1));
    ensure_engine(ctx, std::max(b, ctx->eng.b), ctx->eng.mmax > 0 ? ctx->eng.mmax : auto_mmax(ctx));
    const int mpm = mixed ? mp_mode(ctx) : 0;
    if (mixed) ensure_lf32(ctx, mpm);
    const Engine& g = ctx->eng;
    const int64_t cap = g.ncol / (ctx->seed.k * ctx->seed.k);  // vectors per K1 launch (group 0 buffers)
    int* zero = nullptr;
    if (mixed) {  // no VERIFY positions: every vector takes the 3xTF32 product
      zero = dalloc<int>(ctx, 1);
      if (!ctx->eng.umctr) throw Fail{LYAP_ECUDA};
    }
    for (int64_t v0 = 0; v0 < nvec; v0 += cap) {
      const int nb = (int)std::min<int64_t>(cap, nvec - v0);
      K1Args a{};
      a.Xin = X + v0 * g.L;
      a.L = g.L;
      a.nslot = nb;
      a.mode = 0;
      a.sigma = sigma ? sigma + v0 * ctx->seed.k : nullptr;
      a.Yout = Y + v0 * g.L;
      a.nactive = nullptr;
      a.alist = nullptr;
      a.nver = zero;
      launch_k1(ctx, a, st, nullptr, nullptr, 0, 0, mpm);
      ctx->stats.k1_launches++;
      ctx->stats.k1_vectors += nb;
      if (!mixed) ctx->stats.k1_exact_vectors += nb;
      ctx->stats.k1_flops += 2.0 * (double)ctx->seed.n * ctx->seed.n * ctx->seed.k * ctx->seed.k * nb;
    }
    if (zero) {
      CK(cudaStreamSynchronize(st));
      dfree(zero);
    }
  } catch (Fail f) {
    return f.code;
  }
  return LYAP_OK;
}

int lyap_apply_C(lyap_ctx* ctx, int64_t nvec, const double* X, const double* sigma, double* Y, void* cuda_stream) {
  return apply_C_impl(ctx, nvec, X, sigma, Y, cuda_stream, false);
}

int lyap_apply_C_mixed(lyap_ctx* ctx, int64_t nvec, const double* X, const double* sigma, double* Y,
                       void* cuda_stream) {
  return apply_C_impl(ctx, nvec, X, sigma, Y, cuda_stream, true);
}

int lyap_get_info(const lyap_ctx* ctx, lyap_info* info) {
  if (!ctx || !info) return LYAP_EINVAL;
  *info = ctx->info;
  info->mixed_mode = mp_mode(ctx);
  return LYAP_OK;
}

int lyap_get_stats(const lyap_ctx* ctx, lyap_stats* st) {
  if (!ctx || !st) return LYAP_EINVAL;
  *st = ctx->stats;
  return LYAP_OK;
}

int lyap_reset_stats(lyap_ctx* ctx) {
  if (!ctx) return LYAP_EINVAL;
  ctx->stats = lyap_stats{};
  return LYAP_OK;
}

int lyap_export_state(const lyap_ctx* cctx, double* lam, double* bhr, double* btl, double* F, double* g0,
                      double* hf) {
  lyap_ctx* ctx = const_cast<lyap_ctx*>(cctx);
  if (!ctx) return LYAP_EINVAL;
  try {
    CK(cudaSetDevice(ctx->device));
    const Seed& s = ctx->seed;
    if (lam) CK(cudaMemcpy(lam, s.lam, 2 * s.n * 8, cudaMemcpyDeviceToHost));
    if (bhr) CK(cudaMemcpy(bhr, s.bhr, s.n * s.k * 8, cudaMemcpyDeviceToHost));
    if (btl) CK(cudaMemcpy(btl, s.btl, s.n * s.k * 8, cudaMemcpyDeviceToHost));
    if (F) CK(cudaMemcpy(F, s.F, s.nrep * s.k * s.k * 2 * 8, cudaMemcpyDeviceToHost));
    if (g0) CK(cudaMemcpy(g0, s.g0, s.k * s.npad * 8, cudaMemcpyDeviceToHost));
    if (hf) CK(cudaMemcpy(hf, s.hf, s.k * s.npad * 8, cudaMemcpyDeviceToHost));
  } catch (Fail f) {
    return f.code;
  }
  return LYAP_OK;
}

}  // extern "C"

#include "ek.inc"
