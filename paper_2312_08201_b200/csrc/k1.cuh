// K1 — the Cauchy-fused T-apply: for a batch of folded vectors X (one per slot)
//
//   U_{(s,t),j} = sum_i L_ij (B^r_is X_ti)                     (dense Cauchy coupling, eqs. (N2M1),
//                                                                (N1M2))
//   (T X)_sj    = sum_t B~l_jt U_{(s,t),j} + sum_t F_j[s,t] X_tj  (T_d: eq. (N1M1) and the (2,2)
//                                                                block)
//   out         = sigma_s X_sj - (T X)_sj                        (C(v) = Delta(v) - T)
//
// in real pair-folded coordinates: U = Lf * Bop is one real FP64 GEMM (M = K = npad, N = slots*k^2)
// on the DMMA tensor pipe (mma.sync.m8n8k4.f64), with a prologue kernel that builds the B operand
// (B^r o X outer products) and an epilogue kernel that contracts over t and adds T_d.
#pragma once
#include <cuda_fp16.h>

#include "common.cuh"

namespace lyap {

constexpr int K1_TILE_C = 32;  // coordinates per prologue / epilogue tile
constexpr int K1_THREADS = 256;  // prologue / epilogue block size: compile-time strides let the
                                 // staging loops unroll, so each thread's loads are in flight together

template <int K>
struct K1Tile {
  static constexpr int TS = (64 / (K * K)) > 0 ? (64 / (K * K)) : 1;  // slots per tile
  static constexpr int NC = TS * K * K;                                // GEMM columns per tile
};

// Per-launch arguments of the prologue / epilogue (engine mode or standalone apply mode).
struct K1Args {
  const double* Xin;   // nslot x L  (input vectors, slot-major)
  int64_t L;           // k * npad
  int nslot;
  int mode;            // 0 = apply (Yout = sigma o X - T X), 1 = engine
  const double* sigma; // nslot x k (apply mode: may be null -> 0)
  const double* mask;  // nslot x k (engine mode) 1 = v_t != 0
  const int* phase;    // engine: slot phases
  const int* m;        // engine: current Krylov index per slot
  double* Qb;          // engine: basis (nslot x (mmax+1) x L)
  float* Qf;           // engine, mixed precision: the basis in FP32 (then Qb is null)
  int64_t qstride;     // (mmax+1) * L
  double* Yout;        // apply mode output (nslot x L)
  const int* nactive;  // engine: number of active slots (null: all nslot vectors are active)
  const int* alist;    // engine: active slot ids, compacted (null: identity)
  const double* rhs;   // engine, v-linear Q: per-slot right-hand side (nslot x L); null: g0
  // mixed precision (engine mode): active positions [0, *nver) are VERIFY slots (exact
  // FP64 apply through the DMMA GEMM), positions [*nver, *nactive) ITER slots (apply through the
  // FP32-accurate tensor-core GEMM on the float planes B32 / U32).  nver == null: all FP64.
  const int* nver;
  // 3xFP16: power-of-two operand scales -- per slot and parameter t the max |X_t| (xmax: accumulated by
  // k_prec in the engine, k_xmax in apply mode), per s max |B^r_s| (bmax), the exponent of Lf's scale
  // (eA); k1_gen16 writes each column's unscale factor 2^-(eA + e_n) to colscale
  const float *xmax, *bmax;
  int eA;
  float* colscale;
};

// float split of a double for the 3xTF32 GEMM: hi = x rounded to TF32 (10-bit mantissa), lo = x - hi
__device__ __forceinline__ float tf32_rn(float f) {
  return __uint_as_float((__float_as_uint(f) + 0x1000u) & 0xFFFFE000u);
}

// Fused-epilogue arguments of the K1 GEMM (EPI = k > 0): the k1_epi contraction done from the CTA's
// accumulator tile in shared memory, so U never goes to global memory and k1_epi is not launched.
struct K1EpiArgs {
  K1Args a;
  const double *btl, *F, *g0;
  int npad, two_np, npairs, n;
};

// GEMM column block p (of k^2 columns) belongs to active position p -> slot alist[p]
__device__ __forceinline__ int k1_nact(const K1Args& a) { return a.nactive ? *a.nactive : a.nslot; }
__device__ __forceinline__ int k1_slot(const K1Args& a, int pos) { return a.alist ? a.alist[pos] : pos; }

enum : int { PH_FREE = 0, PH_IDLE = 1, PH_VERIFY = 2, PH_ITER = 3, PH_XUPD = 4, PH_START = 5 };

// ------------------------------------------------------------------------------------------
// K1a prologue: Bop[i][(slot*k + s)*k + t] = folded (B^r_is * X_ti)   (the Hadamard B operand)
// one element of the B operand: fold(B^r_is X_ti) at tile row r (x: the slot's X_t tile, bs: B^r tile)
template <int K>
__device__ __forceinline__ double k1_bval(const double* x, const double (*bs)[K], int r, int s, bool pair) {
  if (pair) {  // conjugate pair: (br + i bi)(x + i y)
    const int ce = r & ~1;
    const double xr = x[ce], yi = x[ce + 1];
    const double br = bs[ce][s], bi = bs[ce + 1][s];
    return (r & 1) ? (br * yi + bi * xr) : (br * xr - bi * yi);
  }
  return bs[r][s] * x[r];
}

// MP = 0: FP64 operand only.  MP = 1 (3xTF32) / 2 (one float plane): also the float operand B32, K-major
// (2 ncol x npad: rows [0, ncol) lo parts, rows [ncol, 2 ncol) hi parts; umma.cuh) for every active
// position, and the FP64 operand only for the VERIFY positions [0, nver).
template <int K, int MP = 0>
__global__ void __launch_bounds__(256) k1_gen(K1Args a, const double* __restrict__ bhr, int npad,
                                               int two_np, double* __restrict__ Bop, int64_t ncol,
                                               float* __restrict__ B32 = nullptr) {
  static_assert(MP <= 2, "3xFP16 operands: k1_gen16");
  constexpr int TS = K1Tile<K>::TS, NC = K1Tile<K>::NC, TC = K1_TILE_C;
  const int nact = k1_nact(a);
  const int nver = MP ? *a.nver : nact;
  const int i0 = blockIdx.x * TC, s0 = blockIdx.y * TS;
  if (s0 >= nact) return;
  __shared__ double xs[TS][K][TC];
  __shared__ double bs[TC][K];
#pragma unroll
  for (int idx = threadIdx.x; idx < TS * K * TC; idx += K1_THREADS) {
    int sl = idx / (K * TC), t = (idx / TC) % K, c = idx % TC;
    xs[sl][t][c] = (s0 + sl < nact) ? a.Xin[(int64_t)k1_slot(a, s0 + sl) * a.L + (int64_t)t * npad + i0 + c] : 0.0;
  }
#pragma unroll
  for (int idx = threadIdx.x; idx < TC * K; idx += K1_THREADS) bs[idx / K][idx % K] = bhr[(int64_t)i0 * K + idx];
  __syncthreads();
  if constexpr (MP == 0) {
#pragma unroll
    for (int idx = threadIdx.x; idx < TC * NC; idx += K1_THREADS) {
      int r = idx / NC, col = idx % NC;
      int sl = col / (K * K), s = (col / K) % K, t = col % K;
      if (s0 + sl >= nact) continue;
      Bop[(int64_t)(i0 + r) * ncol + (int64_t)(s0 + sl) * K * K + col % (K * K)] =
          k1_bval<K>(xs[sl][t], bs, r, s, i0 + r < two_np);
    }
  } else {
    // float planes, K-major (row = GEMM column n, contiguous along the coordinate): consecutive threads
    // take consecutive coordinates, so the stores coalesce
#pragma unroll
    for (int idx = threadIdx.x; idx < TC * NC; idx += K1_THREADS) {
      const int r = idx % TC, col = idx / TC;
      const int sl = col / (K * K), s = (col / K) % K, t = col % K;
      if (s0 + sl >= nact) continue;
      const double val = k1_bval<K>(xs[sl][t], bs, r, s, i0 + r < two_np);
      const int64_t nn = (int64_t)(s0 + sl) * K * K + col % (K * K);
      if (s0 + sl < nver) Bop[(int64_t)(i0 + r) * ncol + nn] = val;  // FP64 operand of the exact apply
      const float f = (float)val;
      const float hi = MP == 1 ? tf32_rn(f) : f;
      B32[(ncol + nn) * npad + i0 + r] = hi;
      if (MP == 1) B32[nn * npad + i0 + r] = (float)(val - (double)hi);
    }
  }
}

// 3xFP16 B operand (MP = 3), one active position per blockIdx.y, two consecutive coordinates per thread
// (a conjugate pair's (Re, Im) rows, or two real rows): every value of the pair is formed from one
// 16-byte load of each X_t and the two B^r rows, and the hi / lo planes are written as half2, so a
// warp stores 128 contiguous bytes per (s, t) column.  Column scale 2^e_n (e_n from max|B^r_s|
// max|X_t|, the same bound as k1_gen<K, 3>) is formed once per block; unscale 2^-(eA + e_n) goes to
// colscale.  The FP64 operand is written for the VERIFY positions [0, nver) only.
constexpr int K1G16_THREADS = 256;
template <int K>
__global__ void __launch_bounds__(K1G16_THREADS) k1_gen16(K1Args a, const double* __restrict__ bhr, int npad,
                                                          int two_np, double* __restrict__ Bop, int64_t ncol,
                                                          __half* __restrict__ B16) {
  const int pos = blockIdx.y;
  const int nact = k1_nact(a);
  if (pos >= nact) return;
  const int nver = *a.nver;
  const int slot = k1_slot(a, pos);
  __shared__ double scl[K * K];
  if (threadIdx.x < K * K) {
    const int s = threadIdx.x / K, t = threadIdx.x % K;
    const float bound = a.bmax[s] * a.xmax[slot * K + t] * 1.5f;
    const int e = bound > 0.f ? 13 - (int)ceilf(log2f(bound)) : 0;
    scl[threadIdx.x] = ldexp(1.0, e);
    if (blockIdx.x == 0) a.colscale[(int64_t)pos * K * K + threadIdx.x] = ldexpf(1.f, -(a.eA + e));
  }
  __syncthreads();
  const int c = 2 * (blockIdx.x * K1G16_THREADS + threadIdx.x);
  if (c >= npad) return;
  const double* x = a.Xin + (int64_t)slot * a.L;
  double2 xv[K];
#pragma unroll
  for (int t = 0; t < K; ++t) xv[t] = *reinterpret_cast<const double2*>(x + (int64_t)t * npad + c);
  double b0[K], b1[K];
#pragma unroll
  for (int s = 0; s < K; ++s) {
    b0[s] = bhr[(int64_t)c * K + s];
    b1[s] = bhr[(int64_t)(c + 1) * K + s];
  }
  const bool pair = c < two_np;
  const int64_t nb = (int64_t)pos * K * K;
#pragma unroll
  for (int s = 0; s < K; ++s) {
#pragma unroll
    for (int t = 0; t < K; ++t) {
      double v0, v1;
      if (pair) {  // (br + i bi)(x + i y): Re row c, Im row c + 1
        v0 = b0[s] * xv[t].x - b1[s] * xv[t].y;
        v1 = b0[s] * xv[t].y + b1[s] * xv[t].x;
      } else {
        v0 = b0[s] * xv[t].x;
        v1 = b1[s] * xv[t].y;
      }
      const int64_t nn = nb + s * K + t;
      if (pos < nver) {
        Bop[(int64_t)c * ncol + nn] = v0;
        Bop[(int64_t)(c + 1) * ncol + nn] = v1;
      }
      const double sc = scl[s * K + t];
      const double y0 = v0 * sc, y1 = v1 * sc;
      const __half h0 = __double2half(y0), h1 = __double2half(y1);
      const __half l0 = __double2half(y0 - (double)__half2float(h0));
      const __half l1 = __double2half(y1 - (double)__half2float(h1));
      *reinterpret_cast<__half2*>(B16 + (ncol + nn) * npad + c) = __halves2half2(h0, h1);
      *reinterpret_cast<__half2*>(B16 + nn * npad + c) = __halves2half2(l0, l1);
    }
  }
}

// mixed precision: Lf32 = [hi | lo] float planes of the folded Cauchy matrix (npad x 2 npad row-major;
// MP = 2: lo = 0), built once per seed
template <int MP>
__global__ void k_split_Lf(const double* __restrict__ Lf, int64_t npad, float* __restrict__ Lf32) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < npad * npad;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / npad, i = e % npad;
    const double x = Lf[e];
    const float f = (float)x;
    const float hi = MP == 1 ? tf32_rn(f) : f;
    Lf32[j * 2 * npad + i] = hi;
    Lf32[j * 2 * npad + npad + i] = MP == 1 ? (float)(x - (double)hi) : 0.f;
  }
}

// 3xFP16: Lf16 = [hi | lo] half planes of 2^eA Lf (npad x 2 npad row-major)
__global__ void k_split_Lf16(const double* __restrict__ Lf, int64_t npad, int eA, __half* __restrict__ Lf16) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < npad * npad;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / npad, i = e % npad;
    const double x = ldexp(Lf[e], eA);
    const __half hi = __double2half(x);
    Lf16[j * 2 * npad + i] = hi;
    Lf16[j * 2 * npad + npad + i] = __double2half(x - (double)__half2float(hi));
  }
}
// max |x| over cnt doubles into *out (one block; float result, rounded up)
__global__ void k_absmax(const double* __restrict__ x, int64_t cnt, float* __restrict__ out) {
  __shared__ double red[32];
  double m = 0.0;
  for (int64_t i = threadIdx.x; i < cnt; i += blockDim.x) m = fmax(m, fabs(x[i]));
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, red[w]);
    *out = __double2float_ru(fmax(m, red[0]));
  }
}
// per-parameter max |B^r_s| (complex modulus over a pair's two coordinates): bmax[s], one block per s
__global__ void k_bmax(const double* __restrict__ bhr, int64_t npad, int k, int two_np, float* __restrict__ bmax) {
  __shared__ double red[32];
  const int s = blockIdx.x;
  double m = 0.0;
  for (int64_t c = threadIdx.x; c < npad; c += blockDim.x) {
    const double v = bhr[c * k + s];
    const double w = (c < two_np) ? bhr[(c ^ 1) * k + s] : 0.0;
    m = fmax(m, sqrt(v * v + w * w));
  }
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, red[w]);
    bmax[s] = __double2float_ru(fmax(m, red[0]));
  }
}
// per active position: xmax[slot * K + t] = max_c |Xin[slot][t][c]| (one block per position)
template <int K>
__global__ void __launch_bounds__(256) k_xmax(K1Args a, int npad, float* __restrict__ xmax) {
  __shared__ double red[K][8];
  const int pos = blockIdx.x;
  if (pos >= k1_nact(a)) return;
  const int slot = k1_slot(a, pos);
  const double* x = a.Xin + (int64_t)slot * a.L;
  double m[K];
#pragma unroll
  for (int t = 0; t < K; ++t) m[t] = 0.0;
  for (int c = threadIdx.x; c < npad; c += blockDim.x)
#pragma unroll
    for (int t = 0; t < K; ++t) m[t] = fmax(m[t], fabs(x[(int64_t)t * npad + c]));
#pragma unroll
  for (int t = 0; t < K; ++t) {
    for (int o = 16; o > 0; o >>= 1) m[t] = fmax(m[t], __shfl_xor_sync(0xffffffffu, m[t], o));
    if ((threadIdx.x & 31) == 0) red[t][threadIdx.x >> 5] = m[t];
  }
  __syncthreads();
  if (threadIdx.x < K) {
    double v = 0.0;
    for (int w = 0; w < 8; ++w) v = fmax(v, red[threadIdx.x][w]);
    xmax[slot * K + threadIdx.x] = __double2float_ru(v);
  }
}

// ------------------------------------------------------------------------------------------
// K1b: C = A * B, FP64, A: M x Kd (row stride lda; the folded Cauchy matrix Lf), B: Kd x N
// row-major, C: M x N row-major.  M % BM == N % BN == Kd % 16 == 0.  STAGES-deep cp.async pipeline, warp
// tile WM x WN of m8n8k4 DMMA fragments.  Shared-memory strides 20 / BN+4 doubles make every
// fragment load conflict-free (lane -> (row l/4, k l%4) maps onto 16 distinct 8-byte banks per
// half-warp).
template <int BM, int BN, int WM, int WN, int STAGES, int BK_ = 16>
struct DgemmCfg {
  static constexpr int BK = BK_, AST = BK + 4, BST = BN + 4;
  static constexpr int WARPS_N = BN / WN, WARPS = (BM / WM) * (BN / WN), THREADS = WARPS * 32;
  static constexpr int A_STAGE = BM * AST, B_STAGE = BK * BST;
  static constexpr size_t SMEM = (size_t)STAGES * (A_STAGE + B_STAGE) * sizeof(double);
};

// Output layouts (OUT): 0 plain C[row * N + col]; the batched full-solution path (lyap_solution,
// DESIGN.md §2.5) uses 1 = "vertical stack -> horizontal stack": row = v * blk + r is written to
// C[r * (N * nblk) + v * N + col] (blk = N, nblk = M / N), and 2 = "horizontal stack -> compact":
// col = v * blk + c is written to C[(v * no + r) * no + c] for r, c < no (the unpadded order).
struct DgemmOut {
  int blk, nblk, no;
};

// destination of a K1 output row: FP64 (d) or, for the FP32 basis of the mixed-precision engine, f
struct K1Dst {
  double* d;
  float* f;
  __device__ __forceinline__ void put(int64_t i, double v) const {
    if (f)
      f[i] = (float)v;
    else
      d[i] = v;
  }
};

template <int K>
__device__ __forceinline__ void k1_out_element(const K1EpiArgs& ep, int slot, int s, int c, const double* ur,
                                               const double* ur1, int ust);

// EPI > 0: fused K1 epilogue for k = EPI (OUT ignored, C unused): see K1EpiArgs.
template <int BM, int BN, int WM, int WN, int STAGES, int BK_ = 16, int OUT = 0, int EPI = 0>
__global__ void __launch_bounds__(DgemmCfg<BM, BN, WM, WN, STAGES, BK_>::THREADS,
                                  DgemmCfg<BM, BN, WM, WN, STAGES, BK_>::THREADS <= 128 ? 3 : 1)
    k1_dgemm(const double* __restrict__ A, const double* __restrict__ B, double* __restrict__ C, int M,
             int N, int Kd, int lda, const int* __restrict__ nactive, int cols_per_active, DgemmOut om = {},
             K1EpiArgs ep = {}) {
  using Cfg = DgemmCfg<BM, BN, WM, WN, STAGES, BK_>;
  constexpr int BK = Cfg::BK, AST = Cfg::AST, BST = Cfg::BST, NT = Cfg::THREADS;
  constexpr int MT = WM / 8, NTL = WN / 8;
  // grouped rasterisation (1-D grid): GROUP_M M-tiles share each sweep over the N-tiles, so the
  // A panels (Lf rows) and the B panels in flight fit in L2 and each operand byte is read from
  // DRAM about once (c5: 1.34 GB -> ~0.4 GB per launch)
  constexpr int GROUP_M = 16;
  const int ntn = N / BN, ntm = M / BM;
  const int bid = blockIdx.x;
  const int group = bid / (GROUP_M * ntn), first_m = group * GROUP_M;
  const int gsz = min(ntm - first_m, GROUP_M);
  const int local = bid - group * GROUP_M * ntn;
  const int mt = first_m + local % gsz, nt = local / gsz;
  if (nactive && nt * BN >= (*nactive) * cols_per_active) return;  // no active column
  extern __shared__ __align__(16) double smem[];
  double* As = smem;
  double* Bs = smem + STAGES * Cfg::A_STAGE;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wm = warp / Cfg::WARPS_N, wn = warp % Cfg::WARPS_N;
  const int m0 = mt * BM, n0 = nt * BN;

  double acc[MT][NTL][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NTL; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  auto load_stage = [&](int stage, int kt) {
    const double* Ag = A + (int64_t)m0 * lda + (int64_t)kt * BK;
    double* as = As + stage * Cfg::A_STAGE;
#pragma unroll
    for (int c = tid; c < BM * BK / 2; c += NT) {
      int r = c / (BK / 2), cc = (c % (BK / 2)) * 2;
      cp_async16(as + r * AST + cc, Ag + (int64_t)r * lda + cc);
    }
    const double* Bg = B + (int64_t)kt * BK * N + n0;
    double* bs = Bs + stage * Cfg::B_STAGE;
#pragma unroll
    for (int c = tid; c < BK * BN / 2; c += NT) {
      int r = c / (BN / 2), cc = (c % (BN / 2)) * 2;
      cp_async16(bs + r * BST + cc, Bg + (int64_t)r * N + cc);
    }
  };

  const int KT = Kd / BK;
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < KT) load_stage(s, s);
    cp_async_commit();
  }
  const int ar = wm * WM + (lane >> 2), ac = lane & 3;
  const int bc = wn * WN + (lane >> 2), br = lane & 3;
  for (int kt = 0; kt < KT; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      int nk = kt + STAGES - 1;
      if (nk < KT) load_stage(nk % STAGES, nk);
      cp_async_commit();
    }
    const double* as = As + (kt % STAGES) * Cfg::A_STAGE;
    const double* bs = Bs + (kt % STAGES) * Cfg::B_STAGE;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[MT], bf[NTL];
#pragma unroll
      for (int i = 0; i < MT; ++i) af[i] = as[(ar + i * 8) * AST + kk + ac];
#pragma unroll
      for (int j = 0; j < NTL; ++j) bf[j] = bs[(kk + br) * BST + bc + j * 8];
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NTL; ++j) dmma_884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();
  if constexpr (EPI > 0) {
    // fused epilogue: accumulator tile -> shared memory, then the k1_epi contraction per (slot, s, row)
    constexpr int UST = BN + 1, KK = EPI * EPI, NPOS = BN / KK;
    static_assert(BN % KK == 0, "a slot's k^2 columns must not straddle tiles");
    __syncthreads();  // every warp is done with the pipeline buffers
    double* Us = smem;
#pragma unroll
    for (int i = 0; i < MT; ++i) {
      const int rl = wm * WM + i * 8 + (lane >> 2);
#pragma unroll
      for (int j = 0; j < NTL; ++j) {
        const int cl = wn * WN + j * 8 + (lane & 3) * 2;
        Us[rl * UST + cl] = acc[i][j][0];
        Us[rl * UST + cl + 1] = acc[i][j][1];
      }
    }
    __syncthreads();
    const int nact = k1_nact(ep.a), p0 = n0 / KK;
    for (int idx = tid; idx < NPOS * EPI * BM; idx += NT) {
      const int r = idx % BM, s = (idx / BM) % EPI, pp = idx / (BM * EPI);
      if (p0 + pp >= nact) continue;
      const int slot = k1_slot(ep.a, p0 + pp);
      const double* ur = Us + r * UST + pp * KK + s * EPI;  // U[(s, t), row r], t = 0..k-1
      k1_out_element<EPI>(ep, slot, s, m0 + r, ur, ur + UST, UST);
    }
  } else {
    // store: lane holds C[row][2c], C[row][2c+1]
#pragma unroll
    for (int i = 0; i < MT; ++i) {
      int row = m0 + wm * WM + i * 8 + (lane >> 2);
#pragma unroll
      for (int j = 0; j < NTL; ++j) {
        int col = n0 + wn * WN + j * 8 + (lane & 3) * 2;
        if (OUT == 0) {
          *reinterpret_cast<double2*>(C + (int64_t)row * N + col) = make_double2(acc[i][j][0], acc[i][j][1]);
        } else if (OUT == 1) {
          const int v = row / om.blk, r = row % om.blk;
          *reinterpret_cast<double2*>(C + (int64_t)r * N * om.nblk + (int64_t)v * N + col) =
              make_double2(acc[i][j][0], acc[i][j][1]);
        } else {
          const int v = col / om.blk, c = col % om.blk;
          if (row < om.no) {
            double* dst = C + ((int64_t)v * om.no + row) * om.no;
            if (c < om.no) dst[c] = acc[i][j][0];
            if (c + 1 < om.no) dst[c + 1] = acc[i][j][1];
          }
        }
      }
    }
  }
}

// One output element of K1 (k1_epi's contraction): row c of parameter s of the slot's vector.
// ur[t] = U[(s, t), c], ur1[t] = U[(s, t), c + 1] (the pair's Im row).  Writes C(v)X (or the VERIFY
// residual) into the slot's Krylov basis, or Y in apply mode.
template <int K>
__device__ __forceinline__ void k1_out_element(const K1EpiArgs& ep, int slot, int s, int c, const double* ur,
                                               const double* ur1, int) {
  const K1Args& a = ep.a;
  const int npad = ep.npad;
  const double* gsrc = a.rhs ? a.rhs + (int64_t)slot * a.L : ep.g0;
  const double* x = a.Xin + (int64_t)slot * a.L;
  K1Dst dst;
  bool verify = false;
  double msk = 1.0, sig;
  if (a.mode == 0) {
    dst = K1Dst{a.Yout + (int64_t)slot * a.L + (int64_t)s * npad, nullptr};
    sig = a.sigma ? a.sigma[slot * K + s] : 0.0;
  } else {
    const int ph = a.phase[slot];
    int64_t off;
    if (ph == PH_ITER) {
      off = (int64_t)slot * a.qstride + (int64_t)(a.m[slot] + 1) * a.L + (int64_t)s * npad;
    } else if (ph == PH_VERIFY) {
      off = (int64_t)slot * a.qstride + (int64_t)s * npad;
      verify = true;
    } else {
      return;
    }
    dst = a.Qf ? K1Dst{nullptr, a.Qf + off} : K1Dst{a.Qb + off, nullptr};
    sig = a.sigma[slot * K + s];
    msk = a.mask[slot * K + s];
  }
  if (c >= ep.n) {  // zero padding stays zero
    dst.put(c, 0.0);
    return;
  }
  if (c < ep.two_np) {
    if (c & 1) return;  // the Re-coordinate thread writes both coordinates of the pair
    const int rep = c >> 1;
    cplx y = mk(0.0, 0.0);
#pragma unroll
    for (int t = 0; t < K; ++t) {
      const cplx u = mk(ur[t], ur1[t]);
      const cplx bl = mk(ep.btl[(int64_t)c * K + t], ep.btl[(int64_t)(c + 1) * K + t]);
      const double* f = ep.F + (((int64_t)rep * K + s) * K + t) * 2;
      const cplx xt = mk(x[(int64_t)t * npad + c], x[(int64_t)t * npad + c + 1]);
      y = y + bl * u + mk(f[0], f[1]) * xt;
    }
    const cplx xv = mk(x[(int64_t)s * npad + c], x[(int64_t)s * npad + c + 1]);
    cplx o = (msk != 0.0) ? (sig * xv - y) : xv;
    if (verify) o = mk(msk * gsrc[(int64_t)s * npad + c], msk * gsrc[(int64_t)s * npad + c + 1]) - o;
    dst.put(c, o.re);
    dst.put(c + 1, o.im);
  } else {
    const int rep = c - ep.two_np + ep.npairs;
    double y = 0.0;
#pragma unroll
    for (int t = 0; t < K; ++t) {
      y += ep.btl[(int64_t)c * K + t] * ur[t];
      y += ep.F[(((int64_t)rep * K + s) * K + t) * 2] * x[(int64_t)t * npad + c];
    }
    const double xv = x[(int64_t)s * npad + c];
    double o = (msk != 0.0) ? (sig * xv - y) : xv;
    if (verify) o = msk * gsrc[(int64_t)s * npad + c] - o;
    dst.put(c, o);
  }
}

// ------------------------------------------------------------------------------------------
// K1c epilogue: contract U over t with B~l, add T_d, form C(v) X (or the VERIFY residual).
// MP: positions [0, nver) read the FP64 GEMM output U, the others the float output U32 (same layout)
template <int K, bool MP = false>
__global__ void __launch_bounds__(256) k1_epi(K1Args a, const double* __restrict__ U, int64_t ncol,
                                               const double* __restrict__ btl, const double* __restrict__ F,
                                               const double* __restrict__ g0, int npad, int two_np, int npairs,
                                               int n, const float* __restrict__ U32 = nullptr, int which = 0) {
  constexpr int TS = K1Tile<K>::TS, NC = K1Tile<K>::NC, TC = K1_TILE_C;
  const int nact = k1_nact(a);
  const int i0 = blockIdx.x * TC, s0 = blockIdx.y * TS;
  if (s0 >= nact) return;
  __shared__ double us[TC][NC + 1];
  __shared__ double xs[TS][K][TC];
  const int nver = MP ? *a.nver : nact;
#pragma unroll
  for (int idx = threadIdx.x; idx < TC * NC; idx += K1_THREADS) {
    // MP: the float product is column-major (U32t[n][m]): coordinate-fast mapping for coalesced loads
    const int r = MP ? idx % TC : idx / NC, col = MP ? idx / TC : idx % NC;
    const int pos = s0 + col / (K * K);
    double u = 0.0;
    if (pos < nact) {
      if (MP && pos >= nver)
        u = (double)U32[((int64_t)s0 * K * K + col) * npad + i0 + r];
      else
        u = U[(int64_t)(i0 + r) * ncol + (int64_t)s0 * K * K + col];
    }
    us[r][col] = u;
  }
#pragma unroll
  for (int idx = threadIdx.x; idx < TS * K * TC; idx += K1_THREADS) {
    int sl = idx / (K * TC), t = (idx / TC) % K, c = idx % TC;
    xs[sl][t][c] = (s0 + sl < nact) ? a.Xin[(int64_t)k1_slot(a, s0 + sl) * a.L + (int64_t)t * npad + i0 + c] : 0.0;
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < TS * K * TC; idx += K1_THREADS) {
    int sl = idx / (K * TC), s = (idx / TC) % K, r = idx % TC;
    if (s0 + sl >= nact) continue;
    // MP, which = 1 / 2: only the VERIFY / only the ITER positions (the other part's epilogue is fused)
    if (MP && ((which == 1 && s0 + sl >= nver) || (which == 2 && s0 + sl < nver))) continue;
    const int slot = k1_slot(a, s0 + sl);
    const double* gsrc = a.rhs ? a.rhs + (int64_t)slot * a.L : g0;
    int c = i0 + r;
    K1Dst dst;
    bool verify = false;
    double msk = 1.0, sig;
    if (a.mode == 0) {
      dst = K1Dst{a.Yout + (int64_t)slot * a.L + (int64_t)s * npad, nullptr};
      sig = a.sigma ? a.sigma[slot * K + s] : 0.0;
    } else {
      int ph = a.phase[slot];
      int64_t off;
      if (ph == PH_ITER) {
        off = (int64_t)slot * a.qstride + (int64_t)(a.m[slot] + 1) * a.L + (int64_t)s * npad;
      } else if (ph == PH_VERIFY) {
        off = (int64_t)slot * a.qstride + (int64_t)s * npad;
        verify = true;
      } else {
        continue;
      }
      dst = a.Qf ? K1Dst{nullptr, a.Qf + off} : K1Dst{a.Qb + off, nullptr};
      sig = a.sigma[slot * K + s];
      msk = a.mask[slot * K + s];
    }
    if (c >= n) {  // zero padding stays zero
      dst.put(c, 0.0);
      continue;
    }
    const int colb = sl * K * K + s * K;
    if (c < two_np) {
      if (r & 1) continue;  // the Re-coordinate thread writes both coordinates of the pair
      const int rep = c >> 1;
      cplx y = mk(0.0, 0.0);
#pragma unroll
      for (int t = 0; t < K; ++t) {
        cplx u = mk(us[r][colb + t], us[r + 1][colb + t]);
        cplx bl = mk(btl[(int64_t)c * K + t], btl[(int64_t)(c + 1) * K + t]);
        const double* f = F + (((int64_t)rep * K + s) * K + t) * 2;
        cplx x = mk(xs[sl][t][r], xs[sl][t][r + 1]);
        y = y + bl * u + mk(f[0], f[1]) * x;
      }
      cplx xv = mk(xs[sl][s][r], xs[sl][s][r + 1]);
      cplx o = (msk != 0.0) ? (sig * xv - y) : xv;
      if (verify) {
        o = mk(msk * gsrc[(int64_t)s * npad + c], msk * gsrc[(int64_t)s * npad + c + 1]) - o;
      }
      dst.put(c, o.re);
      dst.put(c + 1, o.im);
    } else {
      const int rep = c - two_np + npairs;
      double y = 0.0;
#pragma unroll
      for (int t = 0; t < K; ++t) {
        y += btl[(int64_t)c * K + t] * us[r][colb + t];
        y += F[(((int64_t)rep * K + s) * K + t) * 2] * xs[sl][t][r];
      }
      double xv = xs[sl][s][r];
      double o = (msk != 0.0) ? (sig * xv - y) : xv;
      if (verify) o = msk * gsrc[(int64_t)s * npad + c] - o;
      dst.put(c, o);
    }
  }
}

}  // namespace lyap
