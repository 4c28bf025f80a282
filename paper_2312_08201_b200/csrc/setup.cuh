// Seed setup kernels (offline stage, Table 1).
//
// A0 = S Lambda S^{-1} is obtained from the real LAPACK-style eigenvector packing S_r of
// cusolverDnXgeev: for a conjugate pair (p, p+1), s_p = S_r e_p + i S_r e_{p+1} and
// s_{p+1} = conj(s_p), i.e. S = S_r J with J = blockdiag([[1, 1], [i, -i]]) on pairs and 1 on
// real eigenvalues.  All n^3 work is real (cuBLAS DGEMM on S_r, S_r^{-1}); the complex seed
// quantities are then produced entrywise from the real products through J:
//   Q~ = S^{-1} Q S^{-T} = J^{-1} Q_r J^{-T},  Q_r = S_r^{-1} Q S_r^{-T}
//   E~ = S^T E S         = J^T E_r J,          E_r = S_r^T E S_r
//   B~l = S^{-1} Bl = J^{-1} (S_r^{-1} Bl),     B^r = S^T Br = J^T (S_r^T Br)
// and, with the Cauchy matrix L_ij = 1/(lambda_i + lambda_j):
//   X~0 = -L o Q~            (seed solve, eq. (seedLE) PAPER.md:154-156 via PAPER.md:226-234)
//   G0_{s,j} = sum_i B^r_is X~0_ij       (v-independent right-hand side)
//   H_{j,t}  = sum_i (E~ o L)_ij B~l_it  (trace weights)
//   F_j[s,t] = sum_i L_ij B^r_is B~l_it  (T_d blocks = eq. (N1M1) / (2,2) block)
//   t0 = sum_ij E~_ij X~0_ij = trace(E X0)
#pragma once
#include "common.cuh"

namespace lyap {

// out (cols x rows, row-major) = in^T, in: rows x cols row-major
__global__ void k_transpose(const double* __restrict__ in, double* __restrict__ out, int64_t rows, int64_t cols) {
  __shared__ double tile[32][33];
  int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    int64_t r = r0 + i, c = c0 + threadIdx.x;
    if (r < rows && c < cols) tile[i][threadIdx.x] = in[r * cols + c];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    int64_t c = c0 + i, r = r0 + threadIdx.x;
    if (r < rows && c < cols) out[c * rows + r] = tile[threadIdx.x][i];
  }
}

// out = (M + M^T) / 2 for square n x n
__global__ void k_symmetrize(const double* __restrict__ M, double* __restrict__ out, int64_t n) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n * n) return;
  int64_t i = idx / n, j = idx % n;
  out[idx] = 0.5 * (M[i * n + j] + M[j * n + i]);
}

// S_r[:, new] = VR[:, perm[new]]  (column-major n x n)
__global__ void k_gather_cols(const double* __restrict__ VR, const int* __restrict__ perm,
                              double* __restrict__ Sr, int64_t n) {
  int64_t col = blockIdx.y;
  const double* src = VR + (int64_t)perm[col] * n;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    Sr[col * n + i] = src[i];
}

// max over columns of sum |M_ij| (1-norm) of a column-major n x n matrix -> *out (as bits)
__global__ void k_norm1(const double* __restrict__ M, int64_t n, unsigned long long* out) {
  __shared__ double red[32];
  int64_t col = blockIdx.x;
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += fabs(M[col * n + i]);
  s = block_sum(s, red);
  if (threadIdx.x == 0) atomicMax(out, (unsigned long long)__double_as_longlong(s));
}

// eigenvalue of eigen index i (folded coordinates: pair -> coords 2r (lambda), 2r+1 (conj))
__device__ __forceinline__ cplx eig_of(const double* lam, int64_t i, int64_t two_np) {
  cplx l = mk(lam[2 * i], lam[2 * i + 1]);
  return (i < two_np && (i & 1)) ? conj(l) : l;
}

// min_{i,j} |lambda_i + lambda_j| and max |lambda| (as bits; positive doubles order like ints)
__global__ void k_lam_extremes(const double* __restrict__ lam, int64_t n, int64_t two_np,
                               unsigned long long* minsum, unsigned long long* maxabs) {
  int64_t i = blockIdx.y;
  cplx li = eig_of(lam, i, two_np);
  double mn = 1e300;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    cplx s = li + eig_of(lam, j, two_np);
    mn = fmin(mn, sqrt(abs2(s)));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
  if ((threadIdx.x & 31) == 0) atomicMin(minsum, (unsigned long long)__double_as_longlong(mn));
  if (blockIdx.x == 0 && threadIdx.x == 0)
    atomicMax(maxabs, (unsigned long long)__double_as_longlong(sqrt(abs2(li))));
}

// J^{-1} row coefficients of eigen index i over its block base coords (a0, a0+1)
__device__ __forceinline__ void jinv_row(int64_t i, int64_t two_np, cplx& c0, cplx& c1, int& w) {
  if (i < two_np) {
    w = 2;
    c0 = mk(0.5, 0.0);
    c1 = (i & 1) ? mk(0.0, 0.5) : mk(0.0, -0.5);
  } else {
    w = 1;
    c0 = mk(1.0, 0.0);
    c1 = mk(0.0, 0.0);
  }
}
// J column coefficients of eigen index i: (1, +-i) on pairs, 1 on reals
__device__ __forceinline__ void j_col(int64_t i, int64_t two_np, cplx& c0, cplx& c1, int& w) {
  if (i < two_np) {
    w = 2;
    c0 = mk(1.0, 0.0);
    c1 = (i & 1) ? mk(0.0, -1.0) : mk(0.0, 1.0);
  } else {
    w = 1;
    c0 = mk(1.0, 0.0);
    c1 = mk(0.0, 0.0);
  }
}

// One block per representative j (pairs: the eigen index with Im > 0; reals): sums over all n
// eigen indices i of G0_{s,j}, H_{j,t}, F_j[s,t] and the t0 contribution; folds the results.
// Qr, Er: column-major n x n symmetric; Blr, Brr: column-major n x k.
template <int K>
__global__ void __launch_bounds__(128) k_seed_rep(const double* __restrict__ lam, const double* __restrict__ Qr,
                                                  const double* __restrict__ Er, const double* __restrict__ Blr,
                                                  const double* __restrict__ Brr, int64_t n, int64_t npad,
                                                  int64_t two_np, int64_t npairs, double* __restrict__ g0,
                                                  double* __restrict__ hf, double* __restrict__ F,
                                                  double* __restrict__ t0part) {
  __shared__ double red[4];
  const int64_t rep = blockIdx.x;
  const int64_t j = rep < npairs ? 2 * rep : rep + npairs;  // eigen index / coordinate of rep
  const cplx lj = eig_of(lam, j, two_np);
  cplx jq0, jq1, je0, je1;
  int wj;
  jinv_row(j, two_np, jq0, jq1, wj);
  j_col(j, two_np, je0, je1, wj);
  cplx G[K], Hs[K], Fs[K][K], T0 = mk(0.0, 0.0);
#pragma unroll
  for (int s = 0; s < K; ++s) {
    G[s] = Hs[s] = mk(0.0, 0.0);
#pragma unroll
    for (int t = 0; t < K; ++t) Fs[s][t] = mk(0.0, 0.0);
  }
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const int64_t a0 = (i < two_np) ? (i & ~(int64_t)1) : i;
    cplx ia0, ia1, ic0, ic1;
    int wi;
    jinv_row(i, two_np, ia0, ia1, wi);
    j_col(i, two_np, ic0, ic1, wi);
    // Q~_ij = sum_{a,c} Jinv_{i,a} Qr[a,c] Jinv_{j,c};  E~_ij = sum J_{a,i} Er[a,c] J_{c,j}
    cplx q = mk(0.0, 0.0), e = mk(0.0, 0.0);
    for (int cc = 0; cc < wj; ++cc) {
      const int64_t c = j + cc;
      cplx qj = cc ? jq1 : jq0, ej = cc ? je1 : je0;
      const double* qcol = Qr + c * n;  // symmetric: Qr[a, c] = Qr[c, a] -> column c, row a
      const double* ecol = Er + c * n;
      cplx qa = ia0 * mk(qcol[a0], 0.0), ea = ic0 * mk(ecol[a0], 0.0);
      if (wi == 2) {
        qa = qa + ia1 * mk(qcol[a0 + 1], 0.0);
        ea = ea + ic1 * mk(ecol[a0 + 1], 0.0);
      }
      q = q + qa * qj;
      e = e + ea * ej;
    }
    const cplx Lij = cinv(eig_of(lam, i, two_np) + lj);
    const cplx x0 = mk(-1.0, 0.0) * (Lij * q);
    cplx bl[K], br[K];
#pragma unroll
    for (int t = 0; t < K; ++t) {
      double b0 = Blr[(int64_t)t * n + a0], c0 = Brr[(int64_t)t * n + a0];
      if (wi == 2) {
        double b1 = Blr[(int64_t)t * n + a0 + 1], c1 = Brr[(int64_t)t * n + a0 + 1];
        bl[t] = ia0 * mk(b0, 0.0) + ia1 * mk(b1, 0.0);
        br[t] = ic0 * mk(c0, 0.0) + ic1 * mk(c1, 0.0);
      } else {
        bl[t] = mk(b0, 0.0);
        br[t] = mk(c0, 0.0);
      }
    }
    const cplx eL = e * Lij;
    T0 = T0 + e * x0;
#pragma unroll
    for (int s = 0; s < K; ++s) {
      G[s] = G[s] + br[s] * x0;
      Hs[s] = Hs[s] + eL * bl[s];
      const cplx lb = Lij * br[s];
#pragma unroll
      for (int t = 0; t < K; ++t) Fs[s][t] = Fs[s][t] + lb * bl[t];
    }
  }
  // block reductions (fixed order) and folding
#pragma unroll
  for (int s = 0; s < K; ++s) {
    G[s].re = block_sum(G[s].re, red);
    G[s].im = block_sum(G[s].im, red);
    Hs[s].re = block_sum(Hs[s].re, red);
    Hs[s].im = block_sum(Hs[s].im, red);
#pragma unroll
    for (int t = 0; t < K; ++t) {
      Fs[s][t].re = block_sum(Fs[s][t].re, red);
      Fs[s][t].im = block_sum(Fs[s][t].im, red);
    }
  }
  T0.re = block_sum(T0.re, red);
  if (threadIdx.x == 0) {
    const bool pair = j < two_np;
#pragma unroll
    for (int s = 0; s < K; ++s) {
      if (pair) {
        g0[s * npad + j] = G[s].re;
        g0[s * npad + j + 1] = G[s].im;
        hf[s * npad + j] = 2.0 * Hs[s].re;
        hf[s * npad + j + 1] = -2.0 * Hs[s].im;
      } else {
        g0[s * npad + j] = G[s].re;
        hf[s * npad + j] = Hs[s].re;
      }
#pragma unroll
      for (int t = 0; t < K; ++t) {
        F[((rep * K + s) * K + t) * 2] = Fs[s][t].re;
        F[((rep * K + s) * K + t) * 2 + 1] = pair ? Fs[s][t].im : 0.0;
      }
    }
    t0part[rep] = (pair ? 2.0 : 1.0) * T0.re;
  }
}

// folded B^r (= S_r^T Br rows as is) and B~l (pairs: (b0/2, -b1/2)); zero padding
__global__ void k_fold_b(const double* __restrict__ Blr, const double* __restrict__ Brr, int64_t n, int64_t npad,
                         int64_t k, int64_t two_np, double* __restrict__ btl, double* __restrict__ bhr) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= npad * k) return;
  int64_t c = idx / k, t = idx % k;
  double vl = 0.0, vr = 0.0;
  if (c < n) {
    vr = Brr[t * n + c];
    vl = Blr[t * n + c];
    if (c < two_np) vl = (c & 1) ? -0.5 * vl : 0.5 * vl;
  }
  btl[c * k + t] = vl;
  bhr[c * k + t] = vr;
}

// Folded Cauchy matrix Lf (npad x npad, row-major): row = output coordinate j, col = input i.
// Pair-pair block (j rows Re/Im, i cols x/y):  a+ib = L(i,j), c+id = L(conj i, j):
//   [[a+c, d-b], [b+d, a-c]];  pair j / real i: [a; b];  real j / pair i: [2a, -2b];  real-real: a.
__global__ void k_build_Lf(const double* __restrict__ lam, int64_t n, int64_t npad, int64_t two_np,
                           double* __restrict__ Lf) {
  int64_t ic = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t jc = blockIdx.y;
  if (ic >= npad) return;
  double val = 0.0;
  if (ic < n && jc < n) {
    const bool pj = jc < two_np, pi = ic < two_np;
    const int64_t jr = pj ? (jc & ~(int64_t)1) : jc, ir = pi ? (ic & ~(int64_t)1) : ic;
    const cplx lj = mk(lam[2 * jr], lam[2 * jr + 1]), li = mk(lam[2 * ir], lam[2 * ir + 1]);
    const cplx L1 = cinv(li + lj);
    const int rj = pj ? (int)(jc & 1) : 0, ri = pi ? (int)(ic & 1) : 0;
    if (pj && pi) {
      const cplx L2 = cinv(conj(li) + lj);
      const double a = L1.re, b = L1.im, c = L2.re, d = L2.im;
      val = rj == 0 ? (ri == 0 ? a + c : d - b) : (ri == 0 ? b + d : a - c);
    } else if (pj) {
      val = rj == 0 ? L1.re : L1.im;
    } else if (pi) {
      val = ri == 0 ? 2.0 * L1.re : -2.0 * L1.im;
    } else {
      val = L1.re;
    }
  }
  Lf[jc * npad + ic] = val;
}


// Per-rep diagonal block of the folded T (the preconditioner's v-independent part, engine.cuh
// k_pfactor): the exact response of K1's operator (k1_gen -> Lf -> k1_epi) at the rep's own
// coordinates to a unit input there -- T_d (F) plus the Cauchy coupling restricted to the rep's own
// folded 2 x 2 block of Lf (for a pair: L_jj and L_{conj j, j} = 1/(2 Re lambda_j)).
// Pb[rep][(2s + a) * 2K + (2t + b)] for pairs (a, b = Re, Im), Pb[rep][s * 2K + t] for reals.
template <int K>
__global__ void k_pblock(const double* __restrict__ Lf, int64_t npad, const double* __restrict__ bhr,
                         const double* __restrict__ btl, const double* __restrict__ F, int64_t npairs, int64_t nrep,
                         double* __restrict__ Pb) {
  const int64_t rep = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (rep >= nrep) return;
  constexpr int RS = 2 * K;
  double* out = Pb + rep * 4 * K * K;
  const bool pair = rep < npairs;
  const int64_t c = pair ? 2 * rep : rep + npairs;
  if (pair) {
    const double l00 = Lf[c * npad + c], l01 = Lf[c * npad + c + 1];
    const double l10 = Lf[(c + 1) * npad + c], l11 = Lf[(c + 1) * npad + c + 1];
    for (int t = 0; t < K; ++t)
      for (int b = 0; b < 2; ++b) {
        const double x = b == 0 ? 1.0 : 0.0, y = b == 0 ? 0.0 : 1.0;  // unit input X_t = e_b
        for (int s = 0; s < K; ++s) {
          const double br = bhr[c * K + s], bi = bhr[(c + 1) * K + s];
          const double p0 = br * x - bi * y, p1 = br * y + bi * x;  // k1_gen: (B^r_s)(x + iy)
          const cplx u = mk(l00 * p0 + l01 * p1, l10 * p0 + l11 * p1);  // Lf block
          const cplx bl = mk(btl[c * K + t], btl[(c + 1) * K + t]);
          const double* f = F + ((rep * K + s) * K + t) * 2;
          const cplx yv = bl * u + mk(f[0], f[1]) * mk(x, y);  // k1_epi
          out[(2 * s) * RS + 2 * t + b] = yv.re;
          out[(2 * s + 1) * RS + 2 * t + b] = yv.im;
        }
      }
  } else {
    const double l = Lf[c * npad + c];
    for (int s = 0; s < K; ++s)
      for (int t = 0; t < K; ++t)
        out[s * RS + t] = btl[c * K + t] * l * bhr[c * K + s] + F[((rep * K + s) * K + t) * 2];
  }
}

// Full solution (NEXT row f2, eq. (Xsmalllastline)): with the solved
// G, X~ = X~0 + L o (B~l G + G^T B~l^T), X~0 = -L o Q~, and X = S X~ S^T = S_r Y S_r^T with the REAL
// matrix Y = J X~ J^T, generated here entrywise for a chunk of parameter vectors, written as a
// vertical stack of np x np blocks (np = n padded to the GEMM tile; padding stays zero):
// Yst[(v np + a) np + b].  The Hadamard product with the Cauchy matrix is formed element by element,
// never as a matrix; g: folded k x npad per v.
// (v-linear Q, nterms > 0: Q~(v) = sum_i v_i Q~_i with the rows of V (chunk offset v0) as weights)
__global__ void k_solution_Ystack(const double* __restrict__ lam, const double* __restrict__ Qr,
                                  const double* __restrict__ btl, const double* __restrict__ g, int64_t n, int64_t npad,
                                  int64_t k, int64_t two_np, int64_t np, double* __restrict__ Yst,
                                  const double* __restrict__ V = nullptr, int64_t v0 = 0, int nterms = 0) {
  const int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t b = blockIdx.y, v = blockIdx.z;
  if (a >= n) return;
  const double* gv = g + v * k * npad;
  auto qr = [&](int64_t idx) -> double {  // Q_r(v) entry
    if (nterms <= 0) return Qr[idx];
    double acc = 0.0;
    for (int i = 0; i < nterms; ++i) acc += V[(v0 + v) * k + i] * Qr[(int64_t)i * n * n + idx];
    return acc;
  };
  auto blk = [&](int64_t c, int64_t* idx, cplx* jc, int& w) {
    if (c < two_np) {
      const int64_t p0 = c & ~(int64_t)1;
      idx[0] = p0;
      idx[1] = p0 + 1;
      w = 2;
      if (c & 1) {
        jc[0] = mk(0.0, 1.0);
        jc[1] = mk(0.0, -1.0);
      } else {
        jc[0] = mk(1.0, 0.0);
        jc[1] = mk(1.0, 0.0);
      }
    } else {
      idx[0] = c;
      jc[0] = mk(1.0, 0.0);
      w = 1;
    }
  };
  auto folded = [&](int64_t t, int64_t i) -> cplx {
    if (i < two_np) {
      const int64_t p0 = i & ~(int64_t)1;
      const cplx z = mk(gv[t * npad + p0], gv[t * npad + p0 + 1]);
      return (i & 1) ? conj(z) : z;
    }
    return mk(gv[t * npad + i], 0.0);
  };
  auto blt = [&](int64_t i, int64_t t) -> cplx {
    if (i < two_np) {
      const int64_t p0 = i & ~(int64_t)1;
      const cplx z = mk(btl[p0 * k + t], btl[(p0 + 1) * k + t]);
      return (i & 1) ? conj(z) : z;
    }
    return mk(btl[i * k + t], 0.0);
  };
  int64_t ia[2], jb[2];
  cplx ja[2], jbv[2];
  int wa, wb;
  blk(a, ia, ja, wa);
  blk(b, jb, jbv, wb);
  cplx acc = mk(0.0, 0.0);
  for (int u = 0; u < wa; ++u) {
    const int64_t i = ia[u];
    cplx ci0, ci1;
    int wi;
    jinv_row(i, two_np, ci0, ci1, wi);
    const int64_t ai0 = (i < two_np) ? (i & ~(int64_t)1) : i;
    for (int q = 0; q < wb; ++q) {
      const int64_t j = jb[q];
      cplx cj0, cj1;
      int wj;
      jinv_row(j, two_np, cj0, cj1, wj);
      const int64_t aj0 = (j < two_np) ? (j & ~(int64_t)1) : j;
      cplx qt = mk(0.0, 0.0);
      for (int x = 0; x < wi; ++x)
        for (int y = 0; y < wj; ++y)
          qt = qt + ((x ? ci1 : ci0) * (y ? cj1 : cj0)) * mk(qr((aj0 + y) * n + ai0 + x), 0.0);
      cplx rhs = mk(-qt.re, -qt.im);
      for (int64_t t = 0; t < k; ++t) rhs = rhs + blt(i, t) * folded(t, j) + folded(t, i) * blt(j, t);
      const cplx L = cinv(eig_of(lam, i, two_np) + eig_of(lam, j, two_np));
      acc = acc + (ja[u] * jbv[q]) * (L * rhs);
    }
  }
  Yst[(v * np + a) * np + b] = acc.re;
}

// padded copies of S_r (column-major n x n) for the batched solution GEMMs: Sc = S_r column-major
// (as a row-major matrix: S_r^T), Sr = S_r row-major; np x np, zero padding
__global__ void k_pad_basis(const double* __restrict__ S, int64_t n, int64_t np, double* __restrict__ Sc,
                            double* __restrict__ Srow) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, r = blockIdx.y;
  if (c >= np) return;
  const bool in = r < n && c < n;
  Sc[r * np + c] = in ? S[r * n + c] : 0.0;    // row r of S_r^T = column r of S_r
  Srow[r * np + c] = in ? S[c * n + r] : 0.0;  // S_r[r][c]
}

// Coarse-space build helpers: unit vectors e_{c0 + j} (j < nb) as nb x L rows
__global__ void k_unit_vectors(double* __restrict__ X, int64_t c0, int64_t nb, int64_t L) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nb * L; i += (int64_t)gridDim.x * blockDim.x)
    X[i] = (i % L == c0 + i / L) ? 1.0 : 0.0;
}
// Tm[:, c0 + j] = -Y[j] (apply_C with sigma = 0 returns -T e)
__global__ void k_neg_copy(const double* __restrict__ Y, double* __restrict__ Tcol, int64_t cnt) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * blockDim.x)
    Tcol[i] = -Y[i];
}
// T_o' = T - (the pair blocks Pb): column-major L x L explicit folded T, one thread per rep
template <int K>
__global__ void k_sub_pblocks(double* __restrict__ Tm, int64_t L, int64_t npad, const double* __restrict__ Pb,
                              int64_t npairs, int64_t nrep) {
  const int64_t rep = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (rep >= nrep) return;
  const bool pair = rep < npairs;
  const int64_t c = pair ? 2 * rep : rep + npairs;
  const int w = pair ? 2 : 1;
  const double* pb = Pb + rep * 4 * K * K;
  for (int t = 0; t < K; ++t)
    for (int a = 0; a < w; ++a)
      for (int u = 0; u < K; ++u)
        for (int b = 0; b < w; ++b) {
          const int64_t row = t * npad + c + a, col = u * npad + c + b;
          const int pr = pair ? 2 * t + a : t, pcol = pair ? 2 * u + b : u;
          Tm[col * L + row] -= pb[pr * 2 * K + pcol];
        }
}

// deterministic sum of t0 partials (one block)
__global__ void k_sum(const double* __restrict__ x, int64_t n, double* out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += x[i];
  s = block_sum(s, red);
  if (threadIdx.x == 0) *out = s;
}

__global__ void k_negate(double* x, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = -x[i];
}

__global__ void k_set_identity(double* M, int64_t n) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx < n * n) M[idx] = (idx / n == idx % n) ? 1.0 : 0.0;
}

}  // namespace lyap
