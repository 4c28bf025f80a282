// Stability filter (NEXT row f4, Example 2: "computed the rightmost eigenvalue of
// A(v) and discarded those configurations for which Re(lambda) >= 0").  DESIGN.md §2.6.
//
// Instead of an eigendecomposition of every A(v) (O(n^3) per v), the number of eigenvalues of A(v)
// in the open right half-plane is counted with the argument principle on the imaginary axis:
//
//   det(A(v) - sI) = det(A0 - sI) g_v(s),   g_v(s) = det(I_k - D(v) G(s)),
//   G(s) = Br^T (A0 - sI)^{-1} Bl = sum_j B^r_j B~l_j^T / (lambda_j - s)          (k x k)
//
// (Sylvester's determinant identity; B^r = S^T Br, B~l = S^{-1} Bl are the seed factors the engine
// already holds).  With Z_R / P_R the right-half-plane eigenvalue counts of A(v) / A0 and no
// eigenvalue on the axis, the phase of g_v along s = i w, w: -inf -> inf, changes by 2 pi (P_R - Z_R);
// g_v(-iw) = conj(g_v(iw)) (real data) and g_v(i inf) = 1, so with S = the unwrapped phase change of
// g_v(iw) for w: 0 -> inf,   Z_R = P_R - S / pi.
// G is v-independent: it is tabulated once on a frequency grid that resolves every pole (points at
// Im lambda_j + m |Re lambda_j|) plus a log-spaced background; per v only k x k determinants remain
// (O(F k^3)).  Beyond the grid, G(iw) = -sum_m M_m / (iw)^{m+1} with the moments
// M_m = sum_j B^r_j B~l_j^T lambda_j^m (w >= 4 max|lambda|), up to w_end(v) where ||D(v) G|| <= 1/2
// (g_v cannot wind around 0 beyond it).  A step whose phase change exceeds pi/4 is subdivided
// (G summed on the fly), twice at most; a zero of g_v on or extremely near the axis (|g_v| < 1e-10
// at a sample, or an unresolved step) reports "marginal" and the v counts as unstable (Re >= 0).
#pragma once
#include "common.cuh"

namespace lyap {

constexpr int STAB_MOMENTS = 40;

// the pole contributions of one rep at s = i w (pair: lambda and conj(lambda))
template <int K>
__device__ __forceinline__ void stab_rep_term(const double* __restrict__ lam, const double* __restrict__ bhr,
                                              const double* __restrict__ btl, int64_t rep, int64_t npairs, double w,
                                              cplx (&acc)[K][K]) {
  const bool pair = rep < npairs;
  const int64_t c = pair ? 2 * rep : rep + npairs;
  const cplx l = mk(lam[2 * c], lam[2 * c + 1]);
  const cplx d1 = cinv(mk(l.re, l.im - w));  // 1 / (lambda - i w)
  if (pair) {
    const cplx d2 = cinv(mk(l.re, -l.im - w));  // 1 / (conj(lambda) - i w)
#pragma unroll
    for (int a = 0; a < K; ++a) {
      const cplx br = mk(bhr[c * K + a], bhr[(c + 1) * K + a]);
#pragma unroll
      for (int b = 0; b < K; ++b) {
        const cplx r = br * mk(btl[c * K + b], btl[(c + 1) * K + b]);
        acc[a][b] = acc[a][b] + r * d1 + conj(r) * d2;
      }
    }
  } else {
#pragma unroll
    for (int a = 0; a < K; ++a)
#pragma unroll
      for (int b = 0; b < K; ++b) acc[a][b] = acc[a][b] + (bhr[c * K + a] * btl[c * K + b]) * d1;
  }
}

// Gf[f] = G(i w_f), one block per frequency (fixed-order reduction: deterministic)
template <int K>
__global__ void __launch_bounds__(128) k_stab_G(const double* __restrict__ lam, const double* __restrict__ bhr,
                                                const double* __restrict__ btl, int64_t nrep, int64_t npairs,
                                                const double* __restrict__ wgrid, double* __restrict__ Gf) {
  __shared__ double red[4];
  const double w = wgrid[blockIdx.x];
  cplx acc[K][K];
#pragma unroll
  for (int a = 0; a < K; ++a)
#pragma unroll
    for (int b = 0; b < K; ++b) acc[a][b] = mk(0.0, 0.0);
  for (int64_t rep = threadIdx.x; rep < nrep; rep += blockDim.x) stab_rep_term<K>(lam, bhr, btl, rep, npairs, w, acc);
  double* out = Gf + (int64_t)blockIdx.x * K * K * 2;
#pragma unroll
  for (int a = 0; a < K; ++a)
#pragma unroll
    for (int b = 0; b < K; ++b) {
      const double re = block_sum(acc[a][b].re, red);
      const double im = block_sum(acc[a][b].im, red);
      if (threadIdx.x == 0) {
        out[(a * K + b) * 2] = re;
        out[(a * K + b) * 2 + 1] = im;
      }
    }
}

// moments M_m = sum_j B^r_j B~l_j^T lambda_j^m, m < STAB_MOMENTS (one block per m)
template <int K>
__global__ void __launch_bounds__(128) k_stab_moments(const double* __restrict__ lam, const double* __restrict__ bhr,
                                                      const double* __restrict__ btl, int64_t nrep, int64_t npairs,
                                                      double scale, double* __restrict__ Mm) {
  __shared__ double red[4];
  const int m = blockIdx.x;
  cplx acc[K][K];
#pragma unroll
  for (int a = 0; a < K; ++a)
#pragma unroll
    for (int b = 0; b < K; ++b) acc[a][b] = mk(0.0, 0.0);
  for (int64_t rep = threadIdx.x; rep < nrep; rep += blockDim.x) {
    const bool pair = rep < npairs;
    const int64_t c = pair ? 2 * rep : rep + npairs;
    const cplx l = mk(lam[2 * c] / scale, lam[2 * c + 1] / scale);  // (lambda / scale)^m: no overflow
    cplx p = mk(1.0, 0.0);
    for (int q = 0; q < m; ++q) p = p * l;
#pragma unroll
    for (int a = 0; a < K; ++a) {
      const cplx br = pair ? mk(bhr[c * K + a], bhr[(c + 1) * K + a]) : mk(bhr[c * K + a], 0.0);
#pragma unroll
      for (int b = 0; b < K; ++b) {
        const cplx bl = pair ? mk(btl[c * K + b], btl[(c + 1) * K + b]) : mk(btl[c * K + b], 0.0);
        const cplx r = br * bl * p;
        acc[a][b] = acc[a][b] + (pair ? mk(2.0 * r.re, 0.0) : mk(r.re, r.im));  // r + conj(r) for a pair
      }
    }
  }
  double* out = Mm + (int64_t)m * K * K * 2;
#pragma unroll
  for (int a = 0; a < K; ++a)
#pragma unroll
    for (int b = 0; b < K; ++b) {
      const double re = block_sum(acc[a][b].re, red);
      const double im = block_sum(acc[a][b].im, red);
      if (threadIdx.x == 0) {
        out[(a * K + b) * 2] = re;
        out[(a * K + b) * 2 + 1] = im;
      }
    }
}

// det(I - D G) for a k x k complex G (row a scaled by v_a); Gaussian elimination, partial pivoting
template <int K>
__device__ __forceinline__ cplx stab_det(const double* __restrict__ v, const cplx (&G)[K][K]) {
  cplx M[K][K];
#pragma unroll
  for (int a = 0; a < K; ++a)
#pragma unroll
    for (int b = 0; b < K; ++b) M[a][b] = mk((a == b ? 1.0 : 0.0) - v[a] * G[a][b].re, -v[a] * G[a][b].im);
  cplx det = mk(1.0, 0.0);
#pragma unroll
  for (int c = 0; c < K; ++c) {
    double best = abs2(M[c][c]);
#pragma unroll
    for (int r = c + 1; r < K; ++r) {
      if (abs2(M[r][c]) > best) {
        best = abs2(M[r][c]);
#pragma unroll
        for (int t = 0; t < K; ++t) {
          const cplx tm = M[c][t];
          M[c][t] = M[r][t];
          M[r][t] = tm;
        }
        det = mk(-det.re, -det.im);
      }
    }
    det = det * M[c][c];
    if (best == 0.0) return mk(0.0, 0.0);
    const cplx inv = cinv(M[c][c]);
#pragma unroll
    for (int r = c + 1; r < K; ++r) {
      const cplx f = M[r][c] * inv;
#pragma unroll
      for (int t = c; t < K; ++t) M[r][t] = M[r][t] - f * M[c][t];
    }
  }
  return det;
}

// G(i w) beyond the grid from the moments (w >= 4 max|lambda|): G = -sum_m M_m / (i w)^{m+1}
template <int K>
__device__ __forceinline__ void stab_G_tail(const double* __restrict__ Mm, double scale, double w, cplx (&G)[K][K]) {
#pragma unroll
  for (int a = 0; a < K; ++a)
#pragma unroll
    for (int b = 0; b < K; ++b) G[a][b] = mk(0.0, 0.0);
  // 1/(i w)^{m+1} * scale^m  (M_m was accumulated with (lambda/scale)^m)
  const cplx z = cinv(mk(0.0, w));  // 1/(iw)
  cplx p = z;
  for (int m = 0; m < STAB_MOMENTS; ++m) {
    const double* M = Mm + (int64_t)m * K * K * 2;
#pragma unroll
    for (int a = 0; a < K; ++a)
#pragma unroll
      for (int b = 0; b < K; ++b) G[a][b] = G[a][b] - mk(M[(a * K + b) * 2], M[(a * K + b) * 2 + 1]) * p;
    p = p * (scale * z);
  }
}

__device__ __forceinline__ double wrap_pi(double d) {
  const double twopi = 6.283185307179586476925286766559;
  d = fmod(d, twopi);
  if (d > 3.14159265358979323846) d -= twopi;
  if (d < -3.14159265358979323846) d += twopi;
  return d;
}

struct StabArgs {
  const double *lam, *bhr, *btl, *wgrid, *Gf, *Mm;
  int64_t nrep, npairs;
  int F;
  double scale, wtail0, rho;  // moment scale, first tail frequency, sum_j |B^r_j| |B~l_j|
  int PR;                     // eigenvalues of A0 in the open right half-plane
  const double* V;
  int nv;
  int32_t* nunstable;  // per v: Z_R, or -1 when marginal / unresolved
};

// G(i w) summed over all reps by the whole warp (used for refinement points)
template <int K>
__device__ void stab_G_warp(const StabArgs& s, double w, cplx (&G)[K][K]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int a = 0; a < K; ++a)
#pragma unroll
    for (int b = 0; b < K; ++b) G[a][b] = mk(0.0, 0.0);
  for (int64_t rep = lane; rep < s.nrep; rep += 32) stab_rep_term<K>(s.lam, s.bhr, s.btl, rep, s.npairs, w, G);
#pragma unroll
  for (int a = 0; a < K; ++a)
#pragma unroll
    for (int b = 0; b < K; ++b) {
      G[a][b].re = warp_sum(G[a][b].re);
      G[a][b].im = warp_sum(G[a][b].im);
    }
}

template <int K>
__device__ __forceinline__ double stab_phase_at(const StabArgs& s, const double* v, double w, bool& tiny) {
  cplx G[K][K];
  if (w >= s.wtail0)
    stab_G_tail<K>(s.Mm, s.scale, w, G);
  else
    stab_G_warp<K>(s, w, G);
  const cplx d = stab_det<K>(v, G);
  tiny = tiny || sqrt(abs2(d)) < 1e-10;
  return atan2(d.im, d.re);
}

// One warp per v: lanes evaluate the tabulated grid in parallel, the warp refines large steps and
// walks the tail.
template <int K>
__global__ void __launch_bounds__(128) k_stab_count(StabArgs s) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= s.nv) return;
  double v[K];
#pragma unroll
  for (int t = 0; t < K; ++t) v[t] = s.V[(int64_t)warp * K + t];
  const double PI = 3.14159265358979323846;
  // 1) phase at every grid point, lane-parallel; per-lane sum of wrapped steps over its points
  const int per = (s.F + 31) / 32;
  const int f0 = lane * per, f1 = min(s.F, f0 + per);
  double sum = 0.0, prev = 0.0, first = 0.0;
  bool tiny = false;
  int bad = 0;
  for (int f = f0; f < f1; ++f) {
    cplx G[K][K];
    const double* g = s.Gf + (int64_t)f * K * K * 2;
#pragma unroll
    for (int a = 0; a < K; ++a)
#pragma unroll
      for (int b = 0; b < K; ++b) G[a][b] = mk(g[(a * K + b) * 2], g[(a * K + b) * 2 + 1]);
    const cplx d = stab_det<K>(v, G);
    tiny = tiny || sqrt(abs2(d)) < 1e-10;
    const double ph = atan2(d.im, d.re);
    if (f == f0) {
      first = ph;
    } else {
      const double dp = wrap_pi(ph - prev);
      if (fabs(dp) > 0.25 * PI) bad = 1;
      sum += dp;
    }
    prev = ph;
  }
  // seams between lanes: step from the last point of lane l to the first of lane l + 1
  const double nfirst = __shfl_down_sync(0xffffffffu, first, 1);
  const bool has_next = lane < 31 && (lane + 1) * per < s.F && f1 > f0;
  if (has_next) {
    const double dp = wrap_pi(nfirst - prev);
    if (fabs(dp) > 0.25 * PI) bad = 1;
    sum += dp;
  }
  sum = warp_sum(sum);
  tiny = __any_sync(0xffffffffu, tiny);
  const int anybad = __any_sync(0xffffffffu, bad);
  // 2) refinement of every step whose wrapped change exceeds pi/4: the warp recomputes the step as
  //    16 sub-steps (and each large sub-step as 16 more)
  bool unresolved = false;
  if (anybad) {
    sum = 0.0;
    double ph_prev = 0.0;
    for (int f = 0; f < s.F; ++f) {
      cplx G[K][K];
      const double* g = s.Gf + (int64_t)f * K * K * 2;
#pragma unroll
      for (int a = 0; a < K; ++a)
#pragma unroll
        for (int b = 0; b < K; ++b) G[a][b] = mk(g[(a * K + b) * 2], g[(a * K + b) * 2 + 1]);
      const cplx d = stab_det<K>(v, G);
      const double ph = atan2(d.im, d.re);
      if (f > 0) {
        double dp = wrap_pi(ph - ph_prev);
        if (fabs(dp) > 0.25 * PI) {
          const double wa = s.wgrid[f - 1], wb = s.wgrid[f];
          double acc = 0.0, pp = ph_prev;
          for (int q = 1; q <= 16; ++q) {
            const double wq = wa + (wb - wa) * q / 16.0;
            const double pq = q == 16 ? ph : stab_phase_at<K>(s, v, wq, tiny);
            double dq = wrap_pi(pq - pp);
            if (fabs(dq) > 0.25 * PI) {  // second level
              const double wqa = wa + (wb - wa) * (q - 1) / 16.0;
              double acc2 = 0.0, p2 = pp;
              for (int r = 1; r <= 16; ++r) {
                const double wr = wqa + (wq - wqa) * r / 16.0;
                const double pr = r == 16 ? pq : stab_phase_at<K>(s, v, wr, tiny);
                const double d2 = wrap_pi(pr - p2);
                if (fabs(d2) > 0.5 * PI) unresolved = true;
                acc2 += d2;
                p2 = pr;
              }
              dq = acc2;
            }
            acc += dq;
            pp = pq;
          }
          dp = acc;
        }
        sum += dp;
      }
      ph_prev = ph;
    }
  }
  // 3) tail: from the last grid point to w_end(v) where ||D G|| <= 1/2, log-spaced (64 per decade),
  //    then to infinity (g -> 1: phase 0)
  double vmax = 0.0;
#pragma unroll
  for (int t = 0; t < K; ++t) vmax = fmax(vmax, fabs(v[t]));
  const double wend = fmax(s.wtail0, 2.0 * s.wtail0 + 2.0 * vmax * s.rho);
  double w = s.wgrid[s.F - 1];
  double ph_prev;
  {
    cplx G[K][K];
    const double* g = s.Gf + (int64_t)(s.F - 1) * K * K * 2;
#pragma unroll
    for (int a = 0; a < K; ++a)
#pragma unroll
      for (int b = 0; b < K; ++b) G[a][b] = mk(g[(a * K + b) * 2], g[(a * K + b) * 2 + 1]);
    const cplx d = stab_det<K>(v, G);
    ph_prev = atan2(d.im, d.re);
  }
  const double ratio = pow(10.0, 1.0 / 64.0);
  while (w < wend) {
    w = fmin(wend, w * ratio);
    const double ph = stab_phase_at<K>(s, v, w, tiny);
    const double dp = wrap_pi(ph - ph_prev);
    if (fabs(dp) > 0.5 * PI) unresolved = true;
    sum += dp;
    ph_prev = ph;
  }
  sum += wrap_pi(0.0 - ph_prev);  // g(i inf) = 1, and |g - 1| <= 1/2 beyond w_end
  if (lane == 0) {
    const double zr = s.PR - sum / PI;
    const int zi = (int)lrint(zr);
    const bool ok = !tiny && !unresolved && fabs(zr - zi) < 0.25 && zi >= 0;
    s.nunstable[warp] = ok ? zi : -1;
  }
}

}  // namespace lyap
