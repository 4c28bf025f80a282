// Batched right-preconditioned GMRES over parameter vectors.
//
// Each of b "slots" solves one capacitance system C(v) g = g0, C(v) = Delta(v) - T (the symmetric
// nk form of eq. (SMW_linearsystem)), right-preconditioned with the exact
// v-dependent block-diagonal part P(v) = Delta(v) - T_d of eq. (prec) (p-bar = 0).
// All slots advance in lock step: one batched K1 launch per iteration applies C(v) to every slot's
// current vector.  A slot walks   VERIFY (true residual of its current iterate, trace, convergence)
// -> ITER (Krylov steps, CGS2) -> XUPD (x += P^{-1} Q y) -> VERIFY ...; a converged slot writes
// tau(v) and takes the next v of the batch (device-side queue, deterministic order).  With
// warm_start the new v starts from the previous v's solution in the slot: neighbouring grid points
// recycle each other's solution (the recycling idea of PAPER.md:375-391, in its simplest form).
// Basis vectors are stored unnormalised (q^_i, with eta_i = ||q^_i||): the grid-wide norm is only
// known one kernel later, so the division is folded into the coefficients that use q_i.
#pragma once
#include "common.cuh"
#include "k1.cuh"

namespace lyap {

constexpr int RED_CE = 1024;  // vector elements per reduction chunk

struct EngArgs {
  int b, mmax, K, nv;
  int64_t L, npad, nrep, npairs, two_np, n;
  int nchunk;
  double tol, tol_inner, t0;
  int max_restarts, warm;
  const double *V, *g0, *hf, *F;
  const int* order;  // queue position -> row of V (null: identity)
  double *X, *Xin, *Qb, *Minv, *sigma, *mask, *eta, *H, *e, *y, *bnorm, *part, *part3;
  int *phase, *m, *vidx, *applies, *restarts, *ctrl, *newv, *alist;
  double* traces;
  int32_t* status;
  int32_t* out_applies;
  double* out_resid;
};

__device__ __forceinline__ int64_t rep_coord(int64_t rep, int64_t npairs) { return rep < npairs ? 2 * rep : rep + npairs; }

// ---------------------------------------------------------------- phase advance + v queue
// One block (b <= 1024 threads): XUPD -> VERIFY; FREE slots take the next v's in slot order.
__global__ void k_assign(EngArgs a) {
  __shared__ int wsum[32];
  __shared__ int base_s;
  const int tid = threadIdx.x;
  int flag = 0;
  if (tid < a.b) {
    a.newv[tid] = 0;
    if (a.phase[tid] == PH_XUPD) a.phase[tid] = PH_VERIFY;
    flag = a.phase[tid] == PH_FREE;
  }
  // block exclusive scan of flag
  const int lane = tid & 31, w = tid >> 5;
  int x = flag;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[w] = x;
  if (tid == 0) base_s = a.ctrl[0];
  __syncthreads();
  int off = 0, total = 0;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {
    if (i < w) off += wsum[i];
    total += wsum[i];
  }
  const int pos = off + x - flag;
  const int base = base_s;
  if (tid < a.b && flag) {
    const int qpos = base + pos;
    if (qpos < a.nv) {
      const int idx = a.order ? a.order[qpos] : qpos;
      a.vidx[tid] = idx;
      for (int t = 0; t < a.K; ++t) {
        const double v = a.V[(int64_t)idx * a.K + t];
        a.mask[tid * a.K + t] = (v != 0.0) ? 1.0 : 0.0;
        a.sigma[tid * a.K + t] = (v != 0.0) ? 1.0 / v : 0.0;
      }
      a.applies[tid] = 0;
      a.restarts[tid] = 0;
      a.newv[tid] = 1;
      a.phase[tid] = PH_VERIFY;
    } else {
      a.phase[tid] = PH_IDLE;
    }
  }
  __syncthreads();
  // active slots after assignment (VERIFY or ITER), compacted in slot order for K1
  int isact = (tid < a.b) ? (a.phase[tid] != PH_IDLE) : 0;
  int xa = isact;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, xa, o);
    if (lane >= o) xa += y;
  }
  __syncthreads();
  if (lane == 31) wsum[w] = xa;
  __syncthreads();
  int offa = 0;
  for (int i = 0; i < w; ++i) offa += wsum[i];
  if (isact) a.alist[offa + xa - 1] = tid;
  const int act = __syncthreads_count(isact);
  if (tid == 0) {
    a.ctrl[0] = base + total;
    a.ctrl[2] = act;
    *reinterpret_cast<unsigned long long*>(a.ctrl + 4) += (unsigned long long)act;  // applied vectors
  }
}

// ---------------------------------------------------------------- preconditioner factor (K2)
// Minv[slot][rep] = (diag(sigma) - F_rep)^{-1}, k x k complex, Gauss-Jordan with partial pivoting;
// rows with v_t = 0 are identity rows (column t absent).  Cold start zeroes X for new v's.
template <int K>
__global__ void __launch_bounds__(128) k_pfactor(EngArgs a) {
  const int slot = blockIdx.y;
  if (!a.newv[slot]) return;
  const int64_t rep = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (rep >= a.nrep) return;
  cplx M[K][K], R[K][K];
#pragma unroll
  for (int s = 0; s < K; ++s) {
    const double msk = a.mask[slot * K + s], sg = a.sigma[slot * K + s];
#pragma unroll
    for (int t = 0; t < K; ++t) {
      const double* f = a.F + ((rep * K + s) * K + t) * 2;
      cplx v = msk != 0.0 ? mk(-f[0], -f[1]) : mk(0.0, 0.0);
      if (s == t) v = msk != 0.0 ? v + mk(sg, 0.0) : mk(1.0, 0.0);
      M[s][t] = v;
      R[s][t] = mk(s == t ? 1.0 : 0.0, 0.0);
    }
  }
#pragma unroll
  for (int c = 0; c < K; ++c) {
    // pivot: largest |M[r][c]|, r >= c (select-swap keeps everything in registers)
    double best = abs2(M[c][c]);
#pragma unroll
    for (int r = c + 1; r < K; ++r) {
      const double v = abs2(M[r][c]);
      if (v > best) {
        best = v;
#pragma unroll
        for (int t = 0; t < K; ++t) {
          cplx tm = M[c][t];
          M[c][t] = M[r][t];
          M[r][t] = tm;
          tm = R[c][t];
          R[c][t] = R[r][t];
          R[r][t] = tm;
        }
      }
    }
    const cplx pinv = cinv(M[c][c]);
#pragma unroll
    for (int t = 0; t < K; ++t) {
      M[c][t] = M[c][t] * pinv;
      R[c][t] = R[c][t] * pinv;
    }
#pragma unroll
    for (int r = 0; r < K; ++r) {
      if (r == c) continue;
      const cplx f = M[r][c];
#pragma unroll
      for (int t = 0; t < K; ++t) {
        M[r][t] = M[r][t] - f * M[c][t];
        R[r][t] = R[r][t] - f * R[c][t];
      }
    }
  }
  double* out = a.Minv + (((int64_t)slot * a.nrep + rep) * K * K) * 2;
#pragma unroll
  for (int s = 0; s < K; ++s)
#pragma unroll
    for (int t = 0; t < K; ++t) {
      out[(s * K + t) * 2] = R[s][t].re;
      out[(s * K + t) * 2 + 1] = R[s][t].im;
    }
  if (!a.warm) {
    const int64_t c = rep_coord(rep, a.npairs);
    const int w = rep < a.npairs ? 2 : 1;
    for (int t = 0; t < K; ++t)
      for (int q = 0; q < w; ++q) a.X[(int64_t)slot * a.L + t * a.npad + c + q] = 0.0;
  }
}

// z = Minv_rep * r (k complex), real reps keep the real part
template <int K>
__device__ __forceinline__ void apply_minv(const double* mi, const cplx (&r)[K], cplx (&z)[K]) {
#pragma unroll
  for (int s = 0; s < K; ++s) {
    cplx acc = mk(0.0, 0.0);
#pragma unroll
    for (int t = 0; t < K; ++t) acc = acc + mk(mi[(s * K + t) * 2], mi[(s * K + t) * 2 + 1]) * r[t];
    z[s] = acc;
  }
}

// ---------------------------------------------------------------- apply input (K2 apply)
// ITER: Xin = P(v)^{-1} (q^_m / eta_m);  VERIFY: Xin = X.
template <int K>
__global__ void __launch_bounds__(128) k_prec(EngArgs a) {
  const int slot = blockIdx.y;
  const int ph = a.phase[slot];
  if (ph != PH_ITER && ph != PH_VERIFY) return;
  const int64_t rep = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (rep >= a.nrep) return;
  const int64_t c = rep_coord(rep, a.npairs);
  const bool pair = rep < a.npairs;
  double* xin = a.Xin + (int64_t)slot * a.L;
  if (ph == PH_VERIFY) {
    const double* x = a.X + (int64_t)slot * a.L;
#pragma unroll
    for (int t = 0; t < K; ++t) {
      xin[t * a.npad + c] = x[t * a.npad + c];
      if (pair) xin[t * a.npad + c + 1] = x[t * a.npad + c + 1];
    }
    return;
  }
  const int m = a.m[slot];
  const double sc = 1.0 / a.eta[(int64_t)slot * (a.mmax + 1) + m];
  const double* q = a.Qb + ((int64_t)slot * (a.mmax + 1) + m) * a.L;
  cplx r[K], z[K];
#pragma unroll
  for (int t = 0; t < K; ++t) r[t] = mk(sc * q[t * a.npad + c], pair ? sc * q[t * a.npad + c + 1] : 0.0);
  apply_minv<K>(a.Minv + (((int64_t)slot * a.nrep + rep) * K * K) * 2, r, z);
#pragma unroll
  for (int t = 0; t < K; ++t) {
    xin[t * a.npad + c] = z[t].re;
    if (pair) xin[t * a.npad + c + 1] = z[t].im;
  }
}

// DGKS criterion ("twice is enough"): reorthogonalise only if ||w'||^2 < ||w||^2 / 2 after the first
// classical Gram-Schmidt pass.  part3[slot][c] = (||w'||^2, ||w||^2, ||w''||^2) partial sums.
__device__ __forceinline__ bool needs_reorth(const EngArgs& a, int slot) {
  const double* p = a.part3 + (int64_t)slot * a.nchunk * 3;
  double s0 = 0.0, s1 = 0.0;
  for (int c = 0; c < a.nchunk; ++c) {
    s0 += p[c * 3];
    s1 += p[c * 3 + 1];
  }
  return s0 < 0.5 * s1;
}

// ---------------------------------------------------------------- CGS2 dot products (K3)
// ITER: part[slot][i][chunk] = q^_i . w over the chunk (w = candidate q^_{m+1}), i <= m.
// VERIFY (pass 1): part3[slot][chunk] = (||R||^2, ||rhs||^2, <hf, X>) with R in q^_0.
__global__ void __launch_bounds__(256) k_dots(EngArgs a, int pass) {
  __shared__ double ws[RED_CE];
  __shared__ double red[8];
  const int slot = blockIdx.y, chunk = blockIdx.x;
  const int ph = a.phase[slot];
  const int64_t e0 = (int64_t)chunk * RED_CE;
  const int64_t qs = (int64_t)(a.mmax + 1) * a.L;
  if (ph == PH_VERIFY) {
    if (pass != 1) return;
    const double* R = a.Qb + slot * qs;
    const double* X = a.X + (int64_t)slot * a.L;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    for (int i = threadIdx.x; i < RED_CE; i += blockDim.x) {
      const int64_t e = e0 + i;
      if (e < a.L) {
        const double r = R[e];
        const int t = (int)(e / a.npad);
        const double rh = a.mask[slot * a.K + t] * a.g0[e];
        s0 += r * r;
        s1 += rh * rh;
        s2 += a.hf[e] * X[e];
      }
    }
    s0 = block_sum(s0, red);
    s1 = block_sum(s1, red);
    s2 = block_sum(s2, red);
    if (threadIdx.x == 0) {
      double* p = a.part3 + ((int64_t)slot * a.nchunk + chunk) * 3;
      p[0] = s0;
      p[1] = s1;
      p[2] = s2;
    }
    return;
  }
  if (ph != PH_ITER) return;
  if (pass == 2 && !needs_reorth(a, slot)) return;
  const int m = a.m[slot];
  const double* w = a.Qb + slot * qs + (int64_t)(m + 1) * a.L;
  double nw = 0.0;
  for (int i = threadIdx.x; i < RED_CE; i += blockDim.x) {
    const int64_t e = e0 + i;
    const double v = e < a.L ? w[e] : 0.0;
    ws[i] = v;
    nw += v * v;
  }
  if (pass == 1) {
    nw = block_sum(nw, red);
    if (threadIdx.x == 0) a.part3[((int64_t)slot * a.nchunk + chunk) * 3 + 1] = nw;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t lim = (a.L - e0) < RED_CE ? (a.L - e0) : RED_CE;
  for (int i = warp; i <= m; i += 8) {
    const double* q = a.Qb + slot * qs + (int64_t)i * a.L + e0;
    double d0 = 0.0, d1 = 0.0;
    int e = lane;
    for (; e + 32 < lim; e += 64) {
      d0 += q[e] * ws[e];
      d1 += q[e + 32] * ws[e + 32];
    }
    if (e < lim) d0 += q[e] * ws[e];
    const double d = warp_sum(d0 + d1);
    if (lane == 0) a.part[((int64_t)slot * (a.mmax + 2) + i) * a.nchunk + chunk] = d;
  }
}

// ---------------------------------------------------------------- CGS2 update (K3)
// h_i = (q^_i . w) / eta_i (the coefficient on the normalised q_i); w -= sum_i (h_i / eta_i) q^_i;
// H[i][m] (=|+=) h_i;  part3[slot][chunk][0] = ||w'||^2 over the chunk.
__global__ void __launch_bounds__(256) k_upd(EngArgs a, int pass) {
  extern __shared__ double cf[];  // mmax + 1
  __shared__ double red[8];
  const int slot = blockIdx.y, chunk = blockIdx.x;
  if (a.phase[slot] != PH_ITER) return;
  if (pass == 2 && !needs_reorth(a, slot)) return;
  const int m = a.m[slot];
  const int64_t qs = (int64_t)(a.mmax + 1) * a.L;
  const double* eta = a.eta + (int64_t)slot * (a.mmax + 1);
  for (int i = threadIdx.x; i <= m; i += blockDim.x) {
    const double* p = a.part + ((int64_t)slot * (a.mmax + 2) + i) * a.nchunk;
    double h = 0.0;
    for (int c = 0; c < a.nchunk; ++c) h += p[c];
    h /= eta[i];
    cf[i] = h / eta[i];
    if (chunk == 0) {
      double* Hc = a.H + (int64_t)slot * (a.mmax + 1) * a.mmax + (int64_t)m * (a.mmax + 1);
      Hc[i] = (pass == 1) ? h : Hc[i] + h;
    }
  }
  __syncthreads();
  double* w = a.Qb + slot * qs + (int64_t)(m + 1) * a.L;
  const double* Q = a.Qb + slot * qs;
  const int64_t e0 = (int64_t)chunk * RED_CE;
  double nrm = 0.0;
  for (int ii = threadIdx.x; ii < RED_CE; ii += blockDim.x) {
    const int64_t e = e0 + ii;
    if (e >= a.L) break;
    double v = w[e];
    double acc0 = 0.0, acc1 = 0.0;
    int i = 0;
    for (; i + 1 <= m; i += 2) {
      acc0 += cf[i] * Q[(int64_t)i * a.L + e];
      acc1 += cf[i + 1] * Q[(int64_t)(i + 1) * a.L + e];
    }
    if (i <= m) acc0 += cf[i] * Q[(int64_t)i * a.L + e];
    v -= acc0 + acc1;
    w[e] = v;
    nrm += v * v;
  }
  nrm = block_sum(nrm, red);
  if (threadIdx.x == 0) a.part3[((int64_t)slot * a.nchunk + chunk) * 3 + (pass == 1 ? 0 : 2)] = nrm;
}

// ---------------------------------------------------------------- per-slot control (K4)
// one warp per slot: VERIFY -> done / restart;  ITER -> Hessenberg column, Givens, cycle end.
__global__ void __launch_bounds__(128) k_ctrl(EngArgs a) {
  const int slot = blockIdx.x * 4 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (slot >= a.b) return;
  const int ph = a.phase[slot];
  const int ld = a.mmax + 1;
  double* H = a.H + (int64_t)slot * ld * a.mmax;
  double* e = a.e + (int64_t)slot * ld;
  double* eta = a.eta + (int64_t)slot * ld;
  double* cs = a.e + (int64_t)a.b * ld + (int64_t)slot * a.mmax;   // cs, sn live after e
  double* sn = cs + (int64_t)a.b * a.mmax;
  const double* p3 = a.part3 + (int64_t)slot * a.nchunk * 3;
  if (ph == PH_VERIFY) {
    if (lane != 0) return;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    for (int c = 0; c < a.nchunk; ++c) {
      s0 += p3[c * 3];
      s1 += p3[c * 3 + 1];
      s2 += p3[c * 3 + 2];
    }
    const double rho = sqrt(s0), bn = sqrt(s1), tr = a.t0 + 2.0 * s2;
    const int ap = ++a.applies[slot];
    const bool bad = !isfinite(rho) || !isfinite(tr);
    const bool conv = rho <= a.tol * bn;
    if (bad || conv || a.restarts[slot] >= a.max_restarts) {
      const int idx = a.vidx[slot];
      a.traces[idx] = bad ? __longlong_as_double(0x7ff8000000000000LL) : tr;
      if (a.status) a.status[idx] = bad ? LYAP_V_NONFINITE : (conv ? LYAP_V_OK : LYAP_V_NOCONV);
      if (a.out_applies) a.out_applies[idx] = ap;
      if (a.out_resid) a.out_resid[idx] = bn > 0.0 ? rho / bn : rho;
      a.phase[slot] = PH_FREE;
      atomicAdd(&a.ctrl[1], 1);
    } else {
      eta[0] = rho;
      e[0] = rho;
      a.m[slot] = 0;
      a.bnorm[slot] = bn;
      a.phase[slot] = PH_ITER;
    }
    return;
  }
  if (ph != PH_ITER) return;
  const int m = a.m[slot];
  double* Hc = H + (int64_t)m * ld;
  int done = 0;
  if (lane == 0) {
    const int col = needs_reorth(a, slot) ? 2 : 0;  // same decision the pass-2 kernels took
    double s = 0.0;
    for (int c = 0; c < a.nchunk; ++c) s += p3[c * 3 + col];
    const double hn = sqrt(s);
    a.applies[slot] += 1;
    eta[m + 1] = hn > 0.0 ? hn : 1.0;
    Hc[m + 1] = hn;
    for (int i = 0; i < m; ++i) {
      const double t1 = cs[i] * Hc[i] + sn[i] * Hc[i + 1];
      const double t2 = -sn[i] * Hc[i] + cs[i] * Hc[i + 1];
      Hc[i] = t1;
      Hc[i + 1] = t2;
    }
    const double x1 = Hc[m], x2 = Hc[m + 1];
    const double r = hypot(x1, x2);
    const double c = r > 0.0 ? x1 / r : 1.0, sv = r > 0.0 ? x2 / r : 0.0;
    cs[m] = c;
    sn[m] = sv;
    Hc[m] = r;
    Hc[m + 1] = 0.0;
    e[m + 1] = -sv * e[m];
    e[m] = c * e[m];
    const double est = fabs(e[m + 1]);
    done = (est <= a.tol_inner * a.bnorm[slot]) || (m + 1 >= a.mmax) || !(hn > 1e-300 * a.bnorm[slot]) ||
           !isfinite(est);
    a.m[slot] = m + 1;
  }
  done = __shfl_sync(0xffffffffu, done, 0);
  if (!done) return;
  // back substitution R y = e (m1 x m1 upper triangular), warp-parallel column sweep
  const int m1 = m + 1;
  double* y = a.y + (int64_t)slot * a.mmax;
  for (int i = lane; i < m1; i += 32) y[i] = e[i];
  __syncwarp();
  for (int j = m1 - 1; j >= 0; --j) {
    const double d = H[(int64_t)j * ld + j];
    const double yj = d != 0.0 ? y[j] / d : 0.0;
    __syncwarp();
    if (lane == 0) y[j] = yj;
    for (int i = lane; i < j; i += 32) y[i] -= H[(int64_t)j * ld + i] * yj;
    __syncwarp();
  }
  for (int i = lane; i < m1; i += 32) y[i] /= eta[i];
  __syncwarp();
  if (lane == 0) {
    a.restarts[slot] += 1;
    a.phase[slot] = PH_XUPD;
  }
}

// ---------------------------------------------------------------- solution update
// XUPD: X += P(v)^{-1} (sum_{i<m} y_i q^_i)   (y already carries the 1/eta_i)
template <int K>
__global__ void __launch_bounds__(128) k_xupd(EngArgs a) {
  const int slot = blockIdx.y;
  if (a.phase[slot] != PH_XUPD) return;
  const int64_t rep = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (rep >= a.nrep) return;
  const int64_t c = rep_coord(rep, a.npairs);
  const bool pair = rep < a.npairs;
  const int m1 = a.m[slot];
  const double* y = a.y + (int64_t)slot * a.mmax;
  const double* Q = a.Qb + (int64_t)slot * (a.mmax + 1) * a.L;
  cplx r[K], z[K];
#pragma unroll
  for (int t = 0; t < K; ++t) r[t] = mk(0.0, 0.0);
  for (int i = 0; i < m1; ++i) {
    const double yi = y[i];
    const double* q = Q + (int64_t)i * a.L + c;
#pragma unroll
    for (int t = 0; t < K; ++t) {
      r[t].re += yi * q[t * a.npad];
      if (pair) r[t].im += yi * q[t * a.npad + 1];
    }
  }
  apply_minv<K>(a.Minv + (((int64_t)slot * a.nrep + rep) * K * K) * 2, r, z);
  double* X = a.X + (int64_t)slot * a.L + c;
#pragma unroll
  for (int t = 0; t < K; ++t) {
    X[t * a.npad] += z[t].re;
    if (pair) X[t * a.npad + 1] += z[t].im;
  }
}

}  // namespace lyap
