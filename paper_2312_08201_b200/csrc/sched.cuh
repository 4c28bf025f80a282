// Device-side scheduling of a lyap_trace_batch call (DESIGN.md §2.4 "Scheduling"): the cost proxy
// of every v, the queue order (a stable descending sort of the proxy, CUB radix sort), the
// bounding box of the batch and the nearest recycle regime per queue position.  All on the
// caller's stream: V never visits the host.
#pragma once
#include <cub/cub.cuh>

#include "common.cuh"

namespace lyap {

// key[i] = sum_t |v_it| w_t (the size of the rank-k perturbation), idx[i] = i; with the stability
// filter (nunstable != null) a filtered v gets key -1 and sorts behind every v to solve
__global__ void k_cost(const double* __restrict__ V, int nv, int k, const double* __restrict__ w,
                       const int32_t* __restrict__ nunstable, double* __restrict__ key, int* __restrict__ idx) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += gridDim.x * blockDim.x) {
    double c = 0.0;
    for (int t = 0; t < k; ++t) c += fabs(V[(int64_t)i * k + t]) * w[t];
    key[i] = (nunstable && nunstable[i] != 0) ? -1.0 : c;
    idx[i] = i;
  }
}

// filtered v (stability filter): trace NaN, status LYAP_V_UNSTABLE, no T-applies; count of the
// others in *nstable (one block)
__global__ void k_mark_unstable(const int32_t* __restrict__ nunstable, int nv, double* traces, int32_t* status,
                                int32_t* applies, double* resid, int* nstable) {
  __shared__ int cnt[32];
  int c = 0;
  for (int i = threadIdx.x; i < nv; i += blockDim.x) {
    if (nunstable[i] != 0) {
      traces[i] = __longlong_as_double(0x7ff8000000000000LL);
      if (status) status[i] = 3;  // LYAP_V_UNSTABLE
      if (applies) applies[i] = 0;
      if (resid) resid[i] = __longlong_as_double(0x7ff8000000000000LL);
    } else {
      ++c;
    }
  }
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0) cnt[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) t += cnt[q];
    *nstable = t;
  }
}

// box[2t] = min_i v_it, box[2t + 1] = max_i v_it (one block per parameter; fixed-order reduction)
__global__ void k_box(const double* __restrict__ V, int nv, int k, double* __restrict__ box) {
  __shared__ double lo_s[256], hi_s[256];
  const int t = blockIdx.x;
  double lo = 1e300, hi = -1e300;
  for (int i = threadIdx.x; i < nv; i += blockDim.x) {
    const double v = V[(int64_t)i * k + t];
    lo = fmin(lo, v);
    hi = fmax(hi, v);
  }
  lo_s[threadIdx.x] = lo;
  hi_s[threadIdx.x] = hi;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      lo_s[threadIdx.x] = fmin(lo_s[threadIdx.x], lo_s[threadIdx.x + s]);
      hi_s[threadIdx.x] = fmax(hi_s[threadIdx.x], hi_s[threadIdx.x + s]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    box[2 * t] = lo_s[0];
    box[2 * t + 1] = hi_s[0];
  }
}

// regq[q] = the regime whose seed is nearest to v = V[order[q]] in log|v| (first on ties)
__global__ void k_regime(const double* __restrict__ V, const int* __restrict__ order, int nv, int k,
                         const double* __restrict__ lseeds, int nreg, int* __restrict__ regq) {
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < nv; q += gridDim.x * blockDim.x) {
    const double* v = V + (int64_t)(order ? order[q] : q) * k;
    double best = 1e300;
    int arg = -1;
    for (int r = 0; r < nreg; ++r) {
      double d2 = 0.0;
      for (int t = 0; t < k; ++t) {
        const double dv = log(fabs(v[t]) + 1e-300) - lseeds[r * k + t];
        d2 += dv * dv;
      }
      if (d2 < best) {
        best = d2;
        arg = r;
      }
    }
    regq[q] = arg;
  }
}

}  // namespace lyap
