// K1 inner GEMM on the 5th-generation tensor cores (tcgen05, TMEM accumulators, TMA operand staging):
// the FP32-accurate T-apply of the mixed-precision Krylov steps.
//
//   U32t[n][m] = sum_k Lf[m][k] * Bop[k][n]      (the dense Cauchy coupling of eqs. (N2M1)/(N1M2),
//                                                 PAPER.md:336-362, for every ITER slot's vector)
//
// evaluated as 3xTF32: with x = x_hi + x_lo (x_hi = x rounded to TF32, x_lo = x - x_hi, both stored
// as float planes by k_split_Lf / k1_gen), A B ~ A_hi B_lo + A_lo B_hi + A_hi B_hi, all three
// products accumulated in one FP32 TMEM accumulator (relative error ~1e-6 instead of TF32's ~1e-3).
//
// Layouts (all K-major, so both operands use the canonical 128-byte-swizzled K-major UMMA layout):
//   A32 : npad x 2 npad fp32 row-major, row m = [hi(m, 0..npad) | lo(m, 0..npad)]
//   B32t: 2 ncol x npad fp32 row-major, rows [0, ncol) lo planes, [ncol, 2 ncol) hi planes (row = GEMM
//         column n, contiguous along k)
//   U32t: ncol x npad fp32 row-major (column n of the product contiguous along m: coalesced epilogue)
// Tile 128 (m) x 256 (n) x 32 (k), one CTA per tile, 4 warps: warp 0 lane 0 issues the TMA loads, warp 1
// lane 0 issues the MMAs (12 tcgen05.mma.kind::tf32 of 128x256x8 per k-block), then all four warps drain
// TMEM (warp w owns TMEM lanes 32w..32w+31 = rows m0 + 32w + lane).
#pragma once
#include <cuda.h>
#include <cstdint>

#include "k1.cuh"

namespace lyap {

constexpr int UM_BM = 128, UM_BK = 32;
constexpr int UM_A_BYTES = UM_BM * UM_BK * 4;  // one A plane per stage: 16 KB
// BN: GEMM columns per CTA (one tcgen05.mma N), STAGES: TMA pipeline depth
// EB: operand element bytes, 4 = TF32 (kind::tf32, 8 k per instruction), 2 = FP16 (kind::f16, 16 k per
// instruction; 3xFP16 with power-of-two operand scaling).  BK counts elements.
template <int BN, int STAGES, int BK = UM_BK, int EB = 4>
struct UmCfg {
  static constexpr int A_BYTES = UM_BM * BK * EB;                      // one A plane per stage
  static constexpr int B_BYTES = BN * BK * EB;                         // one B plane per stage
  static constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
  static constexpr int ROW = BK * EB;                                  // bytes per K-major smem row
  // K-major rows of 128 B (SWIZZLE_128B) or 64 B (SWIZZLE_64B); 8-row atoms
  static constexpr uint32_t LAYOUT = ROW == 128 ? 2u : 4u, SBO = 8 * ROW;
  static constexpr int KI = EB == 4 ? 8 : 16;                          // k per tcgen05.mma
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;       // + alignment slack + barriers
  static constexpr int TMEM_COLS = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;
  // instruction descriptor: D fp32, A/B tf32 (2) or f16 (0), both K-major, M = 128, N = BN
  static constexpr uint32_t FMT = EB == 4 ? 2u : 0u;
  static constexpr uint32_t IDESC = (1u << 4) | (FMT << 7) | (FMT << 10) | ((uint32_t)(BN >> 3) << 17) |
                                    ((uint32_t)(UM_BM >> 4) << 24);
};
// production configuration of the persistent kernel: 128 x 256 tiles, 16-wide k-blocks (64-byte swizzle),
// 4 stages (tools/microbench/umma_tf32x3.cu: 740 TFLOP/s of TF32 work at the c5 shape, vs 663 for
// 32-wide k-blocks in 2 stages and 733 for three cuBLAS TF32 GEMMs)
constexpr int UM_BN = 256, UM_STAGES = 4, UM_BKE = 16;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1)
      : "memory");
}
// UMMA shared-memory matrix descriptor, K-major, swizzled: 8-row atoms SBO bytes apart
template <uint32_t LAYOUT = 2, uint32_t SBO = 1024>
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);        // start address
  d |= (uint64_t)1 << 16;                        // leading byte offset (unused for swizzled K-major)
  d |= (uint64_t)(SBO >> 4) << 32;               // stride byte offset: next 8-row atom
  d |= (uint64_t)1 << 46;                        // descriptor version (sm_100)
  d |= (uint64_t)LAYOUT << 61;                   // layout: 2 = SWIZZLE_128B, 4 = SWIZZLE_64B
  return d;
}
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) { return umma_desc<2, 1024>(saddr); }
template <uint32_t IDESC, int EB = 4>
__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t acc) {
  if constexpr (EB == 4)
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(IDESC), "r"(acc));
  else
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(IDESC), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

// U32t = A32 (3xTF32) B32t over the active columns (n0 < (*nactive) * cpa; nactive null: all).
// grid: (ncol / BN) x (npad / 128); Kd = multiple of 32 (zero rows of the padding skipped).
template <int BN, int STAGES>
__global__ void __launch_bounds__(128, 1)
    k1_umma_tf32x3(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   float* __restrict__ U32t, int npad, int ncol, int Kd, const int* __restrict__ nactive, int cpa) {
  using Cfg = UmCfg<BN, STAGES>;
  constexpr int UM_STAGE_BYTES = Cfg::STAGE_BYTES, UM_B_BYTES = Cfg::B_BYTES, UM_TMEM_COLS = Cfg::TMEM_COLS;
  const int n0 = blockIdx.x * BN, m0 = blockIdx.y * UM_BM;
  if (nactive && n0 >= (*nactive) * cpa) return;
  extern __shared__ __align__(1024) uint8_t um_smem[];
  // 1024-byte aligned operand stages (the 128-byte swizzle pattern repeats every 1024 B)
  const uint32_t base = (smem_u32(um_smem) + 1023) & ~1023u;
  uint8_t* gbase = um_smem + (base - smem_u32(um_smem));
  uint64_t* bars = reinterpret_cast<uint64_t*>(gbase + STAGES * UM_STAGE_BYTES);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 1);
  const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + STAGES), accb = smem_u32(bars + 2 * STAGES);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, 1);
    }
    mbar_init(accb, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(UM_TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  const int KB = Kd / UM_BK;

  if (warp == 0 && lane == 0) {
    // TMA producer: per k-block A_hi, A_lo (x = k, npad + k; y = m0), B_lo, B_hi (x = k; y = n0, ncol + n0)
    for (int kb = 0; kb < KB; ++kb) {
      const int s = kb % STAGES;
      if (kb >= STAGES) mbar_wait(empty0 + 8 * s, ((kb / STAGES) - 1) & 1);
      const uint32_t st = base + s * UM_STAGE_BYTES, fb = full0 + 8 * s;
      mbar_expect_tx(fb, UM_STAGE_BYTES);
      const int k = kb * UM_BK;
      tma_load_2d(st, &tmA, fb, k, m0);
      tma_load_2d(st + UM_A_BYTES, &tmA, fb, npad + k, m0);
      tma_load_2d(st + 2 * UM_A_BYTES, &tmB, fb, k, n0);
      tma_load_2d(st + 2 * UM_A_BYTES + UM_B_BYTES, &tmB, fb, k, ncol + n0);
    }
  } else if (warp == 1 && lane == 0) {
    // MMA issuer: 3 products x 4 k-steps of 8 per k-block into one accumulator
    for (int kb = 0; kb < KB; ++kb) {
      const int s = kb % STAGES;
      mbar_wait(full0 + 8 * s, (kb / STAGES) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t ah = base + s * UM_STAGE_BYTES, al = ah + UM_A_BYTES, bl = ah + 2 * UM_A_BYTES,
                     bh = bl + UM_B_BYTES;
#pragma unroll
      for (int j = 0; j < UM_BK / 8; ++j) {
        const uint32_t o = 32 * j;  // 8 tf32 = 32 bytes along the swizzled 128-byte row
        const uint32_t acc0 = (kb > 0 || j > 0) ? 1u : 0u;
        umma_tf32<Cfg::IDESC>(tmem, umma_desc_sw128(ah + o), umma_desc_sw128(bl + o), acc0);
        umma_tf32<Cfg::IDESC>(tmem, umma_desc_sw128(al + o), umma_desc_sw128(bh + o), 1u);
        umma_tf32<Cfg::IDESC>(tmem, umma_desc_sw128(ah + o), umma_desc_sw128(bh + o), 1u);
      }
      umma_commit(empty0 + 8 * s);  // frees the stage once these MMAs have read it
    }
    umma_commit(accb);  // accumulator complete
  }
  __syncwarp();
  // epilogue: TMEM lane (32 warp + lane) = row m0 + 32 warp + lane; 32 columns per tcgen05.ld
  mbar_wait(accb, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int m = m0 + 32 * warp + lane;
#pragma unroll 1
  for (int c0 = 0; c0 < BN; c0 += 32) {
    uint32_t r[32];
    const uint32_t taddr = tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)c0;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int j = 0; j < 32; ++j) U32t[(int64_t)(n0 + c0 + j) * npad + m] = __uint_as_float(r[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 2) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(UM_TMEM_COLS));
  }
}


// tile index -> (M tile, N tile): grouped rasterisation, UM_GM row tiles share each sweep over the active
// column tiles, so the A panels in flight (UM_GM x 128 rows of [Lf_hi | Lf_lo], 64 MB at c5) stay in L2
// while B streams once per group (M-tile-fastest order re-read all of A, 134 MB, per wave of tiles)
constexpr int UM_GM = 16;
__device__ __forceinline__ void um_tile(int t, int MT, int ntn, int& mt, int& nt) {
  const int gm = t / (UM_GM * ntn), r = t - gm * UM_GM * ntn;
  const int rows = min(UM_GM, MT - gm * UM_GM);
  mt = gm * UM_GM + r % rows;
  nt = r / rows;
}

// Per-thread coordinate data of the fused K1 epilogue, loaded once per tile (the same for every slot):
// B~l_j (K complex, or real) and the T_d block F_j (K x K complex, or real) of coordinate m.
// pair: m is the Re row of a conjugate pair (m + 1 its Im row, handled by this thread); active = the
// thread writes (an Im-row thread of a pair does not); pad: m >= n (zero rows).
template <int K>
struct EpiCoord {
  double blr[K], bli[K], fr[K][K], fi[K][K];
  bool pair, active, pad;
  __device__ __forceinline__ void load(const K1EpiArgs& ep, int m) {
    pair = m < ep.two_np;
    pad = m >= ep.n;
    active = pad || !pair || !(m & 1);
    if (!active || pad) return;
    const int rep = pair ? (m >> 1) : (m - ep.two_np + ep.npairs);
#pragma unroll
    for (int t = 0; t < K; ++t) {
      blr[t] = ep.btl[(int64_t)m * K + t];
      bli[t] = pair ? ep.btl[(int64_t)(m + 1) * K + t] : 0.0;
    }
#pragma unroll
    for (int s = 0; s < K; ++s)
#pragma unroll
      for (int t = 0; t < K; ++t) {
        const double* f = ep.F + (((int64_t)rep * K + s) * K + t) * 2;
        fr[s][t] = f[0];
        fi[s][t] = f[1];
      }
  }
};

// ------------------------------------------------------------------------------------------------
// Persistent, warp-specialised form (the engine's kernel): grid = one CTA per SM; tiles (M-tile fastest,
// only the tiles that hold active columns) are claimed dynamically from a global counter (tctr[0]; the
// last CTA to run dry resets it), so CTAs that start late -- the other slot group's kernels hold some
// SMs -- simply take fewer tiles.  The producer publishes each claimed tile id through a 4-deep shared
// ring (tid_full / tid_empty mbarriers) to the MMA thread and the epilogue warps.  6 warps:
//   warp 0 lane 0: TMA producer over a STAGES-deep shared-memory ring (full / empty mbarriers)
//   warp 1       : TMEM allocation (2 accumulators of BN columns); lane 0 issues the MMAs
//   warps 2..5   : epilogue, warp w draining TMEM lanes 32 (w % 4) .. +31 (the lane quarter a warp may
//                  access), overlapped with the next tile's main loop (accumulator double buffer:
//                  tfull / tempty mbarriers)
// EPI = k (1, 2, 4): the K1 epilogue is fused -- each thread holds row m (coordinate c) of 32
// consecutive GEMM columns = whole (slot, s, t) groups, contracts them with B~l, adds T_d and sigma x
// (k1_out_element, the same code as the DMMA path's fused epilogue) and writes C(v)x straight into the
// slot's Krylov basis; the Im row of a conjugate pair comes from the neighbouring lane (shfl).  VERIFY
// positions [0, nver) are skipped (their exact FP64 apply comes from the DMMA GEMM).  EPI = 0: U32t.
template <int BN, int STAGES, int EPI, int BK = UM_BK, int EB = 4>
__global__ void __launch_bounds__(192, 1)
    k1_umma_persistent(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                       float* __restrict__ U32t, int npad, int ncol, int Kd, const int* __restrict__ nactive, int cpa,
                       const K1EpiArgs ep, int* __restrict__ tctr, const float* __restrict__ colscale = nullptr) {
  using Cfg = UmCfg<BN, STAGES, BK, EB>;
  constexpr int SB = Cfg::STAGE_BYTES, BB = Cfg::B_BYTES, AB = Cfg::A_BYTES, TCOLS = 2 * BN <= 256 ? 256 : 512;
  extern __shared__ __align__(1024) uint8_t um_smem[];
  const uint32_t base = (smem_u32(um_smem) + 1023) & ~1023u;
  uint8_t* gbase = um_smem + (base - smem_u32(um_smem));
  uint64_t* bars = reinterpret_cast<uint64_t*>(gbase + STAGES * SB);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 12);
  int* tile_ring = reinterpret_cast<int*>(bars + 2 * STAGES + 13);
  const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + STAGES);
  const uint32_t tfull0 = smem_u32(bars + 2 * STAGES), tempty0 = smem_u32(bars + 2 * STAGES + 2);
  const uint32_t rfull0 = smem_u32(bars + 2 * STAGES + 4), rempty0 = smem_u32(bars + 2 * STAGES + 8);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int MT = npad / UM_BM;
  const int ncols_act = nactive ? min(ncol, (*nactive) * cpa) : ncol;
  // EPI: column tiles made only of VERIFY positions (exact path) are skipped
  const int nt0 = EPI ? ((*ep.a.nver) * cpa) / BN : 0;
  const int ntn = max(0, (ncols_act + BN - 1) / BN - nt0);  // active column tiles
  const int ntiles = ntn * MT;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull0 + 8 * a, 1);
      mbar_init(tempty0 + 8 * a, 128);
    }
    for (int r = 0; r < 4; ++r) {
      mbar_init(rfull0 + 8 * r, 1);
      mbar_init(rempty0 + 8 * r, 129);  // the MMA thread + 128 epilogue threads
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  const int KB = Kd / BK;

  if (warp == 0) {
    if (lane == 0) {
      int it = 0;
      for (int li = 0;; ++li) {
        const int rs = li & 3;
        if (li >= 4) mbar_wait(rempty0 + 8 * rs, ((li >> 2) - 1) & 1);
        const int t = atomicAdd(tctr, 1);
        tile_ring[rs] = t;
        mbar_arrive(rfull0 + 8 * rs);
        if (t >= ntiles) {
          if (atomicAdd(tctr + 1, 1) == (int)gridDim.x - 1) {  // every CTA has run dry: reset for the next launch
            tctr[0] = 0;
            tctr[1] = 0;
          }
          break;
        }
        int mt, nt;
        um_tile(t, MT, ntn, mt, nt);
        const int m0 = mt * UM_BM, n0 = (nt + nt0) * BN;
        for (int kb = 0; kb < KB; ++kb, ++it) {
          const int s = it % STAGES;
          mbar_wait(empty0 + 8 * s, ((it / STAGES) & 1) ^ 1);
          const uint32_t st = base + s * SB, fb = full0 + 8 * s;
          mbar_expect_tx(fb, SB);
          const int k = kb * BK;
          tma_load_2d(st, &tmA, fb, k, m0);
          tma_load_2d(st + AB, &tmA, fb, npad + k, m0);
          tma_load_2d(st + 2 * AB, &tmB, fb, k, n0);
          tma_load_2d(st + 2 * AB + BB, &tmB, fb, k, ncol + n0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int it = 0;
      for (int li = 0;; ++li) {
        mbar_wait(rfull0 + 8 * (li & 3), (li >> 2) & 1);
        const int t = tile_ring[li & 3];
        mbar_arrive(rempty0 + 8 * (li & 3));
        if (t >= ntiles) break;
        const int acc = li & 1;
        const uint32_t td = tmem + (uint32_t)(acc * BN);
        mbar_wait(tempty0 + 8 * acc, ((li >> 1) & 1) ^ 1);  // the epilogue has drained this accumulator
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        for (int kb = 0; kb < KB; ++kb, ++it) {
          const int s = it % STAGES;
          mbar_wait(full0 + 8 * s, (it / STAGES) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t ah = base + s * SB, al = ah + AB, bl = ah + 2 * AB, bh = bl + BB;
          constexpr uint32_t LY = Cfg::LAYOUT, SO = Cfg::SBO;
#pragma unroll
          for (int j = 0; j < BK / Cfg::KI; ++j) {
            const uint32_t o = 32 * j;  // one instruction's k (8 tf32 / 16 fp16) = 32 bytes along the swizzled row
            umma_tf32<Cfg::IDESC, EB>(td, umma_desc<LY, SO>(ah + o), umma_desc<LY, SO>(bl + o), (kb > 0 || j > 0) ? 1u : 0u);
            umma_tf32<Cfg::IDESC, EB>(td, umma_desc<LY, SO>(al + o), umma_desc<LY, SO>(bh + o), 1u);
            umma_tf32<Cfg::IDESC, EB>(td, umma_desc<LY, SO>(ah + o), umma_desc<LY, SO>(bh + o), 1u);
          }
          umma_commit(empty0 + 8 * s);
        }
        umma_commit(tfull0 + 8 * acc);
      }
    }
  } else {
    // epilogue warps 2..5
    const int q = warp & 3;  // TMEM lane quarter
    const int nver = EPI ? *ep.a.nver : 0;
    const int nact = EPI ? k1_nact(ep.a) : 0;
    for (int li = 0;; ++li) {
      mbar_wait(rfull0 + 8 * (li & 3), (li >> 2) & 1);
      const int t = tile_ring[li & 3];
      mbar_arrive(rempty0 + 8 * (li & 3));
      if (t >= ntiles) break;
      int mt, nt;
      um_tile(t, MT, ntn, mt, nt);
      const int m0 = mt * UM_BM, n0 = (nt + nt0) * BN;
      const int acc = li & 1;
      mbar_wait(tfull0 + 8 * acc, (li >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int m = m0 + 32 * q + lane;
      EpiCoord<EPI ? EPI : 1> ec;
      if constexpr (EPI > 0) ec.load(ep, m);
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        uint32_t r[32];
        const uint32_t taddr = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(acc * BN + c0);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
            "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
              "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
              "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (colscale) {  // FP16 operands: undo the power-of-two operand scales of every column (exact)
#pragma unroll
          for (int j = 0; j < 32; ++j) r[j] = __float_as_uint(__uint_as_float(r[j]) * colscale[n0 + c0 + j]);
        }
        if constexpr (EPI == 0) {
#pragma unroll
          for (int j = 0; j < 32; ++j) U32t[(int64_t)(n0 + c0 + j) * npad + m] = __uint_as_float(r[j]);
        } else {
          // fused K1 epilogue: (T X)_sj = sum_t B~l_jt U[(s,t), j] + sum_t F_j[s,t] X_tj, out = sigma_s X_sj - (T X)_sj
          // (the k1_epi contraction); row m + 1 (the Im row of a pair) comes from the next lane
          constexpr int KK = EPI * EPI, PP = 32 / KK;
          static_assert(32 % KK == 0, "whole (slot, s, t) groups per 32-column chunk");
#pragma unroll
          for (int pp = 0; pp < PP; ++pp) {
            float u1[KK];
#pragma unroll
            for (int j = 0; j < KK; ++j) u1[j] = __shfl_down_sync(0xffffffffu, __uint_as_float(r[pp * KK + j]), 1);
            const int pos = (n0 + c0) / KK + pp;
            if (pos < nver || pos >= nact || !ec.active) continue;  // VERIFY (exact path), inactive, Im lane
            const int slot = k1_slot(ep.a, pos);
            if (ep.a.phase[slot] != PH_ITER) continue;
            const int64_t off = (int64_t)slot * ep.a.qstride + (int64_t)(ep.a.m[slot] + 1) * ep.a.L;
            const K1Dst dst = ep.a.Qf ? K1Dst{nullptr, ep.a.Qf + off} : K1Dst{ep.a.Qb + off, nullptr};
            if (ec.pad) {
#pragma unroll
              for (int s = 0; s < EPI; ++s) dst.put((int64_t)s * npad + m, 0.0);
              continue;
            }
            const double* x = ep.a.Xin + (int64_t)slot * ep.a.L;
            if (ec.pair) {
              double xr[EPI], xi[EPI];
#pragma unroll
              for (int t = 0; t < EPI; ++t) {
                xr[t] = x[(int64_t)t * npad + m];
                xi[t] = x[(int64_t)t * npad + m + 1];
              }
#pragma unroll
              for (int s = 0; s < EPI; ++s) {
                double yr = 0.0, yi = 0.0;
#pragma unroll
                for (int t = 0; t < EPI; ++t) {
                  const double ur = __uint_as_float(r[pp * KK + s * EPI + t]), ui = u1[s * EPI + t];
                  yr += ec.blr[t] * ur - ec.bli[t] * ui + ec.fr[s][t] * xr[t] - ec.fi[s][t] * xi[t];
                  yi += ec.blr[t] * ui + ec.bli[t] * ur + ec.fr[s][t] * xi[t] + ec.fi[s][t] * xr[t];
                }
                const bool on = ep.a.mask[slot * EPI + s] != 0.0;
                const double sg = ep.a.sigma[slot * EPI + s];
                dst.put((int64_t)s * npad + m, on ? sg * xr[s] - yr : xr[s]);
                dst.put((int64_t)s * npad + m + 1, on ? sg * xi[s] - yi : xi[s]);
              }
            } else {  // real eigenvalue
              double xr[EPI];
#pragma unroll
              for (int t = 0; t < EPI; ++t) xr[t] = x[(int64_t)t * npad + m];
#pragma unroll
              for (int s = 0; s < EPI; ++s) {
                double y = 0.0;
#pragma unroll
                for (int t = 0; t < EPI; ++t)
                  y += ec.blr[t] * (double)__uint_as_float(r[pp * KK + s * EPI + t]) + ec.fr[s][t] * xr[t];
                const bool on = ep.a.mask[slot * EPI + s] != 0.0;
                dst.put((int64_t)s * npad + m, on ? ep.a.sigma[slot * EPI + s] * xr[s] - y : xr[s]);
              }
            }
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      mbar_arrive(tempty0 + 8 * acc);
    }
  }
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TCOLS));
  }
}

}  // namespace lyap
