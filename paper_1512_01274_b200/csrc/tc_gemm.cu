// tcgen05 tensor-core GEMM for the bf16 dense path (sm_100a).
//
//   C[M,N] (fp32) = sum_k A(m,k) B(n,k)  (+ bias[n]) then activation
//
// A and B are bf16 in global memory, each either K-major (X[r*ld + k]) or
// MN-major (X[k*ld + r]); the accumulator is fp32 in tensor memory.  This
// one kernel serves every contraction of the conv nets: forward (both
// K-major), data gradient (B MN-major: the weight in its own layout) and
// weight gradient (both MN-major: activations and output gradients in their
// own layouts, the batch*pixels axis is the contraction), so no operand is
// ever transposed in memory.
//
// Persistent and warp-specialised, one CTA per SM, 192 threads:
//   warp 0 (one lane)   TMA producer: 128B-swizzled 64-wide K slices of A
//                       (128 rows) and B (BN rows) into a STAGES-deep ring
//   warp 1 (one lane)   MMA issuer: tcgen05.mma.kind::f16 M128 x BN x K16,
//                       accumulating into one of two TMEM buffers, so the
//                       epilogue of tile i overlaps the mainloop of tile i+1
//   warps 2-5           epilogue: tcgen05.ld 32 lanes x 32 columns, bias +
//                       activation, 128B-swizzled smem staging, TMA store
//                       (direct fp32 stores when C's row pitch is not
//                       16-byte aligned)
// Tiles are scheduled round-robin over (split, m, n) with n fastest, so the
// CTAs working at one time share A rows in L2.  Split-K partial tiles go
// to a workspace and are summed in ascending split order (deterministic).
//
// This is the tolerance path (bf16 operands, fp32 accumulation in hardware
// order); the exact-order fp32 kernels (dense.cu) stay the parity path.

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>

#include <cstring>
#include <mutex>

#include <stdlib.h>

#include "common.cuh"

namespace mgx {
namespace tc {

constexpr int BM = 128, BK = 64, UMMA_K = 16;
constexpr int kThreads = 192;
constexpr int kStageBoxes = 8;  // epilogue staging boxes: 2 per warp (4 warps) or 1 (8)
constexpr int kMnChunkBytes = BK * 128;  // one MN-major TMA box: 64 K rows x 128 B
constexpr int kStageCBytes = 32 * 32 * 4;  // one epilogue staging box (32 x 32 fp32)

template <int BN>
struct Cfg {
  static constexpr int kABytes = BM * BK * 2;
  static constexpr int kBBytes = BN * BK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  // deep rings for the gather-fed implicit GEMM (L2 round trips per stage):
  // 6 x 32 KB (BN 128) / 8 x 24 KB (BN 64) + 32 KB epilogue staging <= 227 KB
  static constexpr int kStages = BN >= 192 ? 4 : (BN >= 128 ? 6 : 8);
  // double-buffered accumulator, rounded up to a power of two columns
  static constexpr int kTmemCols = 2 * BN <= 128 ? 128 : (2 * BN <= 256 ? 256 : 512);
  static constexpr int kSmemBytes =
      1024 + kStages * kStageBytes + kStageBoxes * kStageCBytes + 256;
};

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// the same wait with a suspend-time hint: the warp sleeps in the barrier
// until the phase flips instead of re-polling (waiters that are not on the
// critical issue path -- producers waiting for a free slot, the epilogue
// waiting for an accumulator -- stop stealing issue slots from the gather)
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(1000000)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0,
                                             int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(c0), "r"(c1), "r"(smem_u32(src))
      : "memory");
}

// tcgen05 shared-memory matrix descriptor: K-major, 128-byte swizzle,
// 8-row swizzle atoms 1024 bytes apart (SBO), version 1 (bit 46).
__device__ __forceinline__ uint64_t smem_desc_sw128(const void* p) {
  const uint64_t addr = smem_u32(p);
  uint64_t d = 0;
  d |= (addr >> 4) & 0x3FFFull;               // start address
  d |= (uint64_t(1024 >> 4) & 0x3FFF) << 32;  // SBO
  d |= uint64_t(1) << 46;                     // fixed 0b001
  d |= uint64_t(2) << 61;                     // SWIZZLE_128B
  return d;
}

// MN-major, 128-byte swizzle: 64-element (128 B) MN rows, K rows 128 B
// apart; 8-row K groups 1024 B apart (SBO); 64-wide MN chunks kMnChunkBytes
// apart (LBO).
__device__ __forceinline__ uint64_t smem_desc_mn_sw128(const void* p) {
  const uint64_t addr = smem_u32(p);
  uint64_t d = 0;
  d |= (addr >> 4) & 0x3FFFull;
  d |= (uint64_t(kMnChunkBytes >> 4) & 0x3FFF) << 16;  // LBO: next 64 MN elements
  d |= (uint64_t(1024 >> 4) & 0x3FFF) << 32;           // SBO: next 8 K rows
  d |= uint64_t(1) << 46;
  d |= uint64_t(2) << 61;
  return d;
}

// instruction descriptor kind::f16: D f32, A/B bf16, M128 x BN; bits 15/16
// select an MN-major A / B operand
template <bool A_MN, bool B_MN, int BN>
constexpr uint32_t idesc() {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((A_MN ? 1u : 0u) << 15) | ((B_MN ? 1u : 0u) << 16) |
         (uint32_t(BN >> 3) << 17) | (uint32_t(BM >> 4) << 24);
}

template <bool A_MN, bool B_MN, int BN>
__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc<A_MN, B_MN, BN>()), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

// one ROWS x 64-K operand tile into `dst`: a single K-major box, or
// ROWS/64 MN-major boxes stacked kMnChunkBytes apart
template <bool MN, int ROWS>
__device__ __forceinline__ void load_operand(uint8_t* dst, const CUtensorMap* map, uint64_t* bar,
                                             int k0, int r0) {
  if (!MN) {
    tma_load_2d(dst, map, bar, k0, r0);
  } else {
#pragma unroll
    for (int c = 0; c < ROWS / 64; ++c) tma_load_2d(dst + c * kMnChunkBytes, map, bar, r0 + c * 64, k0);
  }
}

struct Sched {
  int m_tiles, n_tiles, splits, kps, nk, kext;
  __device__ __forceinline__ void tile(int t, int* m0, int* n0, int* z, int* kb0, int* nkb) const {
    const int per_split = m_tiles * n_tiles;
    *z = t / per_split;
    const int r = t - *z * per_split;
    *m0 = (r / n_tiles) * BM;
    *n0 = (r - (r / n_tiles) * n_tiles);
    *kb0 = *z * kps;
    *nkb = min(nk, *kb0 + kps) - *kb0;
  }
};

// Implicit-GEMM operand: G[m, k] = src[b, oh*sh - ph + i, ow*sw - pw + j, c]
// for output pixel m = (b, oh, ow) and k = (i*kw + j)*C + c, zero outside
// the input or beyond K = kh*kw*C; src is a compact bf16 NHWC tensor with
// C % 8 == 0, so 8 consecutive k are one 16-byte load.
struct Gather {
  const __nv_bfloat16* src;
  int B, H, W, C, kh, kw, sh, sw, ph, pw, Ho, Wo;
  // dil 2: the source is read as if dilated by 2 (zeros between its pixels;
  // the data gradient of a stride-2 convolution as a stride-1 transposed
  // one): virtual position v is source position v / 2 when v is even
  int dil;
  // n / d as __umul64hi(n, mul) for the runtime divisors (exact for any
  // 32-bit n; mul = 2^64 / d rounded up, 0 for d == 1)
  uint64_t mul_hw, mul_wo, mul_c, mul_kw;
};

__host__ inline uint64_t fastdiv_mul(int d) { return d <= 1 ? 0 : ~uint64_t(0) / uint64_t(d) + 1; }
__device__ __forceinline__ int fdiv_u(int n, uint64_t mul) {
  return mul ? static_cast<int>(__umul64hi(static_cast<uint64_t>(static_cast<uint32_t>(n)), mul))
             : n;
}

constexpr int kGatherThreads = 128;  // warps 6..9

__device__ __forceinline__ void cp_async16_zfill(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
               "r"(valid ? 16 : 0)
               : "memory");
}

// GM: 0 plain (both operands by TMA); 1 A gathered (K-major: forward /
// data gradient of a convolution); 2 B gathered (MN-major: weight gradient)
// GM 3: A (K-major) loaded by TMA in im2col mode -- no gather warps
// GM 6: the weight gradient transposed (D[kconv, F] = im2col(x)^T . dY, its
// tiles stored transposed into C[F, kconv]): A (MN-major) by TMA im2col,
// B = dY (MN-major) by TMA -- for few filters F (the 128-row M tile would
// be mostly padding in GM 4's orientation)
// GM 7: GM 6 with the im2col operand gathered by the cp.async warps (C %
// 64 != 0)
// GM 4: B (MN-major: weight gradient) loaded by TMA in im2col mode, one
// 64-pixel x 64-channel box per 64 columns (tap, channel block)
template <int GM>
constexpr bool gathered() {
  return GM == 1 || GM == 2 || GM == 7;
}
// block: TMA producer warp, MMA warp, EPI epilogue warps (4, or 8 with the
// columns of a tile split between two warps per TMEM lane quadrant), then
// the gather warps of the implicit modes (EPI 4 there)
template <int GM, int EPI>
constexpr int threads_for() {
  return 64 + 32 * EPI + (gathered<GM>() ? kGatherThreads : 0);
}

// in-place warp reduce-scatter of 32 per-lane values: afterwards a[0] in
// lane l holds the sum over all lanes of their a[l] (butterfly halving)
__device__ __forceinline__ void warp_reduce_scatter32(float (&a)[32], int lane) {
#pragma unroll
  for (int w = 16; w >= 1; w >>= 1) {
    const bool up = (lane & w) != 0;
#pragma unroll
    for (int i = 0; i < w; ++i) {
      const float send = up ? a[i] : a[i + w];
      const float keep = up ? a[i + w] : a[i];
      a[i] = fadd(keep, __shfl_xor_sync(0xffffffffu, send, w));
    }
  }
}

// ACTK: 0 no activation, 1 relu, 2 any (runtime code; cold path)
template <bool A_MN, bool B_MN, int BN, int ACTK, int GM, int EPI>
__global__ void __launch_bounds__(threads_for<GM, EPI>(), 1)
tc_gemm_bf16_kernel(const __grid_constant__ CUtensorMap map_a,
                    const __grid_constant__ CUtensorMap map_b,
                    const __grid_constant__ CUtensorMap map_c, const float* __restrict__ bias,
                    float* __restrict__ C, int ldc, int M, int N, int act, Sched sc,
                    int64_t split_stride, int use_tma_store, const __grid_constant__ Gather ga,
                    float2* __restrict__ colstats) {
  using G = Cfg<BN>;
  static_assert(EPI == 4 || (EPI == 8 && !gathered<GM>()), "8 epilogue warps: TMA-fed modes only");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* stage_c = smem + G::kStages * G::kStageBytes;  // [4 warps][2 bufs][4 KB]
  uint64_t* full = reinterpret_cast<uint64_t*>(stage_c + kStageBoxes * kStageCBytes);
  uint64_t* empty = full + G::kStages;
  uint64_t* tfull = empty + G::kStages;   // [2]
  uint64_t* tempty = tfull + 2;           // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntiles = sc.m_tiles * sc.n_tiles * sc.splits;

  if (threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");
    for (int s = 0; s < G::kStages; ++s) {
      // gathered operand: the 128 gather threads arrive (cp.async noinc)
      mbar_init(&full[s], gathered<GM>() ? 1 + kGatherThreads : 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], EPI);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(G::kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer
      int it = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        int m0, nt, z, kb0, nkb;
        sc.tile(t, &m0, &nt, &z, &kb0, &nkb);
        const int n0 = nt * BN;
        // GM 3: the tile's first output pixel -> its window origin (im2col
        // coordinates); (tap, channel block) advanced per k-block
        int iw = 0, ih = 0, in_ = 0, tap = 0, cb = 0;
        if (GM == 3) {
          const int hw = ga.Ho * ga.Wo;
          in_ = m0 / hw;
          const int rem = m0 - in_ * hw;
          const int oh = rem / ga.Wo, ow = rem - (rem / ga.Wo) * ga.Wo;
          ih = oh * ga.sh - ga.ph;
          iw = ow * ga.sw - ga.pw;
          const int k0 = kb0 * BK;
          tap = k0 / ga.C;
          cb = k0 - tap * ga.C;
        }
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % G::kStages;
          const uint32_t ph = (it / G::kStages) & 1;
          mbar_wait_sleep(&empty[s], ph ^ 1);
          uint8_t* sa = smem + s * G::kStageBytes;
          mbar_expect_tx(&full[s], (GM == 1 || GM == 7) ? G::kBBytes
                                   : GM == 2              ? G::kABytes
                                                          : G::kStageBytes);
          if (GM == 6) {
            // A = im2col(x)[pixels (K), (tap, c) (M)], as GM 4's B
            const int p0 = (kb0 + kb) * BK;
            const int hw = ga.Ho * ga.Wo;
            const int pn = p0 / hw, prem = p0 - pn * hw;
            const int poh = prem / ga.Wo, pow_ = prem - (prem / ga.Wo) * ga.Wo;
            const int piw = pow_ * ga.sw - ga.pw, pih = poh * ga.sh - ga.ph;
#pragma unroll
            for (int c = 0; c < BM / 64; ++c) {
              const int col = min(m0 + c * 64, M - 64);
              const int ctap = col / ga.C, ccb = col - ctap * ga.C;
              const int ci = ctap / ga.kw, cj = ctap - ci * ga.kw;
              asm volatile(
                  "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::"
                  "bytes [%0], [%1, {%2, %3, %4, %5}], [%6], {%7, %8};" ::"r"(
                      smem_u32(sa + c * kMnChunkBytes)),
                  "l"(reinterpret_cast<uint64_t>(&map_a)), "r"(ccb), "r"(piw), "r"(pih), "r"(pn),
                  "r"(smem_u32(&full[s])), "h"(static_cast<uint16_t>(cj)),
                  "h"(static_cast<uint16_t>(ci))
                  : "memory");
            }
          }
          if (GM == 4) {
            // B = im2col(x)[pixels (K), (tap, c) (N)]: the 64 pixels of this
            // k-block -> their first output position; per 64-column chunk
            // its (tap, channel block), clamped to the last chunk past N
            // (columns never stored)
            const int p0 = (kb0 + kb) * BK;
            const int hw = ga.Ho * ga.Wo;
            const int pn = p0 / hw, prem = p0 - pn * hw;
            const int poh = prem / ga.Wo, pow_ = prem - (prem / ga.Wo) * ga.Wo;
            const int piw = pow_ * ga.sw - ga.pw, pih = poh * ga.sh - ga.ph;
#pragma unroll
            for (int c = 0; c < BN / 64; ++c) {
              const int col = min(n0 + c * 64, N - 64);
              const int ctap = col / ga.C, ccb = col - ctap * ga.C;
              const int ci = ctap / ga.kw, cj = ctap - ci * ga.kw;
              asm volatile(
                  "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::"
                  "bytes [%0], [%1, {%2, %3, %4, %5}], [%6], {%7, %8};" ::"r"(
                      smem_u32(sa + G::kABytes + c * kMnChunkBytes)),
                  "l"(reinterpret_cast<uint64_t>(&map_b)), "r"(ccb), "r"(piw), "r"(pih), "r"(pn),
                  "r"(smem_u32(&full[s])), "h"(static_cast<uint16_t>(cj)),
                  "h"(static_cast<uint16_t>(ci))
                  : "memory");
            }
          }
          if (GM == 3) {
            const int ti = tap / ga.kw, tj = tap - (tap / ga.kw) * ga.kw;
            asm volatile(
                "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%2, %3, %4, %5}], [%6], {%7, %8};" ::"r"(smem_u32(sa)),
                "l"(reinterpret_cast<uint64_t>(&map_a)), "r"(cb), "r"(iw), "r"(ih), "r"(in_),
                "r"(smem_u32(&full[s])), "h"(static_cast<uint16_t>(tj)),
                "h"(static_cast<uint16_t>(ti))
                : "memory");
            cb += BK;
            if (cb == ga.C) {
              cb = 0;
              ++tap;
            }
          } else if (GM != 1 && GM != 6 && GM != 7) {
            load_operand<A_MN, BM>(sa, &map_a, &full[s], (kb0 + kb) * BK, m0);
          }
          if (GM != 2 && GM != 4)
            load_operand<B_MN, BN>(sa + G::kABytes, &map_b, &full[s], (kb0 + kb) * BK, n0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer
      int it = 0, local = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++local) {
        int m0, nt, z, kb0, nkb;
        sc.tile(t, &m0, &nt, &z, &kb0, &nkb);
        const int acc = local & 1;
        const uint32_t aph = (local >> 1) & 1;
        mbar_wait(&tempty[acc], aph ^ 1);  // epilogue drained this buffer
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t dst = tmem + uint32_t(acc * BN);
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % G::kStages;
          const uint32_t ph = (it / G::kStages) & 1;
          mbar_wait(&full[s], ph);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          // cp.async (generic proxy) writes -> tcgen05.mma (async proxy) reads
          if (gathered<GM>()) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          const uint8_t* sa = smem + s * G::kStageBytes;
          const uint64_t adesc = A_MN ? smem_desc_mn_sw128(sa) : smem_desc_sw128(sa);
          const uint64_t bdesc = B_MN ? smem_desc_mn_sw128(sa + G::kABytes)
                                      : smem_desc_sw128(sa + G::kABytes);
#pragma unroll
          for (int k = 0; k < BK / UMMA_K; ++k) {
            // K-major: +32 bytes per K16 step inside the 128-byte swizzle
            // row (>>4 -> +2); MN-major: +16 K rows of 128 bytes (+128)
            const uint64_t da = A_MN ? 128ull * k : 2ull * k;
            const uint64_t db = B_MN ? 128ull * k : 2ull * k;
            umma_bf16<A_MN, B_MN, BN>(dst, adesc + da, bdesc + db, (kb > 0 || k > 0) ? 1u : 0u);
          }
          umma_commit(&empty[s]);
        }
        umma_commit(&tfull[acc]);
      }
    }
  } else if (gathered<GM>() && warp >= 2 + EPI) {
    // ---------------- gather producers (implicit GEMM): cp.async 16-byte
    // chunks straight into the 128B-swizzled operand tile, zero-filled
    // outside the input; the mbarrier arrival fires when they land
    const int g = threadIdx.x - (64 + 32 * EPI);
    int it = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      int m0, nt, z, kb0, nkb;
      sc.tile(t, &m0, &nt, &z, &kb0, &nkb);
      const int n0 = nt * BN;
      if (GM == 1) {
        // A tile (K-major): lanes cover the 8 16-byte chunks of a 128-byte
        // row, so a warp instruction fills 4 whole rows (coalesced); thread
        // (q = g & 7, r0 = g >> 3) owns rows r0 + 16*i, i < 8
        const int q = g & 7, r0 = g >> 3;
        const int hw = ga.Ho * ga.Wo;
        int hb[8], wb[8];
        const __nv_bfloat16* rowp[8];  // element (hb, wb, 0) of the row's window (may be virtual)
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int m = m0 + r0 + 16 * i;
          const int b = m < M ? fdiv_u(m, ga.mul_hw) : -1;
          const int rem = m - (b < 0 ? 0 : b) * hw;
          const int oh = fdiv_u(rem, ga.mul_wo), ow = rem - oh * ga.Wo;
          hb[i] = b < 0 ? -(1 << 20) : oh * ga.sh - ga.ph;  // invalid row: always out of range
          wb[i] = ow * ga.sw - ga.pw;
          // dil 1: element (hb, wb, 0) of the row's window (may be virtual);
          // dil 2: the row's image base
          rowp[i] = ga.dil == 1
                        ? ga.src + (int64_t(b < 0 ? 0 : b) * ga.H * ga.W +
                                    int64_t(hb[i] < 0 && b < 0 ? 0 : hb[i]) * ga.W + wb[i]) * ga.C
                        : ga.src + int64_t(b < 0 ? 0 : b) * ga.H * ga.W * ga.C;
        }
        const int K = ga.kh * ga.kw * ga.C;
        // (tap row ti, tap column tj, channel c) of this thread's 8 K
        // columns, advanced by BK per k-block without dividing; koff is
        // their offset from a row's window origin in the NHWC source
        int k = kb0 * BK + q * 8;
        const int tap0 = fdiv_u(k, ga.mul_c);
        int c = k - tap0 * ga.C;
        int ti = fdiv_u(tap0, ga.mul_kw), tj = tap0 - ti * ga.kw;
        int64_t koff = (int64_t(ti) * ga.W + tj) * ga.C + c;
        const int64_t wskip = int64_t(ga.W - ga.kw) * ga.C;
        const uint32_t dbase = uint32_t(r0 * 128 + ((q ^ (r0 & 7)) << 4));
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % G::kStages;
          const uint32_t ph = (it / G::kStages) & 1;
          mbar_wait_sleep(&empty[s], ph ^ 1);
          const uint32_t tile = smem_u32(smem + s * G::kStageBytes) + dbase;
          const bool kv = k < K;
          if (ga.dil == 1) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int h = hb[i] + ti, w = wb[i] + tj;
              const bool v = kv && static_cast<unsigned>(h) < static_cast<unsigned>(ga.H) &&
                             static_cast<unsigned>(w) < static_cast<unsigned>(ga.W);
              const void* src = v ? static_cast<const void*>(rowp[i] + koff)
                                  : static_cast<const void*>(ga.src);
              cp_async16_zfill(tile + uint32_t(i * 16 * 128), src, v);
            }
          } else {
            // dilated by 2: even virtual positions only, halved
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int h = hb[i] + ti, w = wb[i] + tj;
              const bool v = kv && h >= 0 && w >= 0 && ((h | w) & 1) == 0 && (h >> 1) < ga.H &&
                             (w >> 1) < ga.W;
              const void* src =
                  v ? static_cast<const void*>(rowp[i] + (int64_t(h >> 1) * ga.W + (w >> 1)) * ga.C + c)
                    : static_cast<const void*>(ga.src);
              cp_async16_zfill(tile + uint32_t(i * 16 * 128), src, v);
            }
          }
          asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(
                           smem_u32(&full[s]))
                       : "memory");
          k += BK;
          c += BK;
          koff += BK;
          while (c >= ga.C) {
            c -= ga.C;
            if (++tj == ga.kw) {
              tj = 0;
              ++ti;
              koff += wskip;
            }
          }
        }
      } else {
        // B tile (MN-major): 64 K rows (pixels) x BN columns in 64-column
        // groups of 128-byte rows; lanes cover the 8 chunks of a row; thread
        // (q = g & 7, r0 = g >> 3) owns rows r0 + 16*i (i < 4) of every group
        // (GM 7: the A tile, BM columns from m0)
        const int q = g & 7, r0 = g >> 3;
        constexpr int NG = (GM == 7 ? BM : BN) / 64;
        const int col0 = GM == 7 ? m0 : n0, ncol = GM == 7 ? M : N;
        int gi[NG], gj[NG], gc[NG];
#pragma unroll
        for (int cg = 0; cg < NG; ++cg) {
          const int n = col0 + cg * 64 + q * 8;
          const int tap = n / ga.C;
          gc[cg] = n < ncol ? n - tap * ga.C : -1;
          gi[cg] = tap / ga.kw;
          gj[cg] = tap - gi[cg] * ga.kw;
        }
        const int hw = ga.Ho * ga.Wo;
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % G::kStages;
          const uint32_t ph = (it / G::kStages) & 1;
          mbar_wait_sleep(&empty[s], ph ^ 1);
          const uint32_t tile =
              smem_u32(smem + s * G::kStageBytes + (GM == 7 ? 0 : G::kABytes));
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int kr = r0 + 16 * i;
            const int m = (kb0 + kb) * BK + kr;
            const bool mv = m < sc.kext;
            const int b = mv ? fdiv_u(m, ga.mul_hw) : 0;
            const int rem = m - b * hw;
            const int oh = fdiv_u(rem, ga.mul_wo), ow = rem - oh * ga.Wo;
            const int hb = oh * ga.sh - ga.ph, wb = ow * ga.sw - ga.pw;
            const __nv_bfloat16* img = ga.src + int64_t(b) * ga.H * ga.W * ga.C;
#pragma unroll
            for (int cg = 0; cg < NG; ++cg) {
              const int h = hb + gi[cg], w = wb + gj[cg];
              const bool v = mv && gc[cg] >= 0 && h >= 0 && h < ga.H && w >= 0 && w < ga.W;
              const void* src =
                  v ? static_cast<const void*>(img + (int64_t(h) * ga.W + w) * ga.C + gc[cg])
                    : static_cast<const void*>(ga.src);
              cp_async16_zfill(tile + uint32_t(cg * kMnChunkBytes + kr * 128 + ((q ^ (kr & 7)) << 4)),
                               src, v);
            }
          }
          asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(
                           smem_u32(&full[s]))
                       : "memory");
        }
      }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  } else if (warp >= 2) {
    // ---------------- epilogue warps: TMEM lanes 32*(warp%4) .. +31; with
    // 8 warps, warp ew takes the 32-column chunks h, h+2, ... (h = ew / 4)
    // and stages through one 4 KB box instead of two
    constexpr int NB = 8 / EPI;           // staging boxes per warp
    constexpr int CSTEP = 32 * (EPI / 4);  // column step between a warp's chunks
    const int ew = warp - 2;
    const int lane_base = (warp & 3) * 32;
    uint8_t* cbuf = stage_c + ew * NB * kStageCBytes;
    int local = 0, nbuf = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++local) {
      int m0, nt, z, kb0, nkb;
      sc.tile(t, &m0, &nt, &z, &kb0, &nkb);
      const int n0 = nt * BN;
      const int acc = local & 1;
      const uint32_t aph = (local >> 1) & 1;
      float* Cz = C + int64_t(z) * split_stride;
      mbar_wait_sleep(&tfull[acc], aph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int row0 = m0 + lane_base;
      for (int c0 = 32 * (ew / 4); c0 < BN; c0 += CSTEP) {
        uint32_t r[32];
        const uint32_t taddr = tmem + (uint32_t(lane_base) << 16) + uint32_t(acc * BN + c0);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
            "%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
              "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
              "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
              "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
              "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
              "=r"(r[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (c0 + CSTEP >= BN) {
          // all of this accumulator is in registers: hand TMEM back early
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[acc]);
        }
        // warp-uniform epilogue variants: the generic activation code
        // (double-precision exp/tanh) stays out of the common loops
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = nkb > 0 ? __uint_as_float(r[j]) : 0.0f;
        if (bias) {
          const int nb = n0 + c0;
          if (nb + 32 <= N && (N & 3) == 0) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const float4 b4 = __ldg(reinterpret_cast<const float4*>(bias + nb) + j);
              v[4 * j] = fadd(v[4 * j], b4.x);
              v[4 * j + 1] = fadd(v[4 * j + 1], b4.y);
              v[4 * j + 2] = fadd(v[4 * j + 2], b4.z);
              v[4 * j + 3] = fadd(v[4 * j + 3], b4.w);
            }
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = fadd(v[j], nb + j < N ? __ldg(bias + nb + j) : 0.0f);
          }
        }
        if (ACTK == 1) {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = relu(v[j]);
        } else if (ACTK == 2) {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = act_forward(act, v[j]);
        }
        if (use_tma_store) {
          if (row0 >= M) continue;  // warp-uniform: nothing of this box is in C
          // transposed: this chunk's columns are rows of C; past N they would
          // land in the next split's rows of the workspace (N % 32 == 0)
          if ((GM == 6 || GM == 7) && n0 + c0 >= N) continue;
          uint8_t* buf = cbuf + nbuf * kStageCBytes;
          // the store that last read this buffer (NB chunks ago) is done
          if (lane == 0) {
            if (NB == 2)
              asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            else
              asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          }
          __syncwarp();
          if (GM == 6 || GM == 7) {
            // transposed box: row j = column n0 + c0 + j of D, element lane
            // = row row0 + lane (128-byte swizzle: 16-byte chunk ^ row & 7)
#pragma unroll
            for (int j = 0; j < 32; ++j)
              *reinterpret_cast<float*>(buf + j * 128 + ((((lane >> 2) ^ (j & 7)) << 4) |
                                                         ((lane & 3) << 2))) = v[j];
          } else {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              float4 q = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
              *reinterpret_cast<float4*>(buf + lane * 128 + ((j ^ (lane & 7)) << 4)) = q;
            }
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            if (GM == 6 || GM == 7)
              tma_store_2d(&map_c, buf, row0, int(int64_t(z) * N) + n0 + c0);
            else
              tma_store_2d(&map_c, buf, n0 + c0, int(int64_t(z) * M) + row0);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
          if (colstats) {
            // per-column (mean, M2) of this warp's valid rows (lane = row):
            // values shifted by the block's first row, then two warp
            // reduce-scatter butterflies leave column c0 + lane's sums in
            // lane `lane` (fixed tree order: deterministic) -- the
            // BatchNorm statistics of the convolution output, merged later
            // in a fixed order (bn_stats_from_tiles)
            const int nrows = min(32, M - row0);
            const int col = n0 + c0 + lane;
            const bool valid = lane < nrows;
            float x0 = 0.0f;
            float sq[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const float t = __shfl_sync(0xffffffffu, v[j], 0);
              if (lane == j) x0 = t;
              const float d = valid ? v[j] - t : 0.0f;
              v[j] = d;
              sq[j] = d * d;
            }
            warp_reduce_scatter32(v, lane);
            warp_reduce_scatter32(sq, lane);
            const float s1 = v[0], s2 = sq[0];
            const float inv = 1.0f / float(nrows);
            const float dm = s1 * inv;
            const float m2 = fmaxf(s2 - s1 * dm, 0.0f);
            if (col < N) colstats[int64_t(row0 >> 5) * N + col] = make_float2(x0 + dm, m2);
          }
          if (NB == 2) nbuf ^= 1;
        } else {
          const int row = row0 + lane;
          if (row < M) {
            float* crow = Cz + int64_t(row) * ldc;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const int n = n0 + c0 + j;
              if (n < N) crow[n] = v[j];
            }
          }
        }
      }
    }
    if (use_tma_store && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(G::kTmemCols));
  }
}

// Split-K epilogue: C[m, n] = act(sum_z ws[z][m, n] (+ bias[n])), partial
// tiles summed in ascending split order (deterministic).
__global__ void splitk_reduce_kernel(const float* __restrict__ ws, int splits, int64_t split_stride,
                                     const float* __restrict__ bias, float* __restrict__ C,
                                     int64_t ldc, int64_t M, int64_t N, int act) {
  const int64_t total = M * N;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += stride) {
    const int64_t m = i / N, n = i - m * N;
    const int64_t o = m * N + n;
    float v = ws[o];
    for (int z = 1; z < splits; ++z) v = fadd(v, ws[z * split_stride + o]);
    if (bias) v = fadd(v, __ldg(bias + n));
    C[m * ldc + n] = act_forward(act, v);
  }
}

// float4 form (N % 4 == 0, ldc % 4 == 0, aligned), parallel over the
// splits too: a block owns VB output vectors x SL split lanes (SL * VB =
// 256); lane l sums splits l, l + SL, ... in ascending order, then the SL
// lane sums meet in ascending lane order through shared memory -- a fixed
// association (deterministic) with every split load in flight across the
// block, so a tall split count over a small output is not a serial chain.
__global__ void __launch_bounds__(256)
splitk_reduce4_kernel(const float4* __restrict__ ws, int splits, int64_t split_stride4,
                      const float* __restrict__ bias, float4* __restrict__ C, int64_t ldc4,
                      int64_t M, int64_t N4, int act, int SL) {
  __shared__ float4 part[256];
  const int VB = blockDim.x / SL;
  const int lane = threadIdx.x / VB, v = threadIdx.x - (threadIdx.x / VB) * VB;
  const int64_t total = M * N4;
  for (int64_t base = int64_t(blockIdx.x) * VB; base < total; base += int64_t(gridDim.x) * VB) {
    const int64_t i = base + v;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    bool first = true;
    if (i < total) {
      constexpr int B = 4;
      for (int z0 = lane; z0 < splits; z0 += B * SL) {
        float4 p[B];
#pragma unroll
        for (int u = 0; u < B; ++u)
          if (z0 + u * SL < splits) p[u] = ws[(z0 + u * SL) * split_stride4 + i];
#pragma unroll
        for (int u = 0; u < B; ++u)
          if (z0 + u * SL < splits) {
            if (first) {
              acc = p[u];
              first = false;
            } else {
              acc.x = fadd(acc.x, p[u].x);
              acc.y = fadd(acc.y, p[u].y);
              acc.z = fadd(acc.z, p[u].z);
              acc.w = fadd(acc.w, p[u].w);
            }
          }
      }
    }
    part[threadIdx.x] = acc;
    __syncthreads();
    if (lane == 0 && i < total) {
      float4 t = part[v];
      for (int l = 1; l < SL && l < splits; ++l) {
        const float4 q = part[l * VB + v];
        t.x = fadd(t.x, q.x);
        t.y = fadd(t.y, q.y);
        t.z = fadd(t.z, q.z);
        t.w = fadd(t.w, q.w);
      }
      const int64_t m = i / N4, n4 = i - m * N4;
      if (bias) {
        const float4 b = __ldg(reinterpret_cast<const float4*>(bias) + n4);
        t.x = fadd(t.x, b.x);
        t.y = fadd(t.y, b.y);
        t.z = fadd(t.z, b.z);
        t.w = fadd(t.w, b.w);
      }
      t.x = act_forward(act, t.x);
      t.y = act_forward(act, t.y);
      t.z = act_forward(act, t.z);
      t.w = act_forward(act, t.w);
      C[m * ldc4 + n4] = t;
    }
    __syncthreads();
  }
}

__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}

// y (bf16, rows x ldo) = x (fp32, R x C, row stride ldi), zero-filled
// beyond the source extent (the K padding of a tensor-core operand).  8
// output columns per thread (one 16-byte store).
// rows x vectors launch shape (RowsIdx): a thread owns an 8-column group
__global__ void cast_rows_kernel(const float* __restrict__ x, int64_t R, int64_t C, int64_t ldi,
                                 __nv_bfloat16* __restrict__ y, int64_t rows, int64_t ldo) {
  const RowsIdx ri(static_cast<int>(ldo / 8));
  if (!ri.active) return;
  const int64_t c0 = int64_t(ri.v) * 8;
  const bool vec = ((ldi & 3) == 0) && ((reinterpret_cast<uintptr_t>(x) & 15) == 0);
  for (int64_t r = ri.r; r < rows; r += ri.rstep) {
    float v[8];
    if (r < R && vec && c0 + 8 <= C) {
      const float4 a = __ldg(reinterpret_cast<const float4*>(x + r * ldi + c0));
      const float4 b = __ldg(reinterpret_cast<const float4*>(x + r * ldi + c0 + 4));
      v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
      v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = (r < R && c0 + j < C) ? __ldg(x + r * ldi + c0 + j) : 0.0f;
    }
    uint4 o;
    o.x = pack2(v[0], v[1]);
    o.y = pack2(v[2], v[3]);
    o.z = pack2(v[4], v[5]);
    o.w = pack2(v[6], v[7]);
    *reinterpret_cast<uint4*>(y + r * ldo + c0) = o;
  }
}

// transposed cast: y[c, r] (bf16, rows x ldo) = x[r, c], zero beyond the
// source; 32x32 tiles through shared memory
__global__ void cast_transpose_kernel(const float* __restrict__ x, int64_t R, int64_t C,
                                      int64_t ldi, __nv_bfloat16* __restrict__ y, int64_t rows,
                                      int64_t ldo) {
  __shared__ float tile[32][33];
  const int64_t tr = int64_t(blockIdx.y) * 32, tc = int64_t(blockIdx.x) * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t r = tr + i, c = tc + threadIdx.x;
    tile[i][threadIdx.x] = (r < R && c < C) ? __ldg(x + r * ldi + c) : 0.0f;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t orow = tc + i, ocol = tr + threadIdx.x;
    if (orow < rows && ocol < ldo) y[orow * ldo + ocol] = __float2bfloat16_rn(tile[threadIdx.x][i]);
  }
}

__global__ void cast_f32_bf16_kernel(const float* __restrict__ x, __nv_bfloat16* __restrict__ y,
                                     int64_t n) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    y[i] = __float2bfloat16_rn(x[i]);
}

// ---------------------------------------------------------------- host

static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
static std::once_flag g_encode_once;

typedef CUresult (*PFN_encode_im2col)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                       const cuuint64_t*, const cuuint64_t*, const int*,
                                       const int*, cuuint32_t, cuuint32_t, const cuuint32_t*,
                                       CUtensorMapInterleave, CUtensorMapSwizzle,
                                       CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static PFN_encode_im2col g_encode_im2col = nullptr;
static std::once_flag g_im2col_once;

// TMA im2col map of a bf16 NHWC tensor for a k x k / stride s / pad p
// convolution: each load gives 128 consecutive output pixels x 64 channels
// of one filter tap (offsets in the instruction), zero in the padding
static int encode_im2col(CUtensorMap* map, const void* src, int B, int H, int W, int C, int kh,
                         int kw, int sh, int sw, int ph, int pw, int pixels = BM) {
  std::call_once(g_im2col_once, [] {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &fn, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode_im2col = reinterpret_cast<PFN_encode_im2col>(fn);
  });
  if (!g_encode_im2col) {
    set_error("cuTensorMapEncodeIm2col unavailable from the driver");
    return MGX_INTERNAL;
  }
  cuuint64_t dims[4] = {cuuint64_t(C), cuuint64_t(W), cuuint64_t(H), cuuint64_t(B)};
  cuuint64_t strides[3] = {cuuint64_t(C) * 2, cuuint64_t(W) * C * 2, cuuint64_t(H) * W * C * 2};
  int lower[2] = {-pw, -ph};
  int upper[2] = {pw - (kw - 1), ph - (kh - 1)};
  cuuint32_t estr[4] = {1, cuuint32_t(sw), cuuint32_t(sh), 1};
  CUresult r = g_encode_im2col(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(src),
                               dims, strides, lower, upper, BK, pixels, estr,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeIm2col failed (%d)", static_cast<int>(r));
    return MGX_INTERNAL;
  }
  return MGX_OK;
}

static int get_encode() {
  std::call_once(g_encode_once, [] {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  if (!g_encode) {
    set_error("cuTensorMapEncodeTiled unavailable from the driver");
    return MGX_INTERNAL;
  }
  return MGX_OK;
}

static int encode(CUtensorMap* map, CUtensorMapDataType dt, const void* base, cuuint64_t d0,
                  cuuint64_t d1, cuuint64_t stride_bytes, cuuint32_t b0, cuuint32_t b1) {
  cuuint64_t dims[2] = {d0, d1};
  cuuint64_t strides[1] = {stride_bytes};
  cuuint32_t box[2] = {b0, b1};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(map, dt, 2, const_cast<void*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d)", static_cast<int>(r));
    return MGX_INTERNAL;
  }
  return MGX_OK;
}

// K-major operand: dims {K, rows}, box {64, box_rows}; MN-major: dims
// {rows, K} (rows contiguous), box {64, 64}
static int make_map(CUtensorMap* map, const void* base, int64_t rows, int64_t K, int64_t ld,
                    bool mn, int box_rows) {
  if (!mn)
    return encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, base, K, rows, ld * 2, BK, box_rows);
  return encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, base, rows, K, ld * 2, 64, BK);
}

template <bool A_MN, bool B_MN, int BN, int ACTK, int GM, int EPI>
static int launch_epi(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mc,
                      int grid, const float* bias, float* C, int ldc, int M, int N, int act,
                      const Sched& sc, int64_t split_stride, int tma_store, const Gather& ga,
                      float2* colstats, cudaStream_t st) {
  using G = Cfg<BN>;
  static bool configured = false;
  if (!configured) {
    MGX_CUDA(cudaFuncSetAttribute(tc_gemm_bf16_kernel<A_MN, B_MN, BN, ACTK, GM, EPI>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, G::kSmemBytes));
    configured = true;
  }
  tc_gemm_bf16_kernel<A_MN, B_MN, BN, ACTK, GM, EPI>
      <<<grid, threads_for<GM, EPI>(), G::kSmemBytes, st>>>(
          ma, mb, mc, bias, C, ldc, M, N, act, sc, split_stride, tma_store, ga, colstats);
  MGX_LAUNCHED();
  return MGX_OK;
}

// 8 epilogue warps for the TMA-fed modes (env MGX_GEMM_EPI=4: four)
template <bool A_MN, bool B_MN, int BN, int ACTK, int GM>
static int launch_act(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mc,
                      int grid, const float* bias, float* C, int ldc, int M, int N, int act,
                      const Sched& sc, int64_t split_stride, int tma_store, const Gather& ga,
                      float2* colstats, cudaStream_t st) {
  static const bool epi8 = [] {
    const char* v = getenv("MGX_GEMM_EPI");
    return !(v && atoi(v) == 4);
  }();
  if constexpr (!gathered<GM>()) {
    if (epi8)
      return launch_epi<A_MN, B_MN, BN, ACTK, GM, 8>(ma, mb, mc, grid, bias, C, ldc, M, N, act,
                                                     sc, split_stride, tma_store, ga, colstats,
                                                     st);
  }
  return launch_epi<A_MN, B_MN, BN, ACTK, GM, 4>(ma, mb, mc, grid, bias, C, ldc, M, N, act, sc,
                                                 split_stride, tma_store, ga, colstats, st);
}

struct Launch {
  CUtensorMap ma, mb, mc;
  int grid;
  const float* bias;
  float* C;
  int ldc, M, N, act;
  Sched sc;
  int64_t sstride;
  int tma;
  Gather ga;
  float2* colstats;
};

template <bool A_MN, bool B_MN, int BN, int GM>
static int launch_acts(const Launch& l, cudaStream_t st) {
  if (l.act == MGX_ACT_NONE)
    return launch_act<A_MN, B_MN, BN, 0, GM>(l.ma, l.mb, l.mc, l.grid, l.bias, l.C, l.ldc, l.M, l.N,
                                             l.act, l.sc, l.sstride, l.tma, l.ga, l.colstats, st);
  if (l.act == MGX_ACT_RELU)
    return launch_act<A_MN, B_MN, BN, 1, GM>(l.ma, l.mb, l.mc, l.grid, l.bias, l.C, l.ldc, l.M, l.N,
                                             l.act, l.sc, l.sstride, l.tma, l.ga, l.colstats, st);
  return launch_act<A_MN, B_MN, BN, 2, GM>(l.ma, l.mb, l.mc, l.grid, l.bias, l.C, l.ldc, l.M, l.N,
                                           l.act, l.sc, l.sstride, l.tma, l.ga, l.colstats, st);
}

template <int BN>
static int launch_bn(int a_mn, int b_mn, int gm, const Launch& l, cudaStream_t st) {
  if (gm == 1) return launch_acts<false, false, BN, 1>(l, st);  // implicit A, B K-major
  if (gm == 3) return launch_acts<false, false, BN, 3>(l, st);  // A by TMA im2col, B K-major
  if (gm == 2) return launch_acts<true, true, BN, 2>(l, st);    // A MN-major, implicit B
  if (gm == 4) return launch_acts<true, true, BN, 4>(l, st);    // A MN-major, B by TMA im2col
  if (gm == 6) return launch_acts<true, true, BN, 6>(l, st);    // transposed weight gradient
  if (gm == 7) return launch_acts<true, true, BN, 7>(l, st);    // ... its A gathered
  if (!a_mn && !b_mn) return launch_acts<false, false, BN, 0>(l, st);
  if (!a_mn && b_mn) return launch_acts<false, true, BN, 0>(l, st);
  if (a_mn && !b_mn) return launch_acts<true, false, BN, 0>(l, st);
  return launch_acts<true, true, BN, 0>(l, st);
}

static thread_local int t_cta_cap = 0;

// split-K count: about `target` CTAs per GEMM (0: env MGX_SPLIT_TARGET,
// default 128 -- a GEMM alone on the GPU fills it; the executor passes a
// lower per-network target when independent branches run side by side:
// Inception-BN A/B 128 -> 4.83, 64 -> 4.76, 32 -> 4.67, 16 -> 4.79
// ms/step), each split at least `min_kb` k-blocks (env MGX_SPLIT_MINK,
// default 16: short splits are all prologue, epilogue and workspace
// traffic), and -- for accuracy -- at most kMaxKbPerSplit k-blocks per
// split (fp32 accumulation runs of <= 8192 products, like the default
// target gives the long-K weight gradients).  Never depends on t_cta_cap:
// results are the same on every lane schedule, bitwise.
constexpr int64_t kMaxKbPerSplit = 128;

static int auto_splits(int64_t tiles, int64_t nk, int64_t target = 0) {
  static const int64_t target_env = [] {
    const char* v = getenv("MGX_SPLIT_TARGET");
    return int64_t(v && *v ? atoi(v) : 128);
  }();
  static const int64_t min_kb = [] {
    const char* v = getenv("MGX_SPLIT_MINK");
    return int64_t(v && *v ? atoi(v) : 16);
  }();
  if (target <= 0) target = target_env;
  int64_t s = 1;
  if (tiles < target) {
    const int64_t want = target / tiles, most = nk / min_kb;
    s = want < most ? want : most;
  }
  const int64_t floor_s = ceil_div(nk, kMaxKbPerSplit);
  if (s < floor_s) s = floor_s;
  return static_cast<int>(s < 1 ? 1 : s);
}

// N tile: the width in {64, 128, 192, 256} minimising n_tiles * (BN + 64):
// the columns computed (padding included) plus a fixed per-tile cost worth
// ~64 columns (operand A re-load / re-gather, pipeline fill, epilogue) --
// narrow tiles multiply that cost and issue 4x more, smaller MMAs; ties go
// to the wider tile.  (env MGX_BN_TILE_COST overrides the 64.)
static int pick_bn(int64_t M, int64_t N) {
  (void)M;
  static const int64_t over = [] {
    const char* v = getenv("MGX_BN_TILE_COST");
    return int64_t(v && *v ? atoi(v) : 64);
  }();
  int best = 64;
  int64_t cost = ceil_div(N, 64) * (64 + over);
  for (int bn : {128, 192, 256}) {
    const int64_t c = ceil_div(N, bn) * (bn + over);
    if (c <= cost) {
      cost = c;
      best = bn;
    }
  }
  return best;
}

}  // namespace tc
}  // namespace mgx

namespace mgx {
namespace tc {

// shared implementation: gm 0 plain, 1 implicit A (ga describes it), 2
// implicit B
static int gemm_impl(const void* A, int64_t lda, int a_mn, const void* B, int64_t ldb, int b_mn,
                     const float* bias, float* C, int64_t ldc, int64_t M, int64_t N, int64_t K,
                     int act, int splits, float* workspace, int gm, const Gather& ga,
                     float* colstats, cudaStream_t st) {
  MGX_REQUIRE(C && M > 0 && N > 0 && K > 0, "mgx_gemm_bf16_tc: bad arguments");
  const bool a_impl = gm == 1 || gm == 3 || gm == 6 || gm == 7;  // A gathered / TMA im2col
  const bool trans = gm == 6 || gm == 7;  // D = C^T: C[N, ldc] holds the transposed tiles
  const bool b_impl = gm == 2 || gm == 4;  // B gathered / by TMA im2col
  MGX_REQUIRE((a_impl || A) && (b_impl || B), "mgx_gemm_bf16_tc: missing operand");
  MGX_REQUIRE((a_impl || lda % 8 == 0) && (b_impl || ldb % 8 == 0),
              "mgx_gemm_bf16_tc: leading dimensions must be multiples of 8");
  MGX_REQUIRE((a_impl || lda >= (a_mn ? M : K)) && (b_impl || ldb >= (b_mn ? N : K)),
              "mgx_gemm_bf16_tc: leading dimension smaller than the operand row");
  MGX_REQUIRE((a_impl || mgx::aligned16(A)) && (b_impl || mgx::aligned16(B)),
              "mgx_gemm_bf16_tc: operands not 16-byte aligned");
  MGX_REQUIRE(M < (1ll << 31) && N < (1ll << 31) && K < (1ll << 31) && ldc < (1ll << 31),
              "mgx_gemm_bf16_tc: dimensions exceed 2^31");
  MGX_REQUIRE(splits >= 0, "mgx_gemm_bf16_tc: negative split count");
  MGX_TRY(get_encode());
  const int bn = pick_bn(M, N);
  const int64_t m_tiles = mgx::ceil_div(M, BM), n_tiles = mgx::ceil_div(N, bn);
  const int64_t nk = mgx::ceil_div(K, BK);
  if (splits == 0) splits = workspace ? auto_splits(m_tiles * n_tiles, nk) : 1;
  MGX_REQUIRE(splits == 1 || workspace, "mgx_gemm_bf16_tc: split-K needs a workspace");
  int kps = static_cast<int>(mgx::ceil_div(nk, splits));
  splits = static_cast<int>(mgx::ceil_div(nk, kps));
  MGX_REQUIRE(int64_t(splits) * M < (1ll << 31), "mgx_gemm_bf16_tc: split workspace too tall");
  Launch l;
  std::memset(&l, 0, sizeof(l));
  if (gm == 3)
    MGX_TRY(encode_im2col(&l.ma, ga.src, ga.B, ga.H, ga.W, ga.C, ga.kh, ga.kw, ga.sh, ga.sw,
                          ga.ph, ga.pw));
  else if (gm == 6)
    MGX_TRY(encode_im2col(&l.ma, ga.src, ga.B, ga.H, ga.W, ga.C, ga.kh, ga.kw, ga.sh, ga.sw,
                          ga.ph, ga.pw, BK));
  else if (gm != 1 && gm != 7)
    MGX_TRY(make_map(&l.ma, A, M, K, lda, a_mn != 0, BM));
  if (gm == 4)
    MGX_TRY(encode_im2col(&l.mb, ga.src, ga.B, ga.H, ga.W, ga.C, ga.kh, ga.kw, ga.sh, ga.sw,
                          ga.ph, ga.pw, BK));
  else if (gm != 2)
    MGX_TRY(make_map(&l.mb, B, N, K, ldb, b_mn != 0, bn));
  float* out = splits == 1 ? C : workspace;
  // the stored matrix: M x N, or N x M for the transposed weight gradient
  const int64_t orows = trans ? N : M, ocols = trans ? M : N;
  const int64_t oldc = splits == 1 ? ldc : ocols;
  // TMA store needs a 16-byte row pitch and base; the map spans all splits
  // (partial 32-row boxes of a split would spill into the next split's rows)
  l.tma = (oldc % 4 == 0) && mgx::aligned16(out) && (splits == 1 || orows % 32 == 0);
  MGX_REQUIRE(l.tma || !trans, "mgx_gemm_bf16_tc: the transposed form needs a TMA store");
  if (l.tma)
    MGX_TRY(mgx::tc::encode(&l.mc, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, out, ocols,
                            int64_t(splits) * orows, oldc * 4, 32, 32));
  l.sc = Sched{static_cast<int>(m_tiles), static_cast<int>(n_tiles), splits, kps,
               static_cast<int>(nk), static_cast<int>(K)};
  const int64_t total = m_tiles * n_tiles * splits;
  // persistent CTAs: at most one per SM (env MGX_GEMM_MAX_CTAS caps it lower:
  // concurrent branches of the graph share the GPU)
  static const int64_t max_ctas = [] {
    const char* v = getenv("MGX_GEMM_MAX_CTAS");
    const int64_t c = v && *v ? atoi(v) : mgx::kNumSMs;
    return c < 1 ? 1 : (c > mgx::kNumSMs ? int64_t(mgx::kNumSMs) : c);
  }();
  const int64_t cap = t_cta_cap > 0 && t_cta_cap < max_ctas ? t_cta_cap : max_ctas;
  l.grid = static_cast<int>(total < cap ? total : cap);
  l.sstride = M * N;
  l.bias = splits == 1 ? bias : nullptr;
  l.act = splits == 1 ? act : 0;
  l.C = out;
  l.ldc = static_cast<int>(oldc);
  l.M = static_cast<int>(M);
  l.N = static_cast<int>(N);
  l.ga = ga;
  l.colstats = reinterpret_cast<float2*>(colstats);
  MGX_REQUIRE(!colstats || (splits == 1 && l.tma && mgx::aligned16(colstats)),
              "mgx_gemm_bf16_tc: column statistics need one split and a 16-byte aligned C pitch");
  int rc = bn == 64    ? launch_bn<64>(a_mn, b_mn, gm, l, st)
           : bn == 128 ? launch_bn<128>(a_mn, b_mn, gm, l, st)
           : bn == 192 ? launch_bn<192>(a_mn, b_mn, gm, l, st)
                       : launch_bn<256>(a_mn, b_mn, gm, l, st);
  if (rc != MGX_OK || splits == 1) return rc;
  MGX_REQUIRE(!trans || !bias, "mgx_gemm_bf16_tc: the transposed form takes no bias");
  if (ocols % 4 == 0 && ldc % 4 == 0 && l.sstride % 4 == 0 && mgx::aligned16(C) &&
      mgx::aligned16(workspace) && (!bias || mgx::aligned16(bias))) {
    // split lanes: enough to put ~4 split loads per thread in flight
    int SL = 1;
    while (SL < 32 && SL * 4 < splits) SL *= 2;
    const int VB = 256 / SL;
    int64_t blocks = mgx::ceil_div(M * N / 4, VB);
    if (blocks > 148 * 8) blocks = 148 * 8;
    splitk_reduce4_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(
        reinterpret_cast<const float4*>(workspace), splits, l.sstride / 4, bias,
        reinterpret_cast<float4*>(C), ldc / 4, orows, ocols / 4, act, SL);
    MGX_LAUNCHED();
    return MGX_OK;
  }
  int64_t blocks = mgx::ceil_div(M * N, 256);
  if (blocks > 148 * 8) blocks = 148 * 8;
  splitk_reduce_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(workspace, splits, l.sstride,
                                                                      bias, C, ldc, orows, ocols,
                                                                      act);
  MGX_LAUNCHED();
  return MGX_OK;
}

}  // namespace tc

void set_gemm_cta_cap(int cap) { tc::t_cta_cap = cap < 0 ? 0 : cap; }

}  // namespace mgx

extern "C" int mgx_gemm_bf16_tc_ex(const void* A, int64_t lda, int a_mn, const void* B,
                                   int64_t ldb, int b_mn, const float* bias, float* C, int64_t ldc,
                                   int64_t M, int64_t N, int64_t K, int act, int splits,
                                   float* workspace, float* colstats, uintptr_t stream) {
  mgx::tc::Gather none;
  std::memset(&none, 0, sizeof(none));
  return mgx::tc::gemm_impl(A, lda, a_mn, B, ldb, b_mn, bias, C, ldc, M, N, K, act, splits,
                            workspace, 0, none, colstats, mgx::as_stream(stream));
}

extern "C" int mgx_gemm_bf16_conv(int mode, const void* src, const int64_t* geom, const void* op,
                                  int64_t ldop, const float* bias, float* C, int64_t ldc,
                                  int64_t M, int64_t N, int64_t K, int act, int splits,
                                  float* workspace, float* colstats, uintptr_t stream) {
  using namespace mgx::tc;
  MGX_REQUIRE(src && geom && op && (mode >= 1 && mode <= 3), "mgx_gemm_bf16_conv: bad arguments");
  MGX_REQUIRE(mgx::aligned16(src), "mgx_gemm_bf16_conv: source not 16-byte aligned");
  Gather ga;
  ga.src = static_cast<const __nv_bfloat16*>(src);
  ga.B = static_cast<int>(geom[0]);
  ga.H = static_cast<int>(geom[1]);
  ga.W = static_cast<int>(geom[2]);
  ga.C = static_cast<int>(geom[3]);
  ga.kh = static_cast<int>(geom[4] >> 16);
  ga.kw = static_cast<int>(geom[4] & 0xFFFF);
  ga.sh = static_cast<int>(geom[5] >> 16);
  ga.sw = static_cast<int>(geom[5] & 0xFFFF);
  ga.ph = static_cast<int>(geom[6] >> 16);
  ga.pw = static_cast<int>(geom[6] & 0xFFFF);
  ga.Ho = (ga.H + 2 * ga.ph - ga.kh) / ga.sh + 1;
  ga.Wo = (ga.W + 2 * ga.pw - ga.kw) / ga.sw + 1;
  ga.dil = 1;
  if (mode == 3) {
    // data gradient of a stride-2 convolution whose FORWARD geometry is
    // `geom` (input B x H x W x C): src = dY [B, Ho, Wo, F] read dilated by
    // 2 with pad k-1-p, op = the flipped weights [C, kh*kw*F], output
    // dX [B*H*W, C] -- no column matrix, no col2im
    MGX_REQUIRE(ga.sh == 2 && ga.sw == 2 && ga.ph < ga.kh && ga.pw < ga.kw && K % (ga.kh * ga.kw) == 0,
                "mgx_gemm_bf16_conv: mode 3 needs stride 2 and pad < kernel");
    const int F = static_cast<int>(K / (ga.kh * ga.kw));
    const int H = ga.H, W = ga.W, Ho = ga.Ho, Wo = ga.Wo;
    MGX_REQUIRE(F % 8 == 0 && M == int64_t(ga.B) * H * W && N == ga.C,
                "mgx_gemm_bf16_conv: mode 3 shapes (F %% 8 == 0, M = B*H*W, N = C)");
    ga.H = Ho;
    ga.W = Wo;
    ga.C = F;
    ga.sh = ga.sw = 1;
    ga.ph = ga.kh - 1 - ga.ph;
    ga.pw = ga.kw - 1 - ga.pw;
    ga.Ho = H;
    ga.Wo = W;
    ga.dil = 2;
    ga.mul_hw = fastdiv_mul(H * W);
    ga.mul_wo = fastdiv_mul(W);
    ga.mul_c = fastdiv_mul(F);
    ga.mul_kw = fastdiv_mul(ga.kw);
    return gemm_impl(nullptr, 0, 0, op, ldop, 0, bias, C, ldc, M, N, K, act, splits, workspace, 1,
                     ga, colstats, mgx::as_stream(stream));
  }
  MGX_REQUIRE(ga.C % 8 == 0 && ga.C > 0 && ga.Ho > 0 && ga.Wo > 0 && ga.B > 0,
              "mgx_gemm_bf16_conv: the gathered tensor needs C %% 8 == 0");
  ga.mul_hw = fastdiv_mul(ga.Ho * ga.Wo);
  ga.mul_wo = fastdiv_mul(ga.Wo);
  ga.mul_c = fastdiv_mul(ga.C);
  ga.mul_kw = fastdiv_mul(ga.kw);
  const int64_t pixels = int64_t(ga.B) * ga.Ho * ga.Wo;
  const int64_t kconv = int64_t(ga.kh) * ga.kw * ga.C;
  if (mode == 1) {
    // C[pixels, N] = gather(src)[pixels, kconv] . op[N, kconv]^T
    MGX_REQUIRE(M == pixels && K == kconv, "mgx_gemm_bf16_conv: M/K do not match the geometry");
    // whole 64-channel blocks per tap: the A tile by one TMA im2col load per
    // k-block instead of the gather warps (env MGX_TMA_IM2COL=0 disables)
    static const bool tma_im2col = [] {
      const char* v = getenv("MGX_TMA_IM2COL");
      return !(v && *v == '0');
    }();
    const bool use_tma = tma_im2col && ga.C % BK == 0 && ga.ph <= 127 && ga.pw <= 127 &&
                         ga.kh - 1 - ga.ph <= 128 && ga.kw - 1 - ga.pw <= 128 && ga.sh <= 8 &&
                         ga.sw <= 8;
    return gemm_impl(nullptr, 0, 0, op, ldop, 0, bias, C, ldc, M, N, K, act, splits, workspace,
                     use_tma ? 3 : 1, ga, colstats, mgx::as_stream(stream));
  }
  // C[M, kconv] = op[pixels, M]^T (MN-major) . gather(src)[pixels, kconv];
  // whole 64-channel blocks per tap: B by TMA im2col boxes of 64 pixels x 64
  // channels (MN-major chunks) instead of the gather warps
  MGX_REQUIRE(K == pixels && N == kconv, "mgx_gemm_bf16_conv: N/K do not match the geometry");
  static const bool tma_dw = [] {
    const char* v = getenv("MGX_TMA_IM2COL_DW");
    return !(v && *v == '0');
  }();
  const bool use_tma = tma_dw && ga.C % BK == 0 && ga.ph <= 127 && ga.pw <= 127 &&
                       ga.kh - 1 - ga.ph <= 128 && ga.kw - 1 - ga.pw <= 128 && ga.sh <= 8 &&
                       ga.sw <= 8 && N >= 64;
  // few filters: the transposed product D[kconv, F] fills the 128-row M
  // tiles better (e.g. F = 160: 62 % of the M tile used, transposed 83 %);
  // its tiles are stored transposed (GEMM mode 6; env MGX_DW_SWAP=0: off)
  static const bool dw_swap = [] {
    const char* v = getenv("MGX_DW_SWAP");
    return !(v && *v == '0');
  }();
  if (dw_swap && !bias && !colstats && M % 32 == 0 && N % 4 == 0 && N >= 64 && ldc % 4 == 0 &&
      mgx::aligned16(C) && (!workspace || mgx::aligned16(workspace))) {
    auto fill = [](int64_t m, int64_t n) {
      const int64_t bn = pick_bn(m, n);
      return double(m) / double(mgx::ceil_div(m, int64_t(BM)) * BM) * double(n) /
             double(mgx::ceil_div(n, bn) * bn);
    };
    if (fill(N, M) > 1.1 * fill(M, N))
      return gemm_impl(nullptr, 0, 1, op, ldop, 1, nullptr, C, ldc, N, M, K, act, splits,
                       workspace, use_tma ? 6 : 7, ga, nullptr, mgx::as_stream(stream));
  }
  return gemm_impl(op, ldop, 1, nullptr, 0, 1, bias, C, ldc, M, N, K, act, splits, workspace,
                   use_tma ? 4 : 2, ga, colstats, mgx::as_stream(stream));
}

extern "C" int mgx_gemm_bf16_tc(const void* A, int64_t lda, const void* B, int64_t ldb,
                                const float* bias, float* C, int64_t ldc, int64_t M, int64_t N,
                                int64_t K, int act, uintptr_t stream) {
  return mgx_gemm_bf16_tc_ex(A, lda, 0, B, ldb, 0, bias, C, ldc, M, N, K, act, 1, nullptr, nullptr,
                             stream);
}

extern "C" int mgx_gemm_split_plan(int64_t M, int64_t N, int64_t K, int32_t target,
                                   int32_t* splits_out, int64_t* out_floats) {
  using namespace mgx::tc;
  MGX_REQUIRE(splits_out && out_floats && M > 0 && N > 0 && K > 0,
              "mgx_gemm_split_plan: bad arguments");
  const int64_t tiles = mgx::ceil_div(N, pick_bn(M, N)) * mgx::ceil_div(M, BM);
  const int64_t nk = mgx::ceil_div(K, BK);
  int64_t splits = auto_splits(tiles, nk, target);
  if (splits > 1) {
    const int64_t kps = mgx::ceil_div(nk, splits);
    splits = mgx::ceil_div(nk, kps);
  }
  *splits_out = static_cast<int32_t>(splits);
  *out_floats = splits > 1 ? splits * M * N : 0;
  return MGX_OK;
}

extern "C" int mgx_gemm_splitk_workspace(int64_t M, int64_t N, int64_t K, int64_t* out_floats) {
  int32_t splits = 1;
  return mgx_gemm_split_plan(M, N, K, 0, &splits, out_floats);
}

extern "C" int mgx_cast_bf16_2d(const float* x, int64_t R, int64_t C, int64_t ldi, void* y,
                                int64_t rows, int64_t ldo, int transpose, uintptr_t stream) {
  MGX_REQUIRE(x && y && R > 0 && C > 0 && rows > 0 && ldo > 0, "mgx_cast_bf16_2d: bad arguments");
  MGX_REQUIRE(transpose ? (rows >= C && ldo >= R) : (rows >= R && ldo >= C),
              "mgx_cast_bf16_2d: destination smaller than the source");
  cudaStream_t st = mgx::as_stream(stream);
  if (!transpose && ldo % 8 == 0 && mgx::aligned16(y)) {
    mgx::tc::cast_rows_kernel<<<mgx::rows_grid(rows, ldo / 8), mgx::rows_block(ldo / 8), 0, st>>>(
        x, R, C, ldi, static_cast<__nv_bfloat16*>(y), rows, ldo);
  } else if (!transpose) {
    MGX_REQUIRE(false, "mgx_cast_bf16_2d: ldo must be a multiple of 8 and y 16-byte aligned");
  } else {
    dim3 grid(static_cast<unsigned>(mgx::ceil_div(rows, 32)),
              static_cast<unsigned>(mgx::ceil_div(ldo, 32)));
    mgx::tc::cast_transpose_kernel<<<grid, dim3(32, 8), 0, st>>>(
        x, R, C, ldi, static_cast<__nv_bfloat16*>(y), rows, ldo);
  }
  MGX_LAUNCHED();
  return MGX_OK;
}

extern "C" int mgx_cast_f32_bf16(const float* x, void* y, int64_t n, uintptr_t stream) {
  MGX_REQUIRE(n >= 0 && (n == 0 || (x && y)), "mgx_cast_f32_bf16: bad arguments");
  if (n == 0) return MGX_OK;
  int64_t blocks = mgx::ceil_div(n, 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  mgx::tc::cast_f32_bf16_kernel<<<static_cast<unsigned>(blocks), 256, 0, mgx::as_stream(stream)>>>(
      x, static_cast<__nv_bfloat16*>(y), n);
  MGX_LAUNCHED();
  return MGX_OK;
}
