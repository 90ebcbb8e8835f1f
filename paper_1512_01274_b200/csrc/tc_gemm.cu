// tcgen05 tensor-core GEMM for the bf16 dense path (sm_100a).
//
//   C[M,N] (fp32) = A[M,K] . B[N,K]^T (+ bias[N]) then activation
//
// A and B are bf16, K-major ("TN": FC forward x[B,F] . w[H,F]^T), the
// accumulator is fp32 in tensor memory.  One 128x128 output tile per CTA,
// 4 warps:
//   warp 0 (one lane)  TMA producer: 128B-swizzled 128x64 bf16 tiles of A and
//                      B into a 4-stage shared-memory ring (mbarrier tx)
//   warp 1 (one lane)  MMA issuer: 4 x tcgen05.mma.kind::f16 (M128 N128 K16)
//                      per stage, tcgen05.commit frees the stage
//   warps 0-3          epilogue: tcgen05.ld 32 lanes x 16 columns at a time,
//                      bias + activation, fp32 stores
// This is the tolerance path (bf16 operands, fp32 accumulate in hardware
// order): used for the large FC layers of configs 3-5, never for the
// exact-order fp32 parity path.

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>

#include <mutex>

#include "common.cuh"

namespace mgx {
namespace tc {

constexpr int BM = 128, BN = 128, BK = 64, STAGES = 4, UMMA_K = 16;
constexpr int kTileBytes = BM * BK * 2;               // 16 KB (A or B)
constexpr int kStageBytes = 2 * kTileBytes;            // 32 KB
constexpr int kSmemBytes = STAGES * kStageBytes + 1024 + 256;

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
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
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// tcgen05 shared-memory matrix descriptor: K-major, 128-byte swizzle,
// 8-row swizzle atoms 1024 bytes apart (SBO), version 1 (bit 46).
__device__ __forceinline__ uint64_t smem_desc_sw128(const void* p) {
  const uint64_t addr = smem_u32(p);
  uint64_t d = 0;
  d |= (addr >> 4) & 0x3FFFull;          // start address
  d |= (uint64_t(0) & 0x3FFF) << 16;     // LBO (unused for swizzled K-major)
  d |= (uint64_t(1024 >> 4) & 0x3FFF) << 32;  // SBO
  d |= uint64_t(1) << 46;                // fixed 0b001
  d |= uint64_t(2) << 61;                // SWIZZLE_128B
  return d;
}

// tcgen05 shared-memory matrix descriptor, MN-major, 128-byte swizzle:
// 64-element (128 B) MN rows, K rows 128 B apart; 8-row K groups 1024 B
// apart (SBO); 64-wide MN chunks kMnChunkBytes apart (LBO).
constexpr int kMnChunkBytes = BK * 128;  // one TMA box: 64 K rows x 128 B
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

// instruction descriptor kind::f16: D f32, A/B bf16, M128 N128; bit 15 / 16
// select an MN-major A / B operand
template <bool A_MN, bool B_MN>
constexpr uint32_t idesc() {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((A_MN ? 1u : 0u) << 15) | ((B_MN ? 1u : 0u) << 16) |
         ((BN >> 3) << 17) | ((BM >> 4) << 24);
}

template <bool A_MN, bool B_MN>
__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc<A_MN, B_MN>()), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

// one 128-row x 64-K operand tile into `dst`: a single K-major box, or two
// MN-major boxes (MN 0..63, 64..127) stacked kMnChunkBytes apart
template <bool MN>
__device__ __forceinline__ void load_operand(uint8_t* dst, const CUtensorMap* map, uint64_t* bar,
                                             int k0, int r0) {
  if (!MN) {
    tma_load_2d(dst, map, bar, k0, r0);
  } else {
    tma_load_2d(dst, map, bar, r0, k0);
    tma_load_2d(dst + kMnChunkBytes, map, bar, r0 + 64, k0);
  }
}

// C[M,N] (+bias, act) = sum_k A(m,k) B(n,k).  K-major operand X: X[r*ld + k];
// MN-major: X[k*ld + r].  Split-K: blockIdx.z takes K blocks
// [z*kps, (z+1)*kps) and writes its partial tile to C + z*split_stride.
template <bool A_MN, bool B_MN>
__global__ void __launch_bounds__(128, 1)
tc_gemm_bf16_kernel(const __grid_constant__ CUtensorMap map_a,
                    const __grid_constant__ CUtensorMap map_b, const float* __restrict__ bias,
                    float* __restrict__ C, int ldc, int M, int N, int K, int act, int kps,
                    int64_t split_stride) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte aligned stage ring (SW128 atoms need it)
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * kStageBytes);
  uint64_t* empty = full + STAGES;
  uint64_t* done = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int nk_all = (K + BK - 1) / BK;
  const int kb0 = blockIdx.z * kps;
  const int nk = min(nk_all, kb0 + kps) - kb0;
  C += int64_t(blockIdx.z) * split_stride;

  if (threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % STAGES;
      const uint32_t ph = (kb / STAGES) & 1;
      mbar_wait(&empty[s], ph ^ 1);
      uint8_t* sa = smem + s * kStageBytes;
      mbar_expect_tx(&full[s], kStageBytes);
      load_operand<A_MN>(sa, &map_a, &full[s], (kb0 + kb) * BK, m0);
      load_operand<B_MN>(sa + kTileBytes, &map_b, &full[s], (kb0 + kb) * BK, n0);
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % STAGES;
      const uint32_t ph = (kb / STAGES) & 1;
      mbar_wait(&full[s], ph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint8_t* sa = smem + s * kStageBytes;
      const uint64_t adesc = A_MN ? smem_desc_mn_sw128(sa) : smem_desc_sw128(sa);
      const uint64_t bdesc = B_MN ? smem_desc_mn_sw128(sa + kTileBytes) : smem_desc_sw128(sa + kTileBytes);
#pragma unroll
      for (int k = 0; k < BK / UMMA_K; ++k) {
        // K-major: +32 bytes per K16 step inside the 128-byte swizzle row
        // (>>4 -> +2); MN-major: +16 K rows of 128 bytes (>>4 -> +128)
        const uint64_t da = A_MN ? 128ull * k : 2ull * k;
        const uint64_t db = B_MN ? 128ull * k : 2ull * k;
        umma_bf16<A_MN, B_MN>(tmem, adesc + da, bdesc + db, (kb > 0 || k > 0) ? 1u : 0u);
      }
      umma_commit(&empty[s]);
    }
    umma_commit(done);
  }
  __syncwarp();

  // ---------------- epilogue: all 4 warps, warp w owns TMEM lanes 32w..32w+31
  mbar_wait(done, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int row = m0 + warp * 32 + lane;
  for (int c0 = 0; c0 < BN; c0 += 16) {
    uint32_t r[16];
    const uint32_t taddr = tmem + (uint32_t(warp * 32) << 16) + uint32_t(c0);
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (row < M) {
      float* crow = C + int64_t(row) * ldc;
      if (nk <= 0) {
#pragma unroll
        for (int j = 0; j < 16; ++j) r[j] = 0u;  // empty split: contributes zeros
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int n = n0 + c0 + j;
        if (n < N) {
          float v = __uint_as_float(r[j]);
          if (bias) v = fadd(v, __ldg(bias + n));
          crow[n] = act_forward(act, v);
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(BN));
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

// y (bf16, rows x ldo) = x (fp32, R x C, row stride ldi), optionally
// transposed (y is C x ldo then), zero-filled beyond the source extent so the
// padded K columns contribute nothing to the tensor-core contraction.
__global__ void cast_2d_kernel(const float* __restrict__ x, int64_t R, int64_t C, int64_t ldi,
                               __nv_bfloat16* __restrict__ y, int64_t rows, int64_t ldo,
                               int transpose) {
  const int64_t n = rows * ldo;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int64_t r = i / ldo, c = i - r * ldo;
    float v = 0.0f;
    if (!transpose) {
      if (r < R && c < C) v = x[r * ldi + c];
    } else {
      if (c < R && r < C) v = x[c * ldi + r];
    }
    y[i] = __float2bfloat16_rn(v);
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

// K-major operand: dims {K, rows}, box {64, 128}; MN-major: dims {rows, K}
// (rows contiguous), box {64, 64} (loaded twice per 128-row tile)
static int make_map(CUtensorMap* map, const void* base, int64_t rows, int64_t K, int64_t ld,
                    bool mn) {
  cuuint64_t dims[2];
  cuuint32_t box[2];
  if (!mn) {
    dims[0] = static_cast<cuuint64_t>(K);
    dims[1] = static_cast<cuuint64_t>(rows);
    box[0] = BK;
    box[1] = BM;
  } else {
    dims[0] = static_cast<cuuint64_t>(rows);
    dims[1] = static_cast<cuuint64_t>(K);
    box[0] = 64;
    box[1] = BK;
  }
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * 2)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d)", static_cast<int>(r));
    return MGX_INTERNAL;
  }
  return MGX_OK;
}

template <bool A_MN, bool B_MN>
static int launch_variant(const CUtensorMap& ma, const CUtensorMap& mb, dim3 grid,
                          const float* bias, float* C, int ldc, int M, int N, int K, int act,
                          int kps, int64_t split_stride, cudaStream_t st) {
  static bool configured = false;
  if (!configured) {
    MGX_CUDA(cudaFuncSetAttribute(tc_gemm_bf16_kernel<A_MN, B_MN>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes));
    configured = true;
  }
  tc_gemm_bf16_kernel<A_MN, B_MN><<<grid, 128, kSmemBytes, st>>>(ma, mb, bias, C, ldc, M, N, K,
                                                                   act, kps, split_stride);
  MGX_LAUNCHED();
  return MGX_OK;
}

}  // namespace tc
}  // namespace mgx

extern "C" int mgx_gemm_bf16_tc_ex(const void* A, int64_t lda, int a_mn, const void* B,
                                   int64_t ldb, int b_mn, const float* bias, float* C, int64_t ldc,
                                   int64_t M, int64_t N, int64_t K, int act, int splits,
                                   float* workspace, uintptr_t stream) {
  using namespace mgx::tc;
  MGX_REQUIRE(A && B && C && M > 0 && N > 0 && K > 0, "mgx_gemm_bf16_tc: bad arguments");
  MGX_REQUIRE(lda % 8 == 0 && ldb % 8 == 0,
              "mgx_gemm_bf16_tc: leading dimensions must be multiples of 8");
  MGX_REQUIRE(lda >= (a_mn ? M : K) && ldb >= (b_mn ? N : K),
              "mgx_gemm_bf16_tc: leading dimension smaller than the operand row");
  MGX_REQUIRE(mgx::aligned16(A) && mgx::aligned16(B), "mgx_gemm_bf16_tc: operands not 16-byte aligned");
  MGX_REQUIRE(M < (1ll << 31) && N < (1ll << 31) && K < (1ll << 31) && ldc < (1ll << 31),
              "mgx_gemm_bf16_tc: dimensions exceed 2^31");
  MGX_REQUIRE(splits >= 0, "mgx_gemm_bf16_tc: negative split count");
  MGX_TRY(get_encode());
  CUtensorMap ma, mb;
  MGX_TRY(make_map(&ma, A, M, K, lda, a_mn != 0));
  MGX_TRY(make_map(&mb, B, N, K, ldb, b_mn != 0));
  const int64_t tiles = mgx::ceil_div(N, BN) * mgx::ceil_div(M, BM);
  const int64_t nk = mgx::ceil_div(K, BK);
  if (splits == 0) {
    // auto: enough K splits to cover the SMs once, each split >= 4 K blocks
    splits = 1;
    if (workspace && tiles < mgx::kNumSMs) {
      int64_t want = mgx::kNumSMs / tiles;
      int64_t most = nk / 4;
      splits = static_cast<int>(want < most ? want : most);
      if (splits < 1) splits = 1;
    }
  }
  MGX_REQUIRE(splits == 1 || workspace, "mgx_gemm_bf16_tc: split-K needs a workspace");
  int kps = static_cast<int>(mgx::ceil_div(nk, splits));
  splits = static_cast<int>(mgx::ceil_div(nk, kps));
  dim3 grid(static_cast<unsigned>(mgx::ceil_div(N, BN)), static_cast<unsigned>(mgx::ceil_div(M, BM)),
            static_cast<unsigned>(splits));
  cudaStream_t st = mgx::as_stream(stream);
  float* out = splits == 1 ? C : workspace;
  const int64_t sstride = M * N;
  const int oldc = splits == 1 ? static_cast<int>(ldc) : static_cast<int>(N);
  const float* ebias = splits == 1 ? bias : nullptr;
  const int eact = splits == 1 ? act : 0;
  const int m = static_cast<int>(M), n = static_cast<int>(N), k = static_cast<int>(K);
  int rc;
  if (!a_mn && !b_mn) rc = launch_variant<false, false>(ma, mb, grid, ebias, out, oldc, m, n, k, eact, kps, sstride, st);
  else if (!a_mn && b_mn) rc = launch_variant<false, true>(ma, mb, grid, ebias, out, oldc, m, n, k, eact, kps, sstride, st);
  else if (a_mn && !b_mn) rc = launch_variant<true, false>(ma, mb, grid, ebias, out, oldc, m, n, k, eact, kps, sstride, st);
  else rc = launch_variant<true, true>(ma, mb, grid, ebias, out, oldc, m, n, k, eact, kps, sstride, st);
  if (rc != MGX_OK || splits == 1) return rc;
  int64_t blocks = mgx::ceil_div(M * N, 256);
  if (blocks > 148 * 8) blocks = 148 * 8;
  splitk_reduce_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(workspace, splits, sstride,
                                                                      bias, C, ldc, M, N, act);
  MGX_LAUNCHED();
  return MGX_OK;
}

extern "C" int mgx_gemm_bf16_tc(const void* A, int64_t lda, const void* B, int64_t ldb,
                                const float* bias, float* C, int64_t ldc, int64_t M, int64_t N,
                                int64_t K, int act, uintptr_t stream) {
  return mgx_gemm_bf16_tc_ex(A, lda, 0, B, ldb, 0, bias, C, ldc, M, N, K, act, 1, nullptr, stream);
}

extern "C" int mgx_gemm_splitk_workspace(int64_t M, int64_t N, int64_t K, int64_t* out_floats) {
  using namespace mgx::tc;
  MGX_REQUIRE(out_floats && M > 0 && N > 0 && K > 0, "mgx_gemm_splitk_workspace: bad arguments");
  const int64_t tiles = mgx::ceil_div(N, BN) * mgx::ceil_div(M, BM);
  const int64_t nk = mgx::ceil_div(K, BK);
  int64_t splits = 1;
  if (tiles < mgx::kNumSMs) {
    int64_t want = mgx::kNumSMs / tiles, most = nk / 4;
    splits = want < most ? want : most;
    if (splits < 1) splits = 1;
  }
  *out_floats = splits > 1 ? splits * M * N : 0;
  return MGX_OK;
}

extern "C" int mgx_cast_bf16_2d(const float* x, int64_t R, int64_t C, int64_t ldi, void* y,
                                int64_t rows, int64_t ldo, int transpose, uintptr_t stream) {
  MGX_REQUIRE(x && y && R > 0 && C > 0 && rows > 0 && ldo > 0, "mgx_cast_bf16_2d: bad arguments");
  MGX_REQUIRE(transpose ? (rows >= C && ldo >= R) : (rows >= R && ldo >= C),
              "mgx_cast_bf16_2d: destination smaller than the source");
  int64_t blocks = mgx::ceil_div(rows * ldo, 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  mgx::tc::cast_2d_kernel<<<static_cast<unsigned>(blocks), 256, 0, mgx::as_stream(stream)>>>(
      x, R, C, ldi, static_cast<__nv_bfloat16*>(y), rows, ldo, transpose);
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
