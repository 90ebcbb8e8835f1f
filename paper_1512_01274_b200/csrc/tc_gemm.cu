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

// instruction descriptor kind::f16: D f32, A/B bf16, both K-major, M128 N128
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((BN >> 3) << 17) | ((BM >> 4) << 24);

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(kIdesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__global__ void __launch_bounds__(128, 1)
tc_gemm_bf16_kernel(const __grid_constant__ CUtensorMap map_a,
                    const __grid_constant__ CUtensorMap map_b, const float* __restrict__ bias,
                    float* __restrict__ C, int ldc, int M, int N, int K, int act) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte aligned stage ring (SW128 atoms need it)
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * kStageBytes);
  uint64_t* empty = full + STAGES;
  uint64_t* done = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int nk = (K + BK - 1) / BK;

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
      tma_load_2d(sa, &map_a, &full[s], kb * BK, m0);
      tma_load_2d(sa + kTileBytes, &map_b, &full[s], kb * BK, n0);
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % STAGES;
      const uint32_t ph = (kb / STAGES) & 1;
      mbar_wait(&full[s], ph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint8_t* sa = smem + s * kStageBytes;
      const uint64_t adesc = smem_desc_sw128(sa);
      const uint64_t bdesc = smem_desc_sw128(sa + kTileBytes);
#pragma unroll
      for (int k = 0; k < BK / UMMA_K; ++k) {
        // +32 bytes per K16 step inside the 128-byte swizzle row (>>4 -> +2)
        umma_bf16(tmem, adesc + 2 * k, bdesc + 2 * k, (kb > 0 || k > 0) ? 1u : 0u);
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

static int make_map(CUtensorMap* map, const void* base, int64_t rows, int64_t K, int64_t ld) {
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * 2)};
  cuuint32_t box[2] = {BK, BM};
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

}  // namespace tc
}  // namespace mgx

extern "C" int mgx_gemm_bf16_tc(const void* A, int64_t lda, const void* B, int64_t ldb,
                                const float* bias, float* C, int64_t ldc, int64_t M, int64_t N,
                                int64_t K, int act, uintptr_t stream) {
  using namespace mgx::tc;
  MGX_REQUIRE(A && B && C && M > 0 && N > 0 && K > 0, "mgx_gemm_bf16_tc: bad arguments");
  MGX_REQUIRE(K % 8 == 0 && lda % 8 == 0 && ldb % 8 == 0,
              "mgx_gemm_bf16_tc: K and leading dimensions must be multiples of 8");
  MGX_REQUIRE(mgx::aligned16(A) && mgx::aligned16(B), "mgx_gemm_bf16_tc: operands not 16-byte aligned");
  MGX_REQUIRE(M < (1ll << 31) && N < (1ll << 31) && K < (1ll << 31) && ldc < (1ll << 31),
              "mgx_gemm_bf16_tc: dimensions exceed 2^31");
  MGX_TRY(get_encode());
  CUtensorMap ma, mb;
  MGX_TRY(make_map(&ma, A, M, K, lda));
  MGX_TRY(make_map(&mb, B, N, K, ldb));
  static bool configured = false;
  if (!configured) {
    MGX_CUDA(cudaFuncSetAttribute(tc_gemm_bf16_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  kSmemBytes));
    configured = true;
  }
  dim3 grid(static_cast<unsigned>(mgx::ceil_div(N, BN)), static_cast<unsigned>(mgx::ceil_div(M, BM)));
  tc_gemm_bf16_kernel<<<grid, 128, kSmemBytes, mgx::as_stream(stream)>>>(
      ma, mb, bias, C, static_cast<int>(ldc), static_cast<int>(M), static_cast<int>(N),
      static_cast<int>(K), act);
  MGX_LAUNCHED();
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
