// Exact-order fp32 dense kernels for FullyConnected / MatMul.
//
// The reference computes every contraction with numpy broadcast-multiply +
// add.reduce (kernels.py:20-29) and batch reductions with a balanced
// power-of-two tree (kernels.py:32-47).  These kernels reproduce those
// reduction orders bit-for-bit (products rounded, adds rounded, no FMA):
//
//   gemm_pairwise   C = pairwise_k(A[m,k]*B[n,k])     FC forward (ops.py:102-106),
//                                                     MatMul backward slot 0
//   gemm_sequential C = sequential_k(A[m,k]*B[k,n])   FC dX (ops.py:111-112),
//                                                     MatMul forward/bwd slot 1
//   fc_dw_db        dW = tree_b(og[b,h]*x[b,f]), db = tree_b(og[b,h])
//                                                     FC dW/db (ops.py:113-116)
//
// numpy pairwise_sum (the order of add.reduce over a contiguous axis) for n
// elements: n < 8 -> sequential from +0; n <= 128 -> 8 strided accumulators
// r[j] = a[j] + a[j+8] + ..., combined ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)),
// then the n%8 tail added sequentially; n > 128 -> split at
// n2 = n/2 - (n/2)%8 and recurse.  The split tree depends only on n, so the
// host precomputes its leaves once per K (start, length, merges-after) and
// every kernel thread walks the same leaf list.
//
// Lane mapping: a group of 8 consecutive lanes computes one micro-tile of
// outputs; lane j holds accumulator r[j] for every output of the tile, and
// an xor-butterfly over the 8 lanes (masks 1,2,4) produces exactly
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) because each add is commutative.

#include <mutex>
#include <unordered_map>
#include <vector>

#include "common.cuh"

namespace mgx {

// ---------------------------------------------------------------- host side

static void pw_leaves_rec(int64_t s, int64_t n, std::vector<PwLeaf>& out) {
  if (n <= 128) {
    out.push_back(PwLeaf{static_cast<int32_t>(s), static_cast<int32_t>(n), 0, 0});
    return;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  pw_leaves_rec(s, n2, out);
  pw_leaves_rec(s + n2, n - n2, out);
  out.back().merges += 1;
}

std::vector<PwLeaf> pairwise_leaves(int64_t n) {
  std::vector<PwLeaf> out;
  if (n > 0) pw_leaves_rec(0, n, out);
  return out;
}

// Device copies of leaf tables, one per (device, K); small and immutable.
static std::mutex g_leaf_mu;
static std::unordered_map<int64_t, PwLeaf*> g_leaf_tables;

// Chunks of consecutive whole leaves spanning at most kPwChunk elements
// (the pairwise GEMM stages one chunk of K in shared memory at a time).
constexpr int kPwChunk = 512;

static std::vector<PwLeaf> pairwise_chunks(const std::vector<PwLeaf>& leaves) {
  std::vector<PwLeaf> chunks;  // {k0, klen, leaf_begin, leaf_end}
  size_t l = 0;
  while (l < leaves.size()) {
    const int32_t k0 = leaves[l].start;
    size_t e = l;
    while (e < leaves.size() && leaves[e].start + leaves[e].len - k0 <= kPwChunk) ++e;
    if (e == l) ++e;  // a single leaf is at most 128 elements
    chunks.push_back(PwLeaf{k0, leaves[e - 1].start + leaves[e - 1].len - k0,
                            static_cast<int32_t>(l), static_cast<int32_t>(e)});
    l = e;
  }
  return chunks;
}

int pw_leaf_table(int64_t K, const PwLeaf** out, int* nleaves, int* max_depth, int* nchunks) {
  auto leaves = pairwise_leaves(K);
  auto chunks = pairwise_chunks(leaves);
  int depth = 0, cur = 0;
  for (auto& l : leaves) {
    ++cur;
    depth = depth > cur ? depth : cur;
    cur -= l.merges;
  }
  *nleaves = static_cast<int>(leaves.size());
  *max_depth = depth;
  if (nchunks) *nchunks = static_cast<int>(chunks.size());
  int dev = 0;
  MGX_CUDA(cudaGetDevice(&dev));
  int64_t key = (static_cast<int64_t>(dev) << 48) | K;
  std::lock_guard<std::mutex> lock(g_leaf_mu);
  auto it = g_leaf_tables.find(key);
  if (it != g_leaf_tables.end()) {
    *out = it->second;
    return MGX_OK;
  }
  std::vector<PwLeaf> table(leaves);
  table.insert(table.end(), chunks.begin(), chunks.end());
  PwLeaf* d = nullptr;
  size_t bytes = table.size() * sizeof(PwLeaf);
  MGX_CUDA(cudaMalloc(&d, bytes > 0 ? bytes : sizeof(PwLeaf)));
  // Plain synchronous copy: done once per (device, K), before any capture.
  MGX_CUDA(cudaMemcpy(d, table.data(), bytes, cudaMemcpyHostToDevice));
  // a pageable H2D copy may return before the DMA lands; kernels read the
  // table from non-blocking streams
  MGX_CUDA(cudaDeviceSynchronize());
  g_leaf_tables[key] = d;
  *out = d;
  return MGX_OK;
}

}  // namespace mgx

#include "tiles.cuh"

namespace mgx {

template <int TM, int TN, int D>
__global__ void __launch_bounds__(kPwThreads)
gemm_pairwise_kernel(const float* __restrict__ A, int lda, const float* __restrict__ B, int ldb,
                     const float* __restrict__ bias, float* __restrict__ C, int ldc, int M, int N,
                     int K, const PwLeaf* __restrict__ leaves, int nleaves, int nchunks, int act,
                     int kc, bool vecA, bool vecB) {
  extern __shared__ float4 smem_f4[];
  pw_tile<TM, TN, D>(blockIdx.x, blockIdx.y, reinterpret_cast<float*>(smem_f4), A, lda, B, ldb,
                     bias, C, ldc, M, N, K, leaves, nleaves, nchunks, act, kc, vecA, vecB);
}

__global__ void __launch_bounds__(256)
gemm_sequential_kernel(const float* __restrict__ A, int64_t sam, int64_t sak,
                       const float* __restrict__ B, int64_t sbk, int64_t sbn,
                       float* __restrict__ C, int64_t ldc, const float* __restrict__ Y,
                       int act, int64_t M, int64_t N, int64_t K) {
  extern __shared__ float4 smem_f4[];
  seq_tile(blockIdx.x, blockIdx.y, reinterpret_cast<float*>(smem_f4), A, sam, sak, B, sbk, sbn, C,
           ldc, Y, act, M, N, K);
}

template <int LV>
__global__ void __launch_bounds__(256)
fc_dw_db_kernel(const float* __restrict__ og, const float* __restrict__ x, float* __restrict__ dw,
                float* __restrict__ db, int64_t Bn, int64_t H, int64_t F, bool vecO, bool vecX) {
  extern __shared__ float4 smem_f4[];
  dw_tile<LV>(blockIdx.x, blockIdx.y, reinterpret_cast<float*>(smem_f4), og, x, dw, db, Bn, H, F,
              vecO, vecX);
}

int launch_dw_db(const float* og, const float* x, float* dw, float* db, int64_t Bn, int64_t H,
                 int64_t F, cudaStream_t st) {
  const int64_t nch = Bn >> 3;
  dim3 grid(static_cast<unsigned>(dw ? ceil_div(F, kDwBF) : 1),
            static_cast<unsigned>(ceil_div(H, kDwBH)));
  const bool vecO = (H % 4 == 0) && aligned16(og);
  const bool vecX = dw && (F % 4 == 0) && aligned16(x);
  if (nch < (1 << 4)) {
    fc_dw_db_kernel<4><<<grid, 256, kDwSmemFloats * 4, st>>>(og, x, dw, db, Bn, H, F, vecO, vecX);
  } else if (nch < (1 << 10)) {
    fc_dw_db_kernel<10><<<grid, 256, kDwSmemFloats * 4, st>>>(og, x, dw, db, Bn, H, F, vecO, vecX);
  } else if (nch < (1 << 20)) {
    fc_dw_db_kernel<20><<<grid, 256, kDwSmemFloats * 4, st>>>(og, x, dw, db, Bn, H, F, vecO, vecX);
  } else {
    set_error("batch tree: %lld rows exceed the supported 2^23", static_cast<long long>(Bn));
    return MGX_BAD_ARGUMENT;
  }
  MGX_LAUNCHED();
  return MGX_OK;
}

template <int TM, int TN, int D>
static int pw_launch(dim3 grid, size_t smem, cudaStream_t st, const float* A, int64_t lda,
                     const float* B, int64_t ldb, const float* bias, float* C, int64_t ldc,
                     int64_t M, int64_t N, int64_t K, const PwLeaf* leaves, int nleaves,
                     int nchunks, int act, int kc, bool vecA, bool vecB) {
  static bool configured[8] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!configured[dev & 7]) {
    MGX_CUDA(cudaFuncSetAttribute(gemm_pairwise_kernel<TM, TN, D>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  2 * (4 * TM + 8 * TN) * (kPwChunk + 4) * 4));
    configured[dev & 7] = true;
  }
  gemm_pairwise_kernel<TM, TN, D><<<grid, kPwThreads, smem, st>>>(
      A, static_cast<int>(lda), B, static_cast<int>(ldb), bias, C, static_cast<int>(ldc),
      static_cast<int>(M), static_cast<int>(N), static_cast<int>(K), leaves, nleaves, nchunks,
      act, kc, vecA, vecB);
  MGX_LAUNCHED();
  return MGX_OK;
}

int launch_gemm_pairwise(const float* A, int64_t lda, const float* B, int64_t ldb,
                         const float* bias, float* C, int64_t ldc, int64_t M, int64_t N,
                         int64_t K, int act, cudaStream_t st) {
  const PwLeaf* leaves = nullptr;
  int nleaves = 0, depth = 0, nchunks = 0;
  MGX_TRY(pw_leaf_table(K, &leaves, &nleaves, &depth, &nchunks));
  MGX_REQUIRE(M < (int64_t(1) << 31) && N < (int64_t(1) << 31) && K < (int64_t(1) << 31) &&
                  lda < (int64_t(1) << 31) && ldb < (int64_t(1) << 31) && ldc < (int64_t(1) << 31),
              "pairwise GEMM: dimensions exceed 2^31");
  constexpr int TM = 2, TN = 2;
  const int kc = static_cast<int>(K >= kPwChunk ? kPwChunk : ((K + 7) / 8) * 8);
  const bool vecA = (lda % 4 == 0) && (K % 4 == 0) && aligned16(A);
  const bool vecB = (ldb % 4 == 0) && (K % 4 == 0) && aligned16(B);
  const size_t smem = size_t(2) * (4 * TM + 8 * TN) * (kc + 4) * sizeof(float);
  dim3 grid(static_cast<unsigned>(ceil_div(N, 8 * TN)), static_cast<unsigned>(ceil_div(M, 4 * TM)));
#define MGX_PW(Dd) \
  return pw_launch<TM, TN, Dd>(grid, smem, st, A, lda, B, ldb, bias, C, ldc, M, N, K, leaves, \
                               nleaves, nchunks, act, kc, vecA, vecB)
  if (depth <= 1) MGX_PW(1);
  if (depth <= 6) MGX_PW(6);
  if (depth <= 12) MGX_PW(12);
  if (depth <= kPwMaxDepth) MGX_PW(kPwMaxDepth);
#undef MGX_PW
  set_error("pairwise GEMM: K=%lld too deep", static_cast<long long>(K));
  return MGX_BAD_ARGUMENT;
}

int launch_gemm_sequential(const float* A, int64_t sam, int64_t sak, const float* B, int64_t sbk,
                           int64_t sbn, float* C, int64_t ldc, const float* Y, int act, int64_t M,
                           int64_t N, int64_t K, cudaStream_t st) {
  dim3 grid(static_cast<unsigned>(ceil_div(N, kSeqBN)), static_cast<unsigned>(ceil_div(M, kSeqBM)));
  gemm_sequential_kernel<<<grid, 256, kSeqSmemFloats * 4, st>>>(A, sam, sak, B, sbk, sbn, C, ldc, Y, act, M, N, K);
  MGX_LAUNCHED();
  return MGX_OK;
}

}  // namespace mgx

// ------------------------------------------------------------------ C-ABI

extern "C" int mgx_gemm_pairwise(const float* A, int64_t lda, const float* B, int64_t ldb,
                                 const float* bias, float* C, int64_t ldc, int64_t M, int64_t N,
                                 int64_t K, int act, uintptr_t stream) {
  MGX_REQUIRE(A && B && C && M > 0 && N > 0 && K > 0, "mgx_gemm_pairwise: bad arguments");
  MGX_REQUIRE(K < (int64_t(1) << 31), "mgx_gemm_pairwise: K too large");
  return mgx::launch_gemm_pairwise(A, lda, B, ldb, bias, C, ldc, M, N, K, act,
                                   mgx::as_stream(stream));
}

extern "C" int mgx_gemm_sequential(const float* A, int64_t sam, int64_t sak, const float* B,
                                   int64_t sbk, int64_t sbn, float* C, int64_t ldc,
                                   const float* Y, int act, int64_t M, int64_t N, int64_t K,
                                   uintptr_t stream) {
  MGX_REQUIRE(A && B && C && M > 0 && N > 0 && K > 0, "mgx_gemm_sequential: bad arguments");
  MGX_REQUIRE(act == MGX_ACT_NONE || Y, "mgx_gemm_sequential: fused activation needs Y");
  return mgx::launch_gemm_sequential(A, sam, sak, B, sbk, sbn, C, ldc, Y, act, M, N, K,
                                     mgx::as_stream(stream));
}

extern "C" int mgx_fc_dw_db(const float* og, const float* x, float* dw, float* db, int64_t B,
                            int64_t H, int64_t F, uintptr_t stream) {
  MGX_REQUIRE(og && B > 0 && H > 0, "mgx_fc_dw_db: bad arguments");
  MGX_REQUIRE(!dw || (x && F > 0), "mgx_fc_dw_db: dW needs x and F > 0");
  if (!dw && !db) return MGX_OK;
  return mgx::launch_dw_db(og, x, dw, db, B, H, dw ? F : 1, mgx::as_stream(stream));
}

extern "C" int mgx_tree_sum_rows(const float* a, float* out, int64_t rows, int64_t cols,
                                 uintptr_t stream) {
  MGX_REQUIRE(a && out && rows > 0 && cols > 0, "mgx_tree_sum_rows: bad arguments");
  return mgx::launch_dw_db(a, nullptr, nullptr, out, rows, cols, 1, mgx::as_stream(stream));
}
