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
  g_leaf_tables[key] = d;
  *out = d;
  return MGX_OK;
}

// --------------------------------------------------------- tile staging
// Copy rows [r0, r0+R) x cols [c0, c0+kc) of a row-major matrix (row stride
// ld, K valid columns, nrows valid rows) into smem S[R][kcp] with cp.async.
// Out-of-range elements are zero-filled.  `vec` = 16-byte copies (needs ld,
// c0, K multiples of 4 and an aligned base).
__device__ __forceinline__ void stage_rows(float* S, int kcp, const float* G, int64_t ld,
                                           int64_t r0, int R, int64_t nrows, int64_t c0, int kc,
                                           int64_t K, bool vec) {
  if (vec) {
    const int per_row = kc >> 2;
    for (int e = threadIdx.x; e < R * per_row; e += blockDim.x) {
      const int r = e / per_row, c = (e - r * per_row) << 2;
      const int64_t gr = r0 + r, gc = c0 + c;
      const bool ok = gr < nrows && gc < K;
      cp_async16(S + r * kcp + c, ok ? G + gr * ld + gc : G, ok);
    }
  } else {
    for (int e = threadIdx.x; e < R * kc; e += blockDim.x) {
      const int r = e / kc, c = e - r * kc;
      const int64_t gr = r0 + r, gc = c0 + c;
      const bool ok = gr < nrows && gc < K;
      cp_async4(S + r * kcp + c, ok ? G + gr * ld + gc : G, ok);
    }
  }
}

// ----------------------------------------------------- pairwise GEMM kernel
// Block tile (4*TM) x (8*TN) outputs; 32 groups of 8 lanes, group (gm, gn)
// owns a TM x TN micro-tile and lane j of the group is numpy's accumulator
// r[j].  K is staged through shared memory one chunk of whole leaves at a
// time (<= 512 elements, cp.async, double-buffered).  Per leaf the 8-block
// loop is branch-free; leaf results merge on a D-deep stack held in
// registers (predicated updates, no local memory) per the split tree.

constexpr int kPwThreads = 256;
constexpr int kPwMaxDepth = 24;

template <int D, int T>
struct LeafStack {
  // shift register: v[0] is the top; every index is static, so the stack
  // lives in registers
  float v[D][T];
  __device__ __forceinline__ void push(const float (&x)[T]) {
#pragma unroll
    for (int d = D - 1; d > 0; --d)
#pragma unroll
      for (int o = 0; o < T; ++o) v[d][o] = v[d - 1][o];
#pragma unroll
    for (int o = 0; o < T; ++o) v[0][o] = x[o];
  }
  __device__ __forceinline__ void merge() {  // (second + top), popped into one entry
#pragma unroll
    for (int o = 0; o < T; ++o) v[0][o] = fadd(v[1][o], v[0][o]);
#pragma unroll
    for (int d = 1; d + 1 < D; ++d)
#pragma unroll
      for (int o = 0; o < T; ++o) v[d][o] = v[d + 1][o];
  }
};

template <int TM, int TN, int D>
__global__ void __launch_bounds__(kPwThreads)
gemm_pairwise_kernel(const float* __restrict__ A, int lda, const float* __restrict__ B, int ldb,
                     const float* __restrict__ bias, float* __restrict__ C, int ldc, int M, int N,
                     int K, const PwLeaf* __restrict__ leaves, int nleaves, int nchunks, int act,
                     int kc, bool vecA, bool vecB) {
  extern __shared__ float4 smem_f4[];
  float* smem = reinterpret_cast<float*>(smem_f4);
  constexpr int BM = 4 * TM, BN = 8 * TN, T = TM * TN;
  const int kcp = kc + 4;
  // stage s: A rows at smem + s*(BM+BN)*kcp, B rows right after them
  const int stage_floats = (BM + BN) * kcp;
  const PwLeaf* chunks = leaves + nleaves;

  const int lane8 = threadIdx.x & 7;
  const int group = threadIdx.x >> 3;
  const int gm = group >> 3, gn = group & 7;
  const int mb = blockIdx.y * BM, nb = blockIdx.x * BN;

  {
    const PwLeaf c0 = chunks[0];
    stage_rows(smem, kcp, A, lda, mb, BM, M, c0.start, c0.len, K, vecA);
    stage_rows(smem + BM * kcp, kcp, B, ldb, nb, BN, N, c0.start, c0.len, K, vecB);
    cp_async_commit();
  }
  LeafStack<D, T> stk;
  float res[T];

  for (int c = 0; c < nchunks; ++c) {
    const PwLeaf ch = chunks[c];
    if (c + 1 < nchunks) {
      const PwLeaf cn = chunks[c + 1];
      float* nxt = smem + ((c + 1) & 1) * stage_floats;
      stage_rows(nxt, kcp, A, lda, mb, BM, M, cn.start, cn.len, K, vecA);
      stage_rows(nxt + BM * kcp, kcp, B, ldb, nb, BN, N, cn.start, cn.len, K, vecB);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const float* cur = smem + (c & 1) * stage_floats;
    const float* a_s = cur + gm * TM * kcp;
    const float* b_s = cur + BM * kcp + gn * TN * kcp;
    for (int l = ch.merges; l < ch.pad; ++l) {  // leaves [leaf_begin, leaf_end)
      const PwLeaf lf = leaves[l];
      const int base = lf.start - ch.start;
      const int nblk = lf.len >> 3, tail = lf.len & 7;
      float acc[T];
      if (nblk > 0) {
        const float* ap = a_s + base + lane8;
        const float* bp = b_s + base + lane8;
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j) acc[i * TN + j] = fmul(ap[i * kcp], bp[j * kcp]);
#pragma unroll 4
        for (int q = 1; q < nblk; ++q) {
          float a[TM], b[TN];
#pragma unroll
          for (int i = 0; i < TM; ++i) a[i] = ap[i * kcp + 8 * q];
#pragma unroll
          for (int j = 0; j < TN; ++j) b[j] = bp[j * kcp + 8 * q];
#pragma unroll
          for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int j = 0; j < TN; ++j) acc[i * TN + j] = fadd(acc[i * TN + j], fmul(a[i], b[j]));
        }
#pragma unroll
        for (int mask = 1; mask < 8; mask <<= 1)
#pragma unroll
          for (int o = 0; o < T; ++o) acc[o] = fadd(acc[o], __shfl_xor_sync(0xffffffffu, acc[o], mask));
      } else {
#pragma unroll
        for (int o = 0; o < T; ++o) acc[o] = 0.0f;  // n < 8: res = 0. then +=
      }
      for (int t = 0; t < tail; ++t) {
        const int k = base + 8 * nblk + t;
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j)
            acc[i * TN + j] = fadd(acc[i * TN + j], fmul(a_s[i * kcp + k], b_s[j * kcp + k]));
      }
      if constexpr (D == 1) {
#pragma unroll
        for (int o = 0; o < T; ++o) res[o] = acc[o];
      } else {
        stk.push(acc);
        for (int q = 0; q < lf.merges; ++q) stk.merge();
      }
    }
    __syncthreads();
  }
  if constexpr (D > 1) {
#pragma unroll
    for (int o = 0; o < T; ++o) res[o] = stk.v[0][o];
  }
  // lane j of the group stores outputs (i*TN + j) % 8 == j: bias added
  // separately (np.add(res, b), ops.py:106), then the activation
#pragma unroll
  for (int i = 0; i < TM; ++i) {
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      if ((i * TN + j) % 8 != lane8) continue;
      const int m = mb + gm * TM + i, n = nb + gn * TN + j;
      if (m >= M || n >= N) continue;
      float v = res[i * TN + j];
      if (bias) v = fadd(v, __ldg(bias + n));
      C[int64_t(m) * ldc + n] = act_forward(act, v);
    }
  }
}

// --------------------------------------------------- sequential GEMM kernel
// 32x32 output tile, 16x16 threads with 2x2 outputs; A and B chunks of K
// staged in smem with cp.async (double-buffered); every output accumulates
// strictly in k order from -0.0 (the additive identity, so the first step
// yields the first product exactly).

constexpr int kSeqBM = 32, kSeqBN = 32, kSeqKC = 64;

__device__ __forceinline__ void stage_a_seq(float* As, const float* A, int64_t sam, int64_t sak,
                                            int64_t mb, int64_t M, int64_t k0, int64_t K) {
  // As[m][k], row pitch kSeqKC + 1
  for (int e = threadIdx.x; e < kSeqBM * kSeqKC; e += 256) {
    const int kk = sak == 1 ? e % kSeqKC : e / kSeqBM;
    const int mm = sak == 1 ? e / kSeqKC : e % kSeqBM;
    const int64_t m = mb + mm, k = k0 + kk;
    const bool ok = m < M && k < K;
    cp_async4(As + mm * (kSeqKC + 1) + kk, ok ? A + m * sam + k * sak : A, ok);
  }
}

__device__ __forceinline__ void stage_b_seq(float* Bs, const float* B, int64_t sbk, int64_t sbn,
                                            int64_t nb, int64_t N, int64_t k0, int64_t K) {
  // Bs[k][n], row pitch kSeqBN + 1
  for (int e = threadIdx.x; e < kSeqKC * kSeqBN; e += 256) {
    const int nn = sbn == 1 ? e % kSeqBN : e / kSeqKC;
    const int kk = sbn == 1 ? e / kSeqBN : e % kSeqKC;
    const int64_t n = nb + nn, k = k0 + kk;
    const bool ok = n < N && k < K;
    cp_async4(Bs + kk * (kSeqBN + 1) + nn, ok ? B + k * sbk + n * sbn : B, ok);
  }
}

__global__ void __launch_bounds__(256)
gemm_sequential_kernel(const float* __restrict__ A, int64_t sam, int64_t sak,
                       const float* __restrict__ B, int64_t sbk, int64_t sbn,
                       float* __restrict__ C, int64_t ldc, const float* __restrict__ Y,
                       int act, int64_t M, int64_t N, int64_t K) {
  __shared__ float As[2][kSeqBM * (kSeqKC + 1)];
  __shared__ float Bs[2][kSeqKC * (kSeqBN + 1)];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t mb = int64_t(blockIdx.y) * kSeqBM, nb = int64_t(blockIdx.x) * kSeqBN;
  float acc[2][2] = {{-0.0f, -0.0f}, {-0.0f, -0.0f}};
  const int nchunks = static_cast<int>((K + kSeqKC - 1) / kSeqKC);
  stage_a_seq(As[0], A, sam, sak, mb, M, 0, K);
  stage_b_seq(Bs[0], B, sbk, sbn, nb, N, 0, K);
  cp_async_commit();
  for (int c = 0; c < nchunks; ++c) {
    if (c + 1 < nchunks) {
      stage_a_seq(As[(c + 1) & 1], A, sam, sak, mb, M, int64_t(c + 1) * kSeqKC, K);
      stage_b_seq(Bs[(c + 1) & 1], B, sbk, sbn, nb, N, int64_t(c + 1) * kSeqKC, K);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const float* a_s = As[c & 1];
    const float* b_s = Bs[c & 1];
    const int kmax = static_cast<int>(K - int64_t(c) * kSeqKC < kSeqKC ? K - int64_t(c) * kSeqKC
                                                                       : kSeqKC);
#pragma unroll 4
    for (int kk = 0; kk < kmax; ++kk) {
      const float a0 = a_s[ty * (kSeqKC + 1) + kk], a1 = a_s[(ty + 16) * (kSeqKC + 1) + kk];
      const float b0 = b_s[kk * (kSeqBN + 1) + tx], b1 = b_s[kk * (kSeqBN + 1) + tx + 16];
      acc[0][0] = fadd(acc[0][0], fmul(a0, b0));
      acc[0][1] = fadd(acc[0][1], fmul(a0, b1));
      acc[1][0] = fadd(acc[1][0], fmul(a1, b0));
      acc[1][1] = fadd(acc[1][1], fmul(a1, b1));
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int64_t m = mb + ty + 16 * i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int64_t n = nb + tx + 16 * j;
      if (n >= N) continue;
      float v = acc[i][j];
      if (act != MGX_ACT_NONE) v = act_backward(act, Y[m * ldc + n], v);
      C[m * ldc + n] = v;
    }
  }
}

// ------------------------------------------------ batch-tree (dW, db) kernel
// tree_sum (kernels.py:32-42) over n rows equals, for n = sum of distinct
// powers 2^a1 > 2^a2 > ..., T(2^a1) + (T(2^a2) + (... + T(2^ak))) with T a
// perfect pairwise tree over consecutive rows.  Rows are consumed in chunks
// of 8 (a perfect T8 in registers), chunk trees go through a binary counter
// (slot a holds a perfect T(8*2^a)); the n%8 tail rows form T4/T2/T1 by its
// bits; the pieces are then folded right-associatively, smallest first.
// The og and x tiles for up to kDwRows batch rows are staged in smem with
// cp.async (double-buffered over row chunks).

template <int LV, int T>
struct BatchTree {
  float slot[LV][T];
  __device__ __forceinline__ void push(int c, const float (&t8)[T]) {
    float carry[T];
#pragma unroll
    for (int o = 0; o < T; ++o) carry[o] = t8[o];
    bool done = false;
#pragma unroll
    for (int a = 0; a < LV; ++a) {
      if (!done) {
        if ((c >> a) & 1) {
#pragma unroll
          for (int o = 0; o < T; ++o) carry[o] = fadd(slot[a][o], carry[o]);
        } else {
#pragma unroll
          for (int o = 0; o < T; ++o) slot[a][o] = carry[o];
          done = true;
        }
      }
    }
  }
  __device__ __forceinline__ void finish(int nch, bool have_acc, float (&acc)[T]) {
#pragma unroll
    for (int a = 0; a < LV; ++a) {
      if ((nch >> a) & 1) {
        if (have_acc) {
#pragma unroll
          for (int o = 0; o < T; ++o) acc[o] = fadd(slot[a][o], acc[o]);
        } else {
#pragma unroll
          for (int o = 0; o < T; ++o) acc[o] = slot[a][o];
          have_acc = true;
        }
      }
    }
  }
};

template <int N>
__device__ __forceinline__ float perfect_tree(const float* v) {
  if constexpr (N == 1) {
    return v[0];
  } else {
    return fadd(perfect_tree<N / 2>(v), perfect_tree<N / 2>(v + N / 2));
  }
}

constexpr int kDwTH = 2, kDwTF = 2;
constexpr int kDwBH = 16 * kDwTH, kDwBF = 16 * kDwTF;
constexpr int kDwRows = 64;  // rows per staged chunk (multiple of 8)

template <int LV>
__global__ void __launch_bounds__(256)
fc_dw_db_kernel(const float* __restrict__ og, const float* __restrict__ x, float* __restrict__ dw,
                float* __restrict__ db, int64_t Bn, int64_t H, int64_t F, bool vecO, bool vecX) {
  __shared__ __align__(16) float Os[2][kDwRows][kDwBH + 4];
  __shared__ __align__(16) float Xs[2][kDwRows][kDwBF + 4];
  const int tf = threadIdx.x & 15, th = threadIdx.x >> 4;
  const int64_t hb = int64_t(blockIdx.y) * kDwBH, fb = int64_t(blockIdx.x) * kDwBF;
  const bool do_db = db != nullptr && blockIdx.x == 0 && tf == 0;
  const bool do_dw = dw != nullptr;
  constexpr int T = kDwTH * kDwTF;
  BatchTree<LV, T> tw;
  BatchTree<LV, kDwTH> tb;
  const int nrc = static_cast<int>((Bn + kDwRows - 1) / kDwRows);

  auto stage = [&](int buf, int64_t r0) {
    // og rows r0.. (row stride H), columns hb..hb+32; x rows, columns fb..
    stage_rows(&Os[buf][0][0], kDwBH + 4, og - 0, H, r0, kDwRows, Bn, hb, kDwBH, H, vecO);
    if (do_dw) stage_rows(&Xs[buf][0][0], kDwBF + 4, x, F, r0, kDwRows, Bn, fb, kDwBF, F, vecX);
    cp_async_commit();
  };
  // stage_rows indexes columns from c0 = hb; it expects (r0, c0) semantics
  stage(0, 0);
  int buf = 0;
  for (int rc = 0; rc < nrc; ++rc, buf ^= 1) {
    const int64_t r0 = int64_t(rc) * kDwRows;
    if (rc + 1 < nrc) {
      stage(buf ^ 1, r0 + kDwRows);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const int rows = static_cast<int>(Bn - r0 < kDwRows ? Bn - r0 : kDwRows);
    for (int c8 = 0; c8 + 8 <= rows; c8 += 8) {
      const int c = static_cast<int>((r0 + c8) >> 3);
      float p[T][8], q[kDwTH][8];
#pragma unroll
      for (int r = 0; r < 8; ++r) {
#pragma unroll
        for (int i = 0; i < kDwTH; ++i) {
          const float o = Os[buf][c8 + r][th + 16 * i];
          q[i][r] = o;
#pragma unroll
          for (int j = 0; j < kDwTF; ++j) p[i * kDwTF + j][r] = fmul(o, Xs[buf][c8 + r][tf + 16 * j]);
        }
      }
      float t8[T], b8[kDwTH];
#pragma unroll
      for (int o = 0; o < T; ++o) t8[o] = perfect_tree<8>(p[o]);
#pragma unroll
      for (int i = 0; i < kDwTH; ++i) b8[i] = perfect_tree<8>(q[i]);
      if (do_dw) tw.push(c, t8);
      if (do_db) tb.push(c, b8);
    }
    if (rc + 1 < nrc) __syncthreads();
  }
  // tail rows (Bn % 8 of them, all in the last staged chunk, buffer buf^1)
  const int tail = static_cast<int>(Bn & 7);
  const int lbuf = buf ^ 1;
  const int tr0 = static_cast<int>((Bn - tail) - int64_t(nrc - 1) * kDwRows);
  float acc[T], accb[kDwTH];
  bool have = false;
  auto prod = [&](int r, int o) {
    const int i = o / kDwTF, j = o % kDwTF;
    return fmul(Os[lbuf][tr0 + r][th + 16 * i], Xs[lbuf][tr0 + r][tf + 16 * j]);
  };
  auto ogv = [&](int r, int i) { return Os[lbuf][tr0 + r][th + 16 * i]; };
  {
    const int o2 = (tail & 4) ? 4 : 0;
    const int o1 = o2 + ((tail & 2) ? 2 : 0);
    if (tail & 1) {
#pragma unroll
      for (int o = 0; o < T; ++o) acc[o] = do_dw ? prod(o1, o) : 0.0f;
#pragma unroll
      for (int i = 0; i < kDwTH; ++i) accb[i] = ogv(o1, i);
      have = true;
    }
    if (tail & 2) {
#pragma unroll
      for (int o = 0; o < T; ++o) {
        const float t2 = do_dw ? fadd(prod(o2, o), prod(o2 + 1, o)) : 0.0f;
        acc[o] = have ? fadd(t2, acc[o]) : t2;
      }
#pragma unroll
      for (int i = 0; i < kDwTH; ++i) {
        const float t2 = fadd(ogv(o2, i), ogv(o2 + 1, i));
        accb[i] = have ? fadd(t2, accb[i]) : t2;
      }
      have = true;
    }
    if (tail & 4) {
#pragma unroll
      for (int o = 0; o < T; ++o) {
        const float t4 = do_dw ? fadd(fadd(prod(0, o), prod(1, o)), fadd(prod(2, o), prod(3, o)))
                               : 0.0f;
        acc[o] = have ? fadd(t4, acc[o]) : t4;
      }
#pragma unroll
      for (int i = 0; i < kDwTH; ++i) {
        const float t4 = fadd(fadd(ogv(0, i), ogv(1, i)), fadd(ogv(2, i), ogv(3, i)));
        accb[i] = have ? fadd(t4, accb[i]) : t4;
      }
      have = true;
    }
  }
  const int nch = static_cast<int>(Bn >> 3);
  if (do_dw) {
    tw.finish(nch, have, acc);
#pragma unroll
    for (int i = 0; i < kDwTH; ++i) {
      const int64_t h = hb + th + 16 * i;
      if (h >= H) continue;
#pragma unroll
      for (int j = 0; j < kDwTF; ++j) {
        const int64_t f = fb + tf + 16 * j;
        if (f < F) dw[h * F + f] = acc[i * kDwTF + j];
      }
    }
  }
  if (do_db) {
    tb.finish(nch, have, accb);
#pragma unroll
    for (int i = 0; i < kDwTH; ++i) {
      const int64_t h = hb + th + 16 * i;
      if (h < H) db[h] = accb[i];
    }
  }
}

int launch_dw_db(const float* og, const float* x, float* dw, float* db, int64_t Bn, int64_t H,
                 int64_t F, cudaStream_t st) {
  const int64_t nch = Bn >> 3;
  dim3 grid(static_cast<unsigned>(dw ? ceil_div(F, kDwBF) : 1),
            static_cast<unsigned>(ceil_div(H, kDwBH)));
  const bool vecO = (H % 4 == 0) && aligned16(og);
  const bool vecX = dw && (F % 4 == 0) && aligned16(x);
  if (nch < (1 << 4)) {
    fc_dw_db_kernel<4><<<grid, 256, 0, st>>>(og, x, dw, db, Bn, H, F, vecO, vecX);
  } else if (nch < (1 << 10)) {
    fc_dw_db_kernel<10><<<grid, 256, 0, st>>>(og, x, dw, db, Bn, H, F, vecO, vecX);
  } else if (nch < (1 << 20)) {
    fc_dw_db_kernel<20><<<grid, 256, 0, st>>>(og, x, dw, db, Bn, H, F, vecO, vecX);
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
  gemm_sequential_kernel<<<grid, 256, 0, st>>>(A, sam, sak, B, sbk, sbn, C, ldc, Y, act, M, N, K);
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
