// Device tile functions shared by the standalone kernels (dense.cu,
// pointwise.cu) and the persistent program kernel (megakernel.cu).  Each
// tile function computes one block-sized tile; shared memory is passed in
// (the caller owns the allocation), block coordinates are arguments.
#pragma once

#include "common.cuh"

namespace mgx {

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
__device__ __forceinline__ void pw_tile(int bx, int by, float* smem,
                     const float* __restrict__ A, int lda, const float* __restrict__ B, int ldb,
                     const float* __restrict__ bias, float* __restrict__ C, int ldc, int M, int N,
                     int K, const PwLeaf* __restrict__ leaves, int nleaves, int nchunks, int act,
                     int kc, bool vecA, bool vecB) {
  constexpr int BM = 4 * TM, BN = 8 * TN, T = TM * TN;
  const int kcp = kc + 4;
  // stage s: A rows at smem + s*(BM+BN)*kcp, B rows right after them
  const int stage_floats = (BM + BN) * kcp;
  const PwLeaf* chunks = leaves + nleaves;

  const int lane8 = threadIdx.x & 7;
  const int group = threadIdx.x >> 3;
  const int gm = group >> 3, gn = group & 7;
  const int mb = by * BM, nb = bx * BN;

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

constexpr int kSeqSmemFloats = 2 * kSeqBM * (kSeqKC + 1) + 2 * kSeqKC * (kSeqBN + 1);

__device__ __forceinline__ void seq_tile(int bx, int by, float* smem,
                       const float* __restrict__ A, int64_t sam, int64_t sak,
                       const float* __restrict__ B, int64_t sbk, int64_t sbn,
                       float* __restrict__ C, int64_t ldc, const float* __restrict__ Y,
                       int act, int64_t M, int64_t N, int64_t K) {
  auto As = reinterpret_cast<float (*)[kSeqBM * (kSeqKC + 1)]>(smem);
  auto Bs = reinterpret_cast<float (*)[kSeqKC * (kSeqBN + 1)]>(smem + 2 * kSeqBM * (kSeqKC + 1));
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t mb = int64_t(by) * kSeqBM, nb = int64_t(bx) * kSeqBN;
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

constexpr int kDwSmemFloats = 2 * kDwRows * (kDwBH + 4) + 2 * kDwRows * (kDwBF + 4);

template <int LV>
__device__ __forceinline__ void dw_tile(int bx, int by, float* smem, const float* __restrict__ og, const float* __restrict__ x, float* __restrict__ dw,
                float* __restrict__ db, int64_t Bn, int64_t H, int64_t F, bool vecO, bool vecX) {
  auto Os = reinterpret_cast<float (*)[kDwRows][kDwBH + 4]>(smem);
  auto Xs = reinterpret_cast<float (*)[kDwRows][kDwBF + 4]>(smem + 2 * kDwRows * (kDwBH + 4));
  const int tf = threadIdx.x & 15, th = threadIdx.x >> 4;
  const int64_t hb = int64_t(by) * kDwBH, fb = int64_t(bx) * kDwBF;
  const bool do_db = db != nullptr && bx == 0 && tf == 0;
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


// ------------------------------------------------ pointwise / softmax

// Elementwise tile: elements [t*kMapTile, (t+1)*kMapTile) of n; float4 when
// every operand is 16-byte aligned (the element range is then 4-aligned).
constexpr int kMapTile = 4096;

template <typename F>
__device__ __forceinline__ void map_tile(int64_t t, int64_t n, bool vec, const F& f) {
  const int64_t lo = t * kMapTile;
  const int64_t hi = lo + kMapTile < n ? lo + kMapTile : n;
  if (vec) {
    const int64_t hi4 = lo + ((hi - lo) >> 2 << 2);
    for (int64_t i = (lo >> 2) + threadIdx.x; i < (hi4 >> 2); i += blockDim.x) f.vec(i);
    for (int64_t i = hi4 + threadIdx.x; i < hi; i += blockDim.x) f.scalar(i);
  } else {
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) f.scalar(i);
  }
}

struct FillOp {
  float* y;
  float v;
  __device__ void vec(int64_t i) const { reinterpret_cast<float4*>(y)[i] = make_float4(v, v, v, v); }
  __device__ void scalar(int64_t i) const { y[i] = v; }
};

struct CopyOp {
  const float* x;
  float* y;
  __device__ void vec(int64_t i) const {
    reinterpret_cast<float4*>(y)[i] = __ldg(reinterpret_cast<const float4*>(x) + i);
  }
  __device__ void scalar(int64_t i) const { y[i] = x[i]; }
};

// y = y + x*alpha (kernels.py:50-53)
struct AxpyOp {
  const float* x;
  float* y;
  float alpha;
  __device__ float f(float xv, float yv) const { return fadd(yv, fmul(xv, alpha)); }
  __device__ void vec(int64_t i) const {
    const float4 a = reinterpret_cast<const float4*>(x)[i];
    float4 b = reinterpret_cast<float4*>(y)[i];
    b = make_float4(f(a.x, b.x), f(a.y, b.y), f(a.z, b.z), f(a.w, b.w));
    reinterpret_cast<float4*>(y)[i] = b;
  }
  __device__ void scalar(int64_t i) const { y[i] = f(x[i], y[i]); }
};

struct EwOp {
  const float* a;
  const float* b;
  float* out;
  int op;
  __device__ float f(float x, float z) const {
    switch (op) {
      case 0: return fadd(x, z);
      case 1: return fsub(x, z);
      case 2: return fmul(x, z);
      default: return fdiv(x, z);
    }
  }
  __device__ void vec(int64_t i) const {
    const float4 x = reinterpret_cast<const float4*>(a)[i];
    const float4 z = reinterpret_cast<const float4*>(b)[i];
    reinterpret_cast<float4*>(out)[i] = make_float4(f(x.x, z.x), f(x.y, z.y), f(x.z, z.z), f(x.w, z.w));
  }
  __device__ void scalar(int64_t i) const { out[i] = f(a[i], b[i]); }
};

struct ScalarOp {
  const float* a;
  float* out;
  float c;
  int op;
  __device__ float f(float x) const { return op == 0 ? fadd(x, c) : fmul(x, c); }
  __device__ void vec(int64_t i) const {
    const float4 x = reinterpret_cast<const float4*>(a)[i];
    reinterpret_cast<float4*>(out)[i] = make_float4(f(x.x), f(x.y), f(x.z), f(x.w));
  }
  __device__ void scalar(int64_t i) const { out[i] = f(a[i]); }
};

struct ActFwdOp {
  const float* x;
  float* y;
  int act;
  __device__ void vec(int64_t i) const {
    const float4 v = reinterpret_cast<const float4*>(x)[i];
    reinterpret_cast<float4*>(y)[i] = make_float4(act_forward(act, v.x), act_forward(act, v.y),
                                                  act_forward(act, v.z), act_forward(act, v.w));
  }
  __device__ void scalar(int64_t i) const { y[i] = act_forward(act, x[i]); }
};

struct ActBwdOp {
  const float* y;
  const float* og;
  float* g;
  int act;
  __device__ void vec(int64_t i) const {
    const float4 a = reinterpret_cast<const float4*>(y)[i];
    const float4 o = reinterpret_cast<const float4*>(og)[i];
    reinterpret_cast<float4*>(g)[i] =
        make_float4(act_backward(act, a.x, o.x), act_backward(act, a.y, o.y),
                    act_backward(act, a.z, o.z), act_backward(act, a.w, o.w));
  }
  __device__ void scalar(int64_t i) const { g[i] = act_backward(act, y[i], og[i]); }
};

// Momentum SGD tensor path (optim.py:39-50):
//   tmp = g; tmp = tmp + w*wd; v = v*mom; v = v + tmp*(-eta); w = w + v*1
struct SgdOp {
  float* w;
  const float* g;
  float* v;
  float neg_eta, mom, wd;
  __device__ void step(float& wv, float gv, float& vv) const {
    const float tmp = fadd(gv, fmul(wv, wd));
    vv = fmul(vv, mom);
    vv = fadd(vv, fmul(tmp, neg_eta));
    wv = fadd(wv, fmul(vv, 1.0f));
  }
  __device__ void vec(int64_t i) const {
    float4 a = reinterpret_cast<float4*>(w)[i];
    const float4 b = reinterpret_cast<const float4*>(g)[i];
    float4 c = reinterpret_cast<float4*>(v)[i];
    step(a.x, b.x, c.x);
    step(a.y, b.y, c.y);
    step(a.z, b.z, c.z);
    step(a.w, b.w, c.w);
    reinterpret_cast<float4*>(w)[i] = a;
    reinterpret_cast<float4*>(v)[i] = c;
  }
  __device__ void scalar(int64_t i) const { step(w[i], g[i], v[i]); }
};

__device__ __forceinline__ float max_nan(float a, float b) {
  if (a != a) return a;
  if (b != b) return b;
  return a > b ? a : b;
}

__device__ __forceinline__ void softmax_fwd_tile(int bx, const float* __restrict__ x,
                                                 float* __restrict__ p, int64_t Bn, int64_t C,
                                                 const PwLeaf* __restrict__ leaves, int nleaves) {
  const int lane8 = threadIdx.x & 7;
  const int64_t row = int64_t(bx) * 32 + (threadIdx.x >> 3);
  const bool live = row < Bn;
  const float* xr = x + (live ? row : 0) * C;
  float* pr = p + (live ? row : 0) * C;

  float mx = -INFINITY;
  for (int64_t c = lane8; c < C; c += 8) mx = max_nan(mx, xr[c]);
#pragma unroll
  for (int mask = 1; mask < 8; mask <<= 1) mx = max_nan(mx, __shfl_xor_sync(0xffffffffu, mx, mask));
  if (live)
    for (int64_t c = lane8; c < C; c += 8) pr[c] = exp_rn(fsub(xr[c], mx));
  __syncwarp();

  float stk[32];
  int sp = 0;
  float res = 0.0f;
  for (int l = 0; l < nleaves; ++l) {
    const PwLeaf lf = leaves[l];
    const int nb = lf.len >> 3, tail = lf.len & 7;
    float acc;
    if (nb > 0) {
      int64_t c = lf.start + lane8;
      acc = live ? pr[c] : 0.0f;
      for (int bb = 1; bb < nb; ++bb) {
        c += 8;
        acc = fadd(acc, live ? pr[c] : 0.0f);
      }
#pragma unroll
      for (int mask = 1; mask < 8; mask <<= 1) acc = fadd(acc, __shfl_xor_sync(0xffffffffu, acc, mask));
    } else {
      acc = 0.0f;
    }
    for (int t = 0; t < tail; ++t) acc = fadd(acc, live ? pr[lf.start + 8 * nb + t] : 0.0f);
    if (nleaves == 1) {
      res = acc;
    } else {
      stk[sp++] = acc;
      for (int q = 0; q < lf.merges; ++q) {
        --sp;
        stk[sp - 1] = fadd(stk[sp - 1], stk[sp]);
      }
    }
  }
  if (nleaves > 1) res = stk[0];
  __syncwarp();
  if (live)
    for (int64_t c = lane8; c < C; c += 8) pr[c] = fdiv(pr[c], res);
}

// grad = (p - onehot(int64(label))) / f32(B)   (ops.py:188-196)
struct SoftmaxBwdOp {
  const float* p;
  const float* label;
  float* g;
  int64_t C;
  float denom;
  __device__ void scalar(int64_t i) const {
    const int64_t b = i / C, c = i - b * C;
    int64_t cls = static_cast<int64_t>(label[b]);  // astype(int64): truncation
    if (cls < 0) cls += C;                         // numpy negative indexing
    g[i] = fdiv(fsub(p[i], c == cls ? 1.0f : 0.0f), denom);
  }
  __device__ void vec(int64_t i) const {
#pragma unroll
    for (int k = 0; k < 4; ++k) scalar(4 * i + k);
  }
};

}  // namespace mgx
