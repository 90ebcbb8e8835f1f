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

int pw_leaf_table(int64_t K, const PwLeaf** out, int* nleaves, int* max_depth) {
  auto leaves = pairwise_leaves(K);
  int depth = 0, cur = 0;
  for (auto& l : leaves) {
    ++cur;
    depth = depth > cur ? depth : cur;
    cur -= l.merges;
  }
  *nleaves = static_cast<int>(leaves.size());
  *max_depth = depth;
  int dev = 0;
  MGX_CUDA(cudaGetDevice(&dev));
  int64_t key = (static_cast<int64_t>(dev) << 48) | K;
  std::lock_guard<std::mutex> lock(g_leaf_mu);
  auto it = g_leaf_tables.find(key);
  if (it != g_leaf_tables.end()) {
    *out = it->second;
    return MGX_OK;
  }
  PwLeaf* d = nullptr;
  size_t bytes = leaves.size() * sizeof(PwLeaf);
  MGX_CUDA(cudaMalloc(&d, bytes > 0 ? bytes : sizeof(PwLeaf)));
  // Plain synchronous copy: done once per (device, K), before any capture.
  MGX_CUDA(cudaMemcpy(d, leaves.data(), bytes, cudaMemcpyHostToDevice));
  g_leaf_tables[key] = d;
  *out = d;
  return MGX_OK;
}

// ----------------------------------------------------- pairwise GEMM kernel

constexpr int kPwThreads = 256;  // 32 groups of 8 lanes
constexpr int kPwMaxDepth = 24;

template <int TM, int TN, bool kStack>
__global__ void __launch_bounds__(kPwThreads)
gemm_pairwise_kernel(const float* __restrict__ A, int64_t lda, const float* __restrict__ B,
                     int64_t ldb, const float* __restrict__ bias, float* __restrict__ C,
                     int64_t ldc, int64_t M, int64_t N, const PwLeaf* __restrict__ leaves,
                     int nleaves, int act) {
  const int lane8 = threadIdx.x & 7;
  const int group = threadIdx.x >> 3;  // 0..31: 4 (m) x 8 (n)
  const int gm = group >> 3;
  const int gn = group & 7;
  const int64_t m0 = static_cast<int64_t>(blockIdx.y) * (4 * TM) + gm * TM;
  const int64_t n0 = static_cast<int64_t>(blockIdx.x) * (8 * TN) + gn * TN;

  const float* arow[TM];
  const float* brow[TN];
#pragma unroll
  for (int i = 0; i < TM; ++i) arow[i] = A + (m0 + i < M ? m0 + i : M - 1) * lda;
#pragma unroll
  for (int j = 0; j < TN; ++j) brow[j] = B + (n0 + j < N ? n0 + j : N - 1) * ldb;

  float stk[kStack ? kPwMaxDepth : 1][TM][TN];
  float res[TM][TN];
  int sp = 0;

  for (int l = 0; l < nleaves; ++l) {
    const PwLeaf lf = leaves[l];
    const int nb = lf.len >> 3;
    const int tail = lf.len & 7;
    float acc[TM][TN];
    if (nb > 0) {
      int k = lf.start + lane8;
      float a[TM], b[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) a[i] = __ldg(arow[i] + k);
#pragma unroll
      for (int j = 0; j < TN; ++j) b[j] = __ldg(brow[j] + k);
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fmul(a[i], b[j]);
      for (int bb = 1; bb < nb; ++bb) {
        k += 8;
#pragma unroll
        for (int i = 0; i < TM; ++i) a[i] = __ldg(arow[i] + k);
#pragma unroll
        for (int j = 0; j < TN; ++j) b[j] = __ldg(brow[j] + k);
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j) acc[i][j] = fadd(acc[i][j], fmul(a[i], b[j]));
      }
#pragma unroll
      for (int mask = 1; mask < 8; mask <<= 1)
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j)
            acc[i][j] = fadd(acc[i][j], __shfl_xor_sync(0xffffffffu, acc[i][j], mask));
    } else {
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = 0.0f;  // n < 8: res = 0. then +=
    }
    for (int t = 0; t < tail; ++t) {
      const int k = lf.start + 8 * nb + t;
#pragma unroll
      for (int i = 0; i < TM; ++i) {
        const float a = __ldg(arow[i] + k);
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fadd(acc[i][j], fmul(a, __ldg(brow[j] + k)));
      }
    }
    if constexpr (kStack) {
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) stk[sp][i][j] = acc[i][j];
      ++sp;
      for (int q = 0; q < lf.merges; ++q) {
        --sp;
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j) stk[sp - 1][i][j] = fadd(stk[sp - 1][i][j], stk[sp][i][j]);
      }
    } else {
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) res[i][j] = acc[i][j];
    }
  }
  if constexpr (kStack) {
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j) res[i][j] = stk[0][i][j];
  }

  // Epilogue: lane j of the group stores column j of the micro-tile rows,
  // bias added separately (np.add(res, b), ops.py:106), then activation.
#pragma unroll
  for (int i = 0; i < TM; ++i) {
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      if ((i * TN + j) % 8 != lane8) continue;
      const int64_t m = m0 + i, n = n0 + j;
      if (m >= M || n >= N) continue;
      float v = res[i][j];
      if (bias) v = fadd(v, __ldg(bias + n));
      C[m * ldc + n] = act_forward(act, v);
    }
  }
}

// --------------------------------------------------- sequential GEMM kernel
// Classic shared-memory tiled SIMT GEMM; each output accumulates its K
// products strictly in order k = 0..K-1, starting from -0.0 (the additive
// identity, so the first step yields the first product exactly).

constexpr int kSeqBM = 64, kSeqBN = 64, kSeqBK = 16, kSeqTM = 4, kSeqTN = 4;

__global__ void __launch_bounds__(256)
gemm_sequential_kernel(const float* __restrict__ A, int64_t sam, int64_t sak,
                       const float* __restrict__ B, int64_t sbk, int64_t sbn,
                       float* __restrict__ C, int64_t ldc, const float* __restrict__ Y,
                       int act, int64_t M, int64_t N, int64_t K) {
  __shared__ float As[kSeqBK][kSeqBM + 1];
  __shared__ float Bs[kSeqBK][kSeqBN + 1];
  const int tx = threadIdx.x & 15;  // n
  const int ty = threadIdx.x >> 4;  // m
  const int64_t mb = static_cast<int64_t>(blockIdx.y) * kSeqBM;
  const int64_t nb = static_cast<int64_t>(blockIdx.x) * kSeqBN;
  float acc[kSeqTM][kSeqTN];
#pragma unroll
  for (int i = 0; i < kSeqTM; ++i)
#pragma unroll
    for (int j = 0; j < kSeqTN; ++j) acc[i][j] = -0.0f;

  for (int64_t k0 = 0; k0 < K; k0 += kSeqBK) {
    for (int e = threadIdx.x; e < kSeqBK * kSeqBM; e += 256) {
      // coalesce along whichever of A's axes is contiguous
      const int kk = sak == 1 ? e % kSeqBK : e / kSeqBM;
      const int mm = sak == 1 ? e / kSeqBK : e % kSeqBM;
      const int64_t m = mb + mm, k = k0 + kk;
      As[kk][mm] = (m < M && k < K) ? __ldg(A + m * sam + k * sak) : 0.0f;
    }
    for (int e = threadIdx.x; e < kSeqBK * kSeqBN; e += 256) {
      const int kk = sbn == 1 ? e / kSeqBN : e % kSeqBK;
      const int nn = sbn == 1 ? e % kSeqBN : e / kSeqBK;
      const int64_t n = nb + nn, k = k0 + kk;
      Bs[kk][nn] = (n < N && k < K) ? __ldg(B + k * sbk + n * sbn) : 0.0f;
    }
    __syncthreads();
    const int kmax = static_cast<int>(K - k0 < kSeqBK ? K - k0 : kSeqBK);
    for (int kk = 0; kk < kmax; ++kk) {
      float a[kSeqTM], b[kSeqTN];
#pragma unroll
      for (int i = 0; i < kSeqTM; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < kSeqTN; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < kSeqTM; ++i)
#pragma unroll
        for (int j = 0; j < kSeqTN; ++j) acc[i][j] = fadd(acc[i][j], fmul(a[i], b[j]));
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < kSeqTM; ++i) {
    const int64_t m = mb + ty + 16 * i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < kSeqTN; ++j) {
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
  // Fold: tail pieces (already combined, smallest-first into `acc`, valid if
  // have_acc) then slots a = 0..LV-1 for the set bits of nch.
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

// perfect pairwise tree over v[0..2^L) in registers
template <int N>
__device__ __forceinline__ float perfect_tree(const float* v) {
  if constexpr (N == 1) {
    return v[0];
  } else {
    return fadd(perfect_tree<N / 2>(v), perfect_tree<N / 2>(v + N / 2));
  }
}

constexpr int kDwTH = 2, kDwTF = 2;            // outputs per thread
constexpr int kDwBH = 16 * kDwTH, kDwBF = 16 * kDwTF;  // 32 x 32 tile
constexpr int kDwRows = 32;                    // batch rows staged per pass

template <int LV>
__global__ void __launch_bounds__(256)
fc_dw_db_kernel(const float* __restrict__ og, const float* __restrict__ x, float* __restrict__ dw,
                float* __restrict__ db, int64_t Bn, int64_t H, int64_t F) {
  __shared__ float Os[kDwRows][kDwBH];
  __shared__ float Xs[kDwRows][kDwBF + 1];
  const int tf = threadIdx.x & 15;
  const int th = threadIdx.x >> 4;
  const int64_t hb = static_cast<int64_t>(blockIdx.y) * kDwBH;
  const int64_t fb = static_cast<int64_t>(blockIdx.x) * kDwBF;
  const bool do_db = db != nullptr && blockIdx.x == 0 && tf == 0;
  const bool do_dw = dw != nullptr;

  constexpr int T = kDwTH * kDwTF;
  BatchTree<LV, T> tw;
  BatchTree<LV, kDwTH> tb;
  const int64_t nch = Bn >> 3;
  const int tail = static_cast<int>(Bn & 7);
  float tailv[7][T];
  float tailb[7][kDwTH];

  for (int64_t r0 = 0; r0 < Bn; r0 += kDwRows) {
    const int rows = static_cast<int>(Bn - r0 < kDwRows ? Bn - r0 : kDwRows);
    for (int e = threadIdx.x; e < kDwRows * kDwBH; e += 256) {
      const int rr = e / kDwBH, hh = e % kDwBH;
      const int64_t h = hb + hh;
      Os[rr][hh] = (rr < rows && h < H) ? __ldg(og + (r0 + rr) * H + h) : 0.0f;
    }
    for (int e = threadIdx.x; e < kDwRows * kDwBF; e += 256) {
      const int rr = e / kDwBF, ff = e % kDwBF;
      const int64_t f = fb + ff;
      Xs[rr][ff] = (x != nullptr && rr < rows && f < F) ? __ldg(x + (r0 + rr) * F + f) : 0.0f;
    }
    __syncthreads();
    for (int c8 = 0; c8 < rows; c8 += 8) {
      const int64_t chunk = (r0 + c8) >> 3;
      const int nr = rows - c8 < 8 ? rows - c8 : 8;
      float p[T][8];
      float q[kDwTH][8];
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        if (r < nr) {
#pragma unroll
          for (int i = 0; i < kDwTH; ++i) {
            const float o = Os[c8 + r][th + 16 * i];
            q[i][r] = o;
#pragma unroll
            for (int j = 0; j < kDwTF; ++j) p[i * kDwTF + j][r] = fmul(o, Xs[c8 + r][tf + 16 * j]);
          }
        }
      }
      if (nr == 8) {
        float t8[T], b8[kDwTH];
#pragma unroll
        for (int o = 0; o < T; ++o) t8[o] = perfect_tree<8>(p[o]);
#pragma unroll
        for (int i = 0; i < kDwTH; ++i) b8[i] = perfect_tree<8>(q[i]);
        const int c = static_cast<int>(chunk);
        if (do_dw) tw.push(c, t8);
        if (do_db) tb.push(c, b8);
      } else {
#pragma unroll
        for (int r = 0; r < 7; ++r) {
          if (r < nr) {
#pragma unroll
            for (int o = 0; o < T; ++o) tailv[r][o] = p[o][r];
#pragma unroll
            for (int i = 0; i < kDwTH; ++i) tailb[r][i] = q[i][r];
          }
        }
      }
    }
    __syncthreads();
  }

  // Tail pieces by the bits of `tail` (descending sizes from the front):
  // rows [0, 4) if bit 2, then [.., +2) if bit 1, then 1 if bit 0.  Fold
  // smallest first: acc = T1; acc = T2 + acc; acc = T4 + acc.
  float acc[T], accb[kDwTH];
  bool have = false;
  {
    const int o4 = 0;
    const int o2 = (tail & 4) ? 4 : 0;
    const int o1 = o2 + ((tail & 2) ? 2 : 0);
    if (tail & 1) {
#pragma unroll
      for (int o = 0; o < T; ++o) acc[o] = tailv[o1][o];
#pragma unroll
      for (int i = 0; i < kDwTH; ++i) accb[i] = tailb[o1][i];
      have = true;
    }
    if (tail & 2) {
#pragma unroll
      for (int o = 0; o < T; ++o) {
        const float t2 = fadd(tailv[o2][o], tailv[o2 + 1][o]);
        acc[o] = have ? fadd(t2, acc[o]) : t2;
      }
#pragma unroll
      for (int i = 0; i < kDwTH; ++i) {
        const float t2 = fadd(tailb[o2][i], tailb[o2 + 1][i]);
        accb[i] = have ? fadd(t2, accb[i]) : t2;
      }
      have = true;
    }
    if (tail & 4) {
#pragma unroll
      for (int o = 0; o < T; ++o) {
        const float t4 = fadd(fadd(tailv[o4][o], tailv[o4 + 1][o]),
                              fadd(tailv[o4 + 2][o], tailv[o4 + 3][o]));
        acc[o] = have ? fadd(t4, acc[o]) : t4;
      }
#pragma unroll
      for (int i = 0; i < kDwTH; ++i) {
        const float t4 = fadd(fadd(tailb[o4][i], tailb[o4 + 1][i]),
                              fadd(tailb[o4 + 2][i], tailb[o4 + 3][i]));
        accb[i] = have ? fadd(t4, accb[i]) : t4;
      }
      have = true;
    }
  }
  const int nchi = static_cast<int>(nch);
  if (do_dw) {
    tw.finish(nchi, have, acc);
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
    tb.finish(nchi, have, accb);
#pragma unroll
    for (int i = 0; i < kDwTH; ++i) {
      const int64_t h = hb + th + 16 * i;
      if (h < H) db[h] = accb[i];
    }
  }
}

// tree over rows for a plain column reduction: treat it as db with og=a.
int launch_dw_db(const float* og, const float* x, float* dw, float* db, int64_t Bn, int64_t H,
                 int64_t F, cudaStream_t st) {
  const int64_t nch = Bn >> 3;
  dim3 grid(static_cast<unsigned>(dw ? ceil_div(F, kDwBF) : 1),
            static_cast<unsigned>(ceil_div(H, kDwBH)));
  if (nch < (1 << 4)) {
    fc_dw_db_kernel<4><<<grid, 256, 0, st>>>(og, x, dw, db, Bn, H, F);
  } else if (nch < (1 << 10)) {
    fc_dw_db_kernel<10><<<grid, 256, 0, st>>>(og, x, dw, db, Bn, H, F);
  } else if (nch < (1 << 20)) {
    fc_dw_db_kernel<20><<<grid, 256, 0, st>>>(og, x, dw, db, Bn, H, F);
  } else {
    set_error("batch tree: %lld rows exceed the supported 2^23", static_cast<long long>(Bn));
    return MGX_BAD_ARGUMENT;
  }
  MGX_LAUNCHED();
  return MGX_OK;
}

int launch_gemm_pairwise(const float* A, int64_t lda, const float* B, int64_t ldb,
                         const float* bias, float* C, int64_t ldc, int64_t M, int64_t N,
                         int64_t K, int act, cudaStream_t st) {
  const PwLeaf* leaves = nullptr;
  int nleaves = 0, depth = 0;
  MGX_TRY(pw_leaf_table(K, &leaves, &nleaves, &depth));
  if (depth > kPwMaxDepth) {
    set_error("pairwise GEMM: K=%lld too deep", static_cast<long long>(K));
    return MGX_BAD_ARGUMENT;
  }
  constexpr int TM = 2, TN = 2;
  dim3 grid(static_cast<unsigned>(ceil_div(N, 8 * TN)), static_cast<unsigned>(ceil_div(M, 4 * TM)));
  if (nleaves == 1) {
    gemm_pairwise_kernel<TM, TN, false><<<grid, kPwThreads, 0, st>>>(A, lda, B, ldb, bias, C, ldc,
                                                                     M, N, leaves, nleaves, act);
  } else {
    gemm_pairwise_kernel<TM, TN, true><<<grid, kPwThreads, 0, st>>>(A, lda, B, ldb, bias, C, ldc,
                                                                    M, N, leaves, nleaves, act);
  }
  MGX_LAUNCHED();
  return MGX_OK;
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
