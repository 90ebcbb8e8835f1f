// Elementwise, activation, softmax and SGD kernels.
//
// HBM-bound streaming kernels: 128-bit vectorised grid-stride loops sized to
// a multiple of the 148 SMs.  Every arithmetic step is a separately rounded
// fp32 op in the reference's order (tensor.py:169-231, ops.py:138-207,
// optim.py:39-50).

#include "tiles.cuh"

namespace mgx {

namespace {

constexpr int kThreads = 256;

inline unsigned grid_for(int64_t n_vec) {
  int64_t blocks = ceil_div(n_vec, kThreads);
  const int64_t cap = int64_t(kNumSMs) * 8;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  return static_cast<unsigned>(blocks);
}

// Generic vectorised map: out[i] = f(i, in...) over n elements.  Uses float4
// when every pointer is 16-byte aligned, scalar otherwise.
template <typename F>
__global__ void __launch_bounds__(kThreads) map4_kernel(int64_t n, F f) {
  const int64_t n4 = n >> 2;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += stride)
    f.vec(i);
  for (int64_t i = (n4 << 2) + int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    f.scalar(i);
}

template <typename F>
__global__ void __launch_bounds__(kThreads) map1_kernel(int64_t n, F f) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    f.scalar(i);
}

template <typename F>
int launch_map(int64_t n, bool vec_ok, F f, cudaStream_t st) {
  if (n <= 0) return MGX_OK;
  if (vec_ok) {
    map4_kernel<<<grid_for(n >> 2 ? n >> 2 : 1), kThreads, 0, st>>>(n, f);
  } else {
    map1_kernel<<<grid_for(n), kThreads, 0, st>>>(n, f);
  }
  MGX_LAUNCHED();
  return MGX_OK;
}

// --------------------------------------------------------------- softmax
// One group of 8 lanes per row.  shifted = x - rowmax; e = exp(shifted);
// p = e / pairwise_sum(e) (kernels.py:68-76).  The row sum follows numpy's
// pairwise order over the contiguous class axis: per leaf (start multiple of
// 8), lane j accumulates elements start+8i+j, an xor butterfly combines the
// 8 lanes, the tail is added in order, and leaves are merged per the split
// tree (for C <= 128 there is exactly one leaf).

__global__ void __launch_bounds__(256)
softmax_fwd_kernel(const float* __restrict__ x, float* __restrict__ p, int64_t Bn, int64_t C,
                   const PwLeaf* __restrict__ leaves, int nleaves) {
  softmax_fwd_tile(blockIdx.x, x, p, Bn, C, leaves, nleaves);
}

// Wide rows (C >= 256: the 1000-class heads): a 256-thread block per row so
// the elementwise exp and divide passes use the whole block (one group of 8
// lanes per row left a batch of 64 on two SMs); the row maximum is order-
// independent; the sum keeps the exact pairwise order above (one group of 8
// lanes over the block's exponentials).  Bitwise the same result as
// softmax_fwd_kernel.
__global__ void __launch_bounds__(256)
softmax_fwd_row_kernel(const float* __restrict__ x, float* __restrict__ p, int64_t C,
                       const PwLeaf* __restrict__ leaves, int nleaves) {
  __shared__ float red[8];
  __shared__ float total;
  const int64_t row = blockIdx.x;
  const float* xr = x + row * C;
  float* pr = p + row * C;
  float mx = -INFINITY;
  for (int64_t c = threadIdx.x; c < C; c += blockDim.x) mx = max_nan(mx, xr[c]);
#pragma unroll
  for (int mask = 1; mask < 32; mask <<= 1) mx = max_nan(mx, __shfl_xor_sync(0xffffffffu, mx, mask));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  mx = red[0];
  for (int w = 1; w < 8; ++w) mx = max_nan(mx, red[w]);
  for (int64_t c = threadIdx.x; c < C; c += blockDim.x) pr[c] = exp_rn(fsub(xr[c], mx));
  __syncthreads();
  if (threadIdx.x < 8) {
    const int lane8 = threadIdx.x;
    float stk[32];
    int sp = 0;
    float res = 0.0f;
    for (int l = 0; l < nleaves; ++l) {
      const PwLeaf lf = leaves[l];
      const int nb = lf.len >> 3, tail = lf.len & 7;
      float acc;
      if (nb > 0) {
        int64_t c = lf.start + lane8;
        acc = pr[c];
        for (int bb = 1; bb < nb; ++bb) {
          c += 8;
          acc = fadd(acc, pr[c]);
        }
#pragma unroll
        for (int mask = 1; mask < 8; mask <<= 1) acc = fadd(acc, __shfl_xor_sync(0xffu, acc, mask));
      } else {
        acc = 0.0f;
      }
      for (int t = 0; t < tail; ++t) acc = fadd(acc, pr[lf.start + 8 * nb + t]);
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
    if (lane8 == 0) total = res;
  }
  __syncthreads();
  const float res = total;
  for (int64_t c = threadIdx.x; c < C; c += blockDim.x) pr[c] = fdiv(pr[c], res);
}

}  // namespace

int launch_softmax_forward(const float* x, float* p, int64_t Bn, int64_t C, cudaStream_t st) {
  const PwLeaf* leaves = nullptr;
  int nleaves = 0, depth = 0;
  MGX_TRY(pw_leaf_table(C, &leaves, &nleaves, &depth));
  MGX_REQUIRE(depth <= 32, "softmax: %lld classes too deep", static_cast<long long>(C));
  if (C >= 256 && Bn < (int64_t(1) << 31)) {
    softmax_fwd_row_kernel<<<static_cast<unsigned>(Bn), 256, 0, st>>>(x, p, C, leaves, nleaves);
    MGX_LAUNCHED();
    return MGX_OK;
  }
  const unsigned blocks = static_cast<unsigned>(ceil_div(Bn, 32));
  softmax_fwd_kernel<<<blocks, 256, 0, st>>>(x, p, Bn, C, leaves,
                                             nleaves);
  MGX_LAUNCHED();
  return MGX_OK;
}

}  // namespace mgx

using mgx::as_stream;

extern "C" int mgx_fill(float* y, int64_t n, float value, uintptr_t stream) {
  MGX_REQUIRE(n >= 0 && (n == 0 || y), "mgx_fill: bad arguments");
  return mgx::launch_map(n, mgx::aligned16(y), mgx::FillOp{y, value}, as_stream(stream));
}

extern "C" int mgx_copy(const float* x, float* y, int64_t n, uintptr_t stream) {
  MGX_REQUIRE(n >= 0 && (n == 0 || (x && y)), "mgx_copy: bad arguments");
  if (x == y) return MGX_OK;
  return mgx::launch_map(n, mgx::aligned16(x) && mgx::aligned16(y), mgx::CopyOp{x, y},
                         as_stream(stream));
}

extern "C" int mgx_axpy(float alpha, const float* x, float* y, int64_t n, uintptr_t stream) {
  MGX_REQUIRE(n >= 0 && (n == 0 || (x && y)), "mgx_axpy: bad arguments");
  return mgx::launch_map(n, mgx::aligned16(x) && mgx::aligned16(y), mgx::AxpyOp{x, y, alpha},
                         as_stream(stream));
}

extern "C" int mgx_elementwise(int op, const float* a, const float* b, float* out, int64_t n,
                               uintptr_t stream) {
  MGX_REQUIRE(op >= 0 && op <= 3, "mgx_elementwise: unknown op %d", op);
  MGX_REQUIRE(n >= 0 && (n == 0 || (a && b && out)), "mgx_elementwise: bad arguments");
  return mgx::launch_map(n, mgx::aligned16(a) && mgx::aligned16(b) && mgx::aligned16(out),
                         mgx::EwOp{a, b, out, op}, as_stream(stream));
}

extern "C" int mgx_scalar_op(int op, const float* a, float c, float* out, int64_t n,
                             uintptr_t stream) {
  MGX_REQUIRE(op == 0 || op == 1, "mgx_scalar_op: unknown op %d", op);
  MGX_REQUIRE(n >= 0 && (n == 0 || (a && out)), "mgx_scalar_op: bad arguments");
  return mgx::launch_map(n, mgx::aligned16(a) && mgx::aligned16(out), mgx::ScalarOp{a, out, c, op},
                         as_stream(stream));
}

extern "C" int mgx_act_forward(int act, const float* x, float* y, int64_t n, uintptr_t stream) {
  MGX_REQUIRE(act >= 1 && act <= 3, "mgx_act_forward: unknown act %d", act);
  MGX_REQUIRE(n >= 0 && (n == 0 || (x && y)), "mgx_act_forward: bad arguments");
  return mgx::launch_map(n, mgx::aligned16(x) && mgx::aligned16(y), mgx::ActFwdOp{x, y, act},
                         as_stream(stream));
}

extern "C" int mgx_act_backward(int act, const float* y, const float* og, float* g, int64_t n,
                                uintptr_t stream) {
  MGX_REQUIRE(act >= 1 && act <= 3, "mgx_act_backward: unknown act %d", act);
  MGX_REQUIRE(n >= 0 && (n == 0 || (y && og && g)), "mgx_act_backward: bad arguments");
  return mgx::launch_map(n, mgx::aligned16(y) && mgx::aligned16(og) && mgx::aligned16(g),
                         mgx::ActBwdOp{y, og, g, act}, as_stream(stream));
}

extern "C" int mgx_softmax_forward(const float* x, float* p, int64_t B, int64_t C,
                                   uintptr_t stream) {
  MGX_REQUIRE(x && p && B > 0 && C > 0, "mgx_softmax_forward: bad arguments");
  return mgx::launch_softmax_forward(x, p, B, C, as_stream(stream));
}

extern "C" int mgx_softmax_backward(const float* p, const float* label, float* g, int64_t B,
                                    int64_t C, uintptr_t stream) {
  MGX_REQUIRE(p && label && g && B > 0 && C > 0, "mgx_softmax_backward: bad arguments");
  return mgx::launch_map(B * C, false, mgx::SoftmaxBwdOp{p, label, g, C, static_cast<float>(B)},
                         as_stream(stream));
}

extern "C" int mgx_sgd_step(float* w, const float* g, float* v, int64_t n, float eta,
                            float momentum, float weight_decay, uintptr_t stream) {
  MGX_REQUIRE(n >= 0 && (n == 0 || (w && g && v)), "mgx_sgd_step: bad arguments");
  // scalars arrive as float32(cfg.x) exactly like ETYPES[etype](alpha)
  return mgx::launch_map(n, mgx::aligned16(w) && mgx::aligned16(g) && mgx::aligned16(v),
                         mgx::SgdOp{w, g, v, -eta, momentum, weight_decay}, as_stream(stream));
}
