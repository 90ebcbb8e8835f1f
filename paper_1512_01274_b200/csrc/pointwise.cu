// Elementwise, activation, softmax and SGD kernels.
//
// HBM-bound streaming kernels: 128-bit vectorised grid-stride loops sized to
// a multiple of the 148 SMs.  Every arithmetic step is a separately rounded
// fp32 op in the reference's order (tensor.py:169-231, ops.py:138-207,
// optim.py:39-50).

#include "common.cuh"

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

// --------------------------------------------------------------- softmax
// One group of 8 lanes per row.  shifted = x - rowmax; e = exp(shifted);
// p = e / pairwise_sum(e) (kernels.py:68-76).  The row sum follows numpy's
// pairwise order over the contiguous class axis: per leaf (start multiple of
// 8), lane j accumulates elements start+8i+j, an xor butterfly combines the
// 8 lanes, the tail is added in order, and leaves are merged per the split
// tree (for C <= 128 there is exactly one leaf).

__device__ __forceinline__ float max_nan(float a, float b) {
  if (a != a) return a;
  if (b != b) return b;
  return a > b ? a : b;
}

__global__ void __launch_bounds__(256)
softmax_fwd_kernel(const float* __restrict__ x, float* __restrict__ p, int64_t Bn, int64_t C,
                   const PwLeaf* __restrict__ leaves, int nleaves) {
  const int lane8 = threadIdx.x & 7;
  const int64_t row = int64_t(blockIdx.x) * 32 + (threadIdx.x >> 3);
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
__global__ void softmax_bwd_kernel(const float* __restrict__ p, const float* __restrict__ label,
                                   float* __restrict__ g, int64_t Bn, int64_t C) {
  const int64_t n = Bn * C;
  const float denom = static_cast<float>(Bn);
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int64_t b = i / C, c = i % C;
    int64_t cls = static_cast<int64_t>(label[b]);  // astype(int64): truncation
    if (cls < 0) cls += C;                         // numpy negative indexing
    const float hot = (c == cls) ? 1.0f : 0.0f;
    g[i] = fdiv(fsub(p[i], hot), denom);
  }
}

}  // namespace

int launch_softmax_forward(const float* x, float* p, int64_t Bn, int64_t C, cudaStream_t st) {
  const PwLeaf* leaves = nullptr;
  int nleaves = 0, depth = 0;
  MGX_TRY(pw_leaf_table(C, &leaves, &nleaves, &depth));
  MGX_REQUIRE(depth <= 32, "softmax: %lld classes too deep", static_cast<long long>(C));
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
  const unsigned blocks = static_cast<unsigned>(mgx::ceil_div(B * C, 256) < 1184 ? mgx::ceil_div(B * C, 256) : 1184);
  mgx::softmax_bwd_kernel<<<blocks, 256, 0, as_stream(stream)>>>(p, label, g, B, C);
  MGX_LAUNCHED();
  return MGX_OK;
}

extern "C" int mgx_sgd_step(float* w, const float* g, float* v, int64_t n, float eta,
                            float momentum, float weight_decay, uintptr_t stream) {
  MGX_REQUIRE(n >= 0 && (n == 0 || (w && g && v)), "mgx_sgd_step: bad arguments");
  // scalars arrive as float32(cfg.x) exactly like ETYPES[etype](alpha)
  return mgx::launch_map(n, mgx::aligned16(w) && mgx::aligned16(g) && mgx::aligned16(v),
                         mgx::SgdOp{w, g, v, -eta, momentum, weight_decay}, as_stream(stream));
}
