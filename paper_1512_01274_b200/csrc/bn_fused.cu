// Cluster-fused BatchNorm passes for the layers whose rows fit on-chip
// (the 27x27 / 14x14 / 7x7 stages of the convnets: a few thousand to ~50k
// rows).  The unfused chain is statistics-partials -> finalize -> apply in
// the forward and reduce-partials -> finalize -> dx (-> dsum finalize) in
// the backward: 2 and 3-4 launches per layer, each re-reading the tensors
// and most of them latency-bound at these sizes.  Here one kernel does the
// whole pass:
//
//   * a thread-block cluster of CS CTAs (8 portable or 16) owns a slice of
//     W float4 channel vectors (4W channels) and ALL M rows of it, the rows
//     split evenly over its CTAs;
//   * every CTA stages its rows x slice of the input(s) into shared memory
//     with cp.async (the whole tile in flight at once), so HBM is read once;
//   * per-thread fp32 partial sums -> fixed warp xor-tree and warp-order
//     merges in fp64 -> each CTA publishes its partials in shared memory ->
//     barrier.cluster -> every CTA sums the CS partials of the cluster over
//     DSMEM in rank order (the same order everywhere: deterministic, and
//     identical in every CTA, so no broadcast is needed);
//   * the elementwise pass (apply / dx) then runs from shared memory.
//
// Same arithmetic as the unfused kernels (conv.cu: shifted sums against row
// 0 for the statistics, xhat = (x - mean) * rstd, the ReLU mask recomputed
// from x, dx = gamma * rstd * (dy - (s1 + xhat * s2) / M)); only the order of
// the partial sums differs.  Reference semantics: MXNet BatchNorm
// (reference-side operator list in SURVEY.md sec. 8f; oracle/convnet.py).

#include <cooperative_groups.h>
#include <cuda_bf16.h>
#include <stdlib.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace mgx {
namespace bnf {

constexpr int kThreads = 512;
constexpr int kStages = 4;  // cp.async commit groups per tile (load/compute overlap)
constexpr int kWarps = kThreads / 32;
constexpr int kU = 4;  // streaming variant: rows in flight per thread

// Streaming variant (layers whose rows do not fit on-chip): the first pass
// reads with the default policy (the lines stay in L2), the second pass is
// the last use of them.
__device__ __forceinline__ float4 ld_keep(const float4* p) { return __ldg(p); }
__device__ __forceinline__ float4 ld_last(const float4* p) { return __ldcs(p); }

__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}

// ---- cluster exchange without cluster-wide barriers in the hot path: each
// CTA pushes its partials into every peer's receive slot with st.async,
// which completes transaction bytes on the destination's mbarrier; a CTA
// waits only on its own mbarrier (all CS partials arrived), then sums them
// in rank order from local shared memory.  The mbarriers are initialised
// at kernel start and published with one relaxed cluster arrive whose wait
// sits just before the first push (long since satisfied by then).

__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_async_f64(uint32_t raddr, double v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(raddr),
               "l"(__double_as_longlong(v)), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void mbar_init(uint32_t bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void cluster_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
}

// Per-thread fp32 pairs (4 channels each) -> the CTA's per-channel pairs,
// returned by thread j < 2*4W as element j ([2][4W] order): fp32 xor-tree
// over the lanes sharing a channel vector (lane % W), then the warp sums in
// order in fp64.  scratch: [kWarps][2][4W] doubles.
template <int W>
__device__ __forceinline__ double cta_reduce(const float* a, const float* b, double* scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float fa[4], fb[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    fa[q] = a[q];
    fb[q] = b[q];
  }
#pragma unroll
  for (int off = 16; off >= W; off >>= 1) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      fa[q] += __shfl_xor_sync(0xffffffffu, fa[q], off);
      fb[q] += __shfl_xor_sync(0xffffffffu, fb[q], off);
    }
  }
  constexpr int NC = 4 * W;
  if (lane < W) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      scratch[(warp * 2) * NC + lane * 4 + q] = fa[q];
      scratch[(warp * 2 + 1) * NC + lane * 4 + q] = fb[q];
    }
  }
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x < 2 * NC) {
    const int k = threadIdx.x / NC, c = threadIdx.x - (threadIdx.x / NC) * NC;
    double v[kWarps];  // all loads first, then the in-order sum
#pragma unroll
    for (int w = 0; w < kWarps; ++w) v[w] = scratch[(w * 2 + k) * NC + c];
#pragma unroll
    for (int w = 0; w < kWarps; ++w) s += v[w];
  }
  return s;
}

// Cluster sum of the CTA pairs: thread j < 2*4W pushes its value into slot
// [my rank][j] of every CTA's `recv` ([16][2][4W] doubles) on mbarrier `bar`;
// then every CTA waits for its CS * 2 * 4W * 8 bytes and sums the slots in
// rank order into tot[2][4W].
template <int W>
__device__ __forceinline__ void cluster_sum(double v, double* recv, uint64_t* bar, int parity,
                                            unsigned rank, unsigned n, double* tot) {
  constexpr int NC2 = 8 * W;  // 2 * 4W
  const uint32_t rbase = smem_u32(recv), bbase = smem_u32(bar);
  if (threadIdx.x == 0) mbar_expect(bbase, n * NC2 * 8u);
  if (threadIdx.x < NC2) {
    const uint32_t off = (rank * NC2 + threadIdx.x) * 8u;
    for (unsigned r = 0; r < n; ++r) st_async_f64(mapa(rbase + off, r), v, mapa(bbase, r));
  }
  mbar_wait(bbase, parity);
  if (threadIdx.x < NC2) {
    double x[16];
#pragma unroll
    for (unsigned r = 0; r < 16; ++r) x[r] = r < n ? recv[r * NC2 + threadIdx.x] : 0.0;
    double s = 0.0;
#pragma unroll
    for (unsigned r = 0; r < 16; ++r) s += x[r];
    tot[threadIdx.x] = s;
  }
  __syncthreads();
}

struct Slice {
  int r0, r1;  // this CTA's rows
  int c4;      // this thread's channel vector (global)
  int rin, v;  // row phase / vector within the slice
  int per;     // loop iterations per stage (uniform over the CTA)
};

template <int W>
__device__ __forceinline__ Slice slice_of(const cg::cluster_group& cl, int M, int rows_cta) {
  constexpr int RP = kThreads / W;
  Slice s;
  const int rank = static_cast<int>(cl.block_rank());
  s.r0 = rank * rows_cta;
  s.r1 = s.r0 + rows_cta < M ? s.r0 + rows_cta : M;
  s.v = threadIdx.x % W;
  s.rin = threadIdx.x / W;
  s.c4 = blockIdx.y * W + s.v;
  const int iters = (rows_cta + RP - 1) / RP;
  s.per = (iters + kStages - 1) / kStages;
  return s;
}

__device__ __forceinline__ void wait_stage(int left) {
  switch (left) {
    case 0: cp_async_wait<0>(); break;
    case 1: cp_async_wait<1>(); break;
    case 2: cp_async_wait<2>(); break;
    default: cp_async_wait<3>(); break;
  }
}

// Stage the thread's rows of `n` tensors into shared memory: kStages commit
// groups of s.per row-iterations each (local row l = rin + k * RP).
template <int W, int N>
__device__ __forceinline__ void stage_in(const Slice& s, const float4* const (&src)[N],
                                         float4* const (&dst)[N], const int (&ld4)[N]) {
  constexpr int RP = kThreads / W;
  for (int st = 0; st < kStages; ++st) {
    for (int k = st * s.per; k < (st + 1) * s.per; ++k) {
      const int r = s.r0 + s.rin + k * RP;
      if (r >= s.r1) break;
      const int l = (s.rin + k * RP) * W + s.v;
#pragma unroll
      for (int t = 0; t < N; ++t) cp_async16(dst[t] + l, src[t] + r * ld4[t] + s.c4, true);
    }
    cp_async_commit();
  }
}

// Forward: statistics (training, shifted sums against row 0), moving
// averages, apply (+act) -> y (fp32, optional) and y16 (bf16, optional).
template <int W, bool STREAM>
__global__ void __launch_bounds__(kThreads)
bn_fwd_fused_kernel(const float* __restrict__ x, int M, int C, int rows_cta, float eps,
                    float momentum, float* __restrict__ stats, float* __restrict__ mmean,
                    float* __restrict__ mvar, const float* __restrict__ gamma,
                    const float* __restrict__ beta, float* __restrict__ y,
                    __nv_bfloat16* __restrict__ y16, int act, int ldo4) {
  constexpr int RP = kThreads / W;  // rows per pass
  constexpr int NC = 4 * W;
  extern __shared__ __align__(16) unsigned char smem[];
  cg::cluster_group cl = cg::this_cluster();
  const unsigned rank = cl.block_rank(), ncta = cl.num_blocks();
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);                  // [2]
  double* recv = reinterpret_cast<double*>(smem + 16);                 // [ncta][2][NC]
  double* tot = recv + 2 * ncta * 2 * NC;                              // [2][NC]
  double* scratch = tot + 2 * NC;                                      // [kWarps][2][NC]
  float4* tile = reinterpret_cast<float4*>(scratch + kWarps * 2 * NC);  // [rows_cta][W]
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(bars));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cluster_arrive_relaxed();
  const Slice s = slice_of<W>(cl, M, rows_cta);
  const int C4 = C >> 2;
  const float4* x4 = reinterpret_cast<const float4*>(x);
  if (!STREAM) {
    const float4* src[1] = {x4};
    float4* dst[1] = {tile};
    const int ld4[1] = {C4};
    stage_in<W, 1>(s, src, dst, ld4);
  }
  const float4 shv = __ldg(x4 + s.c4);  // row 0: the shift of the sums
  const float sh[4] = {shv.x, shv.y, shv.z, shv.w};
  float s0[4] = {0.f, 0.f, 0.f, 0.f}, s1[4] = {0.f, 0.f, 0.f, 0.f};
  auto acc_stats = [&](const float4& v) {
    const float* pv = &v.x;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float d = pv[q] - sh[q];
      s0[q] += d;
      s1[q] += d * d;
    }
  };
  if (STREAM) {
    // rows straight from global memory, kU loads in flight per thread (the
    // same per-thread row order as the staged path)
    for (int r = s.r0 + s.rin; r < s.r1; r += kU * RP) {
      float4 v[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u)
        if (r + u * RP < s.r1) v[u] = ld_keep(x4 + int64_t(r + u * RP) * C4 + s.c4);
#pragma unroll
      for (int u = 0; u < kU; ++u)
        if (r + u * RP < s.r1) acc_stats(v[u]);
    }
  } else {
    for (int st = 0; st < kStages; ++st) {
      wait_stage(kStages - 1 - st);
      for (int k = st * s.per; k < (st + 1) * s.per; ++k) {
        const int lr = s.rin + k * RP;
        if (s.r0 + lr >= s.r1) break;
        acc_stats(tile[lr * W + s.v]);
      }
    }
  }
  const double part = cta_reduce<W>(s0, s1, scratch);
  cluster_wait();  // every peer's mbarrier is initialised
  cluster_sum<W>(part, recv, bars, 0, rank, ncta, tot);
  cluster_arrive_relaxed();  // all my incoming partials have landed
  // per-channel statistics (same formulas as bn_stats_finalize_kernel)
  float mu[4], rs[4], gm[4], bt[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int cl_ = s.v * 4 + q, c = s.c4 * 4 + q;
    const double dm = tot[cl_] / double(M);
    const double mean = double(sh[q]) + dm;
    double var = tot[NC + cl_] / double(M) - dm * dm;
    if (var < 0.0) var = 0.0;
    mu[q] = static_cast<float>(mean);
    rs[q] = static_cast<float>(1.0 / sqrt(var + double(eps)));
    gm[q] = gamma ? __ldg(gamma + c) : 1.0f;
    bt[q] = __ldg(beta + c);
    if (rank == 0 && s.rin == 0) {
      stats[c] = mu[q];
      stats[C + c] = rs[q];
      if (mmean) mmean[c] = static_cast<float>(double(mmean[c]) * momentum + mean * (1.0 - momentum));
      if (mvar) mvar[c] = static_cast<float>(double(mvar[c]) * momentum + var * (1.0 - momentum));
    }
  }
  auto apply = [&](float4 v, int r) {
    float* pv = &v.x;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float t = (pv[q] - mu[q]) * rs[q] * gm[q] + bt[q];
      pv[q] = act == MGX_ACT_RELU ? relu(t) : act_forward(act, t);
    }
    // outputs may be channel slices of a wider tensor (a Concat written in
    // place): row stride ldo4 float4 / uint2 vectors
    const int64_t i = int64_t(r) * ldo4 + s.c4;
    if (y) reinterpret_cast<float4*>(y)[i] = v;
    if (y16) {
      uint2 h;
      h.x = pack2(v.x, v.y);
      h.y = pack2(v.z, v.w);
      reinterpret_cast<uint2*>(y16)[i] = h;
    }
  };
  if (STREAM) {
    // second read of the rows: L2 hits (this CTA read them moments ago)
    for (int r = s.r0 + s.rin; r < s.r1; r += kU * RP) {
      float4 v[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u)
        if (r + u * RP < s.r1) v[u] = ld_last(x4 + int64_t(r + u * RP) * C4 + s.c4);
#pragma unroll
      for (int u = 0; u < kU; ++u)
        if (r + u * RP < s.r1) apply(v[u], r + u * RP);
    }
  } else {
    for (int r = s.r0 + s.rin; r < s.r1; r += RP) apply(tile[(r - s.r0) * W + s.v], r);
  }
  cluster_wait();  // no CTA leaves while a peer's pushes may be in flight
}

// Backward: s1 = sum dy', s2 = sum dy' * xhat (dy' = dy with the fused ReLU
// mask), dbeta/dgamma/sums, then dx = gamma * rstd * (dy' - (s1 + xhat s2)/M)
// -> dx (fp32, optional) / dx16 (bf16, optional), and dsum = sum dx
// (the bias gradient of the convolution feeding the BatchNorm, optional).
template <int W, bool STREAM>
__global__ void __launch_bounds__(kThreads)
bn_bwd_fused_kernel(const float* __restrict__ dy, int ldd, const float* __restrict__ x,
                    const float* __restrict__ stats, const float* __restrict__ gamma, int M,
                    int C, int rows_cta, const float* __restrict__ relu_gamma,
                    const float* __restrict__ relu_beta, float* __restrict__ dbeta,
                    float* __restrict__ dgamma, int dgamma_zero, float* __restrict__ sums,
                    float* dx, __nv_bfloat16* __restrict__ dx16, float* __restrict__ dsum) {
  constexpr int RP = kThreads / W;
  constexpr int NC = 4 * W;
  extern __shared__ __align__(16) unsigned char smem[];
  cg::cluster_group cl = cg::this_cluster();
  const unsigned rank = cl.block_rank(), ncta = cl.num_blocks();
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);                  // [2]
  double* recv = reinterpret_cast<double*>(smem + 16);                 // [2][ncta][2][NC]
  double* tot = recv + 2 * ncta * 2 * NC;                              // [2][NC]
  double* scratch = tot + 2 * NC;                                      // [kWarps][2][NC]
  float4* tdy = reinterpret_cast<float4*>(scratch + kWarps * 2 * NC);  // [rows_cta][W]
  float4* tx = tdy + rows_cta * W;
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(bars));
    mbar_init(smem_u32(bars + 1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cluster_arrive_relaxed();
  const Slice s = slice_of<W>(cl, M, rows_cta);
  const int C4 = C >> 2;
  const float4* dy4 = reinterpret_cast<const float4*>(dy);
  const float4* x4 = reinterpret_cast<const float4*>(x);
  const int ldd4 = ldd >> 2;
  if (!STREAM) {
    const float4* src[2] = {dy4, x4};
    float4* dst[2] = {tdy, tx};
    const int ld4[2] = {ldd4, C4};
    stage_in<W, 2>(s, src, dst, ld4);
  }
  const bool relu = relu_beta != nullptr;
  float mu[4], rs[4], gm[4], bt[4], g[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int c = s.c4 * 4 + q;
    mu[q] = __ldg(stats + c);
    rs[q] = __ldg(stats + C + c);
    g[q] = gamma ? __ldg(gamma + c) : 1.0f;
    gm[q] = relu && relu_gamma ? __ldg(relu_gamma + c) : 1.0f;
    bt[q] = relu ? __ldg(relu_beta + c) : 0.0f;
  }
  float a0[4] = {0.f, 0.f, 0.f, 0.f}, a1[4] = {0.f, 0.f, 0.f, 0.f};
  auto acc_sums = [&](const float4& d, const float4& xv) {
    const float* pd = &d.x;
    const float* px = &xv.x;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float dq = pd[q];
      if (relu && !((px[q] - mu[q]) * rs[q] * gm[q] + bt[q] > 0.0f)) dq = 0.0f;
      a0[q] += dq;
      a1[q] += dq * ((px[q] - mu[q]) * rs[q]);
    }
  };
  if (STREAM) {
    for (int r = s.r0 + s.rin; r < s.r1; r += kU * RP) {
      float4 d[kU], xv[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        if (r + u * RP < s.r1) {
          d[u] = ld_keep(dy4 + int64_t(r + u * RP) * ldd4 + s.c4);
          xv[u] = ld_keep(x4 + int64_t(r + u * RP) * C4 + s.c4);
        }
      }
#pragma unroll
      for (int u = 0; u < kU; ++u)
        if (r + u * RP < s.r1) acc_sums(d[u], xv[u]);
    }
  } else {
    for (int st = 0; st < kStages; ++st) {
      wait_stage(kStages - 1 - st);
      for (int k = st * s.per; k < (st + 1) * s.per; ++k) {
        const int lr = s.rin + k * RP;
        if (s.r0 + lr >= s.r1) break;
        const int l = lr * W + s.v;
        acc_sums(tdy[l], tx[l]);
      }
    }
  }
  const double part = cta_reduce<W>(a0, a1, scratch);
  cluster_wait();  // every peer's mbarrier is initialised
  cluster_sum<W>(part, recv, bars, 0, rank, ncta, tot);
  if (!dsum) cluster_arrive_relaxed();
  float s1[4], s2[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int cl_ = s.v * 4 + q, c = s.c4 * 4 + q;
    s1[q] = static_cast<float>(tot[cl_]);
    s2[q] = static_cast<float>(tot[NC + cl_]);
    if (rank == 0 && s.rin == 0) {
      if (sums) {
        sums[c] = s1[q];
        sums[C + c] = s2[q];
      }
      if (dbeta) dbeta[c] = s1[q];
      if (dgamma) dgamma[c] = dgamma_zero ? 0.0f : s2[q];
    }
  }
  const float invm = static_cast<float>(1.0 / double(M));
  float ds[4] = {0.f, 0.f, 0.f, 0.f};
  auto dx_row = [&](const float4& d, const float4& xv, int r) {
    const float* pd = &d.x;
    const float* px = &xv.x;
    float4 o;
    float* po = &o.x;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float dq = pd[q];
      if (relu && !((px[q] - mu[q]) * rs[q] * gm[q] + bt[q] > 0.0f)) dq = 0.0f;
      const float xhat = (px[q] - mu[q]) * rs[q];
      po[q] = g[q] * rs[q] * (dq - (s1[q] + xhat * s2[q]) * invm);
      ds[q] += po[q];
    }
    const int64_t i = int64_t(r) * C4 + s.c4;
    if (dx) reinterpret_cast<float4*>(dx)[i] = o;
    if (dx16) {
      uint2 h;
      h.x = pack2(o.x, o.y);
      h.y = pack2(o.z, o.w);
      reinterpret_cast<uint2*>(dx16)[i] = h;
    }
  };
  if (STREAM) {
    for (int r = s.r0 + s.rin; r < s.r1; r += kU * RP) {
      float4 d[kU], xv[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        if (r + u * RP < s.r1) {
          d[u] = ld_last(dy4 + int64_t(r + u * RP) * ldd4 + s.c4);
          xv[u] = ld_last(x4 + int64_t(r + u * RP) * C4 + s.c4);
        }
      }
#pragma unroll
      for (int u = 0; u < kU; ++u)
        if (r + u * RP < s.r1) dx_row(d[u], xv[u], r + u * RP);
    }
  } else {
    for (int r = s.r0 + s.rin; r < s.r1; r += RP) {
      const int l = (r - s.r0) * W + s.v;
      dx_row(tdy[l], tx[l], r);
    }
  }
  if (dsum) {
    const float zero[4] = {0.f, 0.f, 0.f, 0.f};
    __syncthreads();  // scratch / tot reuse
    const double p2 = cta_reduce<W>(ds, zero, scratch);
    cluster_sum<W>(p2, recv + ncta * 2 * NC, bars + 1, 0, rank, ncta, tot);
    cluster_arrive_relaxed();
    if (rank == 0 && threadIdx.x < NC)
      dsum[blockIdx.y * NC + threadIdx.x] = static_cast<float>(tot[threadIdx.x]);
  }
  cluster_wait();  // no CTA leaves while a peer's pushes may be in flight
}

// ------------------------------------------------------------- launch shape

struct Cfg {
  int W = 0, CS = 0;
  int rows_cta = 0;
  size_t smem = 0;
  bool stream = false;  // rows read from global memory twice, not staged
};

inline size_t smem_bytes(int W, int CS, int rows_cta, int tensors) {
  const size_t NC = 4 * size_t(W);
  return 16 + (2 * size_t(CS) * 2 * NC + 2 * NC + kWarps * 2 * NC) * sizeof(double) +
         size_t(rows_cta) * W * 16 * tensors;
}

// Clusters of 8 (portable) then 16, slices of 8/4/2 vectors: the first shape
// whose tile fits `smem_kb` with >= `min_ctas` CTAs, else the fitting shape
// with the most CTAs; none fits -> W == 0 (use the unfused kernels).  A
// deterministic function of (M, C, tensors).
inline int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v && *v ? atoi(v) : dflt;
}

// Streaming shape: slices of W vectors (env MGX_BNS_W, default 4: 64-byte
// fp32 rows), clusters of 16 when fewer than 128 CTAs would run with 8.
// Rows MGX_BNS_MINM..MGX_BNS_MAXM (default 32768..65536: the 27x27 layers
// at batch 64) stream; larger layers keep the unfused multi-CTA passes
// (tools/kbench.py bn / bnf: at 46656 rows x 64 channels the stream runs
// 14.6 / 18.9 us forward / backward against 16.3 staged and 22.3 unfused;
// at 193600 rows it loses to the unfused passes).
inline Cfg pick_stream(int64_t M, int64_t C, int tensors) {
  static const int sw = env_int("MGX_BNS_W", 4);
  static const int max_m = env_int("MGX_BNS_MAXM", 65536);
  Cfg c;
  if (C % 8 != 0 || M < 1 || M > max_m) return c;
  const int64_t C4 = C / 4;
  const int W = (sw == 4 || sw == 8) && C4 % sw == 0 ? sw : 2;
  const int64_t groups = C4 / W;
  static const int cs_env = env_int("MGX_BNS_CS", 0);
  const int CS = cs_env == 8 || cs_env == 16 ? cs_env : (groups * 8 >= 128 ? 8 : 16);
  return Cfg{W, CS, static_cast<int>(ceil_div(M, CS)), smem_bytes(W, CS, 0, tensors), true};
}

inline Cfg pick_staged(int64_t M, int64_t C, int tensors);

// env MGX_BNF_STREAM: 0 never stream, 1 stream from MGX_BNS_MINM rows or
// when the staged tile does not fit (default), 2 always stream
inline Cfg pick(int64_t M, int64_t C, int tensors) {
  static const int mode = env_int("MGX_BNF_STREAM", 1);
  static const int min_m = env_int("MGX_BNS_MINM", 32768);
  if (mode == 2 || (mode == 1 && M >= min_m)) {
    const Cfg c = pick_stream(M, C, tensors);
    if (c.W != 0 || mode == 2) return c;
  }
  const Cfg c = pick_staged(M, C, tensors);
  if (c.W != 0 || mode == 0) return c;
  return pick_stream(M, C, tensors);
}

inline Cfg pick_staged(int64_t M, int64_t C, int tensors) {
  // tuning knobs (read once): narrowest slice, CTA target, smem per CTA
  // defaults measured on Inception-BN (bench sweep): slices of >= 4 vectors
  // (full 32-byte sectors for the bf16 writes), >= 64 CTAs, up to 200 KB
  static const int min_w = env_int("MGX_BNF_MINW", 4);
  static const int min_ctas = env_int("MGX_BNF_MINCTAS", 64);
  static const int smem_kb = env_int("MGX_BNF_SMEM_KB", 200);
  static const int max_m = env_int("MGX_BNF_MAXM", 1 << 30);
  Cfg best;
  if (C % 8 != 0 || M < 1 || M > max_m || M * (C / 4) >= (int64_t(1) << 31)) return best;
  const int64_t C4 = C / 4;
  int64_t best_ctas = 0;
  static const int cs_first = env_int("MGX_BNF_CS_FIRST", 8);
  const int cs_order[2] = {cs_first, cs_first == 8 ? 16 : 8};
  for (int CS : cs_order) {
    for (int W : {8, 4, 2}) {
      if (C4 % W || W < min_w) continue;
      const int rows = static_cast<int>(ceil_div(M, CS));
      const size_t sm = smem_bytes(W, CS, rows, tensors);
      const int64_t ctas = int64_t(CS) * (C4 / W);
      if (sm <= size_t(smem_kb) * 1024 && ctas >= min_ctas) return Cfg{W, CS, rows, sm};
      if (sm <= size_t(200) * 1024 && ctas > best_ctas) {
        best = Cfg{W, CS, rows, sm};
        best_ctas = ctas;
      }
    }
  }
  return best;
}

template <typename... Params>
struct Launcher {
  // one instance (and one attrs_set flag) per kernel
  template <void (*kernel)(Params...), typename... Args>
  static int run(const Cfg& cfg, int64_t C, cudaStream_t st, Args... args);
};

template <typename... Params>
template <void (*kernel)(Params...), typename... Args>
int Launcher<Params...>::run(const Cfg& cfg, int64_t C, cudaStream_t st, Args... args) {
  static bool attrs_set = false;  // per kernel (a static of this instantiation)
  if (!attrs_set) {
    MGX_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  227 * 1024));
    MGX_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    attrs_set = true;
  }
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(cfg.CS, static_cast<unsigned>(C / 4 / cfg.W), 1);
  lc.blockDim = dim3(kThreads, 1, 1);
  lc.dynamicSmemBytes = cfg.smem;
  lc.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cfg.CS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  MGX_CUDA(cudaLaunchKernelEx(&lc, kernel, static_cast<Params>(args)...));
  return MGX_OK;
}

template <int W, typename... Args>
int launch_fwd(const Cfg& cfg, int64_t C, cudaStream_t st, Args... args) {
  using L = Launcher<const float*, int, int, int, float, float, float*, float*, float*,
                     const float*, const float*, float*, __nv_bfloat16*, int, int>;
  return cfg.stream ? L::template run<bn_fwd_fused_kernel<W, true>>(cfg, C, st, args...)
                    : L::template run<bn_fwd_fused_kernel<W, false>>(cfg, C, st, args...);
}

template <int W, typename... Args>
int launch_bwd(const Cfg& cfg, int64_t C, cudaStream_t st, Args... args) {
  using L = Launcher<const float*, int, const float*, const float*, const float*, int, int, int,
                     const float*, const float*, float*, float*, int, float*, float*,
                     __nv_bfloat16*, float*>;
  return cfg.stream ? L::template run<bn_bwd_fused_kernel<W, true>>(cfg, C, st, args...)
                    : L::template run<bn_bwd_fused_kernel<W, false>>(cfg, C, st, args...);
}

}  // namespace bnf
}  // namespace mgx

using mgx::bnf::Cfg;

extern "C" int mgx_bn_fused_ok(int64_t M, int64_t C, int backward, int* ok) {
  MGX_REQUIRE(ok && M > 0 && C > 0, "mgx_bn_fused_ok: bad arguments");
  const Cfg c = mgx::bnf::pick(M, C, backward ? 2 : 1);
  *ok = c.W == 0 ? 0 : (c.stream ? 2 : 1);
  return MGX_OK;
}

extern "C" int mgx_bn_fwd_fused_ld(const float* x, int64_t M, int64_t C, float* stats,
                                   float* moving_mean, float* moving_var, float eps,
                                   float momentum, const float* gamma, const float* beta, float* y,
                                   void* y16, int act, int64_t ldo, uintptr_t stream) {
  MGX_REQUIRE(x && stats && beta && (y || y16) && M > 0 && C > 0 && C <= 65536,
              "mgx_bn_fwd_fused: bad arguments");
  MGX_REQUIRE(mgx::aligned16(x) && (!y || mgx::aligned16(y)) && (!y16 || mgx::aligned16(y16)),
              "mgx_bn_fwd_fused: unaligned tensors");
  if (ldo == 0) ldo = C;
  MGX_REQUIRE(ldo >= C && ldo % 4 == 0 && ldo < 65536 * 4, "mgx_bn_fwd_fused: bad output stride");
  const Cfg cfg = mgx::bnf::pick(M, C, 1);
  MGX_REQUIRE(cfg.W != 0, "mgx_bn_fwd_fused: shape (%lld, %lld) does not fit a cluster",
              static_cast<long long>(M), static_cast<long long>(C));
  cudaStream_t st = mgx::as_stream(stream);
  const int Ci = static_cast<int>(C);
  const int ld4 = static_cast<int>(ldo / 4);
  __nv_bfloat16* h = static_cast<__nv_bfloat16*>(y16);
  switch (cfg.W) {
    case 8:
      return mgx::bnf::launch_fwd<8>(cfg, C, st, x, M, Ci, cfg.rows_cta, eps, momentum, stats,
                                     moving_mean, moving_var, gamma, beta, y, h, act, ld4);
    case 4:
      return mgx::bnf::launch_fwd<4>(cfg, C, st, x, M, Ci, cfg.rows_cta, eps, momentum, stats,
                                     moving_mean, moving_var, gamma, beta, y, h, act, ld4);
    default:
      return mgx::bnf::launch_fwd<2>(cfg, C, st, x, M, Ci, cfg.rows_cta, eps, momentum, stats,
                                     moving_mean, moving_var, gamma, beta, y, h, act, ld4);
  }
}

extern "C" int mgx_bn_fwd_fused(const float* x, int64_t M, int64_t C, float* stats,
                                float* moving_mean, float* moving_var, float eps, float momentum,
                                const float* gamma, const float* beta, float* y, void* y16,
                                int act, uintptr_t stream) {
  return mgx_bn_fwd_fused_ld(x, M, C, stats, moving_mean, moving_var, eps, momentum, gamma, beta,
                             y, y16, act, C, stream);
}

extern "C" int mgx_bn_bwd_fused(const float* dy, int64_t ldd, const float* x, const float* stats,
                                const float* gamma, int64_t M, int64_t C, const float* relu_gamma,
                                const float* relu_beta, float* dbeta, float* dgamma,
                                int dgamma_zero, float* sums, float* dx, void* dx16, float* dsum,
                                uintptr_t stream) {
  MGX_REQUIRE(dy && x && stats && (dx || dx16) && M > 0 && C > 0 && C <= 65536 &&
                  ldd >= C && ldd % 4 == 0 && ldd < (int64_t(1) << 24),
              "mgx_bn_bwd_fused: bad arguments (dy row stride ldd >= C, multiple of 4)");
  MGX_REQUIRE(mgx::aligned16(dy) && mgx::aligned16(x) && (!dx || mgx::aligned16(dx)) &&
                  (!dx16 || mgx::aligned16(dx16)),
              "mgx_bn_bwd_fused: unaligned tensors");
  const Cfg cfg = mgx::bnf::pick(M, C, 2);
  MGX_REQUIRE(cfg.W != 0, "mgx_bn_bwd_fused: shape (%lld, %lld) does not fit a cluster",
              static_cast<long long>(M), static_cast<long long>(C));
  cudaStream_t st = mgx::as_stream(stream);
  const int Ci = static_cast<int>(C);
  __nv_bfloat16* h = static_cast<__nv_bfloat16*>(dx16);
  switch (cfg.W) {
    case 8:
      return mgx::bnf::launch_bwd<8>(cfg, C, st, dy, static_cast<int>(ldd), x, stats, gamma, M,
                              Ci, cfg.rows_cta, relu_gamma, relu_beta, dbeta, dgamma, dgamma_zero,
                              sums, dx, h, dsum);
    case 4:
      return mgx::bnf::launch_bwd<4>(cfg, C, st, dy, static_cast<int>(ldd), x, stats, gamma, M,
                              Ci, cfg.rows_cta, relu_gamma, relu_beta, dbeta, dgamma, dgamma_zero,
                              sums, dx, h, dsum);
    default:
      return mgx::bnf::launch_bwd<2>(cfg, C, st, dy, static_cast<int>(ldd), x, stats, gamma, M,
                              Ci, cfg.rows_cta, relu_gamma, relu_beta, dbeta, dgamma, dgamma_zero,
                              sums, dx, h, dsum);
  }
}
