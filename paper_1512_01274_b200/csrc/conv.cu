// Convolution-net kernels (configs 3-5: LeNet, AlexNet-style, Inception-BN).
//
// The reference has no Convolution/Pooling/BatchNorm/Concat (SURVEY.md §0
// fact 7); these follow MXNet's operator semantics (arXiv
// 1512.01274 §2) in the channels-last layout: activations are NHWC fp32
// [B*H*W rows, C contiguous], convolution weights OHWI [Cout, kh*kw*Cin].
// Convolutions run as tcgen05 GEMMs (tc_gemm.cu) on bf16 operand copies:
//
//   forward  out[M=B*Ho*Wo, Cout] = col[M, K] . W[Cout, K]^T      (both K-major)
//   dgrad    dcol[M, K]           = dY[M, Cout] . W[Cout, K]        (W MN-major)
//   wgrad    dW[Cout, K]          = dY[M, Cout]^T . col[M, K]       (both MN-major)
//
// with K = kh*kw*Cin in (kh, kw, c) order.  The kernels here produce the
// operands (im2col + bf16 cast), scatter dcol back (col2im, a gather with a
// fixed tap order, no atomics), and do the bandwidth-bound work: BatchNorm
// statistics/apply/backward, pooling, channel-offset copies (Concat), and
// per-channel sums (conv bias gradient).  Every reduction has a fixed order
// (row chunks -> fixed-order merge), so results are run-to-run
// deterministic.

#include <cooperative_groups.h>
#include <cuda_bf16.h>

#include "common.cuh"

namespace mgx {
namespace conv {

struct Geom {
  int B, H, W, C, kh, kw, sh, sw, ph, pw, Ho, Wo;
};

// dims: B, H, W, C, (kh<<16|kw), (sh<<16|sw), (ph<<16|pw), then op-specific
__host__ __device__ inline Geom decode(const int64_t* d, bool full = false) {
  Geom g;
  g.B = static_cast<int>(d[0]);
  g.H = static_cast<int>(d[1]);
  g.W = static_cast<int>(d[2]);
  g.C = static_cast<int>(d[3]);
  g.kh = static_cast<int>(d[4] >> 16);
  g.kw = static_cast<int>(d[4] & 0xFFFF);
  g.sh = static_cast<int>(d[5] >> 16);
  g.sw = static_cast<int>(d[5] & 0xFFFF);
  g.ph = static_cast<int>(d[6] >> 16);
  g.pw = static_cast<int>(d[6] & 0xFFFF);
  if (!full) {
    g.Ho = (g.H + 2 * g.ph - g.kh) / g.sh + 1;
    g.Wo = (g.W + 2 * g.pw - g.kw) / g.sw + 1;
  } else {
    g.Ho = (g.H + 2 * g.ph - g.kh + g.sh - 1) / g.sh + 1;
    g.Wo = (g.W + 2 * g.pw - g.kw + g.sw - 1) / g.sw + 1;
  }
  return g;
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}

// ---- max-pooling gradient gathered on the fly (stem fusion): the input
// gradient of a max pooling at pixel r = sum of the pooled output gradient
// over the covering windows whose recorded argmax is r, windows in ascending
// (oh, ow) order -- exactly pool_bwd_vec_kernel's sum, so a BatchNorm
// backward can read its output gradient through the pooling without that
// gradient ever being written (the BatchNorm input is the pooling input).
struct PoolGrad {
  const float4* dy;        // pooled output gradient [B, Ho, Wo, C] as channel vectors
  const uchar4* arg;       // window-local argmax, same shape
  Geom g;                  // pooling geometry (H, W input; Ho, Wo output)
  uint64_t mul_hw, mul_w;  // n / (H W), n / W as __umul64hi(n, mul); 0: divisor 1
};

__host__ inline uint64_t pg_mul(int d) { return d <= 1 ? 0 : ~uint64_t(0) / uint64_t(d) + 1; }
__device__ __forceinline__ int pg_div(int n, uint64_t mul) {
  return mul ? static_cast<int>(__umul64hi(static_cast<uint64_t>(static_cast<uint32_t>(n)), mul))
             : n;
}

// PK: 32 = a 3x3 / stride 2 window (unrolled), 1 = runtime geometry
template <int PK>
__device__ __forceinline__ float4 pool_grad4(const PoolGrad& pg, int r, int c4, int C4) {
  const Geom& g = pg.g;
  const int b = pg_div(r, pg.mul_hw);
  const int rem = r - b * g.H * g.W;
  const int h = pg_div(rem, pg.mul_w), w = rem - h * g.W;
  constexpr int K = PK == 32 ? 3 : 0, S = PK == 32 ? 2 : 0;
  const int kh = K ? K : g.kh, kw = K ? K : g.kw;
  const int sh = K ? S : g.sh, sw = K ? S : g.sw;
  const int nh = h + g.ph - kh + 1, nw = w + g.pw - kw + 1;
  const int oh_lo = nh <= 0 ? 0 : (nh + sh - 1) / sh;
  const int oh_hi = min(g.Ho - 1, (h + g.ph) / sh);
  const int ow_lo = nw <= 0 ? 0 : (nw + sw - 1) / sw;
  const int ow_hi = min(g.Wo - 1, (w + g.pw) / sw);
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  const int64_t ob = int64_t(b) * g.Ho * g.Wo * C4 + c4;
  auto win = [&](int oh, int ow, const float4 d, const uchar4 am) {
    const int li = (h - (oh * sh - g.ph)) * kw + (w - (ow * sw - g.pw));
    const float* pd = &d.x;
    const unsigned char* pa = &am.x;
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (pa[q] == li) acc[q] = fadd(acc[q], pd[q]);
  };
  if constexpr (K > 0) {
    constexpr int NW = (K + S - 1) / S;
    float4 d[NW * NW];
    uchar4 am[NW * NW];
#pragma unroll
    for (int i = 0; i < NW; ++i)
#pragma unroll
      for (int j = 0; j < NW; ++j) {
        const bool ok = oh_lo + i <= oh_hi && ow_lo + j <= ow_hi;
        const int64_t o = ob + (int64_t(oh_lo + i) * g.Wo + ow_lo + j) * C4;
        d[i * NW + j] = ok ? __ldg(pg.dy + o) : make_float4(0.f, 0.f, 0.f, 0.f);
        am[i * NW + j] = ok ? __ldg(pg.arg + o) : make_uchar4(255, 255, 255, 255);
      }
#pragma unroll
    for (int i = 0; i < NW; ++i)
#pragma unroll
      for (int j = 0; j < NW; ++j)
        if (oh_lo + i <= oh_hi && ow_lo + j <= ow_hi)
          win(oh_lo + i, ow_lo + j, d[i * NW + j], am[i * NW + j]);
  } else {
    for (int oh = oh_lo; oh <= oh_hi; ++oh)
      for (int ow = ow_lo; ow <= ow_hi; ++ow) {
        const int64_t o = ob + (int64_t(oh) * g.Wo + ow) * C4;
        win(oh, ow, __ldg(pg.dy + o), __ldg(pg.arg + o));
      }
  }
  return make_float4(acc[0], acc[1], acc[2], acc[3]);
}

// col[m, k] (bf16, row stride ldk >= K, zero beyond K) = x at tap k of output
// pixel m (zero in the padding).  A thread owns the 8 consecutive k of one
// 16-byte store; when C % 8 == 0 they are 8 channels of one tap (two float4
// loads).
__global__ void __launch_bounds__(256)
im2col_kernel(const float* __restrict__ x, __nv_bfloat16* __restrict__ col, Geom g, int64_t ldk) {
  const int K = g.kh * g.kw * g.C;
  const int per_row = static_cast<int>(ldk / 8);
  const RowsIdx ri(per_row);
  if (!ri.active) return;
  const int k0 = ri.v * 8;
  const int M = g.B * g.Ho * g.Wo;
  const int hw = g.Ho * g.Wo;
  const bool vec = (g.C % 8) == 0;
  // per-thread tap decode of its 8 columns
  int ti[8], tj[8], tc[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    const int k = k0 + t;
    const int tap = k / g.C;
    tc[t] = k < K ? k - tap * g.C : -1;
    ti[t] = tap / g.kw;
    tj[t] = tap - ti[t] * g.kw;
  }
  for (int m = ri.r; m < M; m += ri.rstep) {
    const int b = m / hw;
    const int rem = m - b * hw;
    const int oh = rem / g.Wo, ow = rem - (rem / g.Wo) * g.Wo;
    const int hb = oh * g.sh - g.ph, wb = ow * g.sw - g.pw;
    float v8[8];
    if (vec) {
      const int h = hb + ti[0], w = wb + tj[0];
      if (tc[0] >= 0 && h >= 0 && h < g.H && w >= 0 && w < g.W) {
        const float4* src =
            reinterpret_cast<const float4*>(x + ((int64_t(b) * g.H + h) * g.W + w) * g.C + tc[0]);
        const float4 a = __ldg(src), c = __ldg(src + 1);
        v8[0] = a.x; v8[1] = a.y; v8[2] = a.z; v8[3] = a.w;
        v8[4] = c.x; v8[5] = c.y; v8[6] = c.z; v8[7] = c.w;
      } else {
#pragma unroll
        for (int t = 0; t < 8; ++t) v8[t] = 0.0f;
      }
    } else {
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const int h = hb + ti[t], w = wb + tj[t];
        v8[t] = (tc[t] >= 0 && h >= 0 && h < g.H && w >= 0 && w < g.W)
                    ? __ldg(x + ((int64_t(b) * g.H + h) * g.W + w) * g.C + tc[t])
                    : 0.0f;
      }
    }
    uint4 o;
    o.x = pack_bf16(v8[0], v8[1]);
    o.y = pack_bf16(v8[2], v8[3]);
    o.z = pack_bf16(v8[4], v8[5]);
    o.w = pack_bf16(v8[6], v8[7]);
    *reinterpret_cast<uint4*>(col + int64_t(m) * ldk + k0) = o;
  }
}

// im2col for few input channels (the RGB stem), one block per output row
// (b, oh): the kh input rows it touches are staged in shared memory once
// (coalesced, zero-filled in the padding), then every 16-byte store of the
// row's col entries reads its 8 elements from shared memory through a
// per-column offset table -- no per-element tap decode, no redundant global
// reads.  tile: [kh][WT][C] with WT = (Wo - 1) * sw + kw input columns
// starting at w = -pw; lut[k] = (k / (kw C)) * WT * C + k % (kw C), -1 for
// the K padding.
__global__ void __launch_bounds__(256)
im2col_rows_kernel(const float* __restrict__ x, __nv_bfloat16* __restrict__ col, Geom g,
                   int64_t ldk, int WT) {
  extern __shared__ float tile[];
  const int rowlen = WT * g.C;
  int* lut = reinterpret_cast<int*>(tile + g.kh * rowlen);
  const int b = blockIdx.x / g.Ho, oh = blockIdx.x - (blockIdx.x / g.Ho) * g.Ho;
  const int hb = oh * g.sh - g.ph;
  const int K = g.kh * g.kw * g.C, seg = g.kw * g.C;
  for (int k = threadIdx.x; k < ldk; k += blockDim.x)
    lut[k] = k < K ? (k / seg) * rowlen + (k - (k / seg) * seg) : -1;
  const int e_lo = g.pw * g.C, e_hi = (g.W + g.pw) * g.C;  // in-image part of a staged row
  for (int i = 0; i < g.kh; ++i) {
    const int h = hb + i;
    const bool hv = h >= 0 && h < g.H;
    const float* src = x + (int64_t(b) * g.H + (hv ? h : 0)) * g.W * g.C - e_lo;
    for (int e = threadIdx.x; e < rowlen; e += blockDim.x)
      tile[i * rowlen + e] = (hv && e >= e_lo && e < e_hi) ? __ldg(src + e) : 0.0f;
  }
  __syncthreads();
  const int nj = static_cast<int>(ldk / 8);
  const int rpb = blockDim.x / nj;
  const int r = threadIdx.x / nj, j = threadIdx.x - (threadIdx.x / nj) * nj;
  if (r >= rpb) return;
  int off[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) off[t] = lut[j * 8 + t];
  const int step = g.sw * g.C;
  __nv_bfloat16* out = col + (int64_t(b) * g.Ho + oh) * g.Wo * ldk + j * 8;
  for (int ow = r; ow < g.Wo; ow += rpb) {
    float v8[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) v8[t] = off[t] >= 0 ? tile[off[t] + ow * step] : 0.0f;
    uint4 o;
    o.x = pack_bf16(v8[0], v8[1]);
    o.y = pack_bf16(v8[2], v8[3]);
    o.z = pack_bf16(v8[4], v8[5]);
    o.w = pack_bf16(v8[6], v8[7]);
    *reinterpret_cast<uint4*>(out + int64_t(ow) * ldk) = o;
  }
}

// dx[b,h,w,c] = sum over taps (i, j) ascending of dcol[pixel(oh,ow), (i,j,c)]
// for every output pixel whose window covers (h, w): the adjoint of im2col
// as a gather (deterministic, no atomics).
__global__ void col2im_kernel(const float* __restrict__ dcol, int64_t ldk, float* __restrict__ dx,
                              Geom g) {
  const int64_t total = int64_t(g.B) * g.H * g.W * g.C;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; idx < total; idx += stride) {
    const int c = static_cast<int>(idx % g.C);
    int64_t p = idx / g.C;
    const int w = static_cast<int>(p % g.W);
    p /= g.W;
    const int h = static_cast<int>(p % g.H);
    const int b = static_cast<int>(p / g.H);
    float acc = 0.0f;
    for (int i = 0; i < g.kh; ++i) {
      const int hn = h + g.ph - i;
      if (hn < 0 || hn % g.sh) continue;
      const int oh = hn / g.sh;
      if (oh >= g.Ho) continue;
      for (int j = 0; j < g.kw; ++j) {
        const int wn = w + g.pw - j;
        if (wn < 0 || wn % g.sw) continue;
        const int ow = wn / g.sw;
        if (ow >= g.Wo) continue;
        const int64_t m = (int64_t(b) * g.Ho + oh) * g.Wo + ow;
        acc = fadd(acc, __ldg(dcol + m * ldk + (i * g.kw + j) * g.C + c));
      }
    }
    dx[idx] = acc;
  }
}

// The same gather, four channels per thread (C % 4 == 0, ldk % 4 == 0,
// 16-byte aligned): consecutive threads read consecutive 16-byte chunks of
// a dcol row and write consecutive chunks of dx (coalesced); the taps of a
// compile-time kernel/stride are unrolled so every covering window's load
// is issued before the first add (sums still in ascending tap order).
template <int KH, int KW, int SH, int SW>
__global__ void __launch_bounds__(256)
col2im_vec4_kernel(const float4* __restrict__ dcol, int64_t ldk4, float4* __restrict__ dx,
                   Geom g) {
  const int c4n = g.C >> 2;
  const int kh = KH ? KH : g.kh, kw = KW ? KW : g.kw;
  const int sh = SH ? SH : g.sh, sw = SW ? SW : g.sw;
  const int64_t total = int64_t(g.B) * g.H * g.W * c4n;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; idx < total; idx += stride) {
    const int c4 = static_cast<int>(idx % c4n);
    const int64_t pix = idx / c4n;
    const int w = static_cast<int>(pix % g.W);
    const int64_t bh = pix / g.W;
    const int h = static_cast<int>(bh % g.H);
    const int b = static_cast<int>(bh / g.H);
    constexpr int kMax = (KH ? KH : 1) * (KW ? KW : 1);
    if (KH && KW) {
      float4 v[kMax];
      bool ok[kMax];
#pragma unroll
      for (int i = 0; i < KH; ++i) {
#pragma unroll
        for (int j = 0; j < KW; ++j) {
          const int hn = h + g.ph - i, wn = w + g.pw - j;
          const int oh = hn / SH, ow = wn / SW;
          const bool valid = hn >= 0 && wn >= 0 && hn - oh * SH == 0 && wn - ow * SW == 0 &&
                             oh < g.Ho && ow < g.Wo;
          ok[i * KW + j] = valid;
          v[i * KW + j] = make_float4(0.f, 0.f, 0.f, 0.f);
          if (valid) {
            const int64_t m = (int64_t(b) * g.Ho + oh) * g.Wo + ow;
            v[i * KW + j] = __ldg(dcol + m * ldk4 + (i * KW + j) * c4n + c4);
          }
        }
      }
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int t = 0; t < kMax; ++t) {
        if (ok[t]) {
          acc.x = fadd(acc.x, v[t].x);
          acc.y = fadd(acc.y, v[t].y);
          acc.z = fadd(acc.z, v[t].z);
          acc.w = fadd(acc.w, v[t].w);
        }
      }
      dx[idx] = acc;
    } else {
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int i = 0; i < kh; ++i) {
        const int hn = h + g.ph - i;
        if (hn < 0 || hn % sh) continue;
        const int oh = hn / sh;
        if (oh >= g.Ho) continue;
        for (int j = 0; j < kw; ++j) {
          const int wn = w + g.pw - j;
          if (wn < 0 || wn % sw) continue;
          const int ow = wn / sw;
          if (ow >= g.Wo) continue;
          const int64_t m = (int64_t(b) * g.Ho + oh) * g.Wo + ow;
          const float4 t = __ldg(dcol + m * ldk4 + (i * kw + j) * c4n + c4);
          acc.x = fadd(acc.x, t.x);
          acc.y = fadd(acc.y, t.y);
          acc.z = fadd(acc.z, t.z);
          acc.w = fadd(acc.w, t.w);
        }
      }
      dx[idx] = acc;
    }
  }
}

// wf[c, (i*kw + j)*F + f] (bf16, row stride ld, zero beyond kh*kw*F) =
// w[f, kh-1-i, kw-1-j, c]: the weight of the transposed convolution that
// computes a stride-1 data gradient as im2col(dY) . wf^T.
__global__ void weight_flip_kernel(const float* __restrict__ w, int F, int kh, int kw, int C,
                                   __nv_bfloat16* __restrict__ wf, int64_t ld) {
  const int64_t total = int64_t(C) * ld;
  const int K = kh * kw * F;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; idx < total; idx += stride) {
    const int c = static_cast<int>(idx / ld);
    const int k = static_cast<int>(idx - int64_t(c) * ld);
    float v = 0.0f;
    if (k < K) {
      const int tap = k / F, f = k - tap * F;
      const int i = tap / kw, j = tap - (tap / kw) * kw;
      v = __ldg(w + ((int64_t(f) * kh + (kh - 1 - i)) * kw + (kw - 1 - j)) * C + c);
    }
    wf[idx] = __float2bfloat16_rn(v);
  }
}

// Every per-step weight preparation of a program in ONE launch (the bf16
// copies of the convolution weights, row-padded, and the flipped weights of
// the stride-1 data gradients).  The jobs' outputs form one flat space of
// 8-element units (every output row length is a multiple of 8); a thread
// finds its job by binary search over the jobs' first units and writes one
// 16-byte vector.  Same arithmetic as cast_rows_kernel / weight_flip_kernel
// (one rounding to bf16 per element).
constexpr int kPrepMaxJobs = 1024;

__global__ void __launch_bounds__(256)
prep_batch_kernel(const mgx_prep_job* __restrict__ jobs, int njobs, int64_t units) {
  __shared__ int64_t start[kPrepMaxJobs];
  for (int j = threadIdx.x; j < njobs; j += blockDim.x) start[j] = jobs[j].start;
  __syncthreads();
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t u = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; u < units; u += stride) {
    int lo = 0, hi = njobs - 1;  // last job with start <= u
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (start[mid] <= u) lo = mid;
      else hi = mid - 1;
    }
    const mgx_prep_job& jb = jobs[lo];
    const int64_t e0 = (u - start[lo]) * 8;  // first output element of the unit
    float v[8];
    if (jb.kind == 0) {
      // cast rows: dst[r, k] (rows x ldo) = src[r * ldi + k] for r < R, k < C, else 0
      const int64_t R = jb.a, C = jb.b, ldi = jb.c, ldo = jb.e;
      const int64_t r = e0 / ldo, k0 = e0 - r * ldo;
      const float* sp = jb.src + r * ldi + k0;
      if (r < R && k0 + 8 <= C && (reinterpret_cast<uintptr_t>(sp) & 15) == 0) {
        const float4 a = __ldg(reinterpret_cast<const float4*>(sp));
        const float4 c = __ldg(reinterpret_cast<const float4*>(sp) + 1);
        v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
        v[4] = c.x; v[5] = c.y; v[6] = c.z; v[7] = c.w;
      } else {
#pragma unroll
        for (int t = 0; t < 8; ++t)
          v[t] = r < R && k0 + t < C ? __ldg(jb.src + r * ldi + k0 + t) : 0.0f;
      }
    } else {
      // weight flip: dst[c, (i*kw + j)*F + f] (row stride ld) = w[f, kh-1-i, kw-1-j, c]
      const int F = static_cast<int>(jb.a), kh = static_cast<int>(jb.b);
      const int kw = static_cast<int>(jb.c), C = static_cast<int>(jb.d);
      const int64_t ld = jb.e;
      const int K = kh * kw * F;
      const int c = static_cast<int>(e0 / ld);
      const int kb = static_cast<int>(e0 - int64_t(c) * ld);
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const int k = kb + t;
        v[t] = 0.0f;
        if (k < K) {
          const int tap = k / F, f = k - tap * F;
          const int i = tap / kw, j = tap - (tap / kw) * kw;
          v[t] = __ldg(jb.src + ((int64_t(f) * kh + (kh - 1 - i)) * kw + (kw - 1 - j)) * C + c);
        }
      }
    }
    uint4 o;
    o.x = pack_bf16(v[0], v[1]);
    o.y = pack_bf16(v[2], v[3]);
    o.z = pack_bf16(v[4], v[5]);
    o.w = pack_bf16(v[6], v[7]);
    *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(jb.dst) + e0) = o;
  }
}

// ------------------------------------------------------- column reductions
// Per-channel sums over the M rows of an [M, C] matrix, in two fixed-order
// stages: block z reduces rows [z*rpc, (z+1)*rpc) into ws[z][*] (fp64), then
// one thread per channel merges the chunks in ascending z.
//   MODE 0: (sum x, sum x^2)             BatchNorm statistics
//   MODE 1: (sum dy, sum dy*xhat)         BatchNorm backward
//   MODE 2: (sum x)                       conv bias gradient
// xhat = (x - mean) * rstd with stats = [mean C | rstd C].

constexpr int kRedThreads = 256;
constexpr int kMaxChunks = 8 * kNumSMs;

// A ReLU fused in front of a BatchNorm backward: its mask is recomputed
// from the BatchNorm input with the forward's exact arithmetic,
// t = (x - mean) * rstd * gamma + beta > 0, instead of reading the ReLU
// output back.  beta == nullptr: no ReLU; gamma == nullptr: fix_gamma (1).
struct ReluMask {
  const float* gamma;
  const float* beta;
};

template <int MODE>
__global__ void __launch_bounds__(kRedThreads)
colreduce_partial_kernel(const float* __restrict__ a, const float* __restrict__ xs,
                         const float* __restrict__ stats, int64_t M, int C, int64_t rpc,
                         double* __restrict__ ws, ReluMask rm) {
  extern __shared__ double red[];  // [rpp][2*C]
  const int tpr = C < kRedThreads ? C : kRedThreads;  // threads per row
  const int rpp = kRedThreads / tpr;                  // rows per pass
  const int t = threadIdx.x;
  const int r_in = t / tpr, c_in = t - (t / tpr) * tpr;
  const int64_t r0 = int64_t(blockIdx.x) * rpc;
  const int64_t r1 = min(M, r0 + rpc);
  const int nchunk = gridDim.x;
  for (int cb = 0; cb < C; cb += tpr) {
    const int c = cb + c_in;
    double s0 = 0.0, s1 = 0.0;
    if (r_in < rpp && c < C) {
      float mean = 0.0f, rstd = 0.0f, shift = 0.0f, gm = 1.0f, bt = 0.0f;
      if (MODE == 1) {
        mean = __ldg(stats + c);
        rstd = __ldg(stats + C + c);
        if (rm.beta) {
          bt = __ldg(rm.beta + c);
          gm = rm.gamma ? __ldg(rm.gamma + c) : 1.0f;
        }
      }
      if (MODE == 0) shift = __ldg(a + c);  // row 0: shifted sums avoid cancellation
      for (int64_t r = r0 + r_in; r < r1; r += rpp) {
        float v = __ldg(a + r * C + c) - shift;
        if (MODE == 0) {
          s0 += v;
          s1 += double(v) * double(v);
        } else if (MODE == 1) {
          const float xv = __ldg(xs + r * C + c);
          if (rm.beta && !((xv - mean) * rstd * gm + bt > 0.0f)) v = 0.0f;
          s0 += v;
          s1 += double(v) * double((xv - mean) * rstd);
        } else {
          s0 += v;
        }
      }
    }
    if (r_in < rpp) {
      red[r_in * 2 * tpr + c_in] = s0;
      red[r_in * 2 * tpr + tpr + c_in] = s1;
    }
    __syncthreads();
    if (t < tpr && cb + t < C) {
      double u0 = 0.0, u1 = 0.0;
      for (int r = 0; r < rpp; ++r) {
        u0 += red[r * 2 * tpr + t];
        u1 += red[r * 2 * tpr + tpr + t];
      }
      ws[int64_t(blockIdx.x) * C + cb + t] = u0;
      ws[int64_t(nchunk + blockIdx.x) * C + cb + t] = u1;
    }
    __syncthreads();
  }
}

// Vectorised form (C % 4 == 0): a thread owns 4 channels (one float4 per
// row), keeps fp32 partial sums over its rows with kRedUnroll rows of loads
// in flight, then the block merges its threads' partials in fp64 in a fixed
// order.  blockIdx.y tiles channels in groups of 1024.
constexpr int kRedUnroll = 8;

template <int MODE>
__device__ __forceinline__ void red_accum(const float4& v, const float4& xv, const float* sh,
                                          const float* mu, const float* rs, const float* gm,
                                          const float* bt, bool relu, float* s0, float* s1) {
  const float* pv = &v.x;
  const float* px = &xv.x;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    if (MODE == 0) {
      const float d = pv[q] - sh[q];
      s0[q] += d;
      s1[q] += d * d;
    } else if (MODE == 1) {
      float d = pv[q];
      if (relu && !((px[q] - mu[q]) * rs[q] * gm[q] + bt[q] > 0.0f)) d = 0.0f;
      s0[q] += d;
      s1[q] += d * ((px[q] - mu[q]) * rs[q]);
    } else {
      s0[q] += pv[q];
    }
  }
}

template <int MODE>
__global__ void __launch_bounds__(kRedThreads)
colreduce_partial_vec_kernel(const float* __restrict__ a, const float* __restrict__ xs,
                             const float* __restrict__ stats, int64_t M, int C, int64_t rpc,
                             double* __restrict__ ws, ReluMask rm) {
  extern __shared__ double red[];  // [rpp][2][ct]
  const int C4 = C >> 2;
  const int ct4 = C4 < kRedThreads ? C4 : kRedThreads;  // float4 groups per block row
  const int rpp = kRedThreads / ct4;
  const int ct = ct4 * 4;
  const int t = threadIdx.x;
  const int r_in = t / ct4, c_in = t - (t / ct4) * ct4;
  const int c4 = blockIdx.y * ct4 + c_in;
  const bool active = r_in < rpp && c4 < C4;
  const int64_t r0 = int64_t(blockIdx.x) * rpc;
  const int64_t r1 = min(M, r0 + rpc);
  const float4* a4 = reinterpret_cast<const float4*>(a);
  const float4* x4 = reinterpret_cast<const float4*>(xs);
  const bool relu = MODE == 1 && rm.beta != nullptr;
  float s0[4] = {0.f, 0.f, 0.f, 0.f}, s1[4] = {0.f, 0.f, 0.f, 0.f};
  if (active) {
    float sh[4] = {0.f, 0.f, 0.f, 0.f}, mu[4] = {0.f, 0.f, 0.f, 0.f}, rs[4] = {0.f, 0.f, 0.f, 0.f};
    float gm[4] = {1.f, 1.f, 1.f, 1.f}, bt[4] = {0.f, 0.f, 0.f, 0.f};
    if (MODE == 0) {
      const float4 v = __ldg(a4 + c4);
      sh[0] = v.x; sh[1] = v.y; sh[2] = v.z; sh[3] = v.w;
    }
    if (MODE == 1) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int c = c4 * 4 + q;
        mu[q] = __ldg(stats + c);
        rs[q] = __ldg(stats + C + c);
        if (relu) {
          bt[q] = __ldg(rm.beta + c);
          gm[q] = rm.gamma ? __ldg(rm.gamma + c) : 1.0f;
        }
      }
    }
    // rounds of kRedUnroll guarded rows: a short chunk (the small layers'
    // few rows per thread) still has all its loads in flight at once
    for (int64_t r = r0 + r_in; r < r1; r += kRedUnroll * rpp) {
      float4 v[kRedUnroll], xv[kRedUnroll];
#pragma unroll
      for (int u = 0; u < kRedUnroll; ++u) {
        const int64_t rr = r + u * rpp;
        v[u] = rr < r1 ? __ldg(a4 + rr * C4 + c4) : make_float4(0.f, 0.f, 0.f, 0.f);
        if (MODE == 1) xv[u] = rr < r1 ? __ldg(x4 + rr * C4 + c4) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < kRedUnroll; ++u)
        if (r + u * rpp < r1)
          red_accum<MODE>(v[u], MODE == 1 ? xv[u] : v[u], sh, mu, rs, gm, bt, relu, s0, s1);
    }
  }
  if (r_in < rpp) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      red[(r_in * 2) * ct + c_in * 4 + q] = s0[q];
      red[(r_in * 2 + 1) * ct + c_in * 4 + q] = s1[q];
    }
  }
  __syncthreads();
  const int nchunk = gridDim.x;
  for (int c = t; c < ct; c += blockDim.x) {
    const int cg = blockIdx.y * ct + c;
    if (cg >= C) continue;
    double u0 = 0.0, u1 = 0.0;
    for (int rr = 0; rr < rpp; ++rr) {
      u0 += red[(rr * 2) * ct + c];
      u1 += red[(rr * 2 + 1) * ct + c];
    }
    ws[int64_t(blockIdx.x) * C + cg] = u0;
    ws[int64_t(nchunk + blockIdx.x) * C + cg] = u1;
  }
}

// Chunk merge shared by the finalize kernels: a warp per channel (8
// channels per 256-thread block); lane l sums chunks l, l+32, ... in
// ascending order, then the 32 lane sums meet in a fixed xor-butterfly tree
// (the same tree every run: deterministic).
constexpr int kFinChannels = 1;  // channels per 256-thread finalize block

__device__ __forceinline__ void merge_chunks(const double* __restrict__ ws, int nchunk, int C,
                                             int c, bool two, double* s_out, double* q_out) {
  // the whole block on one channel: thread t sums chunks t, t + 256, ...
  // (loads batched 8 deep, ascending), then a fixed xor tree per warp and
  // the 8 warp sums in warp order -- deterministic; valid in thread 0
  __shared__ double wsum[2][8];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  double s = 0.0, q = 0.0;
  if (c < C) {
    constexpr int B = 8;
    for (int z0 = t; z0 < nchunk; z0 += 256 * B) {
      double a[B], b[B];
#pragma unroll
      for (int u = 0; u < B; ++u) {
        const int z = z0 + 256 * u;
        a[u] = z < nchunk ? ws[int64_t(z) * C + c] : 0.0;
        b[u] = (two && z < nchunk) ? ws[int64_t(nchunk + z) * C + c] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < B; ++u) {
        s += a[u];
        q += b[u];
      }
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, off);
    q += __shfl_xor_sync(0xffffffffu, q, off);
  }
  if (lane == 0) {
    wsum[0][warp] = s;
    wsum[1][warp] = q;
  }
  __syncthreads();
  if (t == 0) {
    s = 0.0;
    q = 0.0;
    for (int w = 0; w < 8; ++w) {
      s += wsum[0][w];
      q += wsum[1][w];
    }
  }
  *s_out = s;
  *q_out = q;
}

// BatchNorm dx pass that also reduces its own output per channel (the
// gradient of the bias of the convolution feeding the BatchNorm): the row
// tiling of colreduce_partial_vec_kernel, dx written elementwise, fp32
// partial sums of dx merged per block in fp64 into ws[chunk][C].
// (dy may alias dx: each element is read before it is written.)
__device__ __forceinline__ float4 bn_dx4(const float4& d, const float4& xv, const float* mu,
                                         const float* rs, const float* g, const float* s1,
                                         const float* s2, const float* gm, const float* bt,
                                         bool relu, float invm) {
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
  }
  return o;
}

template <int PK = 0>
__global__ void __launch_bounds__(kRedThreads)
bn_dx_colsum_kernel(const float* dy, const float* __restrict__ x, const float* __restrict__ stats,
                    const float* __restrict__ sums, const float* __restrict__ gamma, float* dx,
                    ReluMask rm, int64_t M, int C, int64_t rpc, double* __restrict__ ws,
                    __nv_bfloat16* __restrict__ dx16, PoolGrad pg) {
  extern __shared__ double red[];  // [rpp][ct]
  const int C4 = C >> 2;
  const int ct4 = C4 < kRedThreads ? C4 : kRedThreads;
  const int rpp = kRedThreads / ct4;
  const int ct = ct4 * 4;
  const int t = threadIdx.x;
  const int r_in = t / ct4, c_in = t - (t / ct4) * ct4;
  const int c4 = blockIdx.y * ct4 + c_in;
  const bool active = r_in < rpp && c4 < C4;
  const int64_t r0 = int64_t(blockIdx.x) * rpc;
  const int64_t r1 = min(M, r0 + rpc);
  const float invm = static_cast<float>(1.0 / double(M));
  const bool relu = rm.beta != nullptr;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  if (active) {
    float mu[4], rs[4], g[4], s1[4], s2[4], gm[4], bt[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int c = c4 * 4 + q;
      mu[q] = __ldg(stats + c);
      rs[q] = __ldg(stats + C + c);
      g[q] = gamma ? __ldg(gamma + c) : 1.0f;
      s1[q] = __ldg(sums + c);
      s2[q] = __ldg(sums + C + c);
      gm[q] = relu && rm.gamma ? __ldg(rm.gamma + c) : 1.0f;
      bt[q] = relu ? __ldg(rm.beta + c) : 0.0f;
    }
    constexpr int U = 4;  // guarded rounds, all loads of a round in flight
    for (int64_t r = r0 + r_in; r < r1; r += U * rpp) {
      float4 d[U], xv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t rr = r + u * rpp;
        const int64_t i = rr * C4 + c4;
        if constexpr (PK != 0)
          d[u] = rr < r1 ? pool_grad4<PK>(pg, static_cast<int>(rr), c4, C4)
                         : make_float4(0.f, 0.f, 0.f, 0.f);
        else
          d[u] = rr < r1 ? reinterpret_cast<const float4*>(dy)[i] : make_float4(0.f, 0.f, 0.f, 0.f);
        xv[u] = rr < r1 ? __ldg(reinterpret_cast<const float4*>(x) + i)
                        : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t rr = r + u * rpp;
        if (rr >= r1) continue;
        const float4 o = bn_dx4(d[u], xv[u], mu, rs, g, s1, s2, gm, bt, relu, invm);
        acc[0] += o.x;
        acc[1] += o.y;
        acc[2] += o.z;
        acc[3] += o.w;
        if (dx) reinterpret_cast<float4*>(dx)[rr * C4 + c4] = o;
        if (dx16) {
          uint2 h;
          h.x = pack_bf16(o.x, o.y);
          h.y = pack_bf16(o.z, o.w);
          reinterpret_cast<uint2*>(dx16)[rr * C4 + c4] = h;
        }
      }
    }
  }
  if (r_in < rpp) {
#pragma unroll
    for (int q = 0; q < 4; ++q) red[r_in * ct + c_in * 4 + q] = acc[q];
  }
  __syncthreads();
  for (int c = t; c < ct; c += blockDim.x) {
    const int cg = blockIdx.y * ct + c;
    if (cg >= C) continue;
    double u = 0.0;
    for (int rr = 0; rr < rpp; ++rr) u += red[rr * ct + c];
    ws[int64_t(blockIdx.x) * C + cg] = u;
  }
}

// MODE 0 finalize: stats = [mean | rstd] (batch statistics, biased variance
// like MXNet), moving averages updated when given.
// use_global: stats from the moving averages (inference).
__global__ void bn_stats_finalize_kernel(const double* __restrict__ ws, int nchunk, int64_t M, int C,
                                         const float* __restrict__ x, float eps, float momentum,
                                         int use_global,
                                         float* __restrict__ stats, float* __restrict__ mmean,
                                         float* __restrict__ mvar) {
  const int c = blockIdx.x;
  if (use_global) {
    if (threadIdx.x == 0 && c < C) {
      stats[c] = mmean[c];
      stats[C + c] = static_cast<float>(1.0 / sqrt(double(mvar[c]) + double(eps)));
    }
    return;
  }
  double s = 0.0, q = 0.0;
  merge_chunks(ws, nchunk, C, c, true, &s, &q);
  if (threadIdx.x != 0 || c >= C) return;
  // sums were taken relative to shift = x[0, c]
  const double dm = s / double(M);
  const double mean = double(x[c]) + dm;
  double var = q / double(M) - dm * dm;
  if (var < 0.0) var = 0.0;
  stats[c] = static_cast<float>(mean);
  stats[C + c] = static_cast<float>(1.0 / sqrt(var + double(eps)));
  if (mmean) mmean[c] = static_cast<float>(double(mmean[c]) * momentum + mean * (1.0 - momentum));
  if (mvar) mvar[c] = static_cast<float>(double(mvar[c]) * momentum + var * (1.0 - momentum));
}

// BatchNorm statistics from the GEMM epilogue's per-32-row (mean, M2)
// pairs of the convolution output: a 1024-thread block per channel; thread
// t sums tiles t, t + 1024, ... (loads batched 8 deep) as shifted sums
// against tile 0's mean -- S1 = sum n_t (mean_t - s), S2 = sum [M2_t +
// n_t (mean_t - s)^2] in fp64, no divisions -- then a fixed xor tree per warp
// and the 32 warp sums in warp order (deterministic):
//   mean = s + S1 / M,  var = S2 / M - (S1 / M)^2.
__global__ void __launch_bounds__(1024)
bn_stats_from_tiles_kernel(const float2* __restrict__ part, int64_t M, int C, float eps,
                           float momentum, float* __restrict__ stats,
                           float* __restrict__ mmean, float* __restrict__ mvar) {
  __shared__ double ws1[32], ws2[32];
  const int c = blockIdx.x;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int nb = static_cast<int>((M + 31) / 32);
  const double sh = double(part[c].x);
  double s1 = 0.0, s2 = 0.0;
  constexpr int B = 8;
  for (int b0 = t; b0 < nb; b0 += 1024 * B) {
    float2 p[B];
#pragma unroll
    for (int u = 0; u < B; ++u) {
      const int b = b0 + 1024 * u;
      p[u] = b < nb ? part[int64_t(b) * C + c] : make_float2(0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < B; ++u) {
      const int b = b0 + 1024 * u;
      if (b >= nb) continue;
      const int64_t left = M - int64_t(b) * 32;
      const double n = double(left < 32 ? left : 32);
      const double d = double(p[u].x) - sh;
      s1 += n * d;
      s2 += double(p[u].y) + n * d * d;
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    s1 += __shfl_xor_sync(0xffffffffu, s1, off);
    s2 += __shfl_xor_sync(0xffffffffu, s2, off);
  }
  if (lane == 0) {
    ws1[warp] = s1;
    ws2[warp] = s2;
  }
  __syncthreads();
  if (t == 0) {
    double a1 = 0.0, a2 = 0.0;
    for (int w = 0; w < 32; ++w) {
      a1 += ws1[w];
      a2 += ws2[w];
    }
    const double dm = a1 / double(M);
    const double mean = sh + dm;
    double var = a2 / double(M) - dm * dm;
    if (var < 0.0) var = 0.0;
    stats[c] = static_cast<float>(mean);
    stats[C + c] = static_cast<float>(1.0 / sqrt(var + double(eps)));
    if (mmean) mmean[c] = static_cast<float>(double(mmean[c]) * momentum + mean * (1.0 - momentum));
    if (mvar) mvar[c] = static_cast<float>(double(mvar[c]) * momentum + var * (1.0 - momentum));
  }
}

// The same statistics with coalesced reads over more SMs: a cluster of CS
// CTAs per 32-channel group, the row blocks split contiguously over the
// cluster's CTAs; in a CTA lane = channel (each warp load is 256 contiguous
// bytes of one row block) and warp w takes blocks w, w + 32, ... in order;
// warp sums merged in warp order, then the CS CTA sums in rank order over
// distributed shared memory by rank 0 (deterministic).  The per-block
// terms are bn_stats_from_tiles_kernel's (shift = tile 0's mean).
template <int CS>
__global__ void __launch_bounds__(1024)
bn_stats_tiles_cluster_kernel(const float2* __restrict__ part, int64_t M, int C, float eps,
                              float momentum, float* __restrict__ stats,
                              float* __restrict__ mmean, float* __restrict__ mvar) {
  namespace cg = cooperative_groups;
  __shared__ double red[2][32][33];
  __shared__ double tot[2][32];
  cg::cluster_group cl = cg::this_cluster();
  const int rank = static_cast<int>(cl.block_rank());
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = blockIdx.y * 32 + lane;
  const bool cv = c < C;
  const int64_t nb = (M + 31) / 32;
  const double sh = cv ? double(part[c].x) : 0.0;
  const int64_t per = (nb + CS - 1) / CS;
  const int64_t b_lo = rank * per, b_hi = b_lo + per < nb ? b_lo + per : nb;
  double s1 = 0.0, s2 = 0.0;
  constexpr int U = 8;
  for (int64_t b0 = b_lo + warp; b0 < b_hi; b0 += 32 * U) {
    float2 p[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t b = b0 + 32 * u;
      p[u] = (cv && b < b_hi) ? part[b * C + c] : make_float2(0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t b = b0 + 32 * u;
      if (!cv || b >= b_hi) continue;
      const int64_t left = M - b * 32;
      const double n = double(left < 32 ? left : 32);
      const double d = double(p[u].x) - sh;
      s1 += n * d;
      s2 += double(p[u].y) + n * d * d;
    }
  }
  red[0][warp][lane] = s1;
  red[1][warp][lane] = s2;
  __syncthreads();
  if (threadIdx.x < 64) {
    const int k = threadIdx.x >> 5, ch = threadIdx.x & 31;
    double a = 0.0;
    for (int w = 0; w < 32; ++w) a += red[k][w][ch];
    tot[k][ch] = a;
  }
  cl.sync();
  if (rank == 0 && threadIdx.x < 32 && cv) {
    double a1 = 0.0, a2 = 0.0;
    for (int r = 0; r < CS; ++r) {
      const double* t = cl.map_shared_rank(&tot[0][0], r);
      a1 += t[lane];
      a2 += t[32 + lane];
    }
    const double dm = a1 / double(M);
    const double mean = sh + dm;
    double var = a2 / double(M) - dm * dm;
    if (var < 0.0) var = 0.0;
    stats[c] = static_cast<float>(mean);
    stats[C + c] = static_cast<float>(1.0 / sqrt(var + double(eps)));
    if (mmean) mmean[c] = static_cast<float>(double(mmean[c]) * momentum + mean * (1.0 - momentum));
    if (mvar) mvar[c] = static_cast<float>(double(mvar[c]) * momentum + var * (1.0 - momentum));
  }
  cl.sync();  // peers' tot stays alive until rank 0 has read it
}

// ---- stem fusion, backward reductions over the pooling WINDOWS: only the
// argmax position of each window receives gradient, so
//   s1 = sum_p mask(p) og(p)        = sum_windows mask(p*) dy(w)
//   s2 = sum_p mask(p) og(p) xhat(p) = sum_windows mask(p*) dy(w) xhat(p*)
// with p* the window's argmax: the pooled gradient, the argmax and one x
// element per window and channel are read -- the full-resolution gradient
// is never formed.  Rows = windows (B Ho Wo), tiled like
// colreduce_partial_vec_kernel; partials per chunk into ws (same layout, so
// colsum_finalize_kernel merges them).
template <int MINB, int U = 4>
__global__ void __launch_bounds__(kRedThreads, MINB)
bn_pool_reduce_kernel(PoolGrad pg, const float* __restrict__ x, const float* __restrict__ stats,
                      ReluMask rm, int64_t Mp, int C, int64_t rpc, double* __restrict__ ws,
                      uint32_t mkw, uint64_t mul_howo, uint64_t mul_wo) {
  extern __shared__ double red[];  // [rpp][2][ct]
  const Geom& g = pg.g;
  const int C4 = C >> 2;
  const int ct4 = C4 < kRedThreads ? C4 : kRedThreads;
  const int rpp = kRedThreads / ct4;
  const int ct = ct4 * 4;
  const int t = threadIdx.x;
  const int r_in = t / ct4, c_in = t - (t / ct4) * ct4;
  const int c4 = blockIdx.y * ct4 + c_in;
  const bool active = r_in < rpp && c4 < C4;
  const int64_t r0 = int64_t(blockIdx.x) * rpc;
  const int64_t r1 = min(Mp, r0 + rpc);
  const bool relu = rm.beta != nullptr;
  float s0[4] = {0.f, 0.f, 0.f, 0.f}, s1[4] = {0.f, 0.f, 0.f, 0.f};
  if (active) {
    float mu[4], rs[4], gm[4], bt[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int c = c4 * 4 + q;
      mu[q] = __ldg(stats + c);
      rs[q] = __ldg(stats + C + c);
      gm[q] = relu && rm.gamma ? __ldg(rm.gamma + c) : 1.0f;
      bt[q] = relu ? __ldg(rm.beta + c) : 0.0f;
    }
    const int howo = g.Ho * g.Wo;
    for (int64_t r = r0 + r_in; r < r1; r += U * rpp) {
      float4 d[U];
      uchar4 am[U];
      float xv[U][4];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t rr = r + u * rpp;
        const bool ok = rr < r1;
        d[u] = ok ? __ldg(pg.dy + rr * C4 + c4) : make_float4(0.f, 0.f, 0.f, 0.f);
        am[u] = ok ? __ldg(pg.arg + rr * C4 + c4) : make_uchar4(0, 0, 0, 0);
        const int ri = static_cast<int>(ok ? rr : r0);
        const int b = pg_div(ri, mul_howo);
        const int rem = ri - b * howo;
        const int oh = pg_div(rem, mul_wo), ow = rem - oh * g.Wo;
        const float* xb = x + (int64_t(b) * g.H * g.W) * C + c4 * 4;
        const unsigned char* pa = &am[u].x;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int li = pa[q];
          const int ti = static_cast<int>((uint32_t(li) * mkw) >> 16), tj = li - ti * g.kw;
          const int h = oh * g.sh - g.ph + ti, w = ow * g.sw - g.pw + tj;
          xv[u][q] = ok ? __ldg(xb + (int64_t(h) * g.W + w) * C + q) : 0.0f;
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (r + u * rpp >= r1) continue;
        const float* pd = &d[u].x;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          float dq = pd[q];
          if (relu && !((xv[u][q] - mu[q]) * rs[q] * gm[q] + bt[q] > 0.0f)) dq = 0.0f;
          s0[q] += dq;
          s1[q] += dq * ((xv[u][q] - mu[q]) * rs[q]);
        }
      }
    }
  }
  if (r_in < rpp) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      red[(r_in * 2) * ct + c_in * 4 + q] = s0[q];
      red[(r_in * 2 + 1) * ct + c_in * 4 + q] = s1[q];
    }
  }
  __syncthreads();
  const int nchunk = gridDim.x;
  for (int c = t; c < ct; c += blockDim.x) {
    const int cg = blockIdx.y * ct + c;
    if (cg >= C) continue;
    double u0 = 0.0, u1 = 0.0;
    for (int rr = 0; rr < rpp; ++rr) {
      u0 += red[(rr * 2) * ct + c];
      u1 += red[(rr * 2 + 1) * ct + c];
    }
    ws[int64_t(blockIdx.x) * C + cg] = u0;
    ws[int64_t(nchunk + blockIdx.x) * C + cg] = u1;
  }
}

// ---- stem fusion, BatchNorm dx through a 3x3 / stride 2 / pad 0 max
// pooling: a thread owns a 2x2 pixel block (rows = blocks) and 4 channels;
// exactly 4 windows cover such a block ((a-1 | a) x (b-1 | b) for block
// (a, b)), so 4 pooled-gradient and argmax loads give the output gradient of
// all 4 pixels (summed in ascending (oh, ow) order like pool_bwd_vec_kernel);
// then dx = gamma rstd (mask og - (s1 + xhat s2) / M) -> dx16, and the
// per-chunk partial sums of dx (conv bias gradient) into ws.
template <int MINB, int UNR = 2>
__global__ void __launch_bounds__(kRedThreads, MINB)
bn_pool_dx_k3s2_kernel(PoolGrad pg, const float* __restrict__ x, const float* __restrict__ stats,
                       const float* __restrict__ sums, const float* __restrict__ gamma,
                       ReluMask rm, int64_t M, int64_t Mb, int C, int64_t rpc,
                       double* __restrict__ ws, __nv_bfloat16* __restrict__ dx16,
                       uint64_t mul_blk, uint64_t mul_wb) {
  extern __shared__ double red[];  // [rpp][ct]
  const Geom& g = pg.g;
  const int C4 = C >> 2;
  const int ct4 = C4 < kRedThreads ? C4 : kRedThreads;
  const int rpp = kRedThreads / ct4;
  const int ct = ct4 * 4;
  const int t = threadIdx.x;
  const int r_in = t / ct4, c_in = t - (t / ct4) * ct4;
  const int c4 = blockIdx.y * ct4 + c_in;
  const bool active = r_in < rpp && c4 < C4;
  const int64_t r0 = int64_t(blockIdx.x) * rpc;
  const int64_t r1 = min(Mb, r0 + rpc);
  const float invm = static_cast<float>(1.0 / double(M));
  const bool relu = rm.beta != nullptr;
  const int Hb = (g.H + 1) >> 1, Wb = (g.W + 1) >> 1;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  if (active) {
    float mu[4], rs[4], gg[4], s1[4], s2[4], gm[4], bt[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int c = c4 * 4 + q;
      mu[q] = __ldg(stats + c);
      rs[q] = __ldg(stats + C + c);
      gg[q] = gamma ? __ldg(gamma + c) : 1.0f;
      s1[q] = __ldg(sums + c);
      s2[q] = __ldg(sums + C + c);
      gm[q] = relu && rm.gamma ? __ldg(rm.gamma + c) : 1.0f;
      bt[q] = relu ? __ldg(rm.beta + c) : 0.0f;
    }
#pragma unroll(UNR)
    for (int64_t r = r0 + r_in; r < r1; r += rpp) {
      const int ri = static_cast<int>(r);
      const int b = pg_div(ri, mul_blk);
      const int rem = ri - b * Hb * Wb;
      const int ba = pg_div(rem, mul_wb), bb = rem - ba * Wb;
      // the 4 covering windows (a-1, b-1), (a-1, b), (a, b-1), (a, b)
      float4 d[4];
      uchar4 am[4];
#pragma unroll
      for (int wi = 0; wi < 4; ++wi) {
        const int oh = ba - 1 + (wi >> 1), ow = bb - 1 + (wi & 1);
        const bool ok = oh >= 0 && oh < g.Ho && ow >= 0 && ow < g.Wo;
        const int64_t o = ((int64_t(b) * g.Ho + oh) * g.Wo + ow) * C4 + c4;
        d[wi] = ok ? __ldg(pg.dy + o) : make_float4(0.f, 0.f, 0.f, 0.f);
        am[wi] = ok ? __ldg(pg.arg + o) : make_uchar4(255, 255, 255, 255);
      }
      // the block's 4 pixels of x, loaded together with the windows' loads
      float4 xq[4];
      bool pin[4];
#pragma unroll
      for (int pi = 0; pi < 4; ++pi) {
        const int h = 2 * ba + (pi >> 1), w = 2 * bb + (pi & 1);
        pin[pi] = h < g.H && w < g.W;
        const int64_t i = ((int64_t(b) * g.H + h) * g.W + w) * C4 + c4;
        xq[pi] = pin[pi] ? __ldg(reinterpret_cast<const float4*>(x) + i)
                         : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int pi = 0; pi < 4; ++pi) {
        const int dh = pi >> 1, dw = pi & 1;
        const int h = 2 * ba + dh, w = 2 * bb + dw;
        if (!pin[pi]) continue;
        const int64_t i = ((int64_t(b) * g.H + h) * g.W + w) * C4 + c4;
        const float4 xv = xq[pi];
        const float* px = &xv.x;
        float og[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int wi = 0; wi < 4; ++wi) {
          const int wh = wi >> 1, ww = wi & 1;
          // window (a-1+wh, b-1+ww) covers this pixel at local (h - 2oh, w - 2ow)
          const int lh = 2 - 2 * wh + dh, lw = 2 - 2 * ww + dw;  // 2*(a - oh) + dh
          if (lh > 2 || lw > 2) continue;
          const int li = lh * 3 + lw;
          const float* pd = &d[wi].x;
          const unsigned char* pa = &am[wi].x;
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (pa[q] == li) og[q] = fadd(og[q], pd[q]);
        }
        float o[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          float dq = og[q];
          if (relu && !((px[q] - mu[q]) * rs[q] * gm[q] + bt[q] > 0.0f)) dq = 0.0f;
          const float xhat = (px[q] - mu[q]) * rs[q];
          o[q] = gg[q] * rs[q] * (dq - (s1[q] + xhat * s2[q]) * invm);
          acc[q] += o[q];
        }
        uint2 hv;
        hv.x = pack_bf16(o[0], o[1]);
        hv.y = pack_bf16(o[2], o[3]);
        reinterpret_cast<uint2*>(dx16)[i] = hv;
      }
    }
  }
  if (r_in < rpp) {
#pragma unroll
    for (int q = 0; q < 4; ++q) red[r_in * ct + c_in * 4 + q] = acc[q];
  }
  __syncthreads();
  for (int c = t; c < ct; c += blockDim.x) {
    const int cg = blockIdx.y * ct + c;
    if (cg >= C) continue;
    double u = 0.0;
    for (int rr = 0; rr < rpp; ++rr) u += red[rr * ct + c];
    ws[int64_t(blockIdx.x) * C + cg] = u;
  }
}

// MODE 1/2 finalize: out[c] = sum0, out[C + c] = sum1 (MODE 1) as fp32;
// optionally also straight into gradient buffers: out0[c] = sum0 and
// out1[c] = sum1 (or 0 when zero1: BatchNorm's fix_gamma)
__global__ void colsum_finalize_kernel(const double* __restrict__ ws, int nchunk, int C, int two,
                                       float* __restrict__ out, float* __restrict__ out0,
                                       float* __restrict__ out1, int zero1) {
  const int c = blockIdx.x;
  double s = 0.0, q = 0.0;
  merge_chunks(ws, nchunk, C, c, two != 0, &s, &q);
  if (threadIdx.x != 0 || c >= C) return;
  out[c] = static_cast<float>(s);
  if (two) out[C + c] = static_cast<float>(q);
  if (out0) out0[c] = static_cast<float>(s);
  if (out1) out1[c] = zero1 ? 0.0f : static_cast<float>(q);
}

// y = (x - mean) * rstd * gamma + beta, then act; gamma == nullptr: fixed 1
__global__ void bn_apply_kernel(const float* __restrict__ x, const float* __restrict__ stats,
                                const float* __restrict__ gamma, const float* __restrict__ beta,
                                float* __restrict__ y, int64_t M, int C, int act,
                                __nv_bfloat16* __restrict__ y16, int64_t ldo4) {
  const int64_t total = M * C;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  if ((C & 3) == 0) {
    // launched with the rows x vectors shape: per-channel constants once
    const int C4 = C >> 2;
    const RowsIdx ri(C4);
    if (!ri.active) return;
    const int c4 = ri.v;
    float mu[4], sc[4], bt[4], gm[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int cc = c4 * 4 + u;
      const float g = gamma ? __ldg(gamma + cc) : 1.0f;
      mu[u] = __ldg(stats + cc);
      sc[u] = __ldg(stats + C + cc);
      gm[u] = g;
      bt[u] = __ldg(beta + cc);
    }
    // outputs may be channel slices of a wider tensor (row stride ldo4)
    auto one = [&](float4 v, int64_t row) {
      const int64_t i = row * ldo4 + c4;
      float* pv = &v.x;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float t = (pv[u] - mu[u]) * sc[u] * gm[u] + bt[u];
        pv[u] = act == MGX_ACT_RELU ? relu(t) : act_forward(act, t);
      }
      if (y) reinterpret_cast<float4*>(y)[i] = v;
      if (y16) {
        uint2 h;
        h.x = pack_bf16(v.x, v.y);
        h.y = pack_bf16(v.z, v.w);
        reinterpret_cast<uint2*>(y16)[i] = h;
      }
    };
    constexpr int U = 4;  // rows in flight per thread
    int64_t r = ri.r;
    for (; r + (U - 1) * int64_t(ri.rstep) < M; r += U * int64_t(ri.rstep)) {
      float4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = __ldg(reinterpret_cast<const float4*>(x) + (r + u * int64_t(ri.rstep)) * C4 + c4);
#pragma unroll
      for (int u = 0; u < U; ++u) one(v[u], r + u * int64_t(ri.rstep));
    }
    for (; r < M; r += ri.rstep) one(__ldg(reinterpret_cast<const float4*>(x) + r * C4 + c4), r);
  } else {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += stride) {
      const int c = static_cast<int>(i % C);
      const float g = gamma ? __ldg(gamma + c) : 1.0f;
      y[i] = act_forward(act, (x[i] - __ldg(stats + c)) * __ldg(stats + C + c) * g + __ldg(beta + c));
    }
  }
}

// dx = gamma * rstd * (dy - (sum_dy + xhat * sum_dyxhat) / M), with an
// optional fused ReLU (mask recomputed from x).  dy may alias dx.
__global__ void bn_bwd_dx_kernel(const float* dy, const float* __restrict__ x,
                                 const float* __restrict__ stats, const float* __restrict__ sums,
                                 const float* __restrict__ gamma, float* dx, int64_t M, int C,
                                 ReluMask rm) {
  const int64_t total = M * C;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  const float invm = static_cast<float>(1.0 / double(M));
  const bool relu = rm.beta != nullptr;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += stride) {
    const int c = static_cast<int>(i % C);
    const float rstd = __ldg(stats + C + c);
    const float mean = __ldg(stats + c);
    const float xv = x[i];
    const float xhat = (xv - mean) * rstd;
    const float g = gamma ? __ldg(gamma + c) : 1.0f;
    float d = dy[i];
    if (relu) {
      const float gm = rm.gamma ? __ldg(rm.gamma + c) : 1.0f;
      if (!((xv - mean) * rstd * gm + __ldg(rm.beta + c) > 0.0f)) d = 0.0f;
    }
    dx[i] = g * rstd * (d - (__ldg(sums + c) + xhat * __ldg(sums + C + c)) * invm);
  }
}

// ------------------------------------------------------------------ pooling
// MXNet pooling semantics: max ignores padding; avg divides by the window
// area clipped to the padded extent (count_include_pad); 'full' convention
// rounds the output size up.

__device__ __forceinline__ float pool_area(const Geom& g, int oh, int ow) {
  const int hs = oh * g.sh - g.ph, ws = ow * g.sw - g.pw;
  const int he = min(hs + g.kh, g.H + g.ph), we = min(ws + g.kw, g.W + g.pw);
  return static_cast<float>((he - hs) * (we - ws));
}

__global__ void pool_fwd_kernel(const float* __restrict__ x, float* __restrict__ y, Geom g,
                                int type) {
  const int64_t total = int64_t(g.B) * g.Ho * g.Wo * g.C;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; idx < total; idx += stride) {
    const int c = static_cast<int>(idx % g.C);
    int64_t p = idx / g.C;
    const int ow = static_cast<int>(p % g.Wo);
    p /= g.Wo;
    const int oh = static_cast<int>(p % g.Ho);
    const int b = static_cast<int>(p / g.Ho);
    const int hs = oh * g.sh - g.ph, ws = ow * g.sw - g.pw;
    const int h0 = max(hs, 0), w0 = max(ws, 0);
    const int h1 = min(hs + g.kh, g.H), w1 = min(ws + g.kw, g.W);
    float acc = type == 0 ? -INFINITY : 0.0f;
    for (int h = h0; h < h1; ++h)
      for (int w = w0; w < w1; ++w) {
        const float v = __ldg(x + ((int64_t(b) * g.H + h) * g.W + w) * g.C + c);
        acc = type == 0 ? (v > acc ? v : acc) : fadd(acc, v);
      }
    y[idx] = type == 0 ? acc : fdiv(acc, pool_area(g, oh, ow));
  }
}

// dx gathered from every window covering the input position.  Max: the
// gradient goes to the FIRST position (row-major window scan, strict >)
// holding the window maximum, like MXNet's unpool; avg: dy / area.
__global__ void pool_bwd_kernel(const float* __restrict__ x, const float* __restrict__ y,
                                const float* __restrict__ dy, float* __restrict__ dx, Geom g,
                                int type) {
  const int64_t total = int64_t(g.B) * g.H * g.W * g.C;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; idx < total; idx += stride) {
    const int c = static_cast<int>(idx % g.C);
    int64_t p = idx / g.C;
    const int w = static_cast<int>(p % g.W);
    p /= g.W;
    const int h = static_cast<int>(p % g.H);
    const int b = static_cast<int>(p / g.H);
    const float xv = type == 0 ? x[idx] : 0.0f;
    // output windows covering h: oh*sh - ph <= h < oh*sh - ph + kh
    const int nh = h + g.ph - g.kh + 1, nw = w + g.pw - g.kw + 1;
    const int oh_lo = nh <= 0 ? 0 : (nh + g.sh - 1) / g.sh;
    const int oh_hi = min(g.Ho - 1, (h + g.ph) / g.sh);
    const int ow_lo = nw <= 0 ? 0 : (nw + g.sw - 1) / g.sw;
    const int ow_hi = min(g.Wo - 1, (w + g.pw) / g.sw);
    float acc = 0.0f;
    for (int oh = oh_lo; oh <= oh_hi; ++oh) {
      const int hs = oh * g.sh - g.ph;
      if (h < hs || h >= hs + g.kh) continue;
      for (int ow = ow_lo; ow <= ow_hi; ++ow) {
        const int ws = ow * g.sw - g.pw;
        if (w < ws || w >= ws + g.kw) continue;
        const int64_t o = ((int64_t(b) * g.Ho + oh) * g.Wo + ow) * g.C + c;
        if (type == 0) {
          const float yv = __ldg(y + o);
          if (xv != yv) continue;
          // first max: no earlier valid window position holds yv
          bool first = true;
          const int h0 = max(hs, 0), w0 = max(ws, 0), w1 = min(ws + g.kw, g.W);
          for (int hh = h0; hh <= h && first; ++hh) {
            const int wend = hh < h ? w1 : w;
            for (int ww = w0; ww < wend; ++ww)
              if (__ldg(x + ((int64_t(b) * g.H + hh) * g.W + ww) * g.C + c) == yv) {
                first = false;
                break;
              }
          }
          if (first) acc = fadd(acc, __ldg(dy + o));
        } else {
          acc = fadd(acc, fdiv(__ldg(dy + o), pool_area(g, oh, ow)));
        }
      }
    }
    dx[idx] = acc;
  }
}

// Channel-vectorised pooling (C % 4 == 0): a thread owns 4 channels of one
// output (forward) or input (backward) pixel, items enumerated linearly over
// (pixel, channel vector) so no lane idles whatever C is.  Max pooling
// records the window-local index of the first maximum (uint8, row-major in
// the window) so the backward is a cheap gather: dx(h,w) = sum of dy over the
// windows whose recorded argmax is (h,w), windows in ascending (oh, ow)
// order.  K, S > 0: a square K x K window with stride S known at compile
// time (the 3x3 / stride 1-2 poolings of the nets): every tap / covering
// window is unrolled with bounds predicates so all loads of a pixel are in
// flight at once; K == 0: runtime geometry.  TYPE 0 max, 1 avg.
// BN: the pooled values are act(BatchNorm(x)) computed on the fly from the
// BatchNorm input x (stem fusion: BatchNorm + ReLU + pooling in one pass;
// the normalised tensor is never written)
struct BnAct {
  const float* stats;  // [mean C | rstd C]
  const float* gamma;  // NULL: 1
  const float* beta;
  int act;
};

template <int K, int S, int TYPE, bool BN = false, int MINB = 1>
__global__ void __launch_bounds__(256, MINB)
pool_fwd_vec_kernel(const float* __restrict__ x, float* __restrict__ y,
                    uint8_t* __restrict__ arg, Geom g, __nv_bfloat16* __restrict__ y16,
                    BnAct bn = BnAct{}) {
  const int C4 = g.C >> 2;
  const int kh = K ? K : g.kh, kw = K ? K : g.kw;
  const int sh = K ? S : g.sh, sw = K ? S : g.sw;
  const int hw = g.Ho * g.Wo;
  const int64_t total = int64_t(g.B) * hw * C4;
  const int64_t step = int64_t(gridDim.x) * blockDim.x;
  const float4* x4 = reinterpret_cast<const float4*>(x);
  for (int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; idx < total; idx += step) {
    const int pix = static_cast<int>(idx / C4);
    const int c4 = static_cast<int>(idx - int64_t(pix) * C4);
    const int b = pix / hw;
    const int rem = pix - b * hw;
    const int oh = rem / g.Wo, ow = rem - (rem / g.Wo) * g.Wo;
    const int hs = oh * sh - g.ph, ws = ow * sw - g.pw;
    float acc[4];
    int ai[4] = {0, 0, 0, 0};
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[q] = TYPE == 0 ? -INFINITY : 0.0f;
    float4 mu4, rs4, gm4, bt4;
    if constexpr (BN) {
      mu4 = __ldg(reinterpret_cast<const float4*>(bn.stats) + c4);
      rs4 = __ldg(reinterpret_cast<const float4*>(bn.stats + g.C) + c4);
      gm4 = bn.gamma ? __ldg(reinterpret_cast<const float4*>(bn.gamma) + c4)
                     : make_float4(1.f, 1.f, 1.f, 1.f);
      bt4 = __ldg(reinterpret_cast<const float4*>(bn.beta) + c4);
    }
    auto tap = [&](float4 v, int li) {
      if constexpr (BN) {  // the same arithmetic as bn_apply_kernel
        const float* pm = &mu4.x;
        const float* pr = &rs4.x;
        const float* pgm = &gm4.x;
        const float* pb = &bt4.x;
        float* pw_ = &v.x;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float t = (pw_[q] - pm[q]) * pr[q] * pgm[q] + pb[q];
          pw_[q] = bn.act == MGX_ACT_RELU ? relu(t) : act_forward(bn.act, t);
        }
      }
      const float* pv = &v.x;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (TYPE == 0) {
          if (pv[q] > acc[q]) {
            acc[q] = pv[q];
            ai[q] = li;
          }
        } else {
          acc[q] = fadd(acc[q], pv[q]);
        }
      }
    };
    const float4* xb = x4 + int64_t(b) * g.H * g.W * C4 + c4;
    if constexpr (K > 0) {
      float4 v[K * K];
      bool ok[K * K];
#pragma unroll
      for (int i = 0; i < K; ++i)
#pragma unroll
        for (int j = 0; j < K; ++j) {
          const int h = hs + i, w = ws + j;
          ok[i * K + j] = h >= 0 && h < g.H && w >= 0 && w < g.W;
          v[i * K + j] = ok[i * K + j] ? __ldg(xb + (int64_t(h) * g.W + w) * C4)
                                       : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
      for (int t = 0; t < K * K; ++t)
        if (ok[t]) tap(v[t], t);
    } else {
      const int h0 = max(hs, 0), w0 = max(ws, 0);
      const int h1 = min(hs + kh, g.H), w1 = min(ws + kw, g.W);
      for (int h = h0; h < h1; ++h)
        for (int w = w0; w < w1; ++w)
          tap(__ldg(xb + (int64_t(h) * g.W + w) * C4), (h - hs) * kw + (w - ws));
    }
    float4 o;
    if (TYPE == 0) {
      o = make_float4(acc[0], acc[1], acc[2], acc[3]);
      if (arg) reinterpret_cast<uchar4*>(arg)[idx] = make_uchar4(ai[0], ai[1], ai[2], ai[3]);
    } else {
      const float inv = __frcp_rn(pool_area(g, oh, ow));
      o = make_float4(acc[0] * inv, acc[1] * inv, acc[2] * inv, acc[3] * inv);
    }
    if (y) reinterpret_cast<float4*>(y)[idx] = o;
    if (y16) {
      uint2 h;
      h.x = pack_bf16(o.x, o.y);
      h.y = pack_bf16(o.z, o.w);
      reinterpret_cast<uint2*>(y16)[idx] = h;
    }
  }
}

// The stem's BatchNorm + ReLU + 3x3 / stride-2 / pad-0 max pooling, two
// horizontally adjacent outputs per thread: their windows share a column,
// so 15 loads and 15 BatchNorm transforms serve 18 taps (vs 18 of each),
// 32-bit indexing throughout.  Same arithmetic and tap order as
// pool_fwd_vec_kernel<3, 2, 0, true> (bitwise).
__global__ void __launch_bounds__(256, 2)
bn_relu_maxpool3s2_kernel(const float4* __restrict__ x, float4* __restrict__ y,
                          uchar4* __restrict__ arg, Geom g, uint2* __restrict__ y16, BnAct bn) {
  const int C4 = g.C >> 2;
  const int wp = (g.Wo + 1) >> 1;  // output pairs per row
  const int total = g.B * g.Ho * wp * C4;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += gridDim.x * blockDim.x) {
    const int c4 = idx % C4;
    const int pp = idx / C4;
    const int owp = pp % wp;
    const int bo = pp / wp;
    const int oh = bo % g.Ho, b = bo / g.Ho;
    const int hs = oh * 2, ws = owp * 4;
    const float4 mu4 = __ldg(reinterpret_cast<const float4*>(bn.stats) + c4);
    const float4 rs4 = __ldg(reinterpret_cast<const float4*>(bn.stats + g.C) + c4);
    const float4 gm4 = bn.gamma ? __ldg(reinterpret_cast<const float4*>(bn.gamma) + c4)
                                : make_float4(1.f, 1.f, 1.f, 1.f);
    const float4 bt4 = __ldg(reinterpret_cast<const float4*>(bn.beta) + c4);
    const float4* xb = x + (b * g.H + hs) * g.W * C4 + c4;
    float4 v[3][5];
    bool okc[5];
#pragma unroll
    for (int j = 0; j < 5; ++j) okc[j] = ws + j < g.W;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 5; ++j)
        v[i][j] = okc[j] ? __ldg(xb + (i * g.W + ws + j) * C4) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 5; ++j) {
        float* pv = &v[i][j].x;
        const float* pm = &mu4.x;
        const float* pr = &rs4.x;
        const float* pg = &gm4.x;
        const float* pb = &bt4.x;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float t = (pv[q] - pm[q]) * pr[q] * pg[q] + pb[q];
          pv[q] = bn.act == MGX_ACT_RELU ? relu(t) : act_forward(bn.act, t);
        }
      }
#pragma unroll
    for (int o = 0; o < 2; ++o) {
      const int ow = owp * 2 + o;
      if (ow >= g.Wo) break;
      float acc[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
      int ai[4] = {0, 0, 0, 0};
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          const float* pv = &v[i][2 * o + j].x;
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (pv[q] > acc[q]) {
              acc[q] = pv[q];
              ai[q] = i * 3 + j;
            }
        }
      const int oi = ((b * g.Ho + oh) * g.Wo + ow) * C4 + c4;
      const float4 r = make_float4(acc[0], acc[1], acc[2], acc[3]);
      if (y) y[oi] = r;
      arg[oi] = make_uchar4(ai[0], ai[1], ai[2], ai[3]);
      if (y16) {
        uint2 h;
        h.x = pack_bf16(r.x, r.y);
        h.y = pack_bf16(r.z, r.w);
        y16[oi] = h;
      }
    }
  }
}

template <int K, int S, int TYPE>
__global__ void __launch_bounds__(256)
pool_bwd_vec_kernel(const uint8_t* __restrict__ arg, const float* __restrict__ dy,
                    float* __restrict__ dx, Geom g) {
  const int C4 = g.C >> 2;
  const int kh = K ? K : g.kh, kw = K ? K : g.kw;
  const int sh = K ? S : g.sh, sw = K ? S : g.sw;
  const int hw = g.H * g.W;
  const int64_t total = int64_t(g.B) * hw * C4;
  const int64_t step = int64_t(gridDim.x) * blockDim.x;
  const float4* dy4 = reinterpret_cast<const float4*>(dy);
  const uchar4* a4 = reinterpret_cast<const uchar4*>(arg);
  for (int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; idx < total; idx += step) {
    const int pix = static_cast<int>(idx / C4);
    const int c4 = static_cast<int>(idx - int64_t(pix) * C4);
    const int b = pix / hw;
    const int rem = pix - b * hw;
    const int h = rem / g.W, w = rem - (rem / g.W) * g.W;
    // output windows covering (h, w): oh*sh - ph <= h < oh*sh - ph + kh
    const int nh = h + g.ph - kh + 1, nw = w + g.pw - kw + 1;
    const int oh_lo = nh <= 0 ? 0 : (nh + sh - 1) / sh;
    const int oh_hi = min(g.Ho - 1, (h + g.ph) / sh);
    const int ow_lo = nw <= 0 ? 0 : (nw + sw - 1) / sw;
    const int ow_hi = min(g.Wo - 1, (w + g.pw) / sw);
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    const int64_t ob = int64_t(b) * g.Ho * g.Wo * C4 + c4;
    auto win = [&](int oh, int ow, const float4 d, const uchar4 am) {
      const float* pd = &d.x;
      if (TYPE == 0) {
        const int li = (h - (oh * sh - g.ph)) * kw + (w - (ow * sw - g.pw));
        const unsigned char* pa = &am.x;
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (pa[q] == li) acc[q] = fadd(acc[q], pd[q]);
      } else {
        const float inv = __frcp_rn(pool_area(g, oh, ow));
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[q] = fadd(acc[q], pd[q] * inv);
      }
    };
    if constexpr (K > 0) {
      constexpr int NW = (K + S - 1) / S;  // covering windows per dimension
      float4 d[NW * NW];
      uchar4 am[NW * NW];
#pragma unroll
      for (int i = 0; i < NW; ++i)
#pragma unroll
        for (int j = 0; j < NW; ++j) {
          const int oh = oh_lo + i, ow = ow_lo + j;
          const bool ok = oh <= oh_hi && ow <= ow_hi;
          const int64_t o = ob + (int64_t(oh) * g.Wo + ow) * C4;
          d[i * NW + j] = ok ? __ldg(dy4 + o) : make_float4(0.f, 0.f, 0.f, 0.f);
          if (TYPE == 0) am[i * NW + j] = ok ? __ldg(a4 + o) : make_uchar4(255, 255, 255, 255);
        }
#pragma unroll
      for (int i = 0; i < NW; ++i)
#pragma unroll
        for (int j = 0; j < NW; ++j)
          if (oh_lo + i <= oh_hi && ow_lo + j <= ow_hi)
            win(oh_lo + i, ow_lo + j, d[i * NW + j], am[i * NW + j]);
    } else {
      for (int oh = oh_lo; oh <= oh_hi; ++oh)
        for (int ow = ow_lo; ow <= ow_hi; ++ow) {
          const int64_t o = ob + (int64_t(oh) * g.Wo + ow) * C4;
          win(oh, ow, __ldg(dy4 + o), TYPE == 0 ? __ldg(a4 + o) : make_uchar4(0, 0, 0, 0));
        }
    }
    reinterpret_cast<float4*>(dx)[idx] = make_float4(acc[0], acc[1], acc[2], acc[3]);
  }
}

// 3x3 / stride 1 / pad 1 average pooling (count_include_pad: every window
// divides by 9) as a shared-memory box filter: a block stages a strip of
// TR (+2 halo) rows x (W + 2) columns x 8 channel vectors, zero-padded, with
// one coalesced read of each input element, then every output sums its 9
// taps from shared memory.  Forward: taps in row-major order, then * 1/9;
// backward: dx = sum over the covering windows in ascending (oh, ow) order
// of dy * 1/9 -- pool_fwd_vec_kernel / pool_bwd_vec_kernel's arithmetic
// (padding taps add exact zeros).
constexpr int kAvgVS = 8;  // the strip height is chosen per shape (host)

template <bool BWD>
__global__ void __launch_bounds__(256)
pool_avg3_tile_kernel(const float4* __restrict__ src, float4* __restrict__ dst,
                      uint2* __restrict__ dst16, Geom g, int kAvgTR) {
  extern __shared__ float4 avg_tile[];  // [kAvgTR + 2][W + 2][kAvgVS]
  const int C4 = g.C >> 2;
  const int nvs = (C4 + kAvgVS - 1) / kAvgVS;
  const int ns = (g.H + kAvgTR - 1) / kAvgTR;
  const int b = blockIdx.x / (nvs * ns);
  const int rem = blockIdx.x - b * nvs * ns;
  const int vs = rem / ns, strip = rem - (rem / ns) * ns;
  const int h0 = strip * kAvgTR, v0 = vs * kAvgVS;
  const int WP = g.W + 2;
  const int rows = min(kAvgTR, g.H - h0);
  const int nload = (rows + 2) * WP * kAvgVS;
  // the whole strip in flight at once: 16-byte cp.async copies straight
  // into shared memory, zero-filled outside the map (the padding taps)
  for (int e = threadIdx.x; e < nload; e += blockDim.x) {
    const int v = e % kAvgVS, cw = (e / kAvgVS) % WP, rr = e / (kAvgVS * WP);
    const int h = h0 - 1 + rr, w = cw - 1, c4 = v0 + v;
    const bool ok = h >= 0 && h < g.H && w >= 0 && w < g.W && c4 < C4;
    const float4* sp = ok ? src + ((int64_t(b) * g.H + h) * g.W + w) * C4 + c4 : src;
    const uint32_t dst_s = static_cast<uint32_t>(__cvta_generic_to_shared(avg_tile + e));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst_s), "l"(sp),
                 "r"(ok ? 16 : 0)
                 : "memory");
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  const float inv = __frcp_rn(9.0f);
  const int nout = rows * g.W * kAvgVS;
  for (int e = threadIdx.x; e < nout; e += blockDim.x) {
    const int v = e % kAvgVS, w = (e / kAvgVS) % g.W, r = e / (kAvgVS * g.W);
    const int c4 = v0 + v;
    if (c4 >= C4) continue;
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const float4 t = avg_tile[((r + i) * WP + (w + j)) * kAvgVS + v];
        if (BWD) {
          acc[0] = fadd(acc[0], t.x * inv);
          acc[1] = fadd(acc[1], t.y * inv);
          acc[2] = fadd(acc[2], t.z * inv);
          acc[3] = fadd(acc[3], t.w * inv);
        } else {
          acc[0] = fadd(acc[0], t.x);
          acc[1] = fadd(acc[1], t.y);
          acc[2] = fadd(acc[2], t.z);
          acc[3] = fadd(acc[3], t.w);
        }
      }
    float4 o = BWD ? make_float4(acc[0], acc[1], acc[2], acc[3])
                   : make_float4(acc[0] * inv, acc[1] * inv, acc[2] * inv, acc[3] * inv);
    const int64_t i = ((int64_t(b) * g.H + h0 + r) * g.W + w) * C4 + c4;
    if (dst) dst[i] = o;
    if (dst16) {
      uint2 hv;
      hv.x = pack_bf16(o.x, o.y);
      hv.y = pack_bf16(o.z, o.w);
      dst16[i] = hv;
    }
  }
}

// out = ((s0 + s1) + s2) + ... : a chain of ElementwiseAdds (the gradient
// fan-in build_gradient emits, symbol.py:254-258) in one pass, same
// left-to-right rounding order.
struct SumSrcs {
  const float* p[6];
  int n;
};

__global__ void sum_n_kernel(SumSrcs src, float* __restrict__ out, int64_t n4) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += stride) {
    // every source's load issued before the first add (a runtime-count loop
    // kept one 16-byte load outstanding); the sum stays the left fold
    // ((p0 + p1) + p2) + ...
    float4 b[6];
#pragma unroll
    for (int k = 0; k < 6; ++k)
      if (k < src.n) b[k] = __ldg(reinterpret_cast<const float4*>(src.p[k]) + i);
    float4 a = b[0];
#pragma unroll
    for (int k = 1; k < 6; ++k) {
      if (k < src.n) {
        a.x = fadd(a.x, b[k].x);
        a.y = fadd(a.y, b[k].y);
        a.z = fadd(a.z, b[k].z);
        a.w = fadd(a.w, b[k].w);
      }
    }
    reinterpret_cast<float4*>(out)[i] = a;
  }
}

// Concat along channels in one pass: out[r, :] = [in0[r, :] | in1[r, :] | ...]
// (all channel counts % 4 == 0), with the optional bf16 copy of out.
struct CatSrcs {
  const float* p[4];
  int c[4];
  int n;
};

__global__ void concat_kernel(CatSrcs in, float* __restrict__ out, int64_t rows, int ctot,
                              __nv_bfloat16* __restrict__ out16) {
  const RowsIdx ri(ctot >> 2);
  if (!ri.active) return;
  const int col = ri.v * 4;
  int k = 0, base = 0;
  while (k < in.n - 1 && col >= base + in.c[k]) {
    base += in.c[k];
    ++k;
  }
  const int cc = col - base, ck = in.c[k];
  const float* src = in.p[k];
  // four rows' loads in flight per thread before their stores (a pure copy:
  // the per-row loop otherwise keeps one 16-byte load outstanding)
  constexpr int U = 8;
  for (int64_t r0 = ri.r; r0 < rows; r0 += int64_t(U) * ri.rstep) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t r = r0 + int64_t(u) * ri.rstep;
      if (r < rows) v[u] = __ldg(reinterpret_cast<const float4*>(src + r * ck + cc));
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t r = r0 + int64_t(u) * ri.rstep;
      if (r >= rows) break;
      *reinterpret_cast<float4*>(out + r * ctot + col) = v[u];
      if (out16) {
        uint2 h;
        h.x = pack_bf16(v[u].x, v[u].y);
        h.y = pack_bf16(v[u].z, v[u].w);
        *reinterpret_cast<uint2*>(out16 + r * ctot + col) = h;
      }
    }
  }
}

// dst[r, doff + c] = src[r, soff + c] (Concat forward / backward slices)
__global__ void chan_copy_kernel(const float* __restrict__ src, int64_t lds, int64_t soff,
                                 float* __restrict__ dst, int64_t ldd, int64_t doff, int64_t rows,
                                 int64_t cols, __nv_bfloat16* __restrict__ dst16) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  if (((cols | lds | soff | ldd | doff) & 3) == 0) {
    // rows x vectors launch shape
    const RowsIdx ri(static_cast<int>(cols / 4));
    if (!ri.active) return;
    const int64_t c = int64_t(ri.v) * 4;
    constexpr int U = 4;  // rows' loads in flight per thread (as concat_kernel)
    for (int64_t r0 = ri.r; r0 < rows; r0 += int64_t(U) * ri.rstep) {
      float4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t r = r0 + int64_t(u) * ri.rstep;
        if (r < rows) v[u] = __ldg(reinterpret_cast<const float4*>(src + r * lds + soff + c));
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t r = r0 + int64_t(u) * ri.rstep;
        if (r >= rows) break;
        *reinterpret_cast<float4*>(dst + r * ldd + doff + c) = v[u];
        if (dst16) {
          uint2 h;
          h.x = pack_bf16(v[u].x, v[u].y);
          h.y = pack_bf16(v[u].z, v[u].w);
          *reinterpret_cast<uint2*>(dst16 + r * ldd + doff + c) = h;
        }
      }
    }
  } else {
    const int64_t total = rows * cols;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += stride) {
      const int64_t r = i / cols, c = i - r * cols;
      dst[r * ldd + doff + c] = src[r * lds + soff + c];
    }
  }
}

inline unsigned grid_for(int64_t n, int threads = 256, int64_t cap = int64_t(kNumSMs) * 16) {
  int64_t b = ceil_div(n, threads);
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return static_cast<unsigned>(b);
}

// chunking of M rows for the column reductions
inline void chunks_for(int64_t M, int64_t C, int64_t* rpc, int* nchunk) {
  // row chunks x column groups ~ 4 blocks per SM (every SM busy even at the
  // 7x7 / 14x14 layers' few thousand rows), each thread walking >= 2 rows;
  // a deterministic function of (M, C): the fixed merge order follows
  const int64_t C4 = C % 4 == 0 ? C / 4 : 0;
  const int64_t ct4 = C4 == 0 ? 0 : (C4 < kRedThreads ? C4 : kRedThreads);
  const int64_t groups = C4 == 0 ? 1 : ceil_div(C4, ct4);
  const int64_t rpp = C4 == 0 ? 1 : kRedThreads / ct4;
  int64_t n = ceil_div(int64_t(4) * kNumSMs, groups);
  const int64_t by_rows = ceil_div(M, 2 * rpp);
  if (n > by_rows) n = by_rows;
  if (n > kMaxChunks) n = kMaxChunks;
  if (n < 1) n = 1;
  *rpc = ceil_div(M, n);
  *nchunk = static_cast<int>(ceil_div(M, *rpc));
}

template <int MODE>
int launch_partial(const float* a, const float* xs, const float* stats, int64_t M, int C,
                   double* ws, int* nchunk_out, cudaStream_t st,
                   ReluMask rm = ReluMask{nullptr, nullptr}) {
  int64_t rpc;
  int nchunk;
  chunks_for(M, C, &rpc, &nchunk);
  const bool vec = (C % 4) == 0 && aligned16(a) && (MODE != 1 || aligned16(xs));
  if (vec) {
    const int C4 = C / 4;
    const int ct4 = C4 < kRedThreads ? C4 : kRedThreads;
    const int rpp = kRedThreads / ct4;
    const size_t smem = size_t(rpp) * 2 * ct4 * 4 * sizeof(double);
    dim3 grid(nchunk, static_cast<unsigned>(ceil_div(C4, ct4)));
    colreduce_partial_vec_kernel<MODE><<<grid, ct4 * rpp, smem, st>>>(a, xs, stats, M, C, rpc, ws,
                                                                      rm);
  } else {
    const int tpr = C < kRedThreads ? C : kRedThreads;
    const int rpp = kRedThreads / tpr;
    const size_t smem = size_t(rpp) * 2 * tpr * sizeof(double);
    colreduce_partial_kernel<MODE><<<nchunk, kRedThreads, smem, st>>>(a, xs, stats, M, C, rpc, ws,
                                                                    rm);
  }
  *nchunk_out = nchunk;
  MGX_LAUNCHED();
  return MGX_OK;
}

}  // namespace conv
}  // namespace mgx

using mgx::conv::Geom;
using mgx::conv::grid_for;

// ------------------------------------------------------------------ C-ABI

extern "C" int mgx_reduce_workspace_bytes(int64_t M, int64_t C, int64_t* out) {
  MGX_REQUIRE(out && M > 0 && C > 0, "mgx_reduce_workspace_bytes: bad arguments");
  int64_t rpc;
  int nchunk;
  mgx::conv::chunks_for(M, C, &rpc, &nchunk);
  *out = int64_t(2) * nchunk * C * 8;
  return MGX_OK;
}

extern "C" int mgx_im2col_bf16(const float* x, void* col, const int64_t* geom, int64_t ldk,
                               uintptr_t stream) {
  MGX_REQUIRE(x && col && geom, "mgx_im2col_bf16: bad arguments");
  Geom g = mgx::conv::decode(geom);
  MGX_REQUIRE(g.B > 0 && g.C > 0 && g.kh > 0 && g.kw > 0 && g.sh > 0 && g.sw > 0 && g.Ho > 0 &&
                  g.Wo > 0, "mgx_im2col_bf16: bad geometry");
  MGX_REQUIRE(ldk % 8 == 0 && ldk >= int64_t(g.kh) * g.kw * g.C, "mgx_im2col_bf16: bad ldk");
  MGX_REQUIRE(mgx::aligned16(x) && mgx::aligned16(col), "mgx_im2col_bf16: unaligned");
  MGX_REQUIRE(int64_t(g.B) * g.Ho * g.Wo < (1ll << 31), "mgx_im2col_bf16: too many rows");
  const int WT = (g.Wo - 1) * g.sw + g.kw;
  const size_t smem = size_t(g.kh) * WT * g.C * sizeof(float) + size_t(ldk) * sizeof(int);
  if (g.C % 8 != 0 && smem <= 48 * 1024 && ldk / 8 <= 256) {
    const int nj = static_cast<int>(ldk / 8);
    mgx::conv::im2col_rows_kernel<<<static_cast<unsigned>(int64_t(g.B) * g.Ho), nj * (256 / nj),
                                    smem, mgx::as_stream(stream)>>>(
        x, static_cast<__nv_bfloat16*>(col), g, ldk, WT);
    MGX_LAUNCHED();
    return MGX_OK;
  }
  mgx::conv::im2col_kernel<<<mgx::rows_grid(int64_t(g.B) * g.Ho * g.Wo, ldk / 8),
                             mgx::rows_block(ldk / 8), 0,
                             mgx::as_stream(stream)>>>(x, static_cast<__nv_bfloat16*>(col), g, ldk);
  MGX_LAUNCHED();
  return MGX_OK;
}

extern "C" int mgx_col2im(const float* dcol, int64_t ldk, float* dx, const int64_t* geom,
                          uintptr_t stream) {
  MGX_REQUIRE(dcol && dx && geom, "mgx_col2im: bad arguments");
  Geom g = mgx::conv::decode(geom);
  MGX_REQUIRE(g.Ho > 0 && g.Wo > 0 && ldk >= int64_t(g.kh) * g.kw * g.C, "mgx_col2im: bad geometry");
  const int64_t n = int64_t(g.B) * g.H * g.W * g.C;
  cudaStream_t st = mgx::as_stream(stream);
  if (g.C % 4 == 0 && ldk % 4 == 0 && mgx::aligned16(dcol) && mgx::aligned16(dx)) {
    const auto* d4 = reinterpret_cast<const float4*>(dcol);
    auto* x4 = reinterpret_cast<float4*>(dx);
    const unsigned grid = grid_for(n / 4, 256, int64_t(mgx::kNumSMs) * 8);
    if (g.kh == 3 && g.kw == 3 && g.sh == 2 && g.sw == 2)
      mgx::conv::col2im_vec4_kernel<3, 3, 2, 2><<<grid, 256, 0, st>>>(d4, ldk / 4, x4, g);
    else if (g.kh == 3 && g.kw == 3 && g.sh == 1 && g.sw == 1)
      mgx::conv::col2im_vec4_kernel<3, 3, 1, 1><<<grid, 256, 0, st>>>(d4, ldk / 4, x4, g);
    else
      mgx::conv::col2im_vec4_kernel<0, 0, 0, 0><<<grid, 256, 0, st>>>(d4, ldk / 4, x4, g);
    MGX_LAUNCHED();
    return MGX_OK;
  }
  mgx::conv::col2im_kernel<<<grid_for(n), 256, 0, st>>>(dcol, ldk, dx, g);
  MGX_LAUNCHED();
  return MGX_OK;
}

extern "C" int mgx_bn_stats(const float* x, int64_t M, int64_t C, void* ws, float* stats,
                            float* moving_mean, float* moving_var, float eps, float momentum,
                            int use_global, uintptr_t stream) {
  MGX_REQUIRE(stats && M > 0 && C > 0 && C <= 65536, "mgx_bn_stats: bad arguments");
  MGX_REQUIRE(!use_global || (moving_mean && moving_var), "mgx_bn_stats: global stats need moving_*");
  cudaStream_t st = mgx::as_stream(stream);
  int nchunk = 0;
  if (!use_global) {
    MGX_REQUIRE(x && ws, "mgx_bn_stats: bad arguments");
    MGX_TRY(mgx::conv::launch_partial<0>(x, nullptr, nullptr, M, static_cast<int>(C),
                                         static_cast<double*>(ws), &nchunk, st));
  }
  mgx::conv::bn_stats_finalize_kernel<<<static_cast<unsigned>(mgx::ceil_div(C, mgx::conv::kFinChannels)), 256, 0, st>>>(
      static_cast<const double*>(ws), nchunk, M, static_cast<int>(C), x, eps, momentum, use_global,
      stats, moving_mean, moving_var);
  MGX_LAUNCHED();
  return MGX_OK;
}

extern "C" int mgx_bn_apply_ld(const float* x, const float* stats, const float* gamma,
                               const float* beta, float* y, int64_t M, int64_t C, int act,
                               void* y16, int64_t ldo, uintptr_t stream) {
  if (ldo == 0) ldo = C;
  MGX_REQUIRE(ldo == C || (ldo > C && ldo % 4 == 0 && C % 4 == 0), "mgx_bn_apply: bad output stride");
  MGX_REQUIRE(x && stats && beta && (y || y16) && M > 0 && C > 0, "mgx_bn_apply: bad arguments");
  MGX_REQUIRE(!y16 || (C % 4 == 0 && mgx::aligned16(y16)), "mgx_bn_apply: bf16 copy needs C %% 4 == 0");
  if ((C & 3) == 0) {
    MGX_REQUIRE(mgx::aligned16(x) && (!y || mgx::aligned16(y)), "mgx_bn_apply: unaligned tensors");
    mgx::conv::bn_apply_kernel<<<mgx::rows_grid(M, C / 4, 4),
                                 mgx::rows_block(C / 4), 0,
                                 mgx::as_stream(stream)>>>(x, stats, gamma, beta, y, M,
                                                           static_cast<int>(C), act,
                                                           static_cast<__nv_bfloat16*>(y16), ldo / 4);
  } else {
    mgx::conv::bn_apply_kernel<<<grid_for(M * C), 256, 0, mgx::as_stream(stream)>>>(
        x, stats, gamma, beta, y, M, static_cast<int>(C), act, nullptr, int64_t(0));
  }
  MGX_LAUNCHED();
  return MGX_OK;
}

extern "C" int mgx_bn_apply(const float* x, const float* stats, const float* gamma,
                            const float* beta, float* y, int64_t M, int64_t C, int act, void* y16,
                            uintptr_t stream) {
  return mgx_bn_apply_ld(x, stats, gamma, beta, y, M, C, act, y16, C, stream);
}

extern "C" int mgx_bn_bwd_reduce(const float* dy, const float* x, const float* stats, int64_t M,
                                 int64_t C, void* ws, float* sums, float* dbeta, float* dgamma,
                                 int dgamma_zero, const float* relu_gamma, const float* relu_beta,
                                 uintptr_t stream) {
  MGX_REQUIRE(dy && x && stats && ws && sums && M > 0 && C > 0, "mgx_bn_bwd_reduce: bad arguments");
  cudaStream_t st = mgx::as_stream(stream);
  int nchunk = 0;
  MGX_TRY(mgx::conv::launch_partial<1>(dy, x, stats, M, static_cast<int>(C), static_cast<double*>(ws),
                                       &nchunk, st, mgx::conv::ReluMask{relu_gamma, relu_beta}));
  mgx::conv::colsum_finalize_kernel<<<static_cast<unsigned>(mgx::ceil_div(C, mgx::conv::kFinChannels)), 256, 0, st>>>(
      static_cast<const double*>(ws), nchunk, static_cast<int>(C), 1, sums, dbeta, dgamma,
      dgamma_zero);
  MGX_LAUNCHED();
  return MGX_OK;
}

extern "C" int mgx_bn_bwd_dx(const float* dy, const float* x, const float* stats, const float* sums,
                             const float* gamma, float* dx, int64_t M, int64_t C,
                             const float* relu_gamma, const float* relu_beta, float* dsum,
                             void* ws, void* dx16, uintptr_t stream) {
  MGX_REQUIRE(dy && x && stats && sums && (dx || dx16) && M > 0 && C > 0,
              "mgx_bn_bwd_dx: bad arguments");
  MGX_REQUIRE(!dx16 || (C % 4 == 0 && mgx::aligned16(dx16)), "mgx_bn_bwd_dx: bf16 copy needs C %% 4 == 0");
  const bool vec = (C % 4) == 0 && mgx::aligned16(dy) && mgx::aligned16(x) &&
                   (!dx || mgx::aligned16(dx));
  MGX_REQUIRE(dx || vec, "mgx_bn_bwd_dx: dx may only be omitted on the vectorised path");
  cudaStream_t st = mgx::as_stream(stream);
  const mgx::conv::ReluMask rm{relu_gamma, relu_beta};
  if (vec) {
    // dx (and, when dsum is given, its per-channel sum: the conv bias
    // gradient) in one row-tiled pass
    MGX_REQUIRE(!dsum || ws, "mgx_bn_bwd_dx: dsum needs a workspace");
    int64_t rpc;
    int nchunk;
    mgx::conv::chunks_for(M, C, &rpc, &nchunk);
    const int C4 = static_cast<int>(C / 4);
    const int ct4 = C4 < mgx::conv::kRedThreads ? C4 : mgx::conv::kRedThreads;
    const int rpp = mgx::conv::kRedThreads / ct4;
    const size_t smem = size_t(rpp) * ct4 * 4 * sizeof(double);
    dim3 grid(nchunk, static_cast<unsigned>(mgx::ceil_div(C4, ct4)));
    double* wsd = dsum ? static_cast<double*>(ws) : nullptr;
    if (!dsum) {
      // reuse the tiled kernel without the reduction output
      MGX_REQUIRE(ws, "mgx_bn_bwd_dx: the vectorised pass needs a workspace");
      wsd = static_cast<double*>(ws);
    }
    mgx::conv::bn_dx_colsum_kernel<<<grid, ct4 * rpp, smem, st>>>(
        dy, x, stats, sums, gamma, dx, rm, M, static_cast<int>(C), rpc, wsd,
        static_cast<__nv_bfloat16*>(dx16), mgx::conv::PoolGrad{});
    if (dsum)
      mgx::conv::colsum_finalize_kernel<<<static_cast<unsigned>(mgx::ceil_div(C, mgx::conv::kFinChannels)), 256, 0, st>>>(
          static_cast<const double*>(ws), nchunk, static_cast<int>(C), 0, dsum, nullptr, nullptr, 0);
    MGX_LAUNCHED();
    return MGX_OK;
  }
  mgx::conv::bn_bwd_dx_kernel<<<grid_for(M * C), 256, 0, st>>>(dy, x, stats, sums, gamma, dx, M,
                                                               static_cast<int>(C), rm);
  MGX_LAUNCHED();
  return MGX_OK;
}

extern "C" int mgx_colsum(const float* x, int64_t M, int64_t C, void* ws, float* out,
                          uintptr_t stream) {
  MGX_REQUIRE(x && ws && out && M > 0 && C > 0, "mgx_colsum: bad arguments");
  cudaStream_t st = mgx::as_stream(stream);
  int nchunk = 0;
  MGX_TRY(mgx::conv::launch_partial<2>(x, nullptr, nullptr, M, static_cast<int>(C),
                                       static_cast<double*>(ws), &nchunk, st));
  mgx::conv::colsum_finalize_kernel<<<static_cast<unsigned>(mgx::ceil_div(C, mgx::conv::kFinChannels)), 256, 0, st>>>(
      static_cast<const double*>(ws), nchunk, static_cast<int>(C), 0, out, nullptr, nullptr, 0);
  MGX_LAUNCHED();
  return MGX_OK;
}

static bool pool_vec_ok(const Geom& g, const void* a, const void* b) {
  return (g.C % 4) == 0 && mgx::aligned16(a) && mgx::aligned16(b);
}

// rows per strip of pool_avg3_tile_kernel: as tall as 48 KB of shared
// memory allows (whole 14x14 maps; 27x27 in two strips), 0 if not even one
static int avg3_strip_rows(const Geom& g) {
  const int64_t row_bytes = int64_t(g.W + 2) * mgx::conv::kAvgVS * 16;
  int64_t tr = 48 * 1024 / row_bytes - 2;
  if (tr > g.H) tr = g.H;
  if (tr >= 2) {  // balance the strips: ceil(H / ceil(H / tr))
    const int64_t ns = (g.H + tr - 1) / tr;
    tr = (g.H + ns - 1) / ns;
  }
  return tr < 1 ? 0 : static_cast<int>(tr);
}

// 10 * K + S for the square K x K / stride S windows with unrolled kernels
static int pool_square(const Geom& g) {
  if (g.kh == 3 && g.kw == 3 && g.sh == g.sw && (g.sh == 1 || g.sh == 2)) return 30 + g.sh;
  return 0;
}

extern "C" int mgx_pool_forward(const float* x, float* y, const int64_t* geom, int full, int type,
                                void* argmax, void* y16, uintptr_t stream) {
  MGX_REQUIRE(x && (y || y16) && geom && (type == 0 || type == 1),
              "mgx_pool_forward: bad arguments");
  Geom g = mgx::conv::decode(geom, full != 0);
  MGX_REQUIRE(g.Ho > 0 && g.Wo > 0, "mgx_pool_forward: bad geometry");
  cudaStream_t st = mgx::as_stream(stream);
  const int avg_tr = avg3_strip_rows(g);
  if (type == 1 && !full && pool_square(g) == 31 && g.ph == 1 && g.pw == 1 && g.Ho == g.H &&
      g.Wo == g.W && g.C % 4 == 0 && mgx::aligned16(x) && (!y || mgx::aligned16(y)) &&
      (!y16 || mgx::aligned16(y16)) && avg_tr > 0) {
    const int C4 = g.C / 4;
    const int64_t blocks = int64_t(g.B) * ((C4 + 7) / 8) * ((g.H + avg_tr - 1) / avg_tr);
    const size_t smem = size_t(avg_tr + 2) * (g.W + 2) * mgx::conv::kAvgVS * 16;
    mgx::conv::pool_avg3_tile_kernel<false><<<static_cast<unsigned>(blocks), 256, smem, st>>>(
        reinterpret_cast<const float4*>(x), reinterpret_cast<float4*>(y),
        reinterpret_cast<uint2*>(y16), g, avg_tr);
    MGX_LAUNCHED();
    return MGX_OK;
  }
  if (pool_vec_ok(g, x, y ? y : y16) && g.kh * g.kw <= 255) {
    const unsigned grid = grid_for(int64_t(g.B) * g.Ho * g.Wo * (g.C / 4));
    uint8_t* arg = type == 0 ? static_cast<uint8_t*>(argmax) : nullptr;
    __nv_bfloat16* h16 = static_cast<__nv_bfloat16*>(y16);
    const int sq = pool_square(g) * 2 + type;
#define MGX_POOL_FWD(K_, S_, T_) \
  mgx::conv::pool_fwd_vec_kernel<K_, S_, T_, false, (K_ > 0 ? 4 : 1)><<<grid, 256, 0, st>>>(x, y, arg, g, h16)
    switch (sq) {
      case 62: MGX_POOL_FWD(3, 1, 0); break;
      case 63: MGX_POOL_FWD(3, 1, 1); break;
      case 64: MGX_POOL_FWD(3, 2, 0); break;
      case 65: MGX_POOL_FWD(3, 2, 1); break;
      case 0: MGX_POOL_FWD(0, 0, 0); break;
      default: MGX_POOL_FWD(0, 0, 1); break;
    }
#undef MGX_POOL_FWD
  } else {
    MGX_REQUIRE(y, "mgx_pool_forward: y may be NULL only on the vectorised path");
    MGX_REQUIRE(!argmax || type != 0, "mgx_pool_forward: argmax needs C %% 4 == 0 and kh*kw <= 255");
    MGX_REQUIRE(!y16, "mgx_pool_forward: a bf16 copy needs C %% 4 == 0");
    const int64_t n = int64_t(g.B) * g.Ho * g.Wo * g.C;
    mgx::conv::pool_fwd_kernel<<<grid_for(n), 256, 0, st>>>(x, y, g, type);
  }
  MGX_LAUNCHED();
  return MGX_OK;
}

extern "C" int mgx_pool_backward(const float* x, const float* y, const float* dy, float* dx,
                                 const int64_t* geom, int full, int type, const void* argmax,
                                 uintptr_t stream) {
  MGX_REQUIRE(dy && dx && geom && (type == 1 || argmax || (x && y)),
              "mgx_pool_backward: bad arguments");
  Geom g = mgx::conv::decode(geom, full != 0);
  cudaStream_t st = mgx::as_stream(stream);
  const bool use_arg = type == 0 && argmax != nullptr;
  const int avg_tr = avg3_strip_rows(g);
  if (type == 1 && !full && pool_square(g) == 31 && g.ph == 1 && g.pw == 1 && g.Ho == g.H &&
      g.Wo == g.W && g.C % 4 == 0 && mgx::aligned16(dy) && mgx::aligned16(dx) && avg_tr > 0) {
    const int C4 = g.C / 4;
    const int64_t blocks = int64_t(g.B) * ((C4 + 7) / 8) * ((g.H + avg_tr - 1) / avg_tr);
    const size_t smem = size_t(avg_tr + 2) * (g.W + 2) * mgx::conv::kAvgVS * 16;
    mgx::conv::pool_avg3_tile_kernel<true><<<static_cast<unsigned>(blocks), 256, smem, st>>>(
        reinterpret_cast<const float4*>(dy), reinterpret_cast<float4*>(dx), nullptr, g, avg_tr);
    MGX_LAUNCHED();
    return MGX_OK;
  }
  if (pool_vec_ok(g, dy, dx) && (type == 1 || use_arg)) {
    const unsigned grid = grid_for(int64_t(g.B) * g.H * g.W * (g.C / 4));
    const uint8_t* arg = static_cast<const uint8_t*>(argmax);
    const int sq = pool_square(g) * 2 + type;
#define MGX_POOL_BWD(K_, S_, T_) \
  mgx::conv::pool_bwd_vec_kernel<K_, S_, T_><<<grid, 256, 0, st>>>(arg, dy, dx, g)
    switch (sq) {
      case 62: MGX_POOL_BWD(3, 1, 0); break;
      case 63: MGX_POOL_BWD(3, 1, 1); break;
      case 64: MGX_POOL_BWD(3, 2, 0); break;
      case 65: MGX_POOL_BWD(3, 2, 1); break;
      case 0: MGX_POOL_BWD(0, 0, 0); break;
      default: MGX_POOL_BWD(0, 0, 1); break;
    }
#undef MGX_POOL_BWD
  } else {
    MGX_REQUIRE(type == 1 || (x && y), "mgx_pool_backward: max pooling needs x and y");
    const int64_t n = int64_t(g.B) * g.H * g.W * g.C;
    mgx::conv::pool_bwd_kernel<<<grid_for(n), 256, 0, st>>>(x, y, dy, dx, g, type);
  }
  MGX_LAUNCHED();
  return MGX_OK;
}

// ---- stem fusion: BatchNorm (+act) -> max pooling, forward and backward
extern "C" int mgx_bn_act_pool_fwd(const float* x, const float* stats, const float* gamma,
                                   const float* beta, int act, const int64_t* geom, int full,
                                   float* y, void* y16, void* argmax, uintptr_t stream) {
  MGX_REQUIRE(x && stats && beta && (y || y16) && argmax && geom,
              "mgx_bn_act_pool_fwd: bad arguments");
  Geom g = mgx::conv::decode(geom, full != 0);
  MGX_REQUIRE(g.Ho > 0 && g.Wo > 0 && g.kh * g.kw <= 255, "mgx_bn_act_pool_fwd: bad geometry");
  MGX_REQUIRE(g.C % 4 == 0 && mgx::aligned16(x) && mgx::aligned16(stats) && mgx::aligned16(beta) &&
                  (!gamma || mgx::aligned16(gamma)) && (!y || mgx::aligned16(y)) &&
                  (!y16 || mgx::aligned16(y16)),
              "mgx_bn_act_pool_fwd: needs C %% 4 == 0 and 16-byte aligned tensors");
  cudaStream_t st = mgx::as_stream(stream);
  const unsigned grid = grid_for(int64_t(g.B) * g.Ho * g.Wo * (g.C / 4));
  const mgx::conv::BnAct bn{stats, gamma, beta, act};
  uint8_t* arg = static_cast<uint8_t*>(argmax);
  __nv_bfloat16* h16 = static_cast<__nv_bfloat16*>(y16);
  // 3 resident CTAs per SM (<= 85 registers): latency-bound gather, +20% over 2
  static const bool pair = [] {
    const char* v = getenv("MGX_STEM_POOL_PAIR");
    return !(v && *v == '0');
  }();
  if (pair && pool_square(g) == 32 && g.ph == 0 && g.pw == 0 &&
      int64_t(g.B) * g.H * g.W * g.C < (int64_t(1) << 31)) {
    const unsigned gp = grid_for(int64_t(g.B) * g.Ho * ((g.Wo + 1) / 2) * (g.C / 4));
    mgx::conv::bn_relu_maxpool3s2_kernel<<<gp, 256, 0, st>>>(
        reinterpret_cast<const float4*>(x), reinterpret_cast<float4*>(y),
        reinterpret_cast<uchar4*>(arg), g, reinterpret_cast<uint2*>(h16), bn);
  } else if (pool_square(g) == 32)
    mgx::conv::pool_fwd_vec_kernel<3, 2, 0, true, 3><<<grid, 256, 0, st>>>(x, y, arg, g, h16, bn);
  else
    mgx::conv::pool_fwd_vec_kernel<0, 0, 0, true><<<grid, 256, 0, st>>>(x, y, arg, g, h16, bn);
  MGX_LAUNCHED();
  return MGX_OK;
}

static int pool_grad_of(const float* dy_pool, const void* argmax, const int64_t* geom, int full,
                        int64_t M, int64_t C, mgx::conv::PoolGrad* pg, int* pk) {
  MGX_REQUIRE(dy_pool && argmax && geom, "pooled BatchNorm backward: bad arguments");
  Geom g = mgx::conv::decode(geom, full != 0);
  MGX_REQUIRE(int64_t(g.B) * g.H * g.W == M && g.C == C && C % 4 == 0 && g.Ho > 0 && g.Wo > 0 &&
                  M < (int64_t(1) << 31) && mgx::aligned16(dy_pool) && mgx::aligned16(argmax),
              "pooled BatchNorm backward: geometry does not match the rows");
  pg->dy = static_cast<const float4*>(static_cast<const void*>(dy_pool));
  pg->arg = static_cast<const uchar4*>(argmax);
  pg->g = g;
  pg->mul_hw = mgx::conv::pg_mul(g.H * g.W);
  pg->mul_w = mgx::conv::pg_mul(g.W);
  *pk = pool_square(g) == 32 ? 32 : 1;
  return MGX_OK;
}

extern "C" int mgx_bn_bwd_reduce_pooled(const float* dy_pool, const void* argmax,
                                        const int64_t* geom, int full, const float* x,
                                        const float* stats, int64_t M, int64_t C, void* ws,
                                        float* sums, float* dbeta, float* dgamma, int dgamma_zero,
                                        const float* relu_gamma, const float* relu_beta,
                                        uintptr_t stream) {
  MGX_REQUIRE(x && stats && ws && sums && M > 0 && C > 0 && mgx::aligned16(x),
              "mgx_bn_bwd_reduce_pooled: bad arguments");
  mgx::conv::PoolGrad pg;
  int pk = 0;
  MGX_TRY(pool_grad_of(dy_pool, argmax, geom, full, M, C, &pg, &pk));
  cudaStream_t st = mgx::as_stream(stream);
  const int64_t Mp = int64_t(pg.g.B) * pg.g.Ho * pg.g.Wo;
  int64_t rpc;
  int nchunk;
  mgx::conv::chunks_for(Mp, C, &rpc, &nchunk);
  const int C4 = static_cast<int>(C / 4);
  const int ct4 = C4 < mgx::conv::kRedThreads ? C4 : mgx::conv::kRedThreads;
  const int rpp = mgx::conv::kRedThreads / ct4;
  const size_t smem = size_t(rpp) * 2 * ct4 * 4 * sizeof(double);
  dim3 grid(nchunk, static_cast<unsigned>(mgx::ceil_div(C4, ct4)));
  double* wsd = static_cast<double*>(ws);
  const uint32_t mkw = static_cast<uint32_t>((65536 + pg.g.kw - 1) / pg.g.kw);
  // 4 resident CTAs per SM with 2 windows in flight per thread
  mgx::conv::bn_pool_reduce_kernel<4, 2><<<grid, ct4 * rpp, smem, st>>>(
      pg, x, stats, mgx::conv::ReluMask{relu_gamma, relu_beta}, Mp, static_cast<int>(C), rpc, wsd,
      mkw, mgx::conv::pg_mul(pg.g.Ho * pg.g.Wo), mgx::conv::pg_mul(pg.g.Wo));
  mgx::conv::colsum_finalize_kernel<<<static_cast<unsigned>(mgx::ceil_div(C, mgx::conv::kFinChannels)), 256, 0, st>>>(
      wsd, nchunk, static_cast<int>(C), 1, sums, dbeta, dgamma, dgamma_zero);
  MGX_LAUNCHED();
  return MGX_OK;
}

extern "C" int mgx_bn_bwd_dx_pooled(const float* dy_pool, const void* argmax, const int64_t* geom,
                                    int full, const float* x, const float* stats,
                                    const float* sums, const float* gamma, int64_t M, int64_t C,
                                    const float* relu_beta, float* dsum, void* ws, float* dx,
                                    void* dx16, uintptr_t stream) {
  MGX_REQUIRE(x && stats && sums && ws && (dx || dx16) && M > 0 && C > 0 &&
                  mgx::aligned16(x) && (!dx || mgx::aligned16(dx)) &&
                  (!dx16 || mgx::aligned16(dx16)),
              "mgx_bn_bwd_dx_pooled: bad arguments");
  mgx::conv::PoolGrad pg;
  int pk = 0;
  MGX_TRY(pool_grad_of(dy_pool, argmax, geom, full, M, C, &pg, &pk));
  cudaStream_t st = mgx::as_stream(stream);
  int64_t rpc;
  int nchunk;
  mgx::conv::chunks_for(M, C, &rpc, &nchunk);
  const int C4 = static_cast<int>(C / 4);
  const int ct4 = C4 < mgx::conv::kRedThreads ? C4 : mgx::conv::kRedThreads;
  const int rpp = mgx::conv::kRedThreads / ct4;
  const size_t smem = size_t(rpp) * ct4 * 4 * sizeof(double);
  dim3 grid(nchunk, static_cast<unsigned>(mgx::ceil_div(C4, ct4)));
  // the ReLU mask uses the BatchNorm gamma (relu_beta non-NULL: fused ReLU)
  const mgx::conv::ReluMask rm{relu_beta ? gamma : nullptr, relu_beta};
  __nv_bfloat16* h16 = static_cast<__nv_bfloat16*>(dx16);
  double* wsd = static_cast<double*>(ws);
  static const bool block_dx = [] {
    const char* v = getenv("MGX_STEM_DX_BLOCK");
    return !(v && *v == '0');
  }();
  if (block_dx && pk == 32 && pg.g.ph == 0 && pg.g.pw == 0 && dx == nullptr && dx16 != nullptr) {
    // 2x2 pixel blocks: 4 windows cover a block
    const int Hb = (pg.g.H + 1) / 2, Wb = (pg.g.W + 1) / 2;
    const int64_t Mb = int64_t(pg.g.B) * Hb * Wb;
    int64_t rpcb;
    int nchunkb;
    mgx::conv::chunks_for(Mb, C, &rpcb, &nchunkb);
    dim3 gridb(nchunkb, static_cast<unsigned>(mgx::ceil_div(C4, ct4)));
    mgx::conv::bn_pool_dx_k3s2_kernel<1><<<gridb, ct4 * rpp, smem, st>>>(
        pg, x, stats, sums, gamma, rm, M, Mb, static_cast<int>(C), rpcb, wsd, h16,
        mgx::conv::pg_mul(Hb * Wb), mgx::conv::pg_mul(Wb));
    if (dsum)
      mgx::conv::colsum_finalize_kernel<<<static_cast<unsigned>(mgx::ceil_div(C, mgx::conv::kFinChannels)), 256, 0, st>>>(
          wsd, nchunkb, static_cast<int>(C), 0, dsum, nullptr, nullptr, 0);
    MGX_LAUNCHED();
    return MGX_OK;
  }
  if (pk == 32)
    mgx::conv::bn_dx_colsum_kernel<32><<<grid, ct4 * rpp, smem, st>>>(
        nullptr, x, stats, sums, gamma, dx, rm, M, static_cast<int>(C), rpc, wsd, h16, pg);
  else
    mgx::conv::bn_dx_colsum_kernel<1><<<grid, ct4 * rpp, smem, st>>>(
        nullptr, x, stats, sums, gamma, dx, rm, M, static_cast<int>(C), rpc, wsd, h16, pg);
  if (dsum)
    mgx::conv::colsum_finalize_kernel<<<static_cast<unsigned>(mgx::ceil_div(C, mgx::conv::kFinChannels)), 256, 0, st>>>(
        wsd, nchunk, static_cast<int>(C), 0, dsum, nullptr, nullptr, 0);
  MGX_LAUNCHED();
  return MGX_OK;
}

extern "C" int mgx_chan_copy(const float* src, int64_t lds, int64_t soff, float* dst, int64_t ldd,
                             int64_t doff, int64_t rows, int64_t cols, void* dst16,
                             uintptr_t stream) {
  MGX_REQUIRE(src && dst && rows >= 0 && cols >= 0, "mgx_chan_copy: bad arguments");
  MGX_REQUIRE(!dst16 || (((cols | lds | soff | ldd | doff) & 3) == 0 && mgx::aligned16(dst16)),
              "mgx_chan_copy: a bf16 copy needs 4-aligned columns");
  if (rows == 0 || cols == 0) return MGX_OK;
  if (((cols | lds | soff | ldd | doff) & 3) == 0)
    mgx::conv::chan_copy_kernel<<<mgx::rows_grid(rows, cols / 4, 4),
                                  mgx::rows_block(cols / 4), 0,
                                  mgx::as_stream(stream)>>>(src, lds, soff, dst, ldd, doff, rows, cols,
                                                            static_cast<__nv_bfloat16*>(dst16));
  else
    mgx::conv::chan_copy_kernel<<<grid_for(rows * cols), 256, 0, mgx::as_stream(stream)>>>(
        src, lds, soff, dst, ldd, doff, rows, cols, nullptr);
  MGX_LAUNCHED();
  return MGX_OK;
}

extern "C" int mgx_weight_flip_bf16(const float* w, int64_t F, int64_t kh, int64_t kw, int64_t C,
                                    void* wf, int64_t ld, uintptr_t stream) {
  MGX_REQUIRE(w && wf && F > 0 && kh > 0 && kw > 0 && C > 0 && ld >= kh * kw * F,
              "mgx_weight_flip_bf16: bad arguments");
  mgx::conv::weight_flip_kernel<<<grid_for(C * ld), 256, 0, mgx::as_stream(stream)>>>(
      w, static_cast<int>(F), static_cast<int>(kh), static_cast<int>(kw), static_cast<int>(C),
      static_cast<__nv_bfloat16*>(wf), ld);
  MGX_LAUNCHED();
  return MGX_OK;
}

extern "C" int mgx_prep_batch(const void* jobs, int64_t njobs, int64_t units, uintptr_t stream) {
  MGX_REQUIRE(jobs && njobs > 0 && njobs <= mgx::conv::kPrepMaxJobs && units > 0,
              "mgx_prep_batch: bad arguments");
  mgx::conv::prep_batch_kernel<<<grid_for(units), 256, 0, mgx::as_stream(stream)>>>(
      static_cast<const mgx_prep_job*>(jobs), static_cast<int>(njobs), units);
  MGX_LAUNCHED();
  return MGX_OK;
}

extern "C" int mgx_bn_stats_from_tiles(const void* part, int64_t M, int64_t C, float* stats,
                                       float* moving_mean, float* moving_var, float eps,
                                       float momentum, uintptr_t stream) {
  MGX_REQUIRE(part && stats && M > 0 && C > 0, "mgx_bn_stats_from_tiles: bad arguments");
  // many row blocks (the stem's 112x112 / 56x56 maps): the cluster kernel
  // (coalesced 32-channel rows over 16 CTAs per channel group); else one
  // block per channel (env MGX_BN_STATS_CLUSTER=0: always the latter)
  static const bool cluster = [] {
    const char* v = getenv("MGX_BN_STATS_CLUSTER");
    return !(v && *v == '0');
  }();
  if (cluster && M >= (int64_t(1) << 16)) {
    constexpr int CS = 16;
    static bool attrs = false;
    if (!attrs) {
      MGX_CUDA(cudaFuncSetAttribute(mgx::conv::bn_stats_tiles_cluster_kernel<CS>,
                                    cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      attrs = true;
    }
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(CS, static_cast<unsigned>(mgx::ceil_div(C, int64_t(32))), 1);
    lc.blockDim = dim3(1024, 1, 1);
    lc.stream = mgx::as_stream(stream);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CS;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    MGX_CUDA(cudaLaunchKernelEx(&lc, mgx::conv::bn_stats_tiles_cluster_kernel<CS>,
                                static_cast<const float2*>(part), M, static_cast<int>(C), eps,
                                momentum, stats, moving_mean, moving_var));
    return MGX_OK;
  }
  mgx::conv::bn_stats_from_tiles_kernel<<<static_cast<unsigned>(C), 1024, 0, mgx::as_stream(stream)>>>(
      static_cast<const float2*>(part), M, static_cast<int>(C), eps, momentum, stats, moving_mean,
      moving_var);
  MGX_LAUNCHED();
  return MGX_OK;
}

extern "C" int mgx_sum_n(const float* const* srcs, int32_t count, float* out, int64_t n,
                         uintptr_t stream) {
  MGX_REQUIRE(srcs && out && count >= 1 && count <= 6 && n >= 0, "mgx_sum_n: bad arguments");
  MGX_REQUIRE(n % 4 == 0 && mgx::aligned16(out), "mgx_sum_n: needs n %% 4 == 0 and aligned data");
  mgx::conv::SumSrcs s;
  s.n = count;
  for (int k = 0; k < 6; ++k) s.p[k] = k < count ? srcs[k] : nullptr;
  for (int k = 0; k < count; ++k)
    MGX_REQUIRE(s.p[k] && mgx::aligned16(s.p[k]), "mgx_sum_n: source %d null or unaligned", k);
  if (n == 0) return MGX_OK;
  mgx::conv::sum_n_kernel<<<grid_for(n / 4), 256, 0, mgx::as_stream(stream)>>>(s, out, n / 4);
  MGX_LAUNCHED();
  return MGX_OK;
}

extern "C" int mgx_concat(const float* const* srcs, const int64_t* channels, int32_t count,
                          float* out, void* out16, int64_t rows, uintptr_t stream) {
  MGX_REQUIRE(srcs && channels && out && count >= 1 && count <= 4 && rows >= 0,
              "mgx_concat: bad arguments");
  mgx::conv::CatSrcs in;
  in.n = count;
  int ctot = 0;
  for (int k = 0; k < 4; ++k) {
    in.p[k] = k < count ? srcs[k] : nullptr;
    in.c[k] = k < count ? static_cast<int>(channels[k]) : 0;
  }
  for (int k = 0; k < count; ++k) {
    MGX_REQUIRE(in.p[k] && in.c[k] > 0 && in.c[k] % 4 == 0 && mgx::aligned16(in.p[k]),
                "mgx_concat: input %d needs channels %% 4 == 0 and aligned data", k);
    ctot += in.c[k];
  }
  MGX_REQUIRE(mgx::aligned16(out) && (!out16 || mgx::aligned16(out16)), "mgx_concat: unaligned output");
  if (rows == 0) return MGX_OK;
  mgx::conv::concat_kernel<<<mgx::rows_grid(rows, ctot / 4, 8), mgx::rows_block(ctot / 4), 0,
                             mgx::as_stream(stream)>>>(in, out, rows, ctot,
                                                       static_cast<__nv_bfloat16*>(out16));
  MGX_LAUNCHED();
  return MGX_OK;
}
