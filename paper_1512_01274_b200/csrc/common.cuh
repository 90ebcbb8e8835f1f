// Shared helpers for the mgx C-ABI implementation.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "mgx.h"

namespace mgx {

void set_error(const char* fmt, ...);
cudaStream_t as_stream(uintptr_t s);

}  // namespace mgx

#define MGX_CUDA(call)                                                        \
  do {                                                                        \
    cudaError_t e_ = (call);                                                  \
    if (e_ != cudaSuccess) {                                                  \
      mgx::set_error("%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_),  \
                     __FILE__, __LINE__);                                     \
      return MGX_INTERNAL;                                                    \
    }                                                                         \
  } while (0)

#define MGX_LAUNCHED() MGX_CUDA(cudaGetLastError())

#define MGX_REQUIRE(cond, ...)      \
  do {                              \
    if (!(cond)) {                  \
      mgx::set_error(__VA_ARGS__);  \
      return MGX_BAD_ARGUMENT;      \
    }                               \
  } while (0)

#define MGX_TRY(call)          \
  do {                         \
    int st_ = (call);          \
    if (st_ != MGX_OK) return st_; \
  } while (0)

namespace mgx {

// Every parity kernel spells out its roundings: one rounding per mul and per
// add, never contracted into an FMA (the reference is numpy, which rounds
// the product array before reducing it).  The library is also compiled with
// -fmad=false as a second line of defence.
__device__ __forceinline__ float fadd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float fsub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float fmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float fdiv(float a, float b) { return __fdiv_rn(a, b); }

// numpy.maximum(x, 0) (ops.py:139): returns x when x >= 0 or x is NaN.
__device__ __forceinline__ float relu(float x) { return (x >= 0.0f || x != x) ? x : 0.0f; }

// float32 exp / tanh rounded from double precision.  numpy's SIMD float32
// exp/tanh are not correctly rounded (probe: ~39% of exp results differ from
// the correctly rounded value), so these ops are tolerance-matched, not
// bitwise; rounding from double keeps the GPU result within 1 ulp of truth.
__device__ __forceinline__ float exp_rn(float x) { return __double2float_rn(exp((double)x)); }
__device__ __forceinline__ float tanh_rn(float x) { return __double2float_rn(tanh((double)x)); }

// sigmoid as written at kernels.py:60: 1.0 / (1.0 + exp(-x)), in float32.
__device__ __forceinline__ float sigmoid(float x) {
  return fdiv(1.0f, fadd(1.0f, exp_rn(-x)));
}

__device__ __forceinline__ float act_forward(int act, float x) {
  switch (act) {
    case MGX_ACT_RELU: return relu(x);
    case MGX_ACT_SIGMOID: return sigmoid(x);
    case MGX_ACT_TANH: return tanh_rn(x);
    default: return x;
  }
}

// Backward through the activation's output y (ops.py:140-147):
//   relu: og * (y > 0)     sigmoid: og * y * (1 - y)     tanh: og * (1 - y*y)
__device__ __forceinline__ float act_backward(int act, float y, float og) {
  switch (act) {
    case MGX_ACT_RELU: return fmul(og, y > 0.0f ? 1.0f : 0.0f);
    case MGX_ACT_SIGMOID: return fmul(fmul(og, y), fsub(1.0f, y));
    case MGX_ACT_TANH: return fmul(og, fsub(1.0f, fmul(y, y)));
    default: return og;
  }
}

constexpr int kNumSMs = 148;

// CTA cap for the tensor-core GEMMs launched by this host thread (0: none):
// the multi-lane program runner sets it for the instructions OFF the
// critical lane, so their persistent grids leave SMs to the critical path
// (tc_gemm.cu; runtime.cu run_range).
void set_gemm_cta_cap(int cap);

// One leaf of numpy's pairwise-summation split tree over n elements
// (see dense.cu); `merges` = number of stack merges after this leaf.
struct PwLeaf {
  int32_t start;
  int32_t len;
  int32_t merges;
  int32_t pad;
};
// Device-resident leaf table for length K (cached per device and K).
// The table holds the leaves followed by `nchunks` chunk records
// {k0, klen, leaf_begin, leaf_end} (runs of whole leaves of <= 512 elements).
int pw_leaf_table(int64_t K, const PwLeaf** out, int* nleaves, int* max_depth,
                  int* nchunks = nullptr);

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// ---- cp.async (LDGSTS) staging helpers: global -> shared without a register
// round trip, so a whole operand tile is in flight at once.  `valid == false`
// zero-fills the destination (src-size 0; the source pointer must still be a
// mapped address).
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src),
               "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_u32(dst)), "l"(src),
               "r"(valid ? 4 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// Row-by-vector launch shape shared by the bandwidth kernels: a thread
// owns one vector column v of the rows (fixed per thread, so its per-column
// constants load once) and walks rows, with tpr = min(V, 256) threads per
// row and rpb = 256 / tpr rows per block pass; the block is tpr * rpb
// threads (rows_block), so no lane idles for any V -- no 64-bit division per
// element either.
constexpr int kRowsThreads = 256;

struct RowsIdx {
  int v, r, rstep;
  bool active;
  __device__ __forceinline__ RowsIdx(int V) {
    const int tpr = V < kRowsThreads ? V : kRowsThreads;
    const int rpb = blockDim.x / tpr;
    const int t = threadIdx.x;
    const int rin = t / tpr;
    v = blockIdx.x * tpr + (t - rin * tpr);
    r = blockIdx.y * rpb + rin;
    rstep = gridDim.y * rpb;
    active = rin < rpb && v < V;
  }
};

inline int rows_block(int64_t vecs) {
  const int64_t tpr = vecs < kRowsThreads ? (vecs < 1 ? 1 : vecs) : kRowsThreads;
  return static_cast<int>(tpr * (kRowsThreads / tpr));
}

// min_rows: rows each thread walks at least (kernels with per-thread setup)
inline dim3 rows_grid(int64_t rows, int64_t vecs, int64_t min_rows = 1) {
  const int64_t tpr = vecs < kRowsThreads ? (vecs < 1 ? 1 : vecs) : kRowsThreads;
  const int64_t rpb = kRowsThreads / tpr;
  const int64_t gx = ceil_div(vecs < 1 ? 1 : vecs, tpr);
  int64_t gy = ceil_div(rows, rpb * (min_rows < 1 ? 1 : min_rows));
  const int64_t cap = ceil_div(int64_t(kNumSMs) * 16, gx);
  if (gy > cap) gy = cap;
  if (gy > 65535) gy = 65535;
  return dim3(static_cast<unsigned>(gx), static_cast<unsigned>(gy < 1 ? 1 : gy));
}


}  // namespace mgx
