// Persistent program kernel: a whole executor pass in ONE launch.
//
// The executor's instruction list (runtime.cu) is split into dependency
// levels on the host: an instruction's level is one more than the highest
// level of any earlier instruction whose byte ranges conflict with it
// (read-after-write, write-after-read, write-after-write).  Instructions of
// one level are independent, so their tiles form one flat tile space.  The
// kernel is launched cooperatively with every block resident; each block
// walks the levels, runs tiles of the current level (tile functions from
// tiles.cuh), and meets the other blocks at a grid barrier before the next
// level.  For the config-1 MLP this turns 10 kernels into one launch with 8
// levels (independent dX and dW/db nodes share a level).

#include <algorithm>
#include <cstring>
#include <map>
#include <mutex>
#include <utility>
#include <vector>

#include "fused.cuh"
#include "tiles.cuh"

namespace mgx {

struct MegaOp {
  int32_t op, act;
  int32_t ntiles, tiles_x;
  int32_t variant;   // pairwise stack depth / batch-tree levels
  int32_t kc, nleaves, nchunks;
  int32_t vec0, vec1;
  const PwLeaf* table;
  int64_t dims[8];
  float fattr[4];
  void* ptr[6];
};

struct MegaLevel {
  int32_t first, count, tiles;
};

__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Grid barrier on a monotonically increasing arrival counter: level k ends
// when (k+1)*gridDim.x blocks have arrived.  The fences make the level's
// global writes visible and drop stale L1 lines before the next level.
__device__ __forceinline__ uint64_t now_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// A block that waits more than 10 s (another kernel holding SMs, so not
// every block became resident) records the failure in host-mapped memory
// and continues instead of hanging the device.
__device__ __forceinline__ void grid_barrier(uint32_t* counter, uint32_t target, uint32_t* err) {
  // release-add publishes this block's writes (ordered before it by the
  // bar.sync), acquire-polling makes the other blocks' writes visible
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(counter) : "memory");
    const uint64_t t0 = now_ns();
    while (ld_acquire_gpu(counter) < target) {
      if (now_ns() - t0 > 10ull * 1000 * 1000 * 1000) {
        atomicExch(err, 1u);
        break;
      }
    }
  }
  __syncthreads();
}

__device__ void run_tile(const MegaOp& o, int t, float* smem) {
  const int64_t* d = o.dims;
  float* p0 = static_cast<float*>(o.ptr[0]);
  float* p1 = static_cast<float*>(o.ptr[1]);
  float* p2 = static_cast<float*>(o.ptr[2]);
  float* p3 = static_cast<float*>(o.ptr[3]);
  switch (o.op) {
    case MGX_OP_GEMM_PW: {
      const int bx = t % o.tiles_x, by = t / o.tiles_x;
#define MGX_PW_TILE(Dd)                                                                         \
  pw_tile<2, 2, Dd>(bx, by, smem, p0, int(d[3]), p1, int(d[4]), p2, p3, int(d[5]), int(d[0]), \
                    int(d[1]), int(d[2]), o.table, o.nleaves, o.nchunks, o.act, o.kc,         \
                    o.vec0 != 0, o.vec1 != 0)
      if (o.variant == 1) MGX_PW_TILE(1);
      else MGX_PW_TILE(6);
#undef MGX_PW_TILE
      break;
    }
    case MGX_OP_GEMM_SEQ: {
      const int bx = t % o.tiles_x, by = t / o.tiles_x;
      seq_tile(bx, by, smem, p0, d[3], d[4], p1, d[5], d[6], p2, d[7], p3, o.act, d[0], d[1],
               d[2]);
      break;
    }
    case MGX_OP_DW_DB: {
      const int bx = t % o.tiles_x, by = t / o.tiles_x;
      dw_tile<8>(bx, by, smem, p0, p1, p2, p3, d[0], d[1], p2 ? d[2] : 1, o.vec0 != 0,
                 o.vec1 != 0);
      break;
    }
    case MGX_OP_SOFTMAX_FWD:
      softmax_fwd_tile(t, p0, p1, d[0], d[1], o.table, o.nleaves);
      break;
    case MGX_OP_SOFTMAX_BWD:
      map_tile(t, d[0] * d[1], false,
               SoftmaxBwdOp{p0, p1, p2, d[1], static_cast<float>(d[0])});
      break;
    case MGX_OP_FILL: map_tile(t, d[0], o.vec0 != 0, FillOp{p0, o.fattr[0]}); break;
    case MGX_OP_COPY: map_tile(t, d[0], o.vec0 != 0, CopyOp{p0, p1}); break;
    case MGX_OP_EW: map_tile(t, d[0], o.vec0 != 0, EwOp{p0, p1, p2, int(d[1])}); break;
    case MGX_OP_SCALAR:
      map_tile(t, d[0], o.vec0 != 0, ScalarOp{p0, p1, o.fattr[0], int(d[1])});
      break;
    case MGX_OP_ACT_FWD: map_tile(t, d[0], o.vec0 != 0, ActFwdOp{p0, p1, o.act}); break;
    case MGX_OP_ACT_BWD: map_tile(t, d[0], o.vec0 != 0, ActBwdOp{p0, p1, p2, o.act}); break;
    case MGX_OP_AXPY: map_tile(t, d[0], o.vec0 != 0, AxpyOp{p0, p1, o.fattr[0]}); break;
    default: break;
  }
}

// The whole op/level table travels as one __grid_constant__ kernel
// parameter: tiles read their descriptors through the constant cache
// (uniform broadcast) instead of dependent global loads.
constexpr int kMaxProgramOps = 48;
constexpr int kMaxProgramLevels = 48;

struct ProgramParams {
  uint32_t* barrier;
  uint32_t* err;
  unsigned long long* times;  // optional: [0] launch start, [1+lv] last block done with level lv
  int32_t nlevels, nops;
  MegaLevel levels[kMaxProgramLevels];
  MegaOp ops[kMaxProgramOps];
};

__global__ void __launch_bounds__(256, 1)
program_kernel(const __grid_constant__ ProgramParams p) {
  extern __shared__ float4 smem_f4[];
  float* smem = reinterpret_cast<float*>(smem_f4);
  uint32_t* barrier = p.barrier;
  if (p.times && threadIdx.x == 0) atomicMin(&p.times[0], static_cast<unsigned long long>(now_ns()));
  for (int lv = 0; lv < p.nlevels; ++lv) {
    const MegaLevel L = p.levels[lv];
    for (int t = blockIdx.x; t < L.tiles; t += gridDim.x) {
      int j = L.first, base = 0;
      while (t - base >= p.ops[j].ntiles) {
        base += p.ops[j].ntiles;
        ++j;
      }
      run_tile(p.ops[j], t - base, smem);
      __syncthreads();
    }
    if (p.times && threadIdx.x == 0)
      atomicMax(&p.times[1 + lv], static_cast<unsigned long long>(now_ns()));
    if (lv + 1 < p.nlevels) grid_barrier(barrier, uint32_t(lv + 1) * gridDim.x, p.err);
  }
  // last block out resets the counters for the next launch
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t prev = atomicAdd(barrier + 1, 1u);
    if (prev == gridDim.x - 1) {
      barrier[0] = 0;
      barrier[1] = 0;
      __threadfence();
    }
  }
}

// ------------------------------------------------------------------ host

// process-wide error word in host-mapped pinned memory (barrier timeouts)
uint32_t* program_error_word() {
  static uint32_t* word = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    if (cudaHostAlloc(&p, 64, cudaHostAllocMapped | cudaHostAllocPortable) == cudaSuccess) {
      std::memset(p, 0, 64);
      word = static_cast<uint32_t*>(p);
    }
  });
  return word;
}

struct Range {
  uintptr_t lo, hi;
};

static void extents(const mgx_instr& in, std::vector<Range>& rd, std::vector<Range>& wr) {
  auto R = [](const void* p, int64_t nfloats) {
    return Range{reinterpret_cast<uintptr_t>(p), reinterpret_cast<uintptr_t>(p) + 4 * uintptr_t(nfloats)};
  };
  const int64_t* d = in.dims;
  switch (in.op) {
    case MGX_OP_FILL: wr.push_back(R(in.ptr[0], d[0])); break;
    case MGX_OP_COPY: rd.push_back(R(in.ptr[0], d[0])); wr.push_back(R(in.ptr[1], d[0])); break;
    case MGX_OP_EW:
      rd.push_back(R(in.ptr[0], d[0]));
      rd.push_back(R(in.ptr[1], d[0]));
      wr.push_back(R(in.ptr[2], d[0]));
      break;
    case MGX_OP_SCALAR:
    case MGX_OP_ACT_FWD:
      rd.push_back(R(in.ptr[0], d[0]));
      wr.push_back(R(in.ptr[1], d[0]));
      break;
    case MGX_OP_ACT_BWD:
      rd.push_back(R(in.ptr[0], d[0]));
      rd.push_back(R(in.ptr[1], d[0]));
      wr.push_back(R(in.ptr[2], d[0]));
      break;
    case MGX_OP_AXPY:
      rd.push_back(R(in.ptr[0], d[0]));
      rd.push_back(R(in.ptr[1], d[0]));
      wr.push_back(R(in.ptr[1], d[0]));
      break;
    case MGX_OP_GEMM_PW:  // M,N,K,lda,ldb,ldc
      rd.push_back(R(in.ptr[0], (d[0] - 1) * d[3] + d[2]));
      rd.push_back(R(in.ptr[1], (d[1] - 1) * d[4] + d[2]));
      if (in.ptr[2]) rd.push_back(R(in.ptr[2], d[1]));
      wr.push_back(R(in.ptr[3], (d[0] - 1) * d[5] + d[1]));
      break;
    case MGX_OP_GEMM_SEQ:  // M,N,K,sam,sak,sbk,sbn,ldc
      rd.push_back(R(in.ptr[0], (d[0] - 1) * d[3] + (d[2] - 1) * d[4] + 1));
      rd.push_back(R(in.ptr[1], (d[2] - 1) * d[5] + (d[1] - 1) * d[6] + 1));
      if (in.ptr[3]) rd.push_back(R(in.ptr[3], (d[0] - 1) * d[7] + d[1]));
      wr.push_back(R(in.ptr[2], (d[0] - 1) * d[7] + d[1]));
      break;
    case MGX_OP_DW_DB:  // B,H,F
      rd.push_back(R(in.ptr[0], d[0] * d[1]));
      if (in.ptr[2]) {
        rd.push_back(R(in.ptr[1], d[0] * d[2]));
        wr.push_back(R(in.ptr[2], d[1] * d[2]));
      }
      if (in.ptr[3]) wr.push_back(R(in.ptr[3], d[1]));
      break;
    case MGX_OP_SOFTMAX_FWD:
      rd.push_back(R(in.ptr[0], d[0] * d[1]));
      wr.push_back(R(in.ptr[1], d[0] * d[1]));
      break;
    case MGX_OP_SOFTMAX_BWD:
      rd.push_back(R(in.ptr[0], d[0] * d[1]));
      rd.push_back(R(in.ptr[1], d[0]));
      wr.push_back(R(in.ptr[2], d[0] * d[1]));
      break;
    default: break;
  }
}

static bool overlaps(const std::vector<Range>& a, const std::vector<Range>& b) {
  for (const auto& x : a)
    for (const auto& y : b)
      if (x.lo < y.hi && y.lo < x.hi) return true;
  return false;
}

static bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// Fill a MegaOp; returns false if the instruction has no megakernel variant.
static int build_op(const mgx_instr& in, MegaOp* o, size_t* smem_need) {
  std::memset(o, 0, sizeof(*o));
  o->op = in.op;
  o->act = in.act;
  std::memcpy(o->dims, in.dims, sizeof(o->dims));
  std::memcpy(o->fattr, in.fattr, sizeof(o->fattr));
  std::memcpy(o->ptr, in.ptr, sizeof(o->ptr));
  const int64_t* d = in.dims;
  auto tiles_of = [](int64_t n) { return static_cast<int32_t>(ceil_div(n, kMapTile)); };
  switch (in.op) {
    case MGX_OP_GEMM_PW: {
      int nl = 0, depth = 0, nc = 0;
      const PwLeaf* t = nullptr;
      MGX_TRY(pw_leaf_table(d[2], &t, &nl, &depth, &nc));
      if (depth > 6) {  // K > ~4096: the per-instruction kernels handle it
        set_error("program kernel: pairwise depth %d unsupported", depth);
        return MGX_BAD_ARGUMENT;
      }
      o->variant = depth <= 1 ? 1 : 6;
      o->table = t;
      o->nleaves = nl;
      o->nchunks = nc;
      o->kc = static_cast<int32_t>(d[2] >= 512 ? 512 : ((d[2] + 7) / 8) * 8);
      o->vec0 = (d[3] % 4 == 0) && (d[2] % 4 == 0) && al16(in.ptr[0]);
      o->vec1 = (d[4] % 4 == 0) && (d[2] % 4 == 0) && al16(in.ptr[1]);
      o->tiles_x = static_cast<int32_t>(ceil_div(d[1], 16));
      o->ntiles = o->tiles_x * static_cast<int32_t>(ceil_div(d[0], 8));
      *smem_need = std::max<size_t>(*smem_need, size_t(2) * 24 * (o->kc + 4) * 4);
      break;
    }
    case MGX_OP_GEMM_SEQ:
      o->tiles_x = static_cast<int32_t>(ceil_div(d[1], kSeqBN));
      o->ntiles = o->tiles_x * static_cast<int32_t>(ceil_div(d[0], kSeqBM));
      *smem_need = std::max<size_t>(*smem_need, kSeqSmemFloats * 4);
      break;
    case MGX_OP_DW_DB: {
      if (!in.ptr[2] && !in.ptr[3]) break;
      const int64_t nch = d[0] >> 3;
      if (nch >= (1 << 8)) {
        set_error("program kernel: batch %lld too large", static_cast<long long>(d[0]));
        return MGX_BAD_ARGUMENT;
      }
      o->variant = 8;
      o->vec0 = (d[1] % 4 == 0) && al16(in.ptr[0]);
      o->vec1 = in.ptr[2] && (d[2] % 4 == 0) && al16(in.ptr[1]);
      o->tiles_x = in.ptr[2] ? static_cast<int32_t>(ceil_div(d[2], kDwBF)) : 1;
      o->ntiles = o->tiles_x * static_cast<int32_t>(ceil_div(d[1], kDwBH));
      *smem_need = std::max<size_t>(*smem_need, kDwSmemFloats * 4);
      break;
    }
    case MGX_OP_SOFTMAX_FWD: {
      int nl = 0, depth = 0;
      const PwLeaf* t = nullptr;
      MGX_TRY(pw_leaf_table(d[1], &t, &nl, &depth));
      o->table = t;
      o->nleaves = nl;
      o->ntiles = static_cast<int32_t>(ceil_div(d[0], 32));
      break;
    }
    case MGX_OP_SOFTMAX_BWD: o->ntiles = tiles_of(d[0] * d[1]); break;
    case MGX_OP_FILL:
      o->vec0 = al16(in.ptr[0]);
      o->ntiles = tiles_of(d[0]);
      break;
    case MGX_OP_COPY:
      o->vec0 = al16(in.ptr[0]) && al16(in.ptr[1]);
      o->ntiles = in.ptr[0] == in.ptr[1] ? 0 : tiles_of(d[0]);
      break;
    case MGX_OP_EW:
    case MGX_OP_ACT_BWD:
      o->vec0 = al16(in.ptr[0]) && al16(in.ptr[1]) && al16(in.ptr[2]);
      o->ntiles = tiles_of(d[0]);
      break;
    case MGX_OP_SCALAR:
    case MGX_OP_ACT_FWD:
    case MGX_OP_AXPY:
      o->vec0 = al16(in.ptr[0]) && al16(in.ptr[1]);
      o->ntiles = tiles_of(d[0]);
      break;
    default:
      set_error("program kernel: opcode %d unsupported", in.op);
      return MGX_BAD_ARGUMENT;
  }
  return MGX_OK;
}

int build_fused(const mgx_instr* instrs, int n, FusedRange* out) {
  // allocate the error word now: a first use inside a stream capture would
  // allocate during capture and invalidate it
  if (!program_error_word()) {
    set_error("program kernel: cannot allocate the host-mapped error word");
    return MGX_INTERNAL;
  }
  std::vector<std::vector<Range>> rd(n), wr(n);
  for (int i = 0; i < n; ++i) extents(instrs[i], rd[i], wr[i]);
  std::vector<int> level(n, 0);
  int nlevels = 0;
  for (int i = 0; i < n; ++i) {
    int lv = 0;
    for (int j = 0; j < i; ++j) {
      if (overlaps(wr[j], rd[i]) || overlaps(wr[j], wr[i]) || overlaps(rd[j], wr[i]))
        lv = std::max(lv, level[j] + 1);
    }
    level[i] = lv;
    nlevels = std::max(nlevels, lv + 1);
  }
  std::vector<MegaOp> ops;
  std::vector<MegaLevel> levels;
  size_t smem = 0;
  int max_tiles = 1;
  for (int lv = 0; lv < nlevels; ++lv) {
    MegaLevel L{static_cast<int32_t>(ops.size()), 0, 0};
    for (int i = 0; i < n; ++i) {
      if (level[i] != lv) continue;
      MegaOp o;
      MGX_TRY(build_op(instrs[i], &o, &smem));
      if (o.ntiles == 0) continue;
      ops.push_back(o);
      ++L.count;
      L.tiles += o.ntiles;
    }
    if (L.count == 0) continue;
    max_tiles = std::max(max_tiles, static_cast<int>(L.tiles));
    levels.push_back(L);
  }
  if (levels.empty()) {
    out->nlevels = 0;
    return MGX_OK;
  }
  int dev = 0, sms = kNumSMs, per_sm = 0;
  MGX_CUDA(cudaGetDevice(&dev));
  MGX_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  {
    // the attribute is per function: only ever raise it, or building one
    // range would shrink the limit another range was built with
    static std::mutex mu;
    static size_t granted[16] = {0};
    std::lock_guard<std::mutex> lock(mu);
    if (smem > granted[dev & 15]) {
      MGX_CUDA(cudaFuncSetAttribute(program_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(smem)));
      granted[dev & 15] = smem;
    }
  }
  MGX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, program_kernel, 256,
                                                         std::max<size_t>(smem, 16)));
  if (per_sm < 1) {
    set_error("program kernel does not fit on an SM (smem %zu)", smem);
    return MGX_INTERNAL;
  }
  if (ops.size() > size_t(kMaxProgramOps) || levels.size() > size_t(kMaxProgramLevels)) {
    set_error("program kernel: %zu ops / %zu levels exceed %d / %d", ops.size(), levels.size(),
              kMaxProgramOps, kMaxProgramLevels);
    return MGX_BAD_ARGUMENT;
  }
  out->grid = std::min(sms, max_tiles);
  out->smem = std::max<size_t>(smem, 16);
  out->nlevels = static_cast<int>(levels.size());
  out->level_of = level;
  MGX_CUDA(cudaMalloc(&out->d_barrier, 2 * sizeof(uint32_t)));
  MGX_CUDA(cudaMemset(out->d_barrier, 0, 2 * sizeof(uint32_t)));
  // the memset rides the legacy stream and may still be in flight; the
  // program kernel launches on a non-blocking stream, so finish it first
  MGX_CUDA(cudaDeviceSynchronize());
  auto* prm = new ProgramParams();
  std::memset(prm, 0, sizeof(*prm));
  prm->barrier = out->d_barrier;
  prm->err = program_error_word();
  prm->nlevels = static_cast<int32_t>(levels.size());
  prm->nops = static_cast<int32_t>(ops.size());
  std::copy(levels.begin(), levels.end(), prm->levels);
  std::copy(ops.begin(), ops.end(), prm->ops);
  out->params = prm;
  return MGX_OK;
}

int launch_fused(const FusedRange& f, cudaStream_t st) {
  if (f.nlevels == 0) return MGX_OK;
  // Plain launch, one block per SM: every block is resident when the stream
  // owns the device (cooperative launches were rejected for this kernel and
  // are not capturable here); the barrier times out instead of hanging.
  program_kernel<<<f.grid, 256, f.smem, st>>>(*f.params);
  MGX_LAUNCHED();
  return MGX_OK;
}

// One instrumented launch: ns from the first block's start to the last block
// finishing each level (includes that level's barrier wait of the previous).
int time_fused(const FusedRange& f, cudaStream_t st, double* ns_out) {
  if (f.nlevels == 0) return MGX_OK;
  // device-resident timestamps (host-mapped atomics would dominate the timing)
  std::vector<unsigned long long> host(f.nlevels + 1, 0);
  host[0] = ~0ull;
  unsigned long long* buf = nullptr;
  MGX_CUDA(cudaMalloc(&buf, host.size() * sizeof(unsigned long long)));
  cudaError_t e = cudaMemcpyAsync(buf, host.data(), host.size() * 8, cudaMemcpyHostToDevice, st);
  ProgramParams prm = *f.params;
  prm.times = buf;
  if (e == cudaSuccess) {
    program_kernel<<<f.grid, 256, f.smem, st>>>(prm);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(host.data(), buf, host.size() * 8, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e == cudaSuccess)
    for (int i = 0; i < f.nlevels; ++i) ns_out[i] = double(host[1 + i] - host[0]);
  cudaFree(buf);
  MGX_CUDA(e);
  return MGX_OK;
}

void free_fused(FusedRange& f) {
  if (f.d_barrier) cudaFree(f.d_barrier);
  delete f.params;
  f = FusedRange();
}

}  // namespace mgx
