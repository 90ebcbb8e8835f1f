// Device KVStore round: fused reduce -> update -> broadcast.
//
// Reference data path (kvstore.py):
//   push        worker copies its gradient to its level-1 server     (:190-211)
//   level 1     tree_sum over the machine's W workers, ascending id   (:328-338)
//   level 2     tree_sum over the M machine aggregates, ascending id  (:390-402)
//   updater     make_sgd_updater -> sgd_arrays (optim.py:53-78), or add (:47-49)
//   broadcast   snapshot copied to every level-1 server, pulls copy   (:373-375, :233-238)
//
// Here all of that is one pass over HBM/NVLink.  The element range of a key
// (or a bucket of small keys) is split into contiguous owner shards; the
// owner reads every worker's gradient for its shard (local HBM or a peer's
// over NVLink via CUDA IPC mappings), sums them with the reference's exact
// two-level balanced tree, applies the updater with its momentum shard, and
// stores the new weight into every worker's replica.  Per element this is the
// reference's float-op sequence, so the result is bitwise identical no matter
// how the range is sharded.
//
// Cross-process ordering: when `flags` is set, each block does a
// release/acquire flag barrier with the same-index block of every peer before
// reading (all gradients final, all peers done reading the previous weights)
// and after writing (all replicas final before anyone's next forward).  The
// grid is at most one resident wave, so every block of every peer is running.

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <utility>

#include "common.cuh"

namespace mgx {

constexpr int kKvThreads = 512;
constexpr int kKvMaxNW = 16;
constexpr int kKvMaxSegs = 256;
constexpr int kKvFlagBlocks = 1024;  // flag-array stride per phase

struct KvParams {
  float* grads[kKvMaxNW];
  float* weights[kKvMaxNW];
  uint32_t* flags[kKvMaxNW];
  float* velocity;
  float* agg_out;
  uint32_t* error_word;
  int32_t nseg;
  int32_t self_replica;
  int32_t updater;
  int32_t rank;
  uint32_t* epoch_ctr;  // device: [completed launches, blocks finished]
  float rescale, neg_eta, momentum, weight_decay;
  mgx_kv_seg segs[kKvMaxSegs];
  // push mode (nscatter > 0)
  int32_t nscatter;
  int64_t stage_slot;
  float* stage[kKvMaxNW];
  mgx_kv_seg scatter[kKvMaxSegs];
  int8_t scatter_owner[kKvMaxSegs];
};

// flat index -> segment: last s with pre[s] <= gi
__device__ __forceinline__ int seg_of(const int64_t* pre, int n, int64_t gi) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (pre[mid] <= gi) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// largest power of two strictly below n (n >= 2): kernels.py:39
__host__ __device__ constexpr int hpow2(int n) {
  int h = 1;
  while (h * 2 < n) h *= 2;
  return h;
}

template <int N>
__device__ __forceinline__ float tree(const float* v) {
  if constexpr (N == 1) {
    return v[0];
  } else {
    constexpr int H = hpow2(N);
    return fadd(tree<H>(v), tree<N - H>(v + H));
  }
}

// level-1 tree per machine over its W workers, then level-2 tree over machines
template <int M, int W>
__device__ __forceinline__ float two_level(const float* v) {
  if constexpr (M == 1) {
    return tree<W>(v);
  } else {
    float agg[M];
#pragma unroll
    for (int m = 0; m < M; ++m) agg[m] = tree<W>(v + m * W);
    return tree<M>(agg);
  }
}

__device__ __forceinline__ float4 ld_nc_v4(const float* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}

// coherent 128-bit load (L2, not the read-only path): for data other GPUs
// stored during this kernel (the push-mode staging buffer)
__device__ __forceinline__ float4 ld_cg_v4(const float* p) {
  float4 r;
  asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p)
               : "memory");
  return r;
}

__device__ __forceinline__ void st_v4(float* p, float4 v) {
  asm volatile("st.global.L1::no_allocate.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w)
               : "memory");
}

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Flag barrier with the same-index block of every peer.  Returns false (for
// the whole block) if a peer did not arrive within 30 s.
template <int NW>
__device__ bool block_barrier(const KvParams& p, int phase, uint32_t epoch) {
  __shared__ int ok;
  __syncthreads();
  if (threadIdx.x == 0) ok = 1;
  __syncthreads();
  if (threadIdx.x < NW) {
    const size_t base = (size_t(phase) * kKvFlagBlocks + blockIdx.x) * NW;
    __threadfence_system();
    st_release_sys(p.flags[threadIdx.x] + base + p.rank, epoch);
    const uint32_t* mine = p.flags[p.rank] + base + threadIdx.x;
    const uint64_t t0 = global_ns();
    while (static_cast<int32_t>(ld_acquire_sys(mine) - epoch) < 0) {
      if (global_ns() - t0 > 30ull * 1000 * 1000 * 1000) {
        atomicExch(p.error_word, 1u);
        ok = 0;
        break;
      }
    }
  }
  __syncthreads();
  return ok != 0;
}

template <int M, int W, int UNROLL, int THREADS>
__global__ void __launch_bounds__(THREADS) kv_round_kernel(const __grid_constant__ KvParams p) {
  constexpr int NW = M * W;
  const bool barrier = p.flags[0] != nullptr;
  // The barrier epoch lives on the device (launch count + 1), so a captured
  // launch replays correctly; the last block to finish advances it.
  __shared__ uint32_t s_epoch;
  if (barrier) {
    if (threadIdx.x == 0) s_epoch = *reinterpret_cast<volatile uint32_t*>(p.epoch_ctr) + 1;
    __syncthreads();
  }
  const bool push = p.nscatter > 0;
  const int64_t stride = int64_t(gridDim.x) * THREADS;
  bool live = true;
  if (push) {
    // phase 1: this rank's gradient values for every owner's shard, stored
    // into that owner's staging slot (remote writes; the previous round's
    // closing barrier guarantees every owner finished reading its stage).
    // The scatter list is owner-major and each owner's part lists its
    // segments exactly as that owner's own list does, and the loop below
    // has phase 2's thread -> element mapping: the element owner r reads in
    // block b after the same-index barrier was written by block b here.
    __shared__ int64_t spre[kKvMaxSegs];
    __shared__ int64_t gtot[kKvMaxNW];
    __shared__ int gq[kKvMaxNW + 1];
    if (threadIdx.x == 0) {
      int q = 0;
      for (int o = 0; o < NW; ++o) {
        gq[o] = q;
        int64_t acc = 0;
        while (q < p.nscatter && p.scatter_owner[q] == o) {
          spre[q] = acc;  // prefix within the owner's group
          acc += (p.scatter[q].len + 3) >> 2;
          ++q;
        }
        gtot[o] = acc;
      }
      gq[NW] = q;
    }
    __syncthreads();
    const float* gsrc = p.grads[p.rank];
    for (int o = 0; o < NW; ++o) {
      const int q0 = gq[o], q1 = gq[o + 1];
      if (q0 == q1) continue;
      const int64_t tot = gtot[o];
      float* const dst_base = p.stage[o];
      for (int64_t base = int64_t(blockIdx.x) * THREADS + threadIdx.x; base < tot;
           base += stride * UNROLL) {
        float4 v[UNROLL];
        float* dst[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
          const int64_t gi = base + u * stride;
          dst[u] = nullptr;
          if (gi < tot) {
            const int q = q0 + seg_of(spre + q0, q1 - q0, gi);
            const int64_t i = gi - spre[q];
            v[u] = ld_nc_v4(gsrc + p.scatter[q].off + 4 * i);
            dst[u] = dst_base + p.scatter[q].voff + 4 * i;
          }
        }
#pragma unroll
        for (int u = 0; u < UNROLL; ++u)
          if (dst[u]) st_v4(dst[u], v[u]);
      }
    }
  }
  if (barrier) live = block_barrier<NW>(p, 0, s_epoch);

  const float* wsrc = p.weights[p.self_replica];
  const float* my_stage = push ? p.stage[p.rank] : nullptr;
  // One flat index space over all segments (float4 units): every thread has
  // UNROLL independent vectors in flight regardless of how many small keys
  // the round holds (a per-segment loop serialised one latency per key).
  __shared__ int64_t pre[kKvMaxSegs + 1];
  if (threadIdx.x == 0) {
    int64_t acc = 0;
    for (int s = 0; s < p.nseg; ++s) {
      pre[s] = acc;
      acc += (p.segs[s].len + 3) >> 2;
    }
    pre[p.nseg] = acc;
  }
  __syncthreads();
  const int64_t total4 = pre[p.nseg];
  for (int64_t base = int64_t(blockIdx.x) * THREADS + threadIdx.x; live && base < total4;
       base += stride * UNROLL) {
    float4 g[UNROLL][NW];
    float4 w[UNROLL];
    float4 v[UNROLL];
    int64_t eoff[UNROLL], evoff[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const int64_t gi = base + u * stride;
      eoff[u] = -1;
      if (gi < total4) {
        // segment of gi: last s with pre[s] <= gi (binary search)
        int lo = 0, hi = p.nseg - 1;
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (pre[mid] <= gi) lo = mid;
          else hi = mid - 1;
        }
        const int64_t i = gi - pre[lo];
        eoff[u] = p.segs[lo].off + 4 * i;
        evoff[u] = p.segs[lo].voff + 4 * i;
        if (push) {
          // every worker's values for this shard are in the local stage
#pragma unroll
          for (int j = 0; j < NW; ++j) g[u][j] = ld_cg_v4(my_stage + j * p.stage_slot + evoff[u]);
        } else {
#pragma unroll
          for (int j = 0; j < NW; ++j) g[u][j] = ld_nc_v4(p.grads[j] + eoff[u]);
        }
        if (p.updater != MGX_KV_AGG) w[u] = ld_nc_v4(wsrc + eoff[u]);
        if (p.updater == MGX_KV_SGD) v[u] = *reinterpret_cast<const float4*>(p.velocity + evoff[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      if (eoff[u] < 0) continue;
      const int64_t off = eoff[u], voff = evoff[u];
      float tot[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        float vals[NW];
#pragma unroll
        for (int j = 0; j < NW; ++j) vals[j] = reinterpret_cast<const float*>(&g[u][j])[c];
        tot[c] = two_level<M, W>(vals);
      }
      if (p.updater == MGX_KV_AGG) {
        *reinterpret_cast<float4*>(p.agg_out + off) = make_float4(tot[0], tot[1], tot[2], tot[3]);
        continue;
      }
      float* wc = reinterpret_cast<float*>(&w[u]);
      if (p.updater == MGX_KV_SGD) {
        // make_sgd_updater (optim.py:72-76) -> sgd_arrays (optim.py:53-61):
        //   g = incoming * f32(1/scale); tmp = g + w*wd; v = v*mom;
        //   v = v + tmp*(-eta); w = w + v*1
        float* vc = reinterpret_cast<float*>(&v[u]);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const float gg = fmul(tot[c], p.rescale);
          const float tmp = fadd(gg, fmul(wc[c], p.weight_decay));
          vc[c] = fmul(vc[c], p.momentum);
          vc[c] = fadd(vc[c], fmul(tmp, p.neg_eta));
          wc[c] = fadd(wc[c], fmul(vc[c], 1.0f));
        }
        *reinterpret_cast<float4*>(p.velocity + voff) = v[u];
      } else {
        // add_updater (kvstore.py:47-49): stored += incoming
#pragma unroll
        for (int c = 0; c < 4; ++c) wc[c] = fadd(wc[c], tot[c]);
      }
#pragma unroll
      for (int j = 0; j < NW; ++j) st_v4(p.weights[j] + off, w[u]);
    }
  }
  if (barrier) {
    if (live) block_barrier<NW>(p, 1, s_epoch);
    if (threadIdx.x == 0) {
      __threadfence();
      const uint32_t prev = atomicAdd(p.epoch_ctr + 1, 1u);
      if (prev == gridDim.x - 1) {
        p.epoch_ctr[1] = 0;
        __threadfence();
        atomicAdd(p.epoch_ctr, 1u);
      }
    }
  }
}

using KvKernel = void (*)(const KvParams);

struct KvVariant {
  KvKernel k;
  int threads, unroll;
};

template <int M, int W, int U, int T>
constexpr KvVariant variant() {
  return KvVariant{kv_round_kernel<M, W, U, T>, T, U};
}

// Launch shape per topology.  For the one-machine topologies the shape can
// be overridden with MGX_KV_VARIANT="<unroll>,<threads>" (unroll 1|2|4,
// threads 256|512|1024) for tuning sweeps.
template <int M, int W>
KvVariant pick_variant() {
  if constexpr (M == 1 && (W == 2 || W == 4 || W == 8)) {
    static const char* env = getenv("MGX_KV_VARIANT");
    if (env) {
      int u = 0, t = 0;
      if (sscanf(env, "%d,%d", &u, &t) == 2) {
#define MGX_KV_V(uu, tt) \
  if (u == uu && t == tt) return variant<M, W, uu, tt>();
        MGX_KV_V(1, 256) MGX_KV_V(1, 512) MGX_KV_V(1, 1024)
        MGX_KV_V(2, 256) MGX_KV_V(2, 512) MGX_KV_V(2, 1024)
        MGX_KV_V(4, 256) MGX_KV_V(4, 512)
#undef MGX_KV_V
      }
    }
  }
  if constexpr (M * W <= 4) return variant<M, W, 2, kKvThreads>();
  else return variant<M, W, 1, kKvThreads>();
}

static KvVariant select_kernel(int M, int W) {
#define MGX_KV_CASE(m, w) \
  if (M == m && W == w) return pick_variant<m, w>();
  MGX_KV_CASE(1, 1) MGX_KV_CASE(1, 2) MGX_KV_CASE(1, 3) MGX_KV_CASE(1, 4)
  MGX_KV_CASE(1, 5) MGX_KV_CASE(1, 6) MGX_KV_CASE(1, 7) MGX_KV_CASE(1, 8)
  MGX_KV_CASE(1, 16)
  MGX_KV_CASE(2, 1) MGX_KV_CASE(2, 2) MGX_KV_CASE(2, 3) MGX_KV_CASE(2, 4) MGX_KV_CASE(2, 8)
  MGX_KV_CASE(3, 1) MGX_KV_CASE(3, 2)
  MGX_KV_CASE(4, 1) MGX_KV_CASE(4, 2) MGX_KV_CASE(4, 4)
  MGX_KV_CASE(8, 1) MGX_KV_CASE(8, 2)
#undef MGX_KV_CASE
  return KvVariant{nullptr, 0, 0};
}

static int kv_capacity(const KvVariant& v, int* out) {
  const KvKernel k = v.k;
  // cached per (kernel, device): no runtime API calls on the launch path,
  // which matters inside stream capture
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> cache;
  int dev0 = 0;
  MGX_CUDA(cudaGetDevice(&dev0));
  const auto key = std::make_pair(reinterpret_cast<const void*>(k), dev0);
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(key);
    if (it != cache.end()) {
      *out = it->second;
      return MGX_OK;
    }
  }
  int per_sm = 0;
  MGX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, v.threads, 0));
  int dev = 0, sms = kNumSMs;
  MGX_CUDA(cudaGetDevice(&dev));
  MGX_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  int cap = per_sm * sms;
  if (cap > kKvFlagBlocks) cap = kKvFlagBlocks;
  *out = cap < 1 ? 1 : cap;
  std::lock_guard<std::mutex> lock(mu);
  cache[key] = *out;
  return MGX_OK;
}

}  // namespace mgx

extern "C" int mgx_kv_max_grid(int32_t machines, int32_t workers, int32_t* out) {
  MGX_REQUIRE(out, "mgx_kv_max_grid: null out");
  mgx::KvVariant v = mgx::select_kernel(machines, workers);
  MGX_REQUIRE(v.k, "mgx_kv_max_grid: unsupported topology %d x %d", machines, workers);
  int cap = 0;
  MGX_TRY(mgx::kv_capacity(v, &cap));
  *out = cap;
  return MGX_OK;
}

extern "C" int mgx_kv_config(int32_t machines, int32_t workers, int32_t* max_grid,
                             int32_t* threads, int32_t* unroll) {
  MGX_REQUIRE(max_grid && threads && unroll, "mgx_kv_config: null out");
  mgx::KvVariant v = mgx::select_kernel(machines, workers);
  MGX_REQUIRE(v.k, "mgx_kv_config: unsupported topology %d x %d", machines, workers);
  int cap = 0;
  MGX_TRY(mgx::kv_capacity(v, &cap));
  *max_grid = cap;
  *threads = v.threads;
  *unroll = v.unroll;
  return MGX_OK;
}

extern "C" int mgx_kv_round(const mgx_kv_round_args* a, uintptr_t stream) {
  MGX_REQUIRE(a && a->segs && a->grads, "mgx_kv_round: null arguments");
  const int M = a->machines, W = a->workers, NW = M * W;
  MGX_REQUIRE(M >= 1 && W >= 1 && NW <= mgx::kKvMaxNW, "mgx_kv_round: bad topology %d x %d", M, W);
  MGX_REQUIRE(a->nseg >= 0 && a->nseg <= mgx::kKvMaxSegs, "mgx_kv_round: nseg %d outside [0, %d]",
              a->nseg, mgx::kKvMaxSegs);
  MGX_REQUIRE(a->updater >= 0 && a->updater <= 2, "mgx_kv_round: unknown updater %d", a->updater);
  MGX_REQUIRE(a->updater == MGX_KV_AGG || a->weights, "mgx_kv_round: weights required");
  MGX_REQUIRE(a->updater != MGX_KV_SGD || a->velocity, "mgx_kv_round: SGD needs velocity");
  MGX_REQUIRE(a->updater != MGX_KV_AGG || a->agg_out, "mgx_kv_round: AGG needs agg_out");
  MGX_REQUIRE(a->self_replica >= 0 && a->self_replica < NW, "mgx_kv_round: bad self_replica");
  mgx::KvVariant var = mgx::select_kernel(M, W);
  MGX_REQUIRE(var.k, "mgx_kv_round: unsupported topology %d x %d", M, W);

  mgx::KvParams p;
  std::memset(&p, 0, sizeof(p));
  int64_t total4 = 0;
  for (int s = 0; s < a->nseg; ++s) {
    const mgx_kv_seg& sg = a->segs[s];
    MGX_REQUIRE(sg.off % 4 == 0 && sg.len >= 0 && sg.voff % 4 == 0,
                "mgx_kv_round: segment %d not 16-byte aligned", s);
    p.segs[s] = sg;
    total4 += (sg.len + 3) / 4;
  }
  for (int j = 0; j < NW; ++j) {
    p.grads[j] = a->grads[j];
    p.weights[j] = a->weights ? a->weights[j] : nullptr;
    p.flags[j] = a->flags ? a->flags[j] : nullptr;
    MGX_REQUIRE(p.grads[j], "mgx_kv_round: null gradient pointer %d", j);
  }
  p.velocity = a->velocity;
  p.agg_out = a->agg_out;
  p.error_word = a->error_word;
  p.nseg = a->nseg;
  p.self_replica = a->self_replica;
  p.updater = a->updater;
  p.rank = a->rank;
  p.epoch_ctr = a->epoch_ctr;
  p.rescale = a->rescale;
  p.neg_eta = a->neg_eta;
  p.momentum = a->momentum;
  p.weight_decay = a->weight_decay;
  p.nscatter = a->nscatter;
  if (a->nscatter > 0) {
    MGX_REQUIRE(a->flags && a->scatter && a->scatter_owner && a->stage && a->stage_slot > 0 &&
                    a->updater != MGX_KV_AGG && a->nscatter <= mgx::kKvMaxSegs,
                "mgx_kv_round: bad push-mode arguments");
    p.stage_slot = a->stage_slot;
    for (int j = 0; j < NW; ++j) {
      p.stage[j] = a->stage[j];
      MGX_REQUIRE(p.stage[j], "mgx_kv_round: null staging pointer %d", j);
    }
    for (int q = 0; q < a->nscatter; ++q) {
      const mgx_kv_seg& sg = a->scatter[q];
      MGX_REQUIRE(sg.off % 4 == 0 && sg.voff % 4 == 0 && sg.len >= 0 && a->scatter_owner[q] >= 0 &&
                      a->scatter_owner[q] < NW,
                  "mgx_kv_round: bad scatter segment %d", q);
      p.scatter[q] = sg;
      p.scatter_owner[q] = static_cast<int8_t>(a->scatter_owner[q]);
    }
    MGX_REQUIRE(a->stage_slot % 4 == 0, "mgx_kv_round: stage slot not 16-byte aligned");
  }

  int cap = 0;
  MGX_TRY(mgx::kv_capacity(var, &cap));
  int grid = a->grid;
  const bool barrier = a->flags != nullptr;
  if (barrier) {
    MGX_REQUIRE(a->error_word && a->epoch_ctr, "mgx_kv_round: barrier needs error_word and epoch_ctr");
    MGX_REQUIRE(a->rank >= 0 && a->rank < NW, "mgx_kv_round: bad rank");
    MGX_REQUIRE(grid >= 1 && grid <= cap,
                "mgx_kv_round: barrier mode needs an explicit grid in [1, %d], got %d", cap, grid);
  } else {
    if (total4 == 0) return MGX_OK;
    if (grid <= 0) {
      int64_t want = mgx::ceil_div(total4, int64_t(var.threads) * var.unroll);
      grid = static_cast<int>(want < cap ? want : cap);
      if (grid < 1) grid = 1;
    }
  }
  var.k<<<grid, var.threads, 0, mgx::as_stream(stream)>>>(p);
  MGX_LAUNCHED();
  return MGX_OK;
}
