/*
 * mgx.h — C-ABI of the B200-native data-parallel training step.
 *
 * This is the drop-in boundary for the reference's hot path (minigraph, the
 * Python restatement of arXiv 1512.01274 under /root/reference/pkg/src).  The
 * reference exposes its flat foreign-call surface in capi.py; every function
 * here follows the same conventions (capi.py:26-29, 102-116):
 *   - return an int status: 0 OK, 1 BAD_HANDLE, 2 BAD_ARGUMENT, 3 INTERNAL;
 *   - results go through out-parameters;
 *   - a thread-local last-error string explains any non-zero status.
 * Pointers are CUDA device pointers (plain addresses, no torch types); streams
 * are cudaStream_t values passed as uintptr_t (0 = legacy default stream).
 *
 * Each entry point cites the reference interface it replaces (file:line,
 * paths relative to /root/reference/pkg/src/minigraph/).
 */
#ifndef MGX_H_
#define MGX_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------ status codes
 * capi.py:26-29 */
#define MGX_OK 0
#define MGX_BAD_HANDLE 1
#define MGX_BAD_ARGUMENT 2
#define MGX_INTERNAL 3

/* Thread-local message for the last failing call (capi.py:95-97). */
const char* mgx_last_error_message(void);
/* ABI version (bumped on any signature change). */
int mgx_abi_version(int* out);

/* ------------------------------------------------------- device & memory
 * Replaces tensor.py Buffer (tensor.py:42-52) and the engine's tags
 * (engine.py:89-92): storage is device memory, ordering is a CUDA stream. */
int mgx_device_count(int* out);
int mgx_set_device(int device);
int mgx_malloc(size_t nbytes, void** out);          /* cudaMalloc: IPC-exportable */
int mgx_free(void* ptr);
int mgx_host_alloc(size_t nbytes, void** out);      /* pinned host memory */
int mgx_host_free(void* ptr);
int mgx_stream_create(uintptr_t* out);
int mgx_stream_destroy(uintptr_t stream);
int mgx_stream_sync(uintptr_t stream);              /* to_host / wait_for sync point (tensor.py:132-137, engine.py:200-209) */
int mgx_memcpy_async(void* dst, const void* src, size_t nbytes, uintptr_t stream); /* load_host / to_host copies (tensor.py:140-147) */
int mgx_memset_async(void* dst, int value, size_t nbytes, uintptr_t stream);
int mgx_event_create(uintptr_t* out);               /* timing-enabled event */
int mgx_event_destroy(uintptr_t ev);
int mgx_event_record(uintptr_t ev, uintptr_t stream);
int mgx_event_elapsed_ms(uintptr_t start, uintptr_t end, float* out);
int mgx_stream_wait_event(uintptr_t stream, uintptr_t ev);

/* CUDA IPC for the multi-process KVStore: peer replicas and barrier flags are
 * mapped into every rank (replaces the L1/L2 queues, kvstore.py:52-82). */
#define MGX_IPC_HANDLE_BYTES 64
int mgx_ipc_get_handle(void* dev_ptr, void* handle_out /* 64 bytes */);
int mgx_ipc_open_handle(const void* handle /* 64 bytes */, void** out);
int mgx_ipc_close_handle(void* dev_ptr);

/* ------------------------------------------------------ tensor primitives
 * tensor.py:103-231 and kernels.py:50-53.  n = element count, fp32. */
int mgx_fill(float* y, int64_t n, float value, uintptr_t stream);             /* zeros/ones, ZerosLike (ops.py:362-373) */
int mgx_copy(const float* x, float* y, int64_t n, uintptr_t stream);          /* copy_to (tensor.py:223-231), Flatten (ops.py:335-357) */
int mgx_axpy(float alpha, const float* x, float* y, int64_t n, uintptr_t stream); /* y = y + x*alpha (kernels.py:50-53) */
/* op: 0 add, 1 sub, 2 mul, 3 div (tensor.py:169-190, ops.py:222-250) */
int mgx_elementwise(int op, const float* a, const float* b, float* out, int64_t n, uintptr_t stream);
/* op: 0 add, 1 mul (tensor.py:193-203, ops.py:281-318) */
int mgx_scalar_op(int op, const float* a, float c, float* out, int64_t n, uintptr_t stream);

/* ------------------------------------------------------- dense operators
 * Exact-order fp32 kernels: they reproduce the reference's numpy reduction
 * orders with separately rounded mul/add. */

/* act: 0 none, 1 relu, 2 sigmoid, 3 tanh (ops.py:138-171). */
#define MGX_ACT_NONE 0
#define MGX_ACT_RELU 1
#define MGX_ACT_SIGMOID 2
#define MGX_ACT_TANH 3

/* C[m,n] = pairwise_k(A[m,k]*B[n,k]) (+ bias[n]) then act.  numpy pairwise
 * summation over k (kernels.py:20-29 via ops.py:102-106: FC forward).
 * lda/ldb/ldc are row strides in elements; bias may be NULL. */
int mgx_gemm_pairwise(const float* A, int64_t lda, const float* B, int64_t ldb,
                      const float* bias, float* C, int64_t ldc,
                      int64_t M, int64_t N, int64_t K, int act, uintptr_t stream);

/* C[m,n] = sequential_k(A[m,k]*B[k,n]); then, if act != NONE, the activation
 * backward against Y (the activation's forward output) is fused:
 * C = C * act'(Y).  (ops.py:111-112 FC dX; ops.py:302-303 MatMul forward;
 * ops.py:164-166 activation backward).  Strides: A[m*sam + k*sak],
 * B[k*sbk + n*sbn], C/Y row stride ldc. */
int mgx_gemm_sequential(const float* A, int64_t sam, int64_t sak,
                        const float* B, int64_t sbk, int64_t sbn,
                        float* C, int64_t ldc, const float* Y, int act,
                        int64_t M, int64_t N, int64_t K, uintptr_t stream);

/* dW[h,f] = tree_b(og[b,h]*x[b,f]); db[h] = tree_b(og[b,h]).  Balanced
 * power-of-two tree over the batch (kernels.py:32-47, ops.py:113-116).
 * dw or db may be NULL. */
int mgx_fc_dw_db(const float* og, const float* x, float* dw, float* db,
                 int64_t B, int64_t H, int64_t F, uintptr_t stream);

/* out[c] = tree_r(a[r, c]) (kernels.py:32-42) over `rows` rows of `cols`. */
int mgx_tree_sum_rows(const float* a, float* out, int64_t rows, int64_t cols, uintptr_t stream);

int mgx_act_forward(int act, const float* x, float* y, int64_t n, uintptr_t stream);          /* ops.py:154-156 */
int mgx_act_backward(int act, const float* y, const float* og, float* g, int64_t n, uintptr_t stream); /* ops.py:159-161 */

/* SoftmaxOutput (ops.py:176-207, kernels.py:68-83).  label holds class ids
 * as fp32 (truncated to int64 like one_hot).  grad = (p - onehot) / f32(B). */
int mgx_softmax_forward(const float* x, float* p, int64_t B, int64_t C, uintptr_t stream);
int mgx_softmax_backward(const float* p, const float* label, float* g, int64_t B, int64_t C, uintptr_t stream);

/* Tensor-core dense path (tolerance, not exact order): C[M,N] fp32 =
 * A[M,K] . B[N,K]^T (+bias) then act, A/B bf16 K-major ("TN"), fp32
 * accumulation in TMEM via tcgen05.mma, operands by TMA.  Replaces the
 * reference's FC forward contraction (ops.py:102-106) for the large FC
 * layers of configs 3-5.  lda, ldb multiples of 8; 16-byte aligned. */
int mgx_gemm_bf16_tc(const void* A, int64_t lda, const void* B, int64_t ldb,
                     const float* bias, float* C, int64_t ldc,
                     int64_t M, int64_t N, int64_t K, int act, uintptr_t stream);
/* y(bf16) = round-to-nearest-even(x(fp32)) */
int mgx_cast_f32_bf16(const float* x, void* y, int64_t n, uintptr_t stream);
/* y (bf16, rows x ldo) = x (fp32, R x C, row stride ldi), transposed if
 * transpose != 0 (y then holds x^T), zero-filled beyond the source extent
 * (the K padding of a tensor-core operand). */
int mgx_cast_bf16_2d(const float* x, int64_t R, int64_t C, int64_t ldi, void* y,
                     int64_t rows, int64_t ldo, int transpose, uintptr_t stream);

/* General tensor-core GEMM: C[M,N] = sum_k A(m,k) B(n,k) (+bias[n]) then
 * act.  a_mn == 0: A[m*lda + k] (K-major), else A[k*lda + m] (MN-major);
 * same for B.  splits: K split count (0 = auto when a workspace is given,
 * 1 = none); partial tiles go to workspace (splits*M*N floats) and are
 * summed in ascending split order (deterministic).  lda/ldb multiples of 8. */
int mgx_gemm_bf16_tc_ex(const void* A, int64_t lda, int a_mn, const void* B, int64_t ldb,
                        int b_mn, const float* bias, float* C, int64_t ldc, int64_t M,
                        int64_t N, int64_t K, int act, int splits, float* workspace,
                        float* colstats, uintptr_t stream);
/* Implicit-GEMM convolution contractions: one operand is gathered on the
 * fly from a compact bf16 NHWC tensor `src` (C % 8 == 0) inside the tcgen05
 * GEMM, never materialised -- by one TMA im2col load per k-block when
 * C % 64 == 0 (mode 1), else by cp.async producer warps:
 *   gather(src)[m, k] = src[b, oh*sh-ph+i, ow*sw-pw+j, c],
 *   m = (b, oh, ow) output pixel, k = (i*kw + j)*C + c  (geom as below).
 * mode 1: C[M=pixels, N] = gather . op[N, K]^T      (op K-major, row stride
 *         ldop: convolution forward / stride-1 data gradient)
 * mode 2: C[M, N=kh*kw*C] = op[K=pixels, M]^T . gather  (op MN-major: the
 *         output gradient; weight gradient)
 * mode 3: data gradient of a stride-2 convolution whose FORWARD geometry is
 *         geom: src = dY [B, Ho, Wo, F] read dilated by 2 with pad k-1-p,
 *         op = the flipped weights [C, kh*kw*F], C[M=B*H*W, N=C].
 * Split-K as mgx_gemm_bf16_tc_ex. */
int mgx_gemm_bf16_conv(int mode, const void* src, const int64_t* geom, const void* op,
                       int64_t ldop, const float* bias, float* C, int64_t ldc, int64_t M,
                       int64_t N, int64_t K, int act, int splits, float* workspace,
                       float* colstats, uintptr_t stream);
/* colstats (optional, both GEMM entry points, one split, C pitch % 4 == 0):
 * the epilogue also writes, for every 32-row block b and column n of C, the
 * pair (mean, M2) of the block's valid rows as float2 colstats[b*N + n] --
 * the BatchNorm statistics of a convolution output without re-reading it.
 * mgx_bn_stats_from_tiles merges them (shifted fp64 sums, fixed order)
 * into stats = [mean | rstd] and updates the moving averages like
 * mgx_bn_stats. */
int mgx_bn_stats_from_tiles(const void* part, int64_t M, int64_t C, float* stats,
                            float* moving_mean, float* moving_var, float eps, float momentum,
                            uintptr_t stream);
/* Workspace (floats) the auto split-K choice needs for an M x N x K GEMM. */
int mgx_gemm_splitk_workspace(int64_t M, int64_t N, int64_t K, int64_t* out_floats);
/* The split-K plan for about `target` CTAs (0: the default): split count
 * (1 = none; at most 128 k-blocks per split) and its workspace floats. */
int mgx_gemm_split_plan(int64_t M, int64_t N, int64_t K, int32_t target, int32_t* splits,
                        int64_t* out_floats);

/* ------------------------------------------------ convolution-net kernels
 * geom = int64[7] {B, H, W, C, kh<<16|kw, sh<<16|sw, ph<<16|pw}. */
/* col[m, k] (bf16, row stride ldk % 8 == 0) = x(NHWC) at tap k = (i, j, c) of
 * output pixel m; zero in the padding and for k >= kh*kw*C. */
int mgx_im2col_bf16(const float* x, void* col, const int64_t* geom, int64_t ldk, uintptr_t stream);
/* wf[c, (i*kw+j)*F + f] (bf16, row stride ld) = w[f, kh-1-i, kw-1-j, c]:
 * the transposed-convolution weight of a stride-1 data gradient
 * dX = im2col(dY, pad kh-1-ph) . wf^T. */
int mgx_weight_flip_bf16(const float* w, int64_t F, int64_t kh, int64_t kw, int64_t C, void* wf,
                         int64_t ld, uintptr_t stream);
/* dx(NHWC) = adjoint of im2col applied to dcol (fp32, row stride ldk). */
int mgx_col2im(const float* dcol, int64_t ldk, float* dx, const int64_t* geom, uintptr_t stream);
/* fp64 workspace bytes for the per-channel reductions of an M x C matrix. */
int mgx_reduce_workspace_bytes(int64_t M, int64_t C, int64_t* out);
/* BatchNorm (MXNet semantics, axis = channels): stats = [mean C | rstd C]
 * from the batch (biased variance) with moving-average update, or from the
 * moving averages when use_global. */
int mgx_bn_stats(const float* x, int64_t M, int64_t C, void* ws, float* stats, float* moving_mean,
                 float* moving_var, float eps, float momentum, int use_global, uintptr_t stream);
/* y = act((x - mean) * rstd * gamma + beta); gamma NULL = fix_gamma (1).
 * y16 (C % 4 == 0): also a bf16 copy; y may then be NULL (copy only). */
/* As mgx_bn_apply / mgx_bn_fwd_fused with an output row stride `ldo`
 * (elements, 0 = C): y / y16 may be channel slices of a wider tensor (a
 * Concat output written in place by its producers). */
int mgx_bn_apply_ld(const float* x, const float* stats, const float* gamma, const float* beta,
                    float* y, int64_t M, int64_t C, int act, void* y16, int64_t ldo,
                    uintptr_t stream);
int mgx_bn_fwd_fused_ld(const float* x, int64_t M, int64_t C, float* stats, float* moving_mean,
                        float* moving_var, float eps, float momentum, const float* gamma,
                        const float* beta, float* y, void* y16, int act, int64_t ldo,
                        uintptr_t stream);
int mgx_bn_apply(const float* x, const float* stats, const float* gamma, const float* beta,
                 float* y, int64_t M, int64_t C, int act, void* y16, uintptr_t stream);
/* sums = [sum dy | sum dy*xhat] per channel; also written to dbeta and
 * dgamma when non-NULL (dgamma zero-filled when dgamma_zero: fix_gamma).
 * relu_beta (optional): a ReLU follows the BatchNorm; dy is then masked by
 * ((x - mean) * rstd * relu_gamma + relu_beta > 0) -- the forward's ReLU
 * decision recomputed from x (relu_gamma NULL = 1) -- so the ReLU backward
 * is fused in and its output never stored. */
int mgx_bn_bwd_reduce(const float* dy, const float* x, const float* stats, int64_t M, int64_t C,
                      void* ws, float* sums, float* dbeta, float* dgamma, int dgamma_zero,
                      const float* relu_gamma, const float* relu_beta, uintptr_t stream);
/* dx = gamma * rstd * (dy - (sum dy + xhat * sum dy*xhat) / M), with the
 * same optional ReLU mask; dy may alias dx.  dx may be NULL when dx16 is
 * given (every consumer reads the bf16 copy).  ws: mgx_reduce_workspace_bytes
 * (needed when C % 4 == 0).  dsum (optional): the per-channel sum of dx
 * over the rows, reduced in the same pass (the bias gradient of the
 * convolution feeding the BatchNorm). */
int mgx_bn_bwd_dx(const float* dy, const float* x, const float* stats, const float* sums,
                  const float* gamma, float* dx, int64_t M, int64_t C, const float* relu_gamma,
                  const float* relu_beta, float* dsum, void* ws, void* dx16, uintptr_t stream);
/* Cluster-fused BatchNorm (training) for layers of up to 65536 rows
 * (bn_fused.cu): a thread-block cluster owns a channel slice and all rows,
 * stages them in shared memory once (or, from 32768 rows, streams them
 * twice through L2), reduces over DSMEM in a fixed order.
 * mgx_bn_fused_ok: *ok = 1 (staged) or 2 (streamed) when (M, C) has such a
 * launch shape (C % 8 == 0), else 0; the fused entry points reject other
 * shapes.
 * fwd: stats [mean | rstd] + moving averages + y = act(bn(x)) -> y (fp32,
 * optional) / y16 (bf16, optional) in one kernel.
 * bwd: dy' = dy masked by the fused ReLU (relu_beta non-NULL: mask
 * (x - mean) rstd relu_gamma + relu_beta > 0); dbeta = sum dy', dgamma =
 * sum dy' xhat (0 when dgamma_zero), sums = [dbeta | dgamma] (optional),
 * dx = gamma rstd (dy' - (dbeta + xhat dgamma) / M) -> dx / dx16 (each
 * optional, one required), dsum = sum dx (optional) in one kernel.  ldd: row
 * stride of dy in floats (C; larger when dy is a channel slice of a wider
 * gradient, e.g. the gradient of a Concat read in place). */
int mgx_bn_fused_ok(int64_t M, int64_t C, int backward, int* ok);
int mgx_bn_fwd_fused(const float* x, int64_t M, int64_t C, float* stats, float* moving_mean,
                     float* moving_var, float eps, float momentum, const float* gamma,
                     const float* beta, float* y, void* y16, int act, uintptr_t stream);
int mgx_bn_bwd_fused(const float* dy, int64_t ldd, const float* x, const float* stats,
                     const float* gamma,
                     int64_t M, int64_t C, const float* relu_gamma, const float* relu_beta,
                     float* dbeta, float* dgamma, int dgamma_zero, float* sums, float* dx,
                     void* dx16, float* dsum, uintptr_t stream);
/* Stem fusion, BatchNorm (+act) feeding a max pooling (argmax recorded):
 * forward: y = maxpool(act(bn(x))) with the argmax, the normalised tensor
 * never written; backward: the BatchNorm gradient passes with their output
 * gradient gathered through the pooling (dy_pool + argmax, the sum
 * mgx_pool_backward computes) instead of read from a materialised tensor.
 * geom/full describe the pooling (its input is the BatchNorm's [M, C]). */
int mgx_bn_act_pool_fwd(const float* x, const float* stats, const float* gamma, const float* beta,
                        int act, const int64_t* geom, int full, float* y, void* y16, void* argmax,
                        uintptr_t stream);
int mgx_bn_bwd_reduce_pooled(const float* dy_pool, const void* argmax, const int64_t* geom,
                             int full, const float* x, const float* stats, int64_t M, int64_t C,
                             void* ws, float* sums, float* dbeta, float* dgamma, int dgamma_zero,
                             const float* relu_gamma, const float* relu_beta, uintptr_t stream);
int mgx_bn_bwd_dx_pooled(const float* dy_pool, const void* argmax, const int64_t* geom, int full,
                         const float* x, const float* stats, const float* sums,
                         const float* gamma, int64_t M, int64_t C, const float* relu_beta,
                         float* dsum, void* ws, float* dx, void* dx16, uintptr_t stream);
/* One launch for all per-step weight preparations of a program: jobs is a
 * DEVICE array of njobs (<= 1024) descriptors (kind 0: bf16 row cast, a..e =
 * R, C, ldi, rows, ldo -- as mgx_cast_bf16_2d; kind 1: flipped bf16 weight,
 * a..e = F, kh, kw, C, ld -- as mgx_weight_flip_bf16).  Each job's output
 * (rows * ldo or C * ld bf16, a multiple of 8, 16-byte aligned) is a run of
 * 8-element units starting at unit `start`; units = the total. */
typedef struct mgx_prep_job {
  const float* src;
  void* dst;
  int64_t a, b, c, d, e;
  int64_t kind;
  int64_t start;
} mgx_prep_job;
int mgx_prep_batch(const void* jobs, int64_t njobs, int64_t units, uintptr_t stream);
/* out[c] = sum over rows of x[r, c] (conv bias gradient). */
int mgx_colsum(const float* x, int64_t M, int64_t C, void* ws, float* out, uintptr_t stream);
/* Pooling, NHWC.  type 0 max (padding ignored), 1 avg (count_include_pad);
 * full != 0: 'full' convention (output size rounded up).  argmax (optional,
 * max only, uint8 per output element, needs C % 4 == 0 and kh*kw <= 255):
 * the window-local index of the first maximum, written by the forward and
 * read by the backward instead of rescanning x.  y16 (C % 4 == 0): a bf16
 * copy of y; y may then be NULL (copy only). */
int mgx_pool_forward(const float* x, float* y, const int64_t* geom, int full, int type,
                     void* argmax, void* y16, uintptr_t stream);
int mgx_pool_backward(const float* x, const float* y, const float* dy, float* dx,
                      const int64_t* geom, int full, int type, const void* argmax,
                      uintptr_t stream);
/* out = ((srcs[0] + srcs[1]) + srcs[2]) + ... (count <= 6, n % 4 == 0): a
 * chain of ElementwiseAdds (ops.py:222-250) in one pass, same order. */
int mgx_sum_n(const float* const* srcs, int32_t count, float* out, int64_t n, uintptr_t stream);
/* Concat along channels in one pass (count <= 4 inputs of rows x channels[k],
 * channels % 4 == 0), with an optional bf16 copy of the output. */
int mgx_concat(const float* const* srcs, const int64_t* channels, int32_t count, float* out,
               void* out16, int64_t rows, uintptr_t stream);
/* dst[r, doff + c] = src[r, soff + c] for r < rows, c < cols (Concat). */
int mgx_chan_copy(const float* src, int64_t lds, int64_t soff, float* dst, int64_t ldd,
                  int64_t doff, int64_t rows, int64_t cols, void* dst16, uintptr_t stream);

/* Momentum SGD, tensor path (optim.py:39-50): 5 separately rounded steps. */
int mgx_sgd_step(float* w, const float* g, float* v, int64_t n,
                 float eta, float momentum, float weight_decay, uintptr_t stream);

/* ---------------------------------------------------------- memory planner
 * plan_memory/_plan_view/_longest_path_order (planner.py:205-348) over a flat
 * index view of the graph (planner.py:164-200).  Node arrays are in topo
 * order.  strategy: 0 none, 1 inplace, 2 coshare, 3 both.
 *   in_ptr/in_idx      CSR of each node's input node indices (with repeats)
 *   ip_ptr/ip_pos      CSR of each node's in-place input positions
 * Outputs: slot_of[n]; slot_bytes/slot_dedicated[*n_slots] (capacity n);
 * edges[2*k] pairs sorted ascending (capacity edge_cap pairs). */
int mgx_plan_memory(int32_t n, const uint8_t* is_var, const int64_t* nbytes,
                    const uint8_t* dedicated, const int32_t* in_ptr,
                    const int32_t* in_idx, const int32_t* ip_ptr,
                    const int32_t* ip_pos, const int32_t* phase, int32_t strategy,
                    int32_t* slot_of, int64_t* slot_bytes, uint8_t* slot_dedicated,
                    int32_t* n_slots, int32_t* edges, int32_t edge_cap,
                    int32_t* n_edges, int64_t* total_internal_bytes,
                    int64_t* visits);
/* Iteration order of CPython's set() over a list of small non-negative ints
 * (the order planner.py:298 frees inputs in); exposed for testing. */
int mgx_py_set_order(const int64_t* keys, int32_t n, int64_t* out, int32_t* n_out);

/* ------------------------------------------------------------ graph builder
 * Reverse-mode gradient structure (replaces symbol.build_gradient,
 * symbol.py:227-298) over the flat form of a forward graph in topo order.
 *   in_ptr/in_idx   CSR of each node's input source indices; the (node, slot)
 *                   pair p = in_ptr[i] + k also indexes role_ptr
 *   role_ptr/role_code  per (node, slot): the values the slot's Backward
 *                   reads: MGX_ROLE_OG, MGX_ROLE_OUT or an input position j
 *   seed_node       nodes seeded by a head-gradient variable (endpoint n + s)
 *   wrt_node        the requested argument nodes
 * Records are emitted in node-creation order (the host names them from its
 * counters): kind MGX_GREC_ADD (a, b = endpoints), MGX_GREC_BACKWARD (a =
 * node, b = slot, inputs in rec_in_ptr/rec_in_idx), MGX_GREC_ZEROS (a = var).
 * Endpoint codes: < n original node, < n + nseed head variable, else record
 * (code - n - nseed); -1 = none (a loss head's output gradient).  wrt_out[j]
 * is the endpoint of argument j's gradient.  A node that needs a gradient but
 * has none sets *bad_node and returns MGX_BAD_ARGUMENT. */
#define MGX_ROLE_OG (-1)
#define MGX_ROLE_OUT (-2)
#define MGX_GREC_ADD 0
#define MGX_GREC_BACKWARD 1
#define MGX_GREC_ZEROS 2
int mgx_grad_build(int32_t n, const uint8_t* is_var, const uint8_t* is_loss,
                   const uint8_t* differentiable, const int32_t* in_ptr, const int32_t* in_idx,
                   int32_t nseed, const int32_t* seed_node, const int32_t* role_ptr,
                   const int32_t* role_code, int32_t nwrt, const int32_t* wrt_node, int32_t cap,
                   int32_t in_cap, int32_t* rec_kind, int64_t* rec_a, int64_t* rec_b,
                   int32_t* rec_in_ptr, int64_t* rec_in_idx, int64_t* wrt_out, int32_t* n_rec,
                   int32_t* bad_node);
/* Launch order of a bound graph (executor.py:143-185): min-heap over
 * (phase, topo index) on the graph's operator edges plus the planner's extra
 * edges (pairs).  Writes every operator node once; non-acyclic input
 * returns MGX_BAD_ARGUMENT. */
int mgx_push_order(int32_t n, const uint8_t* is_var, const int32_t* phase, const int32_t* in_ptr,
                   const int32_t* in_idx, int32_t nextra, const int32_t* extra, int32_t* order,
                   int32_t* n_order);

/* ------------------------------------------------------ executor program
 * The bound graph's push lists (executor.py:143-185) compiled into a native
 * instruction list; forward()/backward() (executor.py:198-215) replay a
 * range of it on a stream, optionally as one captured CUDA graph. */
typedef struct mgx_instr {
  int32_t op;          /* MGX_OP_* */
  int32_t act;         /* activation code for fused epilogues */
  int64_t dims[8];
  float fattr[4];
  void* ptr[6];
} mgx_instr;

#define MGX_OP_FILL 1         /* ptr0=y dims0=n fattr0=value                      */
#define MGX_OP_COPY 2         /* ptr0=x ptr1=y dims0=n                            */
#define MGX_OP_EW 3           /* ptr0=a ptr1=b ptr2=out dims0=n dims1=op          */
#define MGX_OP_SCALAR 4       /* ptr0=a ptr1=out dims0=n dims1=op fattr0=c        */
#define MGX_OP_GEMM_PW 5      /* ptr0=A ptr1=B ptr2=bias ptr3=C act               */
                              /* dims=M,N,K,lda,ldb,ldc                           */
#define MGX_OP_GEMM_SEQ 6     /* ptr0=A ptr1=B ptr2=C ptr3=Y act                  */
                              /* dims=M,N,K,sam,sak,sbk,sbn,ldc                   */
#define MGX_OP_DW_DB 7        /* ptr0=og ptr1=x ptr2=dw ptr3=db dims=B,H,F        */
#define MGX_OP_ACT_FWD 8      /* ptr0=x ptr1=y dims0=n act                        */
#define MGX_OP_ACT_BWD 9      /* ptr0=y ptr1=og ptr2=g dims0=n act                */
#define MGX_OP_SOFTMAX_FWD 10 /* ptr0=x ptr1=p dims=B,C                           */
#define MGX_OP_SOFTMAX_BWD 11 /* ptr0=p ptr1=label ptr2=g dims=B,C                */
#define MGX_OP_AXPY 12        /* ptr0=x ptr1=y dims0=n fattr0=alpha               */
#define MGX_OP_CAST_BF16 13   /* ptr0=x(f32) ptr1=y(bf16) dims=R,C,ldi,rows,ldo,T */
#define MGX_OP_GEMM_TC 14     /* ptr0=A ptr1=B ptr2=bias ptr3=C act (bf16 TN)     */
                              /* dims=M,N,K,lda,ldb,ldc                           */

/* Convolution-net instructions (configs 3-5; no reference oracle: MXNet
 * semantics, NHWC).  "geom" = dims[0..6] = B, H, W, C, kh<<16|kw, sh<<16|sw,
 * ph<<16|pw (input extent and window). */
#define MGX_OP_IM2COL 15      /* ptr0=x ptr1=col(bf16) dims=geom,ldk               */
#define MGX_OP_COL2IM 16      /* ptr0=dcol ptr1=dx dims=geom,ldk                   */
#define MGX_OP_BN_STATS 17    /* ptr0=x ptr1=ws ptr2=stats ptr3=mmean ptr4=mvar    */
                              /* dims=M,C,use_global,from_tiles fattr=eps,momentum */
#define MGX_OP_BN_APPLY 18    /* ptr0=x ptr1=stats ptr2=gamma ptr3=beta ptr4=y     */
                              /* ptr5=y16 (optional bf16 copy) dims=M,C act        */
#define MGX_OP_BN_BWD_REDUCE 19 /* ptr0=dy ptr1=x ptr2=stats ptr3=ws ptr4=sums     */
                              /* ptr5=relu_beta                                    */
                              /* dims=M,C,dbeta*,dgamma*,dgamma_zero,relu_gamma*   */
#define MGX_OP_BN_BWD_DX 20   /* ptr0=dy ptr1=x ptr2=stats ptr3=sums ptr4=gamma    */
                              /* ptr5=dx dims=M,C,relu_beta*,dsum*,ws*,relu_gamma*, */
                              /* dx16* (optional bf16 copy)                        */
                              /* (* = a device address carried in a dim)           */
#define MGX_OP_POOL_FWD 21    /* ptr0=x ptr1=y ptr2=argmax ptr3=y16 dims=geom,full */
#define MGX_OP_POOL_BWD 22    /* ptr0=x ptr1=y ptr2=dy ptr3=dx ptr4=argmax dims=geom,full */
#define MGX_OP_CHAN_COPY 23   /* ptr0=src ptr1=dst ptr2=dst16 dims=rows,cols,lds,    */
                              /* soff,ldd,doff                                     */
#define MGX_OP_COLSUM 24      /* ptr0=x ptr1=ws ptr2=out dims=M,C                  */
#define MGX_OP_GEMM_TC_EX 25  /* ptr0=A ptr1=B ptr2=bias ptr3=C ptr4=workspace     */
                              /* ptr5=colstats act                                 */
                              /* dims=M,N,K,lda,ldb,ldc,(a_mn|b_mn<<1),splits      */
#define MGX_OP_WFLIP 26       /* ptr0=w ptr1=wf(bf16) dims=F,kh,kw,C,ld            */
#define MGX_OP_SUM_N 28       /* ptr0..4=sources ptr5=out dims=n,count             */
#define MGX_OP_CONCAT 29      /* ptr0..3=inputs ptr4=out ptr5=out16                 */
                              /* dims=rows,count,c0,c1,c2,c3                       */
#define MGX_OP_BN_FWD_FUSED 30 /* ptr0=x ptr1=stats ptr2=gamma ptr3=beta ptr4=y    */
                              /* ptr5=y16 dims=M,C,mmean*,mvar* fattr=eps,momentum */
                              /* act                                               */
#define MGX_OP_BN_BWD_FUSED 31 /* ptr0=dy ptr1=x ptr2=stats ptr3=gamma ptr4=dx     */
                              /* ptr5=dx16 dims=M,C,relu_gamma*,relu_beta*,dbeta*, */
                              /* dgamma*,dgamma_zero|ldd<<8,dsum* (ldd 0: C)        */
#define MGX_OP_BN_ACT_POOL 32 /* ptr0=x ptr1=stats ptr2=gamma ptr3=beta ptr4=y     */
                              /* ptr5=y16 act dims=pool geom (7; full at bit 40 of */
                              /* dims6),argmax*                                    */
#define MGX_OP_BN_BWD_REDUCE_POOL 33 /* ptr0=dy_pool ptr1=x ptr2=stats ptr3=ws     */
                              /* ptr4=sums ptr5=argmax act=dgamma_zero dims=M,C,    */
                              /* dbeta*,dgamma*,relu_gamma*,relu_beta*,geom packed  */
                              /* as MGX_OP_GEMM_CONV's (full at bit 48 of dims7)   */
#define MGX_OP_PREP_BATCH 35  /* ptr0=jobs (device mgx_prep_job[]) dims=njobs,units  */
#define MGX_OP_BN_BWD_DX_POOL 34 /* ptr0=dy_pool ptr1=x ptr2=stats ptr3=sums        */
                              /* ptr4=gamma ptr5=argmax dims=M,C,relu_beta*,dsum*, */
                              /* ws*,dx16*,geom packed (bf16 dx only)              */
#define MGX_OP_KV_ROUND 36    /* ptr0=host mgx_kv_round_args (kept alive by the     */
                              /* caller): one fused reduce+update+broadcast round   */
                              /* of a KVStore bucket inside the backward program,   */
                              /* so it overlaps the rest of the backward            */
#define MGX_OP_GEMM_CONV 27   /* ptr0=src(bf16 NHWC) ptr1=op ptr2=bias ptr3=C      */
                              /* ptr4=workspace ptr5=colstats dims=M,N,K,ldop,ldc, */
                              /* mode|splits<<8, B<<48|H<<32|W<<16|C,              */
                              /* kh<<40|kw<<32|sh<<24|sw<<16|ph<<8|pw              */

/* Run instructions eagerly, in order, on stream (no program object). */
int mgx_instr_run(const mgx_instr* instrs, int32_t count, uintptr_t stream);
int mgx_prog_create(const mgx_instr* instrs, int32_t count, uint64_t* out);
/* Launch instructions [begin, end) on stream.  mode 0: one kernel per
 * instruction; 1: those kernels captured once into a CUDA graph (with the
 * multi-lane schedule's side streams) and replayed. */
int mgx_prog_run(uint64_t prog, int32_t begin, int32_t end, uintptr_t stream, int32_t mode);
/* Per-instruction device time of one eager run of [begin,end) (profiling). */
int mgx_prog_profile(uint64_t prog, int32_t begin, int32_t end, uintptr_t stream, float* ms_out);
/* Multi-lane schedule (the dependency engine of engine.py:94-196 as CUDA
 * streams and events): lane[i] in [0, nlanes) for every instruction, and a
 * CSR (dep_ptr[n+1], dep_idx) of earlier instructions on other lanes that
 * instruction i must wait for.  Lane 0 is the caller's stream; a run (or
 * capture) of a range forks the side lanes off it and joins them back.
 * nlanes == 1 restores plain in-order execution.  Set before the first
 * captured run. */
int mgx_prog_set_schedule(uint64_t prog, int32_t nlanes, const int32_t* lane,
                          const int32_t* dep_ptr, const int32_t* dep_idx);
/* Number of kernel launches the range makes (captured once, not run). */
int mgx_prog_kernel_count(uint64_t prog, int32_t begin, int32_t end, uintptr_t stream,
                          int64_t* out);
int mgx_prog_destroy(uint64_t prog);
/* Whole-step graphs: capture what this thread enqueues on `stream` between
 * begin and end (both passes, their lanes, the store's rounds) into one
 * graph instantiated with per-node priorities; launch / destroy by handle. */
int mgx_capture_begin(uintptr_t stream);
int mgx_capture_end(uintptr_t stream, uint64_t* out);
int mgx_graph_launch(uint64_t graph, uintptr_t stream);
int mgx_graph_destroy(uint64_t graph);

/* ------------------------------------------------------------- KVStore
 * Device KVStore (kvstore.py:84-409): push -> level-1 tree aggregate over the
 * W workers of a machine -> level-2 tree over M machines -> updater -> pull.
 * One fused kernel per flushed round: the owner of each element range
 * tree-sums every worker's gradient, applies the updater on its momentum
 * shard, and stores the new weight into every worker replica.
 *
 * Segments are element ranges of the flat key arena this process owns:
 * {arena offset, length, offset into this process's momentum buffer}. */
typedef struct mgx_kv_seg {
  int64_t off;
  int64_t len;
  int64_t voff;
} mgx_kv_seg;

/* updater: 0 = add (kvstore.py:47-49), 1 = fused momentum SGD
 * (optim.py:64-78), 2 = aggregate only (result written to the gradient
 * buffer of worker 0, for custom updaters). */
#define MGX_KV_ADD 0
#define MGX_KV_SGD 1
#define MGX_KV_AGG 2

typedef struct mgx_kv_round_args {
  const mgx_kv_seg* segs;     /* HOST array, nseg <= 256 (copied into the launch) */
  int32_t nseg;
  int32_t machines, workers;  /* M x W gradient sources, ascending worker id */
  float* const* grads;        /* HOST array of M*W device pointers (local or IPC-mapped) */
  float* const* weights;      /* HOST array of M*W replica pointers */
  int32_t self_replica;       /* replica this process reads w from */
  float* velocity;            /* this process's momentum shard (SGD) */
  float* agg_out;             /* AGG: where this process's totals go */
  int32_t updater;
  float rescale, neg_eta, momentum, weight_decay;
  /* cross-process barrier (NULL flags = single process, no barrier):
   * flag arrays are 2 * 1024 * (M*W) uint32 words, zero-initialised once */
  uint32_t* const* flags;     /* HOST array of M*W flag-array pointers */
  int32_t rank;               /* this process's worker id when flags != NULL */
  uint32_t* epoch_ctr;        /* device, 2 words, zero-initialised: the kernel
                                 derives its barrier epoch from it and advances
                                 it, so captured launches replay correctly */
  uint32_t* error_word;       /* device word set non-zero on barrier timeout */
  int32_t grid;               /* 0 = auto; required (same on all ranks) with flags */
  /* push mode (flags != NULL, updater SGD or ADD; nscatter > 0): every
   * NVLink transfer is a remote STORE.  Phase 1 writes this process's
   * gradient values for every owner's segments into that owner's staging
   * buffer; after the barrier each owner reduces its shard from its own
   * staging buffer (local HBM, same tree order) and stores the new weights
   * into every replica.  scatter[i] = {arena offset, length, element offset
   * in stage[scatter_owner[i]]}; this process's staging buffer holds one
   * slot of stage_slot elements per worker, laid out like its momentum
   * shard (segs[].voff). */
  const mgx_kv_seg* scatter;  /* HOST array, nscatter <= 256 */
  const int32_t* scatter_owner;
  int32_t nscatter;
  float* const* stage;        /* HOST array of M*W staging-buffer pointers */
  int64_t stage_slot;
} mgx_kv_round_args;

int mgx_kv_round(const mgx_kv_round_args* args, uintptr_t stream);
/* Largest grid mgx_kv_round will use (flag arrays need grid * M*W words). */
int mgx_kv_max_grid(int32_t machines, int32_t workers, int32_t* out);
#define MGX_KV_FLAG_WORDS_PER_WORKER 2048  /* 2 phases x 1024 blocks */
/* Launch shape of the round kernel for a topology: largest resident grid,
 * threads per block, float4 vectors per thread per iteration. */
int mgx_kv_config(int32_t machines, int32_t workers, int32_t* max_grid, int32_t* threads,
                  int32_t* unroll);

#ifdef __cplusplus
}
#endif
#endif /* MGX_H_ */
