/*
 * fmoe_b200.h -- C-ABI of the B200-native FastMoE MoE-layer hot path.
 *
 * This is the drop-in boundary: plain pointers and sizes, no torch or C++
 * types.  Every entry point replaces one operator of the reference's C++ API
 * (reference: proj/include/fmoe/<name>.hpp) and is cited below.  The C++
 * drop-in headers (include/fmoe/<name>.hpp, libfmoe_dropin.so) and the Python
 * package (paper_2103_13262_b200) are thin hosts over these symbols.
 *
 * Conventions
 *   - Tensor pointers are DEVICE pointers unless the name ends in _host.
 *     Row-major, a row is one sample (matrix.hpp:12-14).
 *   - All work is stream-ordered on the context's stream; no entry point
 *     synchronises the host except where stated (validation, EP count
 *     exchange, *_host copies).
 *   - Indices are int32 on device (the reference uses int64; hosts widen).
 *   - Status: 0 ok, else one of FMOE_ERR_*, mapping 1:1 onto the reference's
 *     exception types (errors.hpp:8-23); fmoe_last_error() (thread-local)
 *     holds the message.  Calls never abort the process.
 *   - dtype selects the arithmetic: FMOE_F64 is the parity mode that
 *     reproduces the reference's fp64 accumulation order (bit-identical on
 *     every operator except softmax's exp); FMOE_F32 is SIMT fp32;
 *     FMOE_BF16 is the product path: bf16 storage, fp32 accumulation on the
 *     tcgen05 tensor cores, fp32 gate scores and fp32 weight gradients.
 */
#ifndef FMOE_B200_H_
#define FMOE_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FMOE_OK 0
#define FMOE_ERR_SHAPE 1     /* fmoe::ShapeError     (errors.hpp:8-11)  */
#define FMOE_ERR_PROTOCOL 2  /* fmoe::ProtocolError  (errors.hpp:13-17) */
#define FMOE_ERR_TRANSPORT 3 /* fmoe::TransportError (errors.hpp:19-23) */
#define FMOE_ERR_CUDA 4      /* CUDA / driver failure (no reference analogue) */

typedef enum { FMOE_F64 = 0, FMOE_F32 = 1, FMOE_BF16 = 2 } fmoe_dtype;

const char* fmoe_last_error(void);
const char* fmoe_version(void);

/* ------------------------------------------------------------------ context */
/* A context binds a device, a stream and a launch counter.  stream may be
 * NULL (legacy default stream) or a cudaStream_t. */
typedef struct fmoe_ctx fmoe_ctx;
int fmoe_ctx_create(int device, void* stream, fmoe_ctx** out);
int fmoe_ctx_destroy(fmoe_ctx* ctx);
int fmoe_ctx_set_stream(fmoe_ctx* ctx, void* stream);
/* Number of kernels this library launched through ctx (for bench accounting). */
int64_t fmoe_ctx_launches(const fmoe_ctx* ctx);
/* Per-stage timing of MoE-layer steps: arm n_steps x N stage events (CUDA
 * events on the context stream, recorded by fmoe_layer_fwd/bwd; n_steps = 0
 * disarms).  profile_read synchronises and returns, per stage, the summed
 * milliseconds between the previous mark and this one over the recorded
 * steps.  Stage order: 0 -, 1 gate, 2 plan, 3 scatter, 4 fc1, 5 fc2,
 * 6 gather_combine, 7 (fwd->bwd gap), 8 gather_combine_bwd, 9 dgrad fc2,
 * 10 wgrad fc2, 11 db2 (bf16: d_b2 column sums + the d_b1 and d_b2 reduce),
 * 12 dgrad fc1, 13 wgrad fc1, 14 db1 (0 on the bf16 path), 15 gate d_wg,
 * 16 gate d_x + scatter_backward. */
int fmoe_ctx_profile(fmoe_ctx* ctx, int n_steps);
int fmoe_ctx_profile_read(fmoe_ctx* ctx, float* stage_ms, int n_stages, int* steps_done);
/* Per profiled step s < n: milliseconds from its first mark to the next
 * step's first mark (the last step: to its own last mark); 0 for steps not
 * recorded.  Marks are graph-capturable (event-record nodes), so steps
 * replayed from a captured CUDA graph are timed too. */
int fmoe_ctx_profile_step_ms(fmoe_ctx* ctx, float* step_ms, int n);
/* Effective SM clock of the expert GEMMs: arm max_launches probe slots
 * (0 disarms); every expert-GEMM launch then records clock64 / globaltimer at
 * the start and end of its first CTA.  probe_read synchronises and returns the
 * cycle-weighted clock over the recorded launches (MHz = sum of cycles / sum
 * of nanoseconds * 1e3) and how many launches were recorded.  Lets a caller
 * state the tensor roofline at the clock the kernels actually ran at (the
 * power-capped B200 runs dense GEMMs well below clocks.max.sm). */
int fmoe_ctx_clock_probe(fmoe_ctx* ctx, int max_launches);
int fmoe_ctx_clock_probe_read(fmoe_ctx* ctx, double* sm_mhz, int* launches);
/* Synchronise the stream and surface any deferred device-side error (e.g. an
 * out-of-range expert index seen by fmoe_plan_build). */
int fmoe_ctx_check(fmoe_ctx* ctx);

/* --------------------------------------------------------------- gate (L1) */
/* gate_forward (gate.hpp:23-27; gate.cpp:23-35): scores = softmax(x * w_g)
 * rowwise, then the k largest scores, descending, ties -> lower expert index
 * (matrix.cpp:172-189).  Selected scores are not renormalised.
 *   x [n_b, d_m] dtype, w_g [d_m, E] dtype
 *   scores [n_b, E] and topk_scores [n_b, k]: f64 when dtype == FMOE_F64, else f32
 *   topk_idx [n_b, k] int32
 * ShapeError when k is not in [1, E]. */
int fmoe_gate_fwd(fmoe_ctx* ctx, fmoe_dtype dtype, const void* x, const void* w_g, int64_t n_b,
                  int64_t d_m, int64_t n_experts, int64_t k, void* scores, int32_t* topk_idx,
                  void* topk_scores);

/* gate_backward (gate.hpp:34-38; gate.cpp:37-65): full softmax Jacobian on
 * the selected scores.  d_topk [n_b, k] (score type), d_wg [d_m, E] (score
 * type, overwritten), d_x [n_b, d_m] dtype (overwritten; may be NULL). */
int fmoe_gate_bwd(fmoe_ctx* ctx, fmoe_dtype dtype, const void* x, const void* w_g,
                  const void* scores, const int32_t* topk_idx, const void* d_topk, int64_t n_b,
                  int64_t d_m, int64_t n_experts, int64_t k, void* d_wg, void* d_x);

/* -------------------------------------------------------- dispatch plan (L1) */
/* DispatchPlan (dispatch.hpp:15-24) on device.  Expert e owns the row block
 * [offsets[e], offsets[e] + counts[e]) of the expanded buffers; with
 * align == 1 offsets are exactly the reference's exclusive prefix sums and
 * capacity == n_b*k.  With align == 128 every block starts on a 128-row
 * tensor-core tile (rows between a block's end and the next start are padding:
 * src_row = -1, zero-filled by fmoe_scatter / fmoe_gather_combine_bwd).
 * Inside a block positions are ordered by (row, slot) ascending, exactly as
 * build_plan's row-major walk (dispatch.cpp:37-45). */
typedef struct {
  int64_t n_b, k, n_experts, align, capacity;
  int32_t* counts;      /* [E]                                              */
  int32_t* offsets;     /* [E+1]  offsets[E] = padded total rows            */
  int32_t* src_row;     /* [capacity] expanded_src_row, -1 for padding      */
  int32_t* slot;        /* [capacity] expanded_slot                         */
  int32_t* inverse_pos; /* [n_b*k]                                          */
  int32_t* tile_expert; /* [capacity/128] (align==128) expert of each tile  */
  int32_t* n_tiles;     /* [1] number of valid 128-row tiles                */
  void* scratch;        /* fmoe_plan_sizes() scratch_bytes                  */
} fmoe_plan;

/* Sizes for a plan: capacity rows and device scratch bytes. */
int fmoe_plan_sizes(int64_t n_b, int64_t k, int64_t n_experts, int64_t align, int64_t* capacity,
                    int64_t* scratch_bytes);
/* build_plan (dispatch.hpp:28; dispatch.cpp:10-47): histogram, exclusive scan
 * and stable (row, slot) ranking on device.  Out-of-range indices are a
 * ShapeError: reported immediately when validate != 0 (one host sync),
 * otherwise by the next fmoe_ctx_check(). */
int fmoe_plan_build(fmoe_ctx* ctx, const int32_t* topk_idx, fmoe_plan* plan, int validate);

/* ------------------------------------------------------------ permutes (L1) */
/* scatter (dispatch.cpp:49-59): xs[p] = x[src_row[p]]; padding rows := 0. */
int fmoe_scatter(fmoe_ctx* ctx, fmoe_dtype dtype, const void* x, int64_t d,
                 const fmoe_plan* plan, void* xs);
/* gather_combine (dispatch.cpp:61-78): y[i] = sum_j w[i,j] * ys[inverse_pos[i,j]],
 * slot order; w in score type. */
int fmoe_gather_combine(fmoe_ctx* ctx, fmoe_dtype dtype, const void* ys, int64_t d,
                        const fmoe_plan* plan, const void* topk_scores, void* y);
/* scatter_backward (dispatch.cpp:80-95): d_x[i] = sum_j d_xs[inverse_pos[i,j]]. */
int fmoe_scatter_bwd(fmoe_ctx* ctx, fmoe_dtype dtype, const void* d_xs, int64_t d,
                     const fmoe_plan* plan, void* d_x);
/* gather_combine_backward (dispatch.cpp:97-126): d_ys[pos] = w * d_y[i];
 * d_topk[i,j] = <d_y[i], ys[pos]>.  Padding rows of d_ys := 0. */
int fmoe_gather_combine_bwd(fmoe_ctx* ctx, fmoe_dtype dtype, const void* d_y, const void* ys,
                            int64_t d, const fmoe_plan* plan, const void* topk_scores,
                            void* d_ys, void* d_topk);

/* ------------------------------------------------------------- experts (L1) */
/* Expert pool parameters, all experts stacked: w1 [E, d_m, d_h], b1 [E, d_h],
 * w2 [E, d_h, d_m], b2 [E, d_m] (expert.hpp:15-21).  Biases are f32 when
 * dtype == FMOE_BF16, else dtype. */
typedef struct {
  const void* w1;
  const void* b1;
  const void* w2;
  const void* b2;
} fmoe_expert_params;
/* Gradients: f32 when dtype == FMOE_BF16, else dtype. */
typedef struct {
  void* d_w1;
  void* d_b1;
  void* d_w2;
  void* d_b2;
} fmoe_expert_grads;

/* multi_expert_forward (expert.hpp:47-53; expert.cpp:85-102): every block of
 * `blocks` (counts/offsets of a plan, or of an EP receive layout) runs
 * expert_forward: hidden = relu(xs*w1 + b1) (cached for backward), ys =
 * hidden*w2 + b2.  Empty blocks are legal.  FMOE_BF16 requires d_m and d_h to
 * be multiples of 64 and blocks->align == 128. */
int fmoe_experts_fwd(fmoe_ctx* ctx, fmoe_dtype dtype, const fmoe_plan* blocks, int64_t d_m,
                     int64_t d_h, fmoe_expert_params params, const void* xs, void* hidden,
                     void* ys);
/* multi_expert_backward (expert.hpp:60-64; expert.cpp:104-125): d_xs and all
 * four gradients (overwritten; empty experts get zero gradients). */
int fmoe_experts_bwd(fmoe_ctx* ctx, fmoe_dtype dtype, const fmoe_plan* blocks, int64_t d_m,
                     int64_t d_h, fmoe_expert_params params, const void* xs, const void* hidden,
                     const void* d_ys, void* d_xs, fmoe_expert_grads grads);

/* Expert operators with the reference's full ForwardCache (expert.hpp:31-35):
 * preact = xs*w1 + b1 is kept next to hidden = relu(preact), and the backward
 * masks with preact > 0 (relu_backward, matrix.cpp:147-153) exactly as
 * expert_backward does (expert.cpp:47-48), so caches built by a host remain
 * valid inputs.  FMOE_F64 / FMOE_F32 only. */
int fmoe_experts_fwd_cached(fmoe_ctx* ctx, fmoe_dtype dtype, const fmoe_plan* blocks, int64_t d_m,
                            int64_t d_h, fmoe_expert_params params, const void* xs, void* preact,
                            void* hidden, void* ys);
int fmoe_experts_bwd_cached(fmoe_ctx* ctx, fmoe_dtype dtype, const fmoe_plan* blocks, int64_t d_m,
                            int64_t d_h, fmoe_expert_params params, const void* xs, const void* preact,
                            const void* hidden, const void* d_ys, void* d_xs, fmoe_expert_grads grads);

/* ------------------------------------------------ dense primitives (L0) */
/* The matrix primitives the gate and experts are composed of, on the same
 * kernels as the FMOE_F64 / FMOE_F32 operators, so compositions reproduce the
 * operators' bits (test_gate.cpp:66-82).  FMOE_F64 / FMOE_F32 only.
 * matmul (matrix.hpp:77; matrix.cpp:96-119): c[m,n] = a[m,p] * b[p,n], one
 * fma chain per element over p ascending from +0.0. */
int fmoe_matmul(fmoe_ctx* ctx, fmoe_dtype dtype, const void* a, const void* b, int64_t m, int64_t p,
                int64_t n, void* c);
/* softmax_rows (matrix.hpp:89; matrix.cpp:155-170). */
int fmoe_softmax_rows(fmoe_ctx* ctx, fmoe_dtype dtype, const void* a, int64_t rows, int64_t cols,
                      void* out);
/* topk_rows (matrix.hpp:91-96; matrix.cpp:172-189): descending, ties -> lower
 * column.  ShapeError when k is not in [1, cols]. */
int fmoe_topk_rows(fmoe_ctx* ctx, fmoe_dtype dtype, const void* a, int64_t rows, int64_t cols,
                   int64_t k, int32_t* idx, void* vals);

/* dst[i] = src[i] converted between dtypes (round to nearest even), on the
 * context's stream; n elements. */
int fmoe_cast(fmoe_ctx* ctx, fmoe_dtype from, const void* src, fmoe_dtype to, void* dst, int64_t n);

/* --------------------------------------------------------- MoE layer (L3) */
/* One rank's slice of the layer (moe_layer.hpp:17-38): config, replicated
 * gate, local experts g = rank*n_e_local + slot, device weights, gradients and
 * all activations/workspace sized for n_b tokens. */
typedef struct {
  int64_t n_b, d_m, d_h, k, n_e_local, world_size, rank;
  uint64_t seed;
  fmoe_dtype dtype;
} fmoe_layer_config;
typedef struct fmoe_layer fmoe_layer;

int fmoe_layer_create(fmoe_ctx* ctx, const fmoe_layer_config* cfg, fmoe_layer** out);
int fmoe_layer_destroy(fmoe_layer* layer);
/* init_state (moe_layer.cpp:28-45): the reference's generators (mt19937_64,
 * stream_seed), bit-identical fp64 values rounded once to the layer dtype. */
int fmoe_layer_init_weights(fmoe_layer* layer);
/* Device pointers of the parameters (w_g, w1, b1, w2, b2) and gradients
 * (d_wg, d_w1, d_b1, d_w2, d_b2) so hosts can read/write them in place. */
int fmoe_layer_params(fmoe_layer* layer, void** w_g, fmoe_expert_params* experts);
int fmoe_layer_grads(fmoe_layer* layer, void** d_wg, fmoe_expert_grads* experts);
/* Activations kept for backward (MoEForwardCache, moe_layer.hpp:42-50). */
int fmoe_layer_routing(fmoe_layer* layer, const int32_t** topk_idx, const void** topk_scores,
                       const void** scores, fmoe_plan* plan);

/* Keep the expert pre-activations x*w1 + b1 of each forward
 * (ForwardCache::preact, expert.hpp:31-35) -- FMOE_F64 / FMOE_F32 layers only
 * (the bf16 path applies relu in the fc1 epilogue); ShapeError otherwise. */
int fmoe_layer_keep_preact(fmoe_layer* layer, int keep);
/* Device pointers of the forward's expert-side activations, in the plan's
 * layout (rows of expert g at plan offsets): xs = scattered inputs, hidden =
 * relu(preact), preact (NULL unless kept), ys = expert outputs.  Layer dtype. */
int fmoe_layer_activations(fmoe_layer* layer, const void** xs, const void** hidden, const void** preact,
                           const void** ys);

/* forward (moe_layer.cpp:67-110): x [n_b, d_m] -> y [n_b, d_m], dtype. */
int fmoe_layer_fwd(fmoe_layer* layer, const void* x, void* y);
/* backward (moe_layer.cpp:112-142): dy -> dx and parameter gradients. */
int fmoe_layer_bwd(fmoe_layer* layer, const void* dy, void* dx);
/* Aliases of fmoe_layer_fwd / fmoe_layer_bwd under the fmoe_moe_* names. */
int fmoe_moe_fwd(fmoe_layer* layer, const void* x, void* y);
int fmoe_moe_bwd(fmoe_layer* layer, const void* dy, void* dx);
/* forward with injected routing (the skewed-gate stress of SURVEY §8d cfg5:
 * a sampled IndexMatrix fed straight into build_plan, dispatch.hpp:28):
 * topk_idx [n_b, k] int32 in [0, E) (checked before any work: out of range ->
 * ShapeError from this call, as build_plan, dispatch.cpp:21-23; the check is
 * the one host synchronisation of the routed step), topk_scores [n_b, k]
 * in the score dtype.  The gate is skipped; the following fmoe_layer_bwd
 * yields d_x = scatter_backward(d_xs) (dispatch.cpp:80-95) with no gate term,
 * a zero gate gradient, and d(topk_scores) (gather_combine_backward's d_w,
 * dispatch.cpp:97-126) through fmoe_layer_routing_grad. */
int fmoe_layer_fwd_routed(fmoe_layer* layer, const void* x, const int32_t* topk_idx, const void* topk_scores,
                          void* y);
/* d(topk_scores) [n_b, k] of the last backward (score dtype, device). */
int fmoe_layer_routing_grad(fmoe_layer* layer, const void** d_topk_scores);
/* Host-buffer step for end-to-end use: H2D x (and dy), forward, backward,
 * D2H y (and dx).  Buffers are host memory (pinned for full speed); dy/dx may
 * be NULL for forward only.  Synchronises before returning. */
int fmoe_layer_step_host(fmoe_layer* layer, const void* x_host, const void* dy_host,
                         void* y_host, void* dx_host);
/* The same step without the final synchronisation, for loops that feed the
 * layer from the host: step t+1's uploads run under step t's kernels and step
 * t's downloads under step t+1's (two device buffer sets, event-ordered).
 * The host buffers of a step must stay untouched until a later
 * fmoe_layer_step_host_wait returns (it waits for every submitted step). */
int fmoe_layer_step_host_async(fmoe_layer* layer, const void* x_host, const void* dy_host,
                               void* y_host, void* dx_host);
int fmoe_layer_step_host_wait(fmoe_layer* layer);

/* train_step (moe_layer.cpp:144-205) on device: forward, mean-squared error
 * against target [n_b, d_m] (dtype) with d_y = 2*(y - target)/n, backward,
 * under EP expert gradients * 1/W and the gate gradient averaged over the
 * world (sync_gradients, param_sync.cpp:46-61, as fmoe_allreduce_sum), then
 * SGD p -= lr*g on every parameter (sgd_step, param_sync.cpp:63-66).  *loss
 * (may be NULL) receives the world-average loss; one host sync per call.
 * FMOE_F64 reproduces the reference's arithmetic; FMOE_BF16 updates fp32
 * master copies of the bf16 weights (widened from the bf16 values on the first
 * step after fmoe_layer_init_weights or fmoe_layer_sync_masters -- call the
 * latter after writing the weights through fmoe_layer_params). */
int fmoe_layer_train_step(fmoe_layer* layer, const void* x, const void* target, double lr, double* loss);
int fmoe_layer_sync_masters(fmoe_layer* layer);

/* Weight checkpoints in the reference's file format ("FMOE-CKPT" v1, f64,
 * checkpoint.hpp:10-16, checkpoint.cpp:63-122).  info reads the header;
 * load_checkpoint reads the gate and this rank's experts straight into the
 * layer (ShapeError unless d_m, d_h and the total expert count match; values
 * rounded once to the layer dtype); save_checkpoint writes every expert and
 * so needs a world_size 1 layer (ShapeError otherwise, as save_checkpoint's
 * expert-list check).  ProtocolError for unreadable / malformed files. */
typedef struct {
  int64_t n_b, d_m, d_h, k, n_e_local, world_size, experts_total;
  uint64_t seed;
} fmoe_ckpt_info;
int fmoe_checkpoint_info(const char* path, fmoe_ckpt_info* out);
int fmoe_layer_load_checkpoint(fmoe_layer* layer, const char* path);
int fmoe_layer_save_checkpoint(fmoe_layer* layer, const char* path);

/* --------------------------------------------- expert parallelism (L2, EP) */
/* A context's transport replaces the reference's Transport (transport.hpp:18-38).
 * Communicator over NCCL (NVLink/NVSwitch), one process per GPU: rank 0
 * creates a 128-byte id, the host broadcasts it out of band (torch.distributed
 * store, MPI, ...), every rank calls fmoe_comm_init.  TransportError on
 * failure. */
int fmoe_comm_unique_id(void* id_out, int64_t id_bytes);
int fmoe_comm_init(fmoe_ctx* ctx, const void* id, int64_t id_bytes, int world, int rank);
/* Use a communicator the caller already has (an ncclComm_t, e.g. the host
 * framework's, one rank per GPU): world and rank are read from it, it stays
 * owned by the caller and must outlive the context's expert-parallel calls. */
int fmoe_comm_attach(fmoe_ctx* ctx, void* nccl_comm);
/* In-process world (InProcWorld, transport.hpp:40-60): `world` ranks run as
 * host threads of one process, each with its own context joined to the world
 * (possibly all on one device).  Used to test the EP path on one GPU. */
typedef struct fmoe_world fmoe_world;
int fmoe_world_create(int world, fmoe_world** out);
int fmoe_world_destroy(fmoe_world* world);
int fmoe_ctx_join_world(fmoe_ctx* ctx, fmoe_world* world, int rank);

/* How an expert-parallel bf16 layer moves its rows (the reference's
 * all_to_all_rows / _reverse, collectives.cpp:146-265):
 *   FMOE_EP_EXCHANGE_PEER (default): fused into the kernels over NVLink peer
 *     memory -- the scatter writes token rows into the expert ranks, the fc2 /
 *     dgrad-fc1 epilogues store rows back into the source ranks, epoch flags
 *     in peer memory order the phases.  Connected on the first step through
 *     the context's transport (raw pointers inside one process, CUDA IPC
 *     across processes); if any rank cannot map its peers, every rank keeps
 *     the transport exchange.
 *   FMOE_EP_EXCHANGE_TRANSPORT: grouped send/recv through the transport
 *     (NCCL or the in-process world) between separate kernels.
 * FMOE_F64 / FMOE_F32 layers always use the transport.  Set before the
 * first forward, identically on every rank. */
/* Host arithmetic of the fused exchange (pure, no device): from the
 * all-gathered counts [world][world*local_experts] (rows rank s routes to
 * global expert g, as exchange_counts delivers them, collectives.cpp:69-109),
 * rank `rank`'s layouts (as fmoe_ep_layout) plus
 *   g_rank[g], g_delta[g]: its send rows of expert g land in rank g_rank[g]'s
 *     receive layout at (send position + g_delta[g]);
 *   route[3][local_experts*world]: for receive chunk c = e*world + s, its first
 *     row, its row count and its first row in rank s's send layout. */
int fmoe_ep_routes(int world, int rank, int64_t local_experts, int64_t align, const int64_t* counts,
                   int64_t* send_off, int64_t* chunk_off, int64_t* block_off, int64_t* rows, int32_t* g_rank,
                   int64_t* g_delta, int32_t* route);
#define FMOE_EP_EXCHANGE_PEER 0
#define FMOE_EP_EXCHANGE_TRANSPORT 1
int fmoe_layer_set_ep_exchange(fmoe_layer* layer, int mode);
/* Host-driven peer setup (instead of the automatic one through the
 * transport): every rank gets its blob (*length bytes; out may be NULL to
 * query), the host all-gathers them in rank order by any means, and every
 * rank connects before its first forward.  A connected bf16 layer then runs
 * expert parallelism with no transport at all.  TransportError if a peer
 * cannot be mapped. */
int fmoe_layer_peer_blob(fmoe_layer* layer, void* out, int64_t capacity, int64_t* length);
int fmoe_layer_peer_connect(fmoe_layer* layer, const void* blobs, int64_t blob_bytes);
/* *fused = 1 when the last forward ran the fused peer-memory exchange. */
int fmoe_layer_ep_exchange_fused(fmoe_layer* layer, int* fused);

/* ExchangePlan (collectives.hpp:16-33), host arrays of world*local_experts
 * entries owned by the caller: send_counts[dest][local expert],
 * recv_counts[source][local expert]. */
typedef struct {
  int64_t world, rank, local_experts;
  int64_t* send_counts;
  int64_t* recv_counts;
  int64_t send_total, recv_total;
} fmoe_exchange_plan;
/* exchange_counts (collectives.hpp:39-40; collectives.cpp:69-109): collective
 * over the context's transport; local_counts is this rank's per-global-expert
 * row count (host, n_counts = world*local_experts).  Synchronises.  ShapeError
 * when n_counts is not divisible by the world size. */
int fmoe_exchange_counts(fmoe_ctx* ctx, const int64_t* local_counts, int64_t n_counts,
                         fmoe_exchange_plan* plan);
/* all_to_all_rows (collectives.hpp:41-47; collectives.cpp:146-203): rows grouped
 * by (dest rank, dest local expert, scatter order) -> rows grouped by (local
 * expert, source rank, source order), device buffers, stream-ordered. */
int fmoe_a2a_rows(fmoe_ctx* ctx, fmoe_dtype dtype, const void* xs, int64_t d,
                  const fmoe_exchange_plan* plan, void* out);
/* Host-only layout of one exchange (no device work): send_off[E] (first row of
 * each (dest rank, its local expert) chunk in the send layout,
 * send_section_offsets collectives.cpp:114-122), chunk_off[el*W] (first row of
 * (local expert e, source s) in the receive layout, recv_chunk_offsets
 * collectives.cpp:126-135, index e*W+s), block_off[el+1] and rows[el] (expert
 * blocks starting on `align`-row boundaries; align 1 = reference layout). */
int fmoe_ep_layout(int world, int64_t local_experts, int64_t align, const int64_t* send_counts,
                   const int64_t* recv_counts, int64_t* send_off, int64_t* chunk_off, int64_t* block_off,
                   int64_t* rows);
/* all_to_all_rows_reverse (collectives.hpp:48-50; collectives.cpp:205-265). */
int fmoe_a2a_rows_reverse(fmoe_ctx* ctx, fmoe_dtype dtype, const void* ys, int64_t d,
                          const fmoe_exchange_plan* plan, void* out);

/* allreduce_sum (collectives.hpp:52-53; collectives.cpp:266-292): in-place
 * sum of n elements over the sorted rank list `group` (which must contain the
 * calling rank), accumulated in ascending rank order so every member holds
 * identical bytes.  ProtocolError for an empty/unsorted group, a caller
 * outside it, or members contributing different element counts.  Every member
 * of the world's transport must enter the call (SPMD).  FMOE_F64 / FMOE_F32. */
int fmoe_allreduce_sum(fmoe_ctx* ctx, fmoe_dtype dtype, void* buf, int64_t n, const int* group,
                       int64_t group_size);

#ifdef __cplusplus
}
#endif
#endif /* FMOE_B200_H_ */
