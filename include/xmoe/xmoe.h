/*
 * xmoe — B200-native (sm_100a) MoE-block hot path of X-MoE (arXiv 2508.13337).
 *
 * C-ABI drop-in boundary.  Plain pointers and sizes only; every operator is
 * stream-ordered on caller-owned DEVICE buffers and returns a status code.
 * Each entry point replaces one operator of the reference simulator's C++ API
 * (namespace moesim, /root/reference/proj/include/moesim/ headers); the citation
 * sits above each declaration.  The reference-shaped C++ adapter
 * (include/xmoe/moesim_compat.hpp) is built on these calls.
 *
 * Conventions
 *   - ids are int32; combine weights are float64 (the reference's `double`);
 *   - XMOE_F64 operands use the reference layouts and reproduce its
 *     arithmetic order bit for bit (parity mode);
 *   - XMOE_F32 keeps fp32 operands in the reference's operation order, the
 *     exact fp32 products accumulated in fp64 and each result rounded once
 *     to fp32 (bar: the reference's own max_rel_diff <= 1e-5, verify.cpp:117);
 *   - XMOE_BF16 operands are the performance path: bf16 storage, fp32
 *     accumulation on tcgen05 tensor cores, weights in the K-major B200
 *     layout documented per call;
 *   - errors: the status codes below map 1:1 onto the reference's exception
 *     types (error.hpp:10-38); xmoe_last_error() returns the reference's
 *     message text (thread-local).
 */
#ifndef XMOE_XMOE_H_
#define XMOE_XMOE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define XMOE_ABI_VERSION 1

/* status codes — moesim::ParseError .. PlanMismatch (error.hpp:10-38) */
#define XMOE_OK 0
#define XMOE_ERR_PARSE 1
#define XMOE_ERR_VALIDATION 2
#define XMOE_ERR_DIMENSION 3
#define XMOE_ERR_INDEX 4
#define XMOE_ERR_COUNT_MISMATCH 5
#define XMOE_ERR_PLAN_MISMATCH 6
#define XMOE_ERR_CUDA 10
#define XMOE_ERR_NCCL 11
#define XMOE_ERR_PEER_TIMEOUT 12 /* a peer rank never reached a cross-GPU flag (XMOE_PEER_TIMEOUT_S) */
#define XMOE_ERR_INTERNAL 99

/* element types */
#define XMOE_F64 0
#define XMOE_BF16 1
#define XMOE_F32 2

/* expert-parallel dispatch modes */
#define XMOE_DISPATCH_NAIVE 0 /* pf_dispatch/pf_combine (pf_pipeline.cpp:12-135) */
#define XMOE_DISPATCH_RBD 1   /* per-GPU redundancy bypass (rbd.cpp:26-358, node_of = rank) */

/* layer flags */
#define XMOE_LAYER_SSMB 1  /* ssmb_forward layer: every rank holds all experts (ssmb.cpp:29-43) */
#define XMOE_LAYER_TRAIN 2 /* keep what xmoe_moe_backward needs (BF16 layers) */
/* token chunks of the pipelined BF16 forward (plain dispatch): chunk c's
 * expert GEMMs overlap chunk c+1's dispatch and chunk c-1's combine.
 * 0 = automatic, 1 = off, 2..8 = that many chunks.  Results are
 * bit-identical for every chunk count. */
#define XMOE_LAYER_CHUNKS(n) ((n) << 8)
#define XMOE_LAYER_CHUNKS_OF(flags) (((flags) >> 8) & 15)
/* Redundancy-bypassing dispatch over nodes of n GPUs (node_of[w] = w / n,
 * the reference's two-tier form, rbd.cpp:83-358): one row per (token,
 * destination node), forwarded inside the node to the replicas' owners.
 * 0 or 1 = one GPU per node. */
#define XMOE_LAYER_GPUS_PER_NODE(n) ((n) << 12)
#define XMOE_LAYER_GPUS_PER_NODE_OF(flags) (((flags) >> 12) & 255)

typedef struct xmoe_ctx xmoe_ctx;
typedef struct xmoe_layer xmoe_layer;

int xmoe_abi_version(void);
const char* xmoe_last_error(void);
/* Number of device kernels this library has launched in the process. */
uint64_t xmoe_kernel_launches(void);

/* ------------------------------------------------------------------ context
 * One context per process and device.  world/rank describe the expert-
 * parallel group (moesim::Comm / WorkerGroup, collectives.hpp:71-76):
 *   rank >= 0 : this process is rank `rank` of `world` processes, one GPU
 *               each; the exchange runs over NCCL on NVLink.  nccl_id is the
 *               128-byte ncclUniqueId from xmoe_nccl_unique_id() on rank 0
 *               (NULL when world == 1).
 *   rank == -1: this process drives all `world` workers itself on `device`
 *               (the reference's SPMD "all ranks in one call" shape,
 *               SURVEY §8(b)); the exchange is an on-device row move.      */
int xmoe_nccl_unique_id(void* out_128_bytes);
int xmoe_ctx_create(int device, int world, int rank, const void* nccl_id, xmoe_ctx** out);
int xmoe_ctx_destroy(xmoe_ctx* ctx);
/* XMOE_OK, or XMOE_ERR_NCCL when the context's communicator reports an
 * asynchronous error (ncclCommGetAsyncError). */
int xmoe_ctx_status(xmoe_ctx* ctx);  /* NCCL async errors; asynchronous checks (once) */

/* ------------------------------------------------------------------ operators */

/* moesim::gate_forward (gating.hpp:35, gating.cpp:14-57).
 * x [S,H]; F64: wg [H,E] (reference layout); BF16: wg [E,H] (K-major).
 * Outputs top_experts [S,k] (descending prob, ties -> lower id) and the raw
 * softmax probabilities weights [S,k]; renorm != 0 divides by their sum
 * (restated beyond the reference).  logits [S,E] fp64 is optional. */
int xmoe_gate_forward(xmoe_ctx* ctx, int dtype, const void* x, const void* wg, int64_t S,
                      int64_t H, int64_t E, int64_t k, int renorm, int32_t* top_experts,
                      double* weights, double* logits, void* stream);

/* moesim::pft_construct (pft.hpp:32-38, pft.cpp:12-60).
 * top [S,k], w [S,k] -> expert-major packed ERI arrays of B <= S*k rows:
 * token_ids[B], expert_ids[B], cw[B], tokens_per_expert[E]; B is written to
 * *B_dev (device int32).  slot_pos [S,k] (optional) receives, per token, the
 * packed rows of its kept copies ascending, padded with -1.  validate != 0
 * checks id range/distinctness (synchronises the stream). */
int xmoe_pft_construct(xmoe_ctx* ctx, const int32_t* top, const double* w, int64_t S, int64_t k,
                       int64_t E, int64_t cap, int32_t* token_ids, int32_t* expert_ids,
                       double* cw, int32_t* tokens_per_expert, int32_t* slot_pos,
                       int32_t* B_dev, int validate, void* stream);

/* moesim::gather_rows (pft.hpp:41, pft.cpp:68-77): out[i] = src[ids[i]]. */
int xmoe_gather_rows(xmoe_ctx* ctx, int dtype, const void* src, int64_t rows, int64_t cols,
                     const int32_t* ids, int64_t n, void* out, int validate, void* stream);

/* moesim::scatter_combine (pft.hpp:45-46, pft.cpp:79-91): out [S,cols] =
 * sum over i ascending of weights[i] * rows[i] into token_ids[i].
 * Deterministic gather-reduce (no atomics); F64 is bit-exact. */
int xmoe_scatter_combine(xmoe_ctx* ctx, int dtype, const void* rows, int64_t n, int64_t cols,
                         const int32_t* token_ids, const double* weights, int64_t S, void* out,
                         int validate, void* stream);

/* moesim::grouped_expert_mlp (pf_pipeline.hpp:38-39, pf_pipeline.cpp:83-105).
 * in [rows,H]; rows_per_expert [G] (device); expert i covers the next
 * rows_per_expert[i] rows and they must sum to `rows` (the reference's
 * CountMismatch, checked on the device without a host sync: the GEMMs run on
 * counts clamped to the buffer and xmoe_ctx_status reports the mismatch).
 * F64: w1 [G,H,F], w2 [G,F,H] (reference layout).
 * BF16: w1 [G,F,H], w2 [G,H,F] (K-major; tcgen05 grouped GEMM). */
int xmoe_grouped_mlp(xmoe_ctx* ctx, int dtype, const void* in, int64_t rows,
                     const int32_t* rows_per_expert, int64_t G, const void* w1, const void* w2,
                     int64_t H, int64_t F, void* out, void* stream);

/* The tcgen05 grouped GEMM itself (BF16): D[rows,N] = A[rows,K] . B_g[N,K]^T
 * per group, optional ReLU epilogue.  Exposed for the numerics tests. */
int xmoe_grouped_gemm_bf16(xmoe_ctx* ctx, const void* A, int64_t rows, int64_t K,
                           const int32_t* rows_per_group, int64_t G, const void* B, int64_t N,
                           void* D, int relu, void* stream);

/* Exchange plan of the plain dispatch for rank `me`, from the all-gathered
 * per-expert counts tpe_all [W, E] (HOST memory; no GPU needed):
 * send_off [E+1]  start of expert e's block in me's packed buffer;
 * recv_off [W*El] grouped row where source s's rows of my local expert le
 *                 start ((local expert, source, position), pf_pipeline.cpp:47-73);
 * recv_per_expert [El].  Any output may be NULL. */
int xmoe_plan_dispatch(int W, int E, const int32_t* tpe_all, int me, int64_t* send_off,
                       int64_t* recv_off, int64_t* recv_per_expert);

/* Grouped weight-gradient GEMM (BF16 in, fp32 out): D_g [M,N] = X_g^T Y_g over
 * the row segments of X [rows,M] and Y [rows,N] (transposed and zero-padded
 * to 64-row multiples on the device, then the grouped-K tcgen05 kernel). */
int xmoe_grouped_wgrad_bf16(xmoe_ctx* ctx, const void* X, const void* Y, int64_t rows,
                             const int32_t* rows_per_group, int64_t G, int64_t M, int64_t N, float* D,
                             void* stream);

/* One weight gradient D [M,N] = X^T Y (BF16 in, fp32 out) over all `rows` of
 * X [rows,M] and Y [rows,N], split along the rows into `splits` (1..32)
 * segments whose fp32 partials are summed in segment order (deterministic).
 * M % 64 == 0, N % 8 == 0 (N is padded to 128 inside; the padding reads as
 * zeros).  This is the layer's shared-expert and gate weight gradient. */
int xmoe_wgrad_split_bf16(xmoe_ctx* ctx, const void* X, const void* Y, int64_t rows, int64_t M, int64_t N,
                          int64_t splits, float* D, void* stream);

/* ------------------------------------------------------------------ split expert-parallel operators
 * The reference's SPMD shape: one call takes EVERY worker's
 * data (rank == -1 context, all W = world workers on this device).  Per-worker
 * arguments are HOST arrays of W DEVICE pointers; counts are host int64
 * arrays.  Packed buffers are a Pft (pft.hpp:17-25): rows x [B_w, H] in
 * expert-major packed order with token_ids / expert_ids / combine weights,
 * tokens_per_expert of all workers as one device [W, E] int32 matrix.  Every
 * copy lands at its owner's grouped row in (local expert, source, position)
 * order (pf_pipeline.cpp:47-73).  dest_rank/dest_row [B_w] receive (or may be
 * scratch when NULL, pf_dispatch only) the owner and grouped row of each copy. */

/* moesim::pf_dispatch (pf_pipeline.hpp:34, pf_pipeline.cpp:12-81).  Outputs:
 * expert_input[j] [n_j, H] (n_j = rows owned by j, sized by the caller from
 * tpe), recv_per_expert [W, E/W] device, arrival_to_grouped[j] [n_j]
 * (optional; NULL entries or NULL array skip it). */
int xmoe_pf_dispatch(xmoe_ctx* ctx, int dtype, int64_t H, int64_t E, const void* const* packed,
                     const int32_t* const* expert_ids, const int64_t* B, const int32_t* tpe, void* const* expert_input,
                     int32_t* recv_per_expert, int32_t* const* dest_rank, int32_t* const* dest_row,
                     int32_t* const* arrival_to_grouped, void* stream);

/* moesim::pf_combine (pf_pipeline.hpp:42-45, pf_pipeline.cpp:107-135): the
 * return trip plus scatter_combine per source: out[w] [seq_lens[w], H] =
 * sum over w's copies in packed order of cw * expert_out[owner][grouped row]
 * (F64: the reference's axpy order, bit-exact). */
int xmoe_pf_combine(xmoe_ctx* ctx, int dtype, int64_t H, int64_t E, const void* const* expert_out,
                    const int32_t* tpe, const int32_t* const* token_ids, const int32_t* const* expert_ids,
                    const double* const* cw, const int64_t* B, const int64_t* seq_lens, void* const* out,
                    void* stream);

/* moesim::select_pilots (rbd.hpp:46-47, rbd.cpp:26-81) for one packed buffer
 * of B copies: groups the copies by (token, node of the expert's owner) with
 * node = owner / gpus_per_node (contiguous blocks, placement.hpp:21-26) and
 * draws one Rng(seed).below(|group|) per group in (token, node) order.
 * S bounds the token ids (< S) and k the copies per token.  pilot_mask [B]
 * (uint8, device); pilot_of [B] (optional) = packed row of each copy's pilot. */
int xmoe_select_pilots(xmoe_ctx* ctx, int64_t B, const int32_t* token_ids, const int32_t* expert_ids, int64_t S,
                       int64_t k, int64_t E, int64_t W, int64_t gpus_per_node, uint64_t seed, uint8_t* pilot_mask,
                       int32_t* pilot_of, void* stream);

/* moesim::rbd_dispatch (rbd.hpp:78-79, rbd.cpp:83-285): stage 1 moves each
 * (token, node) group's pilot row to the pilot's owner (the landing worker),
 * stage 2 re-creates the replicas there from the landed row and stores them
 * at their owners on the same node.  expert_input is bit-identical to
 * xmoe_pf_dispatch's (rbd.hpp:50).  pilot_mask[w] [B_w] is the plan's mask;
 * seq_lens bound the token ids, k the copies per token.  Outputs per source:
 * dest_rank, dest_row and pilot_of [B_w] (all required: they are the
 * bookkeeping the reverse path and the reference's RbdDispatch are built
 * from).  XMOE_ERR_PLAN_MISMATCH when a group has no or several pilots. */
int xmoe_rbd_dispatch(xmoe_ctx* ctx, int dtype, int64_t H, int64_t E, int64_t gpus_per_node,
                      const void* const* packed, const int32_t* const* token_ids, const int32_t* const* expert_ids,
                      const int64_t* B, const int64_t* seq_lens, int64_t k, const int32_t* tpe,
                      const uint8_t* const* pilot_mask, void* const* expert_input, int32_t* recv_per_expert,
                      int32_t* const* dest_rank, int32_t* const* dest_row, int32_t* const* pilot_of, void* stream);

/* moesim::rbd_combine (rbd.hpp:85-88, rbd.cpp:287-358) over the reference's
 * RbdDispatch bookkeeping, flattened: P landed pilots (all landing workers),
 * flat pilot p landed at worker land_of[p], grouped row land_pos[p], multi-copy
 * flag and weight; its replicas' outputs are entries ent_ptr[p]..ent_ptr[p+1]
 * (owner, grouped row, weight) in the reference's slot order.  The landing
 * worker merges: y_p (x w_p when multi) + sum w_r y_r (kernels::scale/axpy);
 * source w then adds, per token in pilot order, merged row f scaled by
 * flat_scale[f] (1 for multi-copy groups, else the pilot weight):
 * src_ptr[w] [seq_lens[w]+1] / src_flat[w] is a token CSR of flat indices.
 * All arrays are DEVICE arrays except seq_lens. */
int xmoe_rbd_combine(xmoe_ctx* ctx, int dtype, int64_t H, const void* const* expert_out, int64_t P,
                     const int32_t* land_of, const int32_t* land_pos, const uint8_t* land_multi, const double* land_w,
                     const int32_t* ent_ptr, const int32_t* ent_owner, const int32_t* ent_pos, const double* ent_w,
                     const int32_t* const* src_ptr, const int32_t* const* src_flat, const double* flat_scale,
                     const int64_t* seq_lens, void* const* out, void* stream);

/* Distinct (token, node) pairs among n copies (moesim::redundancy_rate*,
 * internode_redundancy_counts, rbd.cpp:390-442): node = expert_node[expert]
 * (device [E]), tokens < `tokens`, nodes < `nodes`; copies on skip_node are
 * ignored (-1 = none).  *copies and *groups are host outputs (synchronises). */
int xmoe_route_pairs(xmoe_ctx* ctx, int64_t n, const int32_t* token, const int32_t* expert,
                     const int32_t* expert_node, int64_t E, int64_t nodes, int64_t tokens, int64_t skip_node,
                     int64_t* copies, int64_t* groups, void* stream);

/* ------------------------------------------------------------------ synthetic inputs
 * The reference's generator on the device: outputs [offset, offset+n) of
 * Rng(seed).uniform(lo, hi) (rng.hpp:24-47, xoshiro256** + 53-bit uniform),
 * each snapped to multiples of 1/grid (round half even; grid 0 = none) and
 * stored as dtype (XMOE_F64 | XMOE_F32 | XMOE_BF16, round to nearest even).
 * GF(2) jump-ahead: any offset, no host draws. */
int xmoe_rng_uniform(xmoe_ctx* ctx, uint64_t seed, uint64_t offset, int64_t n, double lo, double hi, double grid,
                     int dtype, void* out, void* stream);
/* The same from an explicit generator state (moesim::Rng's four words), and
 * a host-side jump of such a state by n outputs. */
int xmoe_rng_uniform_state(xmoe_ctx* ctx, const uint64_t* state, uint64_t offset, int64_t n, double lo, double hi,
                           double grid, int dtype, void* out, void* stream);
int xmoe_rng_advance(uint64_t* state, uint64_t n);
/* moesim::salt_seed (rng.hpp:17-19). */
uint64_t xmoe_salt_seed(uint64_t seed, uint64_t a, uint64_t b);
/* moesim::make_layer_weights (padded_pipeline.cpp:13-27) on the device for
 * Rng(seed) advanced by `offset` draws: gate [H,E] (NULL = skip; snapped to
 * gate_grid when > 0) and experts [first_expert, first_expert + n_experts) of
 * w1 [.,H,F] / w2 [.,F,H], in the reference layouts and draw order. */
int xmoe_make_layer_weights(xmoe_ctx* ctx, uint64_t seed, uint64_t offset, int64_t E, int64_t H, int64_t F,
                            int64_t first_expert, int64_t n_experts, double gate_grid, int dtype, void* gate,
                            void* w1, void* w2, void* stream);

/* ------------------------------------------------------------------ layer
 * One MoE layer's weights resident in HBM in the B200 layout, plus the
 * workspace of its forward pass.  Weights are DEVICE pointers in the
 * reference layouts (moe_instance.hpp:17-21) and dtype: gate [H,E],
 * w1 [E_local,H,F], w2 [E_local,F,H], where E_local = E/world experts owned
 * by this rank (all E when rank == -1); shared experts sw1 [n_shared,H,Fs],
 * sw2 [n_shared,Fs,H] (restated beyond the reference; may be NULL). */
typedef struct {
    int64_t num_experts;     /* E */
    int64_t model_dim;       /* H */
    int64_t ffn_dim;         /* F */
    int64_t top_k;           /* k */
    int64_t max_token_count; /* capacity per expert per source rank */
    int64_t n_shared;        /* shared experts (0 = none) */
    int64_t shared_ffn_dim;  /* Fs */
    int64_t max_tokens;      /* S bound per rank (workspace sizing) */
    int32_t dtype;           /* XMOE_F64 | XMOE_BF16 */
    int32_t renorm;          /* top-k renormalisation (0 = reference) */
    int32_t dispatch_mode;   /* XMOE_DISPATCH_NAIVE | XMOE_DISPATCH_RBD */
    int32_t flags;           /* XMOE_LAYER_SSMB | XMOE_LAYER_TRAIN | XMOE_LAYER_CHUNKS(n) */
    uint64_t seed;           /* RBD pilot seed (salted per rank: salt_seed(seed, w, 0)) */
} xmoe_layer_desc;

int xmoe_layer_create(xmoe_ctx* ctx, const xmoe_layer_desc* desc, const void* gate,
                      const void* w1, const void* w2, const void* sw1, const void* sw2,
                      xmoe_layer** out);
/* Collective for one-process-per-GPU layers: every rank must call it (a flag
 * barrier keeps a peer's last NVLink reads off this rank's freed buffers). */
int xmoe_layer_destroy(xmoe_layer* layer);
/* XMOE_OK, XMOE_ERR_NCCL (asynchronous communicator error), or
 * XMOE_ERR_PEER_TIMEOUT when a cross-GPU wait of an earlier pass
 * gave up after XMOE_PEER_TIMEOUT_S seconds (default 300) because a peer never
 * arrived.  The wait does not trap the device: the pass finishes with invalid
 * results and every later forward/backward on the layer returns this code. */
int xmoe_layer_status(xmoe_layer* layer);

/* moesim::pf_moe_forward / rbd_moe_forward (pf_pipeline.hpp:48-49, rbd.hpp:92)
 * selected by desc->dispatch_mode.  x/out: [n_local, S, H] where n_local = 1
 * for a rank >= 0 context and world for rank == -1.  Device buffers. */
int xmoe_moe_forward(xmoe_ctx* ctx, xmoe_layer* layer, const void* x, int64_t S, void* out,
                     void* stream);

/* The same forward with a token count per worker (moe_instance.hpp:27 allows
 * S_w to differ): S_per_worker [n_local] (host); x/out hold the workers'
 * [S_w, H] blocks back to back.  Runs the unchunked pipeline. */
int xmoe_moe_forward_v(xmoe_ctx* ctx, xmoe_layer* layer, const void* x, const int64_t* S_per_worker, void* out,
                       void* stream);

/* moesim::ssmb_forward (ssmb.hpp:23-26, ssmb.cpp:12-46): x_full [S,H] is the
 * whole sequence on every rank; rank g runs rows [g*(S/G), ...) (last rank
 * takes the remainder), then an all-gather restores out_full [S,H] on every
 * rank.  G == world; max_tokens >= the largest shard.
 *   XMOE_LAYER_SSMB layers hold every expert (the reference's replicated
 *   weights, ssmb.cpp:29-43): each shard routes locally.
 *   Expert-parallel layers (no XMOE_LAYER_SSMB; E/world experts per rank):
 *   SSMB composed with EP — the shard's copies go to their owners through the
 *   layer's exchange; same drop sets and, row by row, the same result. */
int xmoe_ssmb_forward(xmoe_ctx* ctx, xmoe_layer* layer, const void* x_full, int64_t S,
                      void* out_full, void* stream);

/* Backward of the last xmoe_moe_forward (restated beyond the reference,
 * which is forward-only).  x is the same input, dy the
 * gradient of the output, both [S, H] bf16 on this rank; writes dx [S, H]
 * bf16 and the layer's fp32 weight gradients, read with xmoe_layer_grads.
 * Routing and capacity drops are constants of the forward (as in the
 * reference's semantics); renorm layers are not supported.  One backward per
 * forward: its cross-rank barriers are keyed by that forward's epoch
 * (XMOE_ERR_VALIDATION otherwise). */
int xmoe_moe_backward(xmoe_ctx* ctx, xmoe_layer* layer, const void* x, const void* dy, int64_t S,
                      void* dx, void* stream);
/* Device pointers (fp32, owned by the layer) to the gradients of the last
 * backward, reference layouts: gate [H,E], w1 [E_local,H,F], w2 [E_local,F,H],
 * shared merged sw1 [H, n_shared*Fs] (expert s = columns s*Fs..), sw2
 * [n_shared*Fs, H].  Any argument may be NULL.
 * Scope with one process per GPU: dw1/dw2 are COMPLETE for this rank's
 * experts (every rank's tokens reach them through the exchange); dgate,
 * dsw1 and dsw2 are PARTIAL sums over this rank's tokens only — all-reduce
 * them over the expert-parallel group before the optimizer step. */
int xmoe_layer_grads(xmoe_layer* layer, float** dgate, float** dw1, float** dw2, float** dsw1,
                     float** dsw2);

/* Replace the layer's weights in place (e.g. after an optimizer step), same
 * layouts and dtype as xmoe_layer_create, this rank's experts only; refreshes
 * the B200-layout copies and, for training layers, the reference-layout
 * copies the backward reads.  Stream-ordered; captured forwards stay valid. */
int xmoe_layer_set_weights(xmoe_layer* layer, const void* gate, const void* w1, const void* w2, const void* sw1,
                           const void* sw2, void* stream);

/* Debug view of the last forward's internal arrays (synchronises the
 * device): *ptr = a DEVICE pointer owned by the layer, *count = elements.
 * `worker` indexes the ranks this context drives (0 for rank >= 0).  Used by
 * the parity tests to compare the routing, the packed order and the grouped
 * dispatch layout bit for bit with the reference's own pf_dispatch /
 * select_pilots. */
#define XMOE_INSPECT_TOP_EXPERTS 0       /* int32 [S,k] (gating.hpp:15-32) */
#define XMOE_INSPECT_WEIGHTS 1           /* f64 [S,k] */
#define XMOE_INSPECT_TOKEN_IDS 2         /* int32 [B] (pft.hpp:17-25) */
#define XMOE_INSPECT_EXPERT_IDS 3        /* int32 [B] */
#define XMOE_INSPECT_COMBINE_WEIGHTS 4   /* f64 [B] */
#define XMOE_INSPECT_TOKENS_PER_EXPERT 5 /* int32 [E] */
#define XMOE_INSPECT_TPE_ALL 6           /* int32 [W,E] all-gathered counts */
#define XMOE_INSPECT_EXPERT_INPUT 7      /* dtype [R_max,H]: PfDispatch::expert_input (unchunked: rows 0..n) */
#define XMOE_INSPECT_EXPERT_OUTPUT 8     /* dtype [R_max,H] */
#define XMOE_INSPECT_RECV_PER_EXPERT 9   /* int32 [E/W] (unchunked layers) */
#define XMOE_INSPECT_TPE_CHUNKS 10       /* int32 [W,C,E] (chunked layers: region c holds chunk c) */
#define XMOE_INSPECT_DEST_RANK 11        /* int32 [B] owner of each packed row */
#define XMOE_INSPECT_DEST_ROW 12         /* int32 [B] its grouped row at the owner */
#define XMOE_INSPECT_SLOT_POS 13         /* int32 [S,k] packed rows of each token's kept copies */
#define XMOE_INSPECT_PILOT_MASK 14       /* uint8 [B] RbdPlan::pilot_mask (rbd.hpp:28-41) */
#define XMOE_INSPECT_SSMB_KEPT 15        /* int32 [G] kept copies per shard of the last ssmb_forward */
int xmoe_layer_inspect(xmoe_layer* layer, int worker, int what, const void** ptr, int64_t* count);

/* Byte ledger of the last forward on this layer (collectives.hpp:31-49):
 * out[0..n) = { dispatch_rows_self, dispatch_rows_offrank,
 *               dispatch_meta_offrank, combine_rows_self,
 *               combine_rows_offrank, routed_copies, unique_rows_offrank,
 *               copies_offrank } summed over this context's ranks. */
int xmoe_layer_ledger(xmoe_layer* layer, uint64_t* out, int n);

/* Topology for the reference-schema ledger (moesim::Topology,
 * config.hpp:30-40): node_of[w] = w / gpus_per_node classifies every
 * message as self, intra-node or inter-node; the alpha-beta model
 * (collectives.cpp:56-76) charges latency + bytes / bandwidth per message
 * to its sender.  dtype_bytes: wire bytes per element (0 = the layer's). */
typedef struct xmoe_topology {
    int64_t gpus_per_node;
    double bw_intra, bw_inter;           /* bytes / s */
    double latency_intra, latency_inter; /* s per message */
    int64_t dtype_bytes;
} xmoe_topology;

/* One collective of the last forward, as moesim::LedgerEntry
 * (collectives.hpp:31-41): the exchanges the reference's pf_moe_forward /
 * rbd_moe_forward / ssmb_forward perform, in its order and with its kinds
 * ("dispatch_counts", "dispatch_rows", "combine_rows", "rbd_dispatch_counts",
 * "rbd_dispatch_meta", "rbd_dispatch_rows1", "rbd_dispatch_meta2",
 * "rbd_dispatch_rows2", "rbd_combine_rows2", "rbd_combine_rows1",
 * "ssmb_gather_rows"), bytes from this layer's actual routing. */
typedef struct xmoe_ledger_entry {
    int64_t id;
    char kind[32];
    uint64_t self_bytes, intra_bytes, inter_bytes, intra_msgs, inter_msgs;
    double time_s;
} xmoe_ledger_entry;

/* Entries of the last forward (topo NULL = the reference defaults:
 * gpus_per_node 8, 200e9 / 25e9 B/s, zero latency).  *n receives the entry
 * count; at most cap are written.  With one process per GPU the per-rank
 * contributions are summed over the group (collective: every rank calls). */
int xmoe_layer_ledger_entries(xmoe_layer* layer, const xmoe_topology* topo, xmoe_ledger_entry* out, int cap,
                              int* n);
/* The same as CostLedger::write_csv (collectives.cpp:26-34):
 * "collective_id,kind,intra_bytes,inter_bytes,modeled_time_s" rows.
 * *len receives the full length; at most cap bytes (NUL-terminated) are
 * written. */
int xmoe_layer_ledger_csv(xmoe_layer* layer, const xmoe_topology* topo, char* buf, int64_t cap, int64_t* len);
/* The padded (GShard) comparator for this layer: the ledger the reference's
 * padded_moe_forward (padded_pipeline.cpp:75-159) charges — every pair moves
 * e_local * max_token_count padded rows each way, whatever the routing —
 * in the same CSV schema ("padded_dispatch_rows", "padded_combine_rows"). */
int xmoe_layer_padded_ledger_csv(xmoe_layer* layer, const xmoe_topology* topo, char* buf, int64_t cap,
                                 int64_t* len);

/* Per-stage device time of the last forward (ms, CUDA events), order:
 * gate, pft, dispatch, experts, shared, combine, total, then the exchange
 * split: counts (all-gather + destination rows), rows_moved (the row kernel), dispatch_barrier,
 * return_wait (merge/barrier before the combine), combine_kernel, and the
 * shared-expert GEMMs.  Timing mode serialises the unchunked forward (the
 * shared-expert GEMMs run in line as the "shared" stage instead of on the
 * side stream), so every stage is an isolated kernel time and "total" is
 * their sum, not the overlapped step.  Chunked layers append, per chunk,
 * the ms from the start to its scatter end, GEMM start, GEMM end and
 * combine end (n = 13 + 4 * chunks).  Requires timing enabled. */
int xmoe_layer_set_timing(xmoe_layer* layer, int enable);
/* Capture the forward as a CUDA graph per (x, out, S) and replay it (the
 * forward has no host synchronisation on the local and NVLink transports). */
int xmoe_layer_set_graph(xmoe_layer* layer, int enable);

/* Token chunks the BF16 forward of this layer is pipelined over (1 = not
 * chunked); see XMOE_LAYER_CHUNKS. */
int xmoe_layer_chunks(const xmoe_layer* layer, int32_t* out);
int xmoe_layer_stage_ms(xmoe_layer* layer, float* out, int n);
/* Per-stage device time of the last backward (ms; timing enabled, training
 * layer), order: dy scatter (+barrier), owner prep (dL/dw, dz), dgrad GEMMs,
 * wgrad GEMMs, token level (transposes + shared experts), gate + dx combine. */
int xmoe_layer_bwd_stage_ms(xmoe_layer* layer, float* out, int n);

#ifdef __cplusplus
}
#endif
#endif /* XMOE_XMOE_H_ */
