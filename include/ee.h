/*
 * ee.h -- C-ABI of the B200-native EE-Tuning exit-head library (libee_b200.so).
 *
 * EE-Tuning (arXiv 2402.00518) tunes early-exit heads attached to a frozen
 * LLM.  This library implements the data-parallel hot path of its Stage 2
 * (§2.2) -- for every exit i: apply the exit head to the
 * cached hidden states h_i, compute the token-level softmax cross-entropy,
 * backpropagate into the exit-head parameters only -- plus the Stage-1
 * initialisers (Copy / Random) and the optimizer (Adam).
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  - Ownership: the caller owns every buffer.  The library never allocates
 *    device memory in these calls; scratch comes from a caller-provided
 *    workspace sized by ee_workspace_size().
 *  - Pointers: "device" pointers must be CUDA device (or managed) memory of the
 *    current device; "host" pointers are ordinary host memory.  Device base
 *    pointers must be 16-byte aligned (EE_ERR_ALIGN otherwise).
 *  - Layout: row-major, C-contiguous.  bf16 = IEEE bfloat16 (uint16 storage).
 *  - Asynchrony: everything is enqueued on `stream` (a cudaStream_t passed as
 *    void*; NULL = legacy default stream).  No call synchronises the host
 *    except ee_get_status().  Argument/shape errors are returned synchronously
 *    and nothing is enqueued; errors only the device can see (target ids out
 *    of range, non-finite losses) are recorded in a status word inside the
 *    workspace and read with ee_get_status().
 *  - Workspace: caller-allocated device scratch of ee_workspace_size() bytes,
 *    ZERO-INITIALISED ONCE before first use (its head holds the device status
 *    word, cleared again by ee_get_status); one workspace per stream.
 *  - Thread safety: calls are re-entrant (distinct workspaces); ee_last_error()
 *    is thread-local; the ee_profile_* instrumentation is process-global.
 *  - Device: the first call caches the current device's properties; use one
 *    device per process (the torchrun model).
 *  - Requires an sm_100a GPU (B200); on anything else ee_tune_step returns
 *    EE_ERR_UNSUPPORTED.  There is no CPU fallback.
 */
#ifndef EE_B200_H
#define EE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  EE_OK = 0,
  EE_ERR_ARG = 1,         /* NULL pointer / invalid enum / negative size          */
  EE_ERR_SHAPE = 2,       /* dimensions unsupported (see ee_head_config)          */
  EE_ERR_ALIGN = 3,       /* base pointer not 16-byte aligned                     */
  EE_ERR_VOCAB = 4,       /* target id outside [-1, V) (device-detected)          */
  EE_ERR_ARCH = 5,        /* tensors present/absent do not match the arch         */
  EE_ERR_STRUCTURE = 6,   /* Copy init: a source module is missing        */
  EE_ERR_DIVERGED = 7,    /* non-finite loss (device-detected, carries exit idx)  */
  EE_ERR_WORKSPACE = 8,   /* workspace NULL or smaller than ee_workspace_size()   */
  EE_ERR_CUDA = 9,        /* a CUDA runtime/driver call failed; device: a decode
                             stream-K fix-up wait timed out (ee_exit_infer)     */
  EE_ERR_NCCL = 10,       /* reserved for the in-library collectives              */
  EE_ERR_UNSUPPORTED = 11,/* no sm_100 device                                     */
  EE_ERR_PEER = 12        /* a peer rank did not reach ee_peer_barrier (device)    */
} ee_status;

/* Exit architectures (§2.1 "Architectures of early exits").
 * EMBEDDING: logits = x W_out^T
 * NORM:      logits = RMSNorm_f(x) W_out^T
 * MLP:       y = x + W_down(silu(W_gate u) * W_up u), u = RMSNorm_a(x);
 *            logits = RMSNorm_f(y) W_out^T   (pre-norm residual P:165-166;
 *            SwiGLU as in the Llama-2 backbone, reading A2)
 * LAYER:     "a complete Transformer layer, with the same structure as those
 *            on the backbone" in front of NORM: the Llama-2 layer
 *            x1 = x + W_o attn(RoPE(W_q u1), RoPE(W_k u1), W_v u1),
 *            u1 = RMSNorm_att(x), causal GQA attention within each sequence of
 *            seq_len tokens (head dim 128), then the MLP exit on x1.  Tokens
 *            couple within a sequence: n_tokens must be whole sequences. */
typedef enum {
  EE_ARCH_EMBEDDING = 0,
  EE_ARCH_NORM = 1,
  EE_ARCH_MLP = 2,
  EE_ARCH_LAYER = 3
} ee_arch;

/* Initialisation of exit parameters. */
typedef enum { EE_INIT_COPY = 0, EE_INIT_RANDOM = 1 } ee_init;

/* Token weights of the exit loss.
 * UNIFORM:    w_t = 1 for valid tokens; L_i = sum_t w_t loss_t / W  (A4).
 * CONFIDENCE: dynamic token-wise weights (App. B.3):
 *             w_t = c_t = max softmax probability of the exit at token t,
 *             detached (a constant in the backward); L_i = sum_t c_t loss_t /
 *             sum_t c_t (normalisation: DESIGN.md A17).  Needs all tokens of
 *             the batch in one call (ee_tune_step without valid_count, the
 *             ee_vp_* phases, or ee_tune_step with a communicator, which
 *             normalises by the global sum); a DP shard with valid_count
 *             returns EE_ERR_UNSUPPORTED.
 * CONFIDENCE_SUM: the same weights, normaliser left to the caller (data
 *             parallelism: sum_t c_t spans every rank's tokens): loss_out =
 *             sum_t c_t loss_t, grads = gradient of alpha sum_t c_t loss_t,
 *             ee_step_aux.weight_sum = sum_t c_t of this call.  The caller sums
 *             the three over ranks and calls ee_normalize_exit. */
/* How the backward obtains dS = dL/dS (a7; A24).
 * RECOMPUTE (default, north_star): a second GEMM recomputes each S tile from
 *   z and W_out and turns it into dS in the epilogue; the logits never reach
 *   HBM in any encoding (SURVEY §7 hard part 3: +2hV FLOPs per token).
 * STORED_P (ablation): the a5 epilogue also stores P~ = exp(S - tile max) as
 *   fp16 [n x V] and a7 is an elementwise pass over it; fewer FLOPs but the
 *   [tokens x vocab] probability matrix is written to HBM. */
typedef enum { EE_DS_RECOMPUTE = 0, EE_DS_STORED_P = 1 } ee_ds_mode;

typedef enum {
  EE_WEIGHT_UNIFORM = 0,
  EE_WEIGHT_CONFIDENCE = 1,
  EE_WEIGHT_CONFIDENCE_SUM = 2
} ee_token_weighting;

/* Element type of Copy-init source tensors. */
typedef enum { EE_DTYPE_BF16 = 0, EE_DTYPE_F32 = 1 } ee_dtype;

/* Shapes of one homogeneous set of exits (all exits share arch and sizes).
 *  hidden       h; multiple of 64, 64 <= h <= 8192.
 *  vocab        V (full vocabulary; targets are ids in [0, V)).
 *  ffn          F, MLP width; multiple of 128 for EE_ARCH_MLP, else ignored.
 *  num_exits    E >= 1.
 *  arch         ee_arch.
 *  norm_eps     RMSNorm epsilon (A3: 1e-5).
 *  vocab_begin, vocab_end
 *               the rows [vocab_begin, vocab_end) of W_out held by this call
 *               (a vocab-parallel shard, 0 <= begin < end <= V, width a
 *               multiple of 8).  ee_tune_step needs the full vocabulary
 *               [0, V) unless it runs with a vocab-parallel communicator
 *               (EE_COMM_VP); shards can also be driven through the ee_vp_*
 *               phases.
 *  token_weighting  ee_token_weighting.
 *  n_heads, n_kv_heads, seq_len, rope_theta
 *               LAYER only (ignored otherwise): query heads (hidden =
 *               n_heads * 128), key/value heads (divides n_heads; GQA),
 *               sequence length T (multiple of 64; token t of row r sits at
 *               position r % T), RoPE base (Llama-2: 10000).
 *  ds_mode      ee_ds_mode (0 = EE_DS_RECOMPUTE). */
typedef struct {
  int32_t hidden, vocab, ffn, num_exits;
  int32_t arch;
  float norm_eps;
  int32_t vocab_begin, vocab_end;
  int32_t token_weighting;
  int32_t n_heads, n_kv_heads, seq_len;
  float rope_theta;
  int32_t ds_mode;
} ee_head_config;

/* Parameters (or gradients, or optimizer moments) of ONE exit.  Device
 * pointers, NULL when the arch has no such tensor.
 *   g_a    [h]     pre-MLP RMSNorm gain       (MLP, LAYER)
 *   w_gate [F x h] SwiGLU gate projection     (MLP, LAYER)
 *   w_up   [F x h] SwiGLU up projection       (MLP, LAYER)
 *   w_down [h x F] down projection            (MLP, LAYER)
 *   g_f    [h]     final RMSNorm gain         (NORM, MLP, LAYER)
 *   w_out  [Vl x h] output embedding, Vl = vocab_end - vocab_begin (all archs);
 *                  the paper's "h x V" matrix stored transposed (A7).
 *   g_att  [h]       pre-attention RMSNorm gain   (LAYER)
 *   w_q    [h x h]   query projection             (LAYER)
 *   w_k    [hkv x h] key projection, hkv = 128 n_kv_heads (LAYER)
 *   w_v    [hkv x h] value projection             (LAYER)
 *   w_o    [h x h]   attention output projection  (LAYER)
 * Element types depend on the role of the struct:
 *   "operand" params: matrices bf16, gains fp32;
 *   master params, grads, Adam m/v: everything fp32. */
typedef struct {
  void *g_a, *w_gate, *w_up, *w_down, *g_f, *w_out;
  void *g_att, *w_q, *w_k, *w_v, *w_o;
} ee_head_tensors;

/* Optional per-token outputs of one exit (device, [n_tokens] each; any may be
 * NULL).  lse = log-sum-exp of the logits; loss_tok = lse - logit[target]
 * (0 for ignored tokens); argmax = lowest index of the max logit (A9);
 * conf = max softmax probability = 1/sum exp(S - max).
 * weight_sum (device float [1]) = the loss normaliser of this call: the valid
 * count W (UNIFORM) or sum_t c_t over valid tokens (CONFIDENCE*). */
typedef struct {
  float* lse;
  float* loss_tok;
  int32_t* argmax;
  float* conf;
  float* weight_sum;
} ee_step_aux;

/* Bytes of workspace ee_tune_step needs for n_tokens tokens with this config.
 * The same workspace may be reused by consecutive calls on the same stream. */
ee_status ee_workspace_size(const ee_head_config* cfg, int64_t n_tokens, size_t* bytes);

/* Stage-1 initialisation of all E exits.
 *   init = EE_INIT_COPY: copy_src[i] holds the backbone modules exit i copies
 *     (element type src_dtype, device): Embedding/Norm -> the final-exit
 *     layer's W_out (and final norm gain g_f); MLP -> the MLP of the
 *     layer the exit is attached to, and that layer's pre-MLP norm gain as g_a
 *     (A10), plus the final g_f and W_out; LAYER -> "the last Transformer
 *     layer of the original LLM" for every exit (attention tensors
 *     and MLP, its pre-MLP gain as g_a), plus g_f and W_out.  A NULL source tensor that
 *     the arch needs -> EE_ERR_STRUCTURE.  Copies are deep.
 *   init = EE_INIT_RANDOM: matrices ~ N(0, std^2) from a counter-based Philox
 *     stream keyed by (seed, exit, tensor); gains = 1 (A12).
 *     copy_src may be NULL.
 *   master_fp32[i]: fp32 master parameters (written).
 *   operand_bf16[i]: bf16 operand copies of the matrices (written); its gain
 *     pointers are fp32 and written too unless they alias the master gains. */
ee_status ee_init_heads(const ee_head_config* cfg, int32_t init, const ee_head_tensors* copy_src,
                        int32_t src_dtype, uint64_t seed, float std,
                        ee_head_tensors* master_fp32, ee_head_tensors* operand_bf16, void* stream);

/* In-library communicator (§2.2 "Support for 3D
 * parallelism").  Opaque; created once per rank by ee_comm_create
 * and passed to ee_tune_step, which then runs a whole data-parallel (DP) or
 * vocab-parallel (VP) step over the `world` ranks of a node in one call.
 * Every exchange is this library's own kernels over NVLink peer memory (CUDA
 * IPC mappings of each rank's symmetric ARENA): stores from the producing
 * GEMM epilogues / norm kernels, rank-ordered (deterministic) reductions of
 * the small vectors, and stream-ordered device barriers (ee_peer_barrier
 * semantics, ~20 s timeout -> EE_ERR_PEER).  No NCCL, no host sync.
 *
 * Setup (per rank, host calls):
 *   1. ee_comm_arena_size(cfg, mode, world, n_local, &bytes);
 *   2. allocate `bytes` of device memory, 256-byte aligned, ZERO-FILLED, and
 *      keep it alive as long as the comm;
 *   3. ee_ipc_get_handle(arena) and exchange the (handle, offset) pairs with
 *      the other ranks by any host transport (a TCP store, MPI, files);
 *      ee_ipc_open each peer's pair (one process per GPU; ranks sharing a
 *      process may pass the peers' device pointers directly);
 *   4. ee_comm_create(&comm, cfg, mode, world, rank, n_local, arenas, bytes)
 *      with arenas[q] = rank q's arena in this process (arenas[rank] = own).
 * Every rank must have completed step 4 before any rank's first step, and
 * all ranks must issue the same sequence of ee_tune_step(comm) calls.
 *
 * DP (EE_COMM_DP; cfg unsharded): hidden/targets are this rank's n_local
 *   tokens (Layer exits: whole sequences).  W = the global valid count
 *   (unless valid_count is given); the weight-gradient GEMM epilogues store
 *   each gradient row into its owner's arena (fused reduce-scatter), the owner
 *   sums the P slots in rank order and every rank gathers the reduced rows:
 *   grads[i] = the gradient over ALL ranks' tokens, bitwise identical on every
 *   rank; loss_out[i] = the global loss.  CONFIDENCE weighting normalises by
 *   the global sum_t c_t (A17).  aux: this rank's tokens.
 * VP (EE_COMM_VP; cfg->vocab_begin/end = this rank's W_out row shard):
 *   hidden/targets are this rank's n_local tokens; the library all-gathers
 *   the targets and z (in the a4 kernel's stores), runs the distributed
 *   softmax-CE (rank-ordered MAX of the (max, argmax) key, SUM of the
 *   rescaled sum-exp and target logit), stores dz rows into their owners'
 *   slots (a8 epilogue) and reduces the exit body's gradients as in DP.
 *   grads[i].w_out = this rank's shard; body grads identical on every rank;
 *   loss_out[i] = the global loss; aux arrays are [world * n_local] (all
 *   tokens).  The workspace must be sized for world * n_local tokens.
 * n_local is fixed at creation; accumulate adds the reduced gradients. */
typedef struct ee_comm ee_comm;
typedef enum { EE_COMM_DP = 0, EE_COMM_VP = 1 } ee_comm_mode;
ee_status ee_comm_arena_size(const ee_head_config* cfg, int32_t mode, int32_t world,
                             int64_t n_local, size_t* bytes);
ee_status ee_comm_create(ee_comm** comm, const ee_head_config* cfg, int32_t mode, int32_t world,
                         int32_t rank, int64_t n_local, void* const* arenas, size_t arena_bytes);
ee_status ee_comm_destroy(ee_comm* comm);

/* One EE-Tuning step over all exits: per exit i, forward of the
 * exit head on hidden[i], softmax cross-entropy against `targets`, and the
 * gradient of exit_weights[i] * L_i w.r.t. the exit's parameters only (the
 * backbone is frozen: no gradient w.r.t. hidden).  Exits are
 * independent.
 *   hidden[i]      device bf16 [n_tokens x h], read-only.
 *   n_tokens       tokens on this rank (N = batch * seq flattened), >= 0;
 *                  LAYER: a multiple of seq_len (whole sequences).
 *   targets        device int32 [n_tokens], next-token ids; -1 = ignore.
 *   exit_weights   host float [E], alpha_i (A5).
 *   params[i]      operand parameters (matrices bf16, gains fp32), read-only.
 *   grads[i]       fp32 gradients, written (accumulate = 0) or added to (1).
 *   loss_out       device float [E]: sum_t w_t loss_t / W (unweighted by
 *                  alpha), i.e. the mean loss over valid tokens on one GPU.
 *   aux            NULL or host array of E ee_step_aux (device buffers).
 *   valid_count    NULL, or device int64 [1] holding W, the GLOBAL number of
 *                  valid tokens (data parallelism, A16).  NULL = count the
 *                  local targets.
 *   workspace      device scratch of ws_bytes >= ee_workspace_size().
 *   comm           NULL = one GPU; else the DP / VP step over the ranks of
 *                  the communicator (ee_comm_create above).
 * Device-detected errors: a target outside [-1, V) -> EE_ERR_VOCAB; a
 * non-finite loss -> EE_ERR_DIVERGED with the exit index (ee_get_status). */
ee_status ee_tune_step(const ee_head_config* cfg, const void* const* hidden, int64_t n_tokens,
                       const int32_t* targets, const float* exit_weights,
                       const ee_head_tensors* params, ee_head_tensors* grads, int32_t accumulate,
                       float* loss_out, const ee_step_aux* aux, const int64_t* valid_count,
                       void* workspace, size_t ws_bytes, const ee_comm* comm, void* stream);

/* Data-parallel confidence weighting (EE_WEIGHT_CONFIDENCE_SUM): after the
 * caller has summed one exit's grads, its loss and weight_sum over the ranks,
 * divide the exit's fp32 gradients (grads: ONE exit, or NULL: the loss only --
 * the sharded DP path divides inside ee_adam_update_sharded) and *loss
 * (device, may be NULL) by *weight_sum (device scalar; <= 0 -> zeros).
 * P:326-336, A17. */
ee_status ee_normalize_exit(const ee_head_config* cfg, ee_head_tensors* grads, float* loss,
                            const float* weight_sum, void* stream);

/* ---- vocab-parallel phases (one exit on one of P ranks) ----
 * W_out is split by rows over P ranks (cfg->vocab_begin/vocab_end = this rank's
 * shard); tokens are split over ranks for the exit body (RMSNorm/MLP) and
 * gathered for the vocab projection.  The caller runs the collectives between
 * the phases, in this order, for each exit i:
 *   1. ee_vp_exit_forward   (a1-a4 on the rank's n_local tokens) -> z_out, which
 *                           should be this rank's slot of z_all [n_all x h] bf16
 *      all-gather z_all
 *   2. ee_vp_vocab_stats    (a5 on the local W_out shard for all n_all tokens)
 *                           -> key [n_all] int64, sums [n_all x 2] fp32
 *      all-reduce MAX (signed int64) on key  -> global row max + lowest argmax
 *   3. ee_vp_rescale        sums[:,0] *= exp(m_local - m_global)
 *      all-reduce SUM on sums                -> global sum-exp, target logit
 *   4. ee_vp_vocab_backward (lse, loss, dS on the shard; dW_out shard = dS^T z_all
 *                           needs no reduction; dz_partial [n_all x h] fp32 =
 *                           dS W_out_shard, NULL for Embedding exits)
 *      reduce-scatter SUM dz_partial -> dz_local [n_local x h]
 *   5. ee_vp_exit_backward  (a10-a13 on local tokens: g_f and MLP grads)
 *      all-reduce SUM of the exit's g_f / MLP gradients (W_out grads stay sharded)
 * The distributed softmax-CE is steps 2-3 (max + argmax key, sum-exp and target
 * logit), the paper's "vocab-parallel" reading of Megatron TP.
 * The workspace must be sized by ee_workspace_size(cfg, n_all) and is shared by
 * the five phases of one exit; exits are processed one after another.
 * loss_out (one float) = sum over ALL tokens of w_t loss_t / W, identical on
 * every rank.  valid_count = W over all tokens (NULL: count targets_all). */
ee_status ee_vp_exit_forward(const ee_head_config* cfg, const void* hidden, int64_t n_local,
                             int64_t n_all, const ee_head_tensors* params, void* z_out,
                             void* workspace, size_t ws_bytes, void* stream);
ee_status ee_vp_vocab_stats(const ee_head_config* cfg, const void* z_all, int64_t n_all,
                            const int32_t* targets_all, const ee_head_tensors* params,
                            int64_t* key_out, float* sums_out, void* workspace, size_t ws_bytes,
                            void* stream);
ee_status ee_vp_rescale(const ee_head_config* cfg, int64_t n_all, const int64_t* key_global,
                        float* sums, void* workspace, size_t ws_bytes, void* stream);
ee_status ee_vp_vocab_backward(const ee_head_config* cfg, const void* z_all, int64_t n_all,
                               const int32_t* targets_all, const int64_t* key_global,
                               const float* sums_global, float exit_weight,
                               const int64_t* valid_count, const ee_head_tensors* params,
                               ee_head_tensors* grads, int32_t accumulate, float* dz_partial,
                               float* loss_out, const ee_step_aux* aux, int32_t exit_index,
                               void* workspace, size_t ws_bytes, void* stream);
ee_status ee_vp_exit_backward(const ee_head_config* cfg, const void* hidden, int64_t n_local,
                              int64_t n_all, const ee_head_tensors* params, const float* dz_local,
                              ee_head_tensors* grads, int32_t accumulate, void* workspace,
                              size_t ws_bytes, void* stream);

/* ---- fused vocab-parallel collectives over peer memory ("fused
 * variants") ----
 * The all-gather of z (after step 1) and the reduce-scatter of dz (after step
 * 4) above move 0.94 GB and 1.88 GB per exit at the 70B shape.  These calls do
 * both inside the producing kernels over NVLink peer memory instead:
 *  - ee_vp_exit_forward_ag: the a4 RMSNorm kernel stores each z row into EVERY
 *    rank's z_all (row rank*n_local + t) -- the all-gather is the kernel's own
 *    stores (Embedding exits: z = x, copied to every rank).
 *  - ee_vp_vocab_backward_rs: as ee_vp_vocab_backward, but the a8 GEMM epilogue
 *    routes row m of this rank's dz partial to the token owner q = m / n_local,
 *    into q's slot buffer at [rank][m - q*n_local][0..h) (no dz_partial).
 *  - ee_vp_exit_backward_slots: as ee_vp_exit_backward with dz_local replaced
 *    by the rank's own slot buffer [n_slots][n_local][h] fp32; the a10 kernel
 *    sums the slots in rank order 0..n_slots-1 (deterministic reduce, fused
 *    into its loads).
 *  - ee_peer_barrier: stream-ordered barrier over all ranks through a signal
 *    array (int32 [EE_MAX_PEERS] per rank): rank r stores `epoch` into slot r
 *    of every rank's array (st.release.sys) and waits until its own array
 *    holds >= epoch in all `world` slots (ld.acquire.sys).  epoch must grow by
 *    one per call.  Required: after each fused all-gather (before step 2),
 *    after each fused reduce-scatter (before step 5), and once per step before
 *    the first exit (the previous step's readers of z_all / slots).  A peer
 *    that does not arrive within ~20 s sets the status word to EE_ERR_PEER
 *    (read it with ee_get_status) instead of hanging.
 * Equal token shards are required (n_all = world * n_local).  Peer pointers
 * (ee_peer_set.ptr[q] = rank q's buffer, mapped into this process; ptr[rank]
 * is the local buffer) come from ee_ipc_get_handle / ee_ipc_open (CUDA IPC,
 * one process per GPU) or, in single-process tests, are plain device
 * buffers.  Results equal the NCCL path's bit for bit except the order of the
 * dz sum (rank order here). */
#define EE_MAX_PEERS 8
typedef struct {
  int32_t rank, world;            /* this rank; number of ranks (1..EE_MAX_PEERS) */
  void* ptr[EE_MAX_PEERS];        /* device pointers valid in this process */
} ee_peer_set;

ee_status ee_vp_exit_forward_ag(const ee_head_config* cfg, const void* hidden, int64_t n_local,
                                int64_t n_all, const ee_head_tensors* params,
                                const ee_peer_set* z_all, void* workspace, size_t ws_bytes,
                                void* stream);
ee_status ee_vp_vocab_backward_rs(const ee_head_config* cfg, const void* z_all, int64_t n_all,
                                  const int32_t* targets_all, const int64_t* key_global,
                                  const float* sums_global, float exit_weight,
                                  const int64_t* valid_count, const ee_head_tensors* params,
                                  ee_head_tensors* grads, int32_t accumulate,
                                  const ee_peer_set* dz_slots, float* loss_out,
                                  const ee_step_aux* aux, int32_t exit_index, void* workspace,
                                  size_t ws_bytes, void* stream);
/* grad_arenas (NULL: gradients into `grads`): the exit body's gradients are
 * routed to their owners' arenas as in ee_tune_step_rs (layout of
 * ee_dp_shard_layout for this cfg; the W_out block is left untouched), for a
 * sharded update of the replicated exit body (ee_adam_update_sharded with a
 * tensor_mask without W_out); accumulate must be 0. */
ee_status ee_vp_exit_backward_slots(const ee_head_config* cfg, const void* hidden,
                                    int64_t n_local, int64_t n_all,
                                    const ee_head_tensors* params, const float* dz_slots,
                                    int32_t n_slots, ee_head_tensors* grads, int32_t accumulate,
                                    const ee_peer_set* grad_arenas, void* workspace,
                                    size_t ws_bytes, void* stream);
ee_status ee_peer_barrier(const ee_peer_set* signals, uint32_t epoch, void* workspace,
                          void* stream);
/* CUDA IPC plumbing for ee_peer_set (host calls, not stream-ordered).
 * ee_ipc_get_handle: 64-byte handle of the allocation containing dev_ptr and
 * the byte offset of dev_ptr inside it.  ee_ipc_open (in another process on
 * any GPU of the node with peer access): maps the allocation and returns
 * base + offset.  ee_ipc_close: unmaps a pointer returned by ee_ipc_open. */
/* ---- data parallel over tokens with the gradient reduce-scatter fused into
 * the weight-gradient GEMMs and a sharded Adam (ZeRO-1) ----
 * The exits' gradients are summed over the P ranks' token shards (the
 * loss is a sum over independent tokens; A16: normalised by the global W).
 * Instead of an all-reduce of full fp32 gradients followed by Adam on every
 * rank, each tensor is split into row blocks of chunk = ceil(R/P) rows (R =
 * rows of the [R x C] tensor; gains are one row of h, owned by rank 0), and
 *  - ee_tune_step_rs: as ee_tune_step (accumulate = 0), but the weight-gradient
 *    GEMM epilogues (a9 dW_out, a11 dW_down, a12 dW_gate|up) and the gain
 *    reductions store each gradient row into its OWNER's arena, slot [rank]
 *    (NVLink stores), instead of a local gradient tensor;
 *  - ee_adam_update_sharded: on each rank, for the rows it owns: g = sum of
 *    the P slots in rank order, Adam on the fp32 master / moment shards, and
 *    the new bf16 operand rows (fp32 for gains) stored into EVERY rank's
 *    operand tensor (the all-gather).
 * Arena of rank q (fp32, one per exit in flight): for each tensor k needed by
 * the arch, in ee_head_tensors order, a block [P][rows_q(k) x C_k] (slot r =
 * rank r's partial); ee_dp_shard_layout gives row_begin / rows of rank's shard
 * of tensor k, the float offset of its block and the arena's total floats.
 * grad_arenas[i] (ee_tune_step_rs): every rank's arena for exit i;
 * grad_arenas[i] (ee_adam_update_sharded): this rank's arena (device ptr);
 * operands[i * 11 + k]: every rank's operand tensor k of exit i (world
 * entries; ignored for tensors the arch lacks).  Barriers (ee_peer_barrier):
 * after the last ee_tune_step_rs writing an arena and before the Adam reading
 * it; before a step's first forward (operand all-gather of the previous
 * update complete); and before an arena is written again (2 arenas
 * alternating exits need no extra barrier).  Results are bitwise equal to
 * ee_tune_step + a rank-ordered fp32 all-reduce + ee_adam_update.
 * Under a vocab shard (cfg->vocab_begin/end not [0, V): vocab-parallel), W_out
 * has no arena block (it is never reduced and its row count differs between
 * ranks); ee_adam_update_sharded then never updates W_out.
 * grad_divisor (device float [E] or NULL): exit i's summed gradient is
 * multiplied by 1/grad_divisor[i] (0 if <= 0) before Adam -- dynamic token
 * weights under DP: ee_tune_step_rs with EE_WEIGHT_CONFIDENCE_SUM, the
 * weight sums all-reduced by the caller, the losses divided with
 * ee_normalize_exit(cfg, NULL, loss, weight_sum) (grads may be NULL there).
 * tensor_mask: bit k (ee_head_tensors order: g_a 0, w_gate 1, w_up 2,
 * w_down 3, g_f 4, w_out 5, g_att 6, w_q 7, w_k 8, w_v 9, w_o 10) selects the
 * tensors ee_adam_update_sharded updates; 0 = all.
 * Uniform token weights; every arch (Layer: also W_q, W_k, W_v, W_o, g_att).
 * Ranks sharing one process (tests): CUDA loads kernels lazily and a load
 * waits for the context's running kernels, so one rank's first launch of a
 * kernel can wait on another rank's spinning barrier; run one world-1 step
 * first (or CUDA_MODULE_LOADING=EAGER).  One process per GPU is unaffected. */
ee_status ee_dp_shard_layout(const ee_head_config* cfg, int32_t world, int32_t rank,
                             int32_t tensor, int64_t* row_begin, int64_t* rows,
                             int64_t* arena_offset_floats, int64_t* arena_total_floats);
ee_status ee_tune_step_rs(const ee_head_config* cfg, const void* const* hidden, int64_t n_tokens,
                          const int32_t* targets, const float* exit_weights,
                          const ee_head_tensors* params, const ee_peer_set* grad_arenas,
                          float* loss_out, const ee_step_aux* aux, const int64_t* valid_count,
                          void* workspace, size_t ws_bytes, void* stream);
ee_status ee_adam_update_sharded(const ee_head_config* cfg, int32_t world, int32_t rank,
                                 const void* const* grad_arenas, ee_head_tensors* master_shard,
                                 ee_head_tensors* m_shard, ee_head_tensors* v_shard,
                                 const ee_peer_set* operands, float lr, float beta1, float beta2,
                                 float eps, float weight_decay, int64_t step, float grad_scale,
                                 uint32_t tensor_mask, const float* grad_divisor, void* stream);

ee_status ee_ipc_get_handle(const void* dev_ptr, void* handle64, uint64_t* offset);
ee_status ee_ipc_open(const void* handle64, uint64_t offset, void** dev_ptr);
ee_status ee_ipc_close(void* dev_ptr, uint64_t offset);

/* Early-exit inference statistics (§3 "Inference"): for
 * each exit i and token t, the exit's greedy next token argmax_out[i][t]
 * (lowest index on ties) and its confidence conf_out[i][t] = max softmax
 * probability; first_exit[t] (may be NULL) = the lowest exit index whose
 * confidence reaches `threshold`, or -1 (threshold 1 disables early exits,
 * P:385).  hidden[i]: device bf16 [n_tokens x h]; outputs device [n_tokens].
 * n_tokens > 16 (or Layer exits): the tuning step's forward kernels (a1-a6).
 * n_tokens <= 16 (decode): weight-streaming "skinny" kernels (TMA-fed
 * shared-memory ring, warp-level bf16 MMA, stream-K over one persistent CTA
 * per SM, fused SwiGLU / residual / per-block online-softmax statistics,
 * programmatic dependent launch) and a wide finalize; same results up to fp32
 * summation order, bitwise reproducible call to call.  No loss, no gradients.
 * The stream-K fix-up uses a library-global pool of 16 slots: at most 16
 * decode calls may EXECUTE concurrently (calls on one stream never overlap);
 * a fix-up wait bounded at 5 s reports EE_ERR_CUDA through ee_get_status.
 * Env EE_INFER_SKINNY=0 forces the GEMM path, EE_PDL=0 plain launches. */
ee_status ee_exit_infer(const ee_head_config* cfg, const void* const* hidden, int64_t n_tokens,
                        const ee_head_tensors* params, float threshold, int32_t* const* argmax_out,
                        float* const* conf_out, int32_t* first_exit, void* workspace,
                        size_t ws_bytes, void* stream);

/* ---- frozen backbone partial forward (NEXT #3) ----
 * "the partial forward pass of the Transformer backbone up to the hidden
 * states connected to the last early exit": Llama-2 pre-norm decoder
 * layers (residual + pre-normalisation), RoPE
 * (rotate-half, base rope_theta), causal GQA attention within sequences of
 * seq_len rows, SwiGLU MLP.  Produces the exits' cached hidden states.
 *  hidden      h = n_heads * 128 (head dim 128, as in every Llama-2 size)
 *  n_kv_heads  divides n_heads (GQA; = n_heads for MHA)
 *  ffn         multiple of 128;  seq_len multiple of 64;  n_tokens multiple
 *              of seq_len (row = sequence * seq_len + position).
 * Layer tensors: gains fp32 [h]; w_q [h x h], w_k, w_v [n_kv*128 x h],
 * w_o [h x h], w_gate, w_up [F x h], w_down [h x F] bf16, row-major.
 * The residual stream is kept in fp32; hidden_out[i] (bf16 [n_tokens x h])
 * receives it after layer exit_after[i] (1-based, ascending); only layers
 * 1..exit_after[num_exits-1] run.  x0: bf16 [n_tokens x h] (the embeddings). */
typedef struct {
  int32_t hidden, n_heads, n_kv_heads, ffn, seq_len;
  float norm_eps, rope_theta;
} ee_backbone_config;
typedef struct {
  void *g_att, *w_q, *w_k, *w_v, *w_o, *g_mlp, *w_gate, *w_up, *w_down;
} ee_layer_tensors;
ee_status ee_backbone_workspace_size(const ee_backbone_config* cfg, int64_t n_tokens, size_t* bytes);
ee_status ee_backbone_forward(const ee_backbone_config* cfg, const ee_layer_tensors* layers,
                              int32_t n_layers, const void* x0, int64_t n_tokens,
                              const int32_t* exit_after, int32_t num_exits,
                              void* const* hidden_out, void* workspace, size_t ws_bytes,
                              void* stream);

/* Number of valid targets (!= -1) -> device int64 out[0]; flags ids outside
 * [-1, V) in the workspace status word.  Used to form the global W under
 * data parallelism (the caller all-reduces out). */
ee_status ee_count_valid(const int32_t* targets, int64_t n_tokens, int32_t vocab, int64_t* out,
                         void* workspace, size_t ws_bytes, void* stream);

/* Adam (Kingma bias correction, eps outside the sqrt, A14) on every
 * tensor present in master[i], for all E exits, elementwise:
 *   g = grad_scale*grad; m = b1 m + (1-b1) g; v = b2 v + (1-b2) g^2;
 *   theta -= lr * (m/(1-b1^t)) / (sqrt(v/(1-b2^t)) + eps) + lr*wd*theta;
 * then operand[i] <- bf16(theta) for matrices (and fp32 gains unless aliased).
 * step = t >= 1.  master, m, v updated in place. */
ee_status ee_adam_update(const ee_head_config* cfg, ee_head_tensors* master,
                         ee_head_tensors* operand_bf16, const ee_head_tensors* grads,
                         ee_head_tensors* m, ee_head_tensors* v, float lr, float beta1,
                         float beta2, float eps, float weight_decay, int64_t step,
                         float grad_scale, void* stream);

/* One tuning step with the Adam update fused into the weight-gradient GEMM
 * epilogues: "forward computation, backward computation, and parameter update
 * for each early-exit layer, without any dependency between early exits"
 * (P:261).  Same as ee_tune_step (accumulate = 0) followed by ee_adam_update
 * with the same arguments, bit for bit, but the matrix gradients are never
 * stored: when a dW_out / dW_down / dW_gate|up tile is final, the epilogue
 * applies Adam to master/m/v at those elements and stores the bf16 operand
 * (the backward GEMMs that read a weight run before the one that updates it).
 * The gains' column-sum gradients go through the workspace and a small Adam.
 * One GPU (the whole gradient is local); every arch (Layer: W_o before L6 and
 * W_q/k/v before L10 are read first); uniform or CONFIDENCE token weights;
 * n_tokens > 0.  operand/master/m/v as in
 * ee_adam_update, [E] each. */
ee_status ee_tune_step_adam(const ee_head_config* cfg, const void* const* hidden,
                            int64_t n_tokens, const int32_t* targets, const float* exit_weights,
                            ee_head_tensors* operand, ee_head_tensors* master, ee_head_tensors* m,
                            ee_head_tensors* v, float lr, float beta1, float beta2, float eps,
                            float weight_decay, int64_t step, float grad_scale, float* loss_out,
                            const ee_step_aux* aux, const int64_t* valid_count, void* workspace,
                            size_t ws_bytes, void* stream);

/* SGD: buf = momentum*buf + g (buf may be NULL iff momentum == 0);
 * theta -= lr * buf; operand refreshed as for Adam. */
ee_status ee_sgd_update(const ee_head_config* cfg, ee_head_tensors* master,
                        ee_head_tensors* operand_bf16, const ee_head_tensors* grads,
                        ee_head_tensors* momentum_buf, float lr, float momentum,
                        float grad_scale, void* stream);

/* Reads (and clears) the device status word in `workspace`; synchronises the
 * stream.  code = EE_OK or the first device error; exit_index = the exit it
 * concerns (-1 if none). */
ee_status ee_get_status(void* workspace, void* stream, int32_t* code, int32_t* exit_index);

/* Learning rate at iteration `iter` of `total` (A14): linear ramp
 * 0 -> lr_max over ceil(warmup_frac*total) iterations, then linear decay to
 * lr_min at `total`.  Pure host function; returns NaN if iter is outside
 * [0, total]. */
double ee_lr_at(int64_t iter, int64_t total, double warmup_frac, double lr_max, double lr_min);

/* Thread-local description of the last non-OK status returned on this thread. */
const char* ee_last_error(void);

/* Library version string. */
const char* ee_version(void);

/* ---- instrumentation (process-global; used by bench.py) ----
 * Between ee_profile_start() and ee_profile_stop(), every kernel launch the
 * library makes is bracketed by a CUDA event pair on its stream.
 * ee_profile_record(i, ...) returns launch i's name (copied into name[0..len)),
 * its device duration in ms (synchronises that event), and its executed FLOPs,
 * algorithmic FLOPs (the recompute GEMM counts 0) and algorithmic HBM bytes.
 * ee_launch_count() = total kernel launches made by the library so far. */
ee_status ee_profile_start(void);
ee_status ee_profile_stop(int32_t* count);
ee_status ee_profile_record(int32_t i, char* name, int32_t name_len, float* ms, double* flops_exec,
                            double* flops_alg, double* bytes);
int64_t ee_launch_count(void);

/* ---- testing hook (used by the GPU parity tests; not part of the step) ----
 * C[M x N] (fp32 row-major, device) = A B^T  (or += if accumulate), where the
 * bf16 device operands are stored A: [M x K] if a_kmajor else [K x M];
 * B: [N x K] if b_kmajor else [K x N].  Runs the same tcgen05 kernel as the
 * step's plain-fp32 GEMMs.  K, and M (N) when MN-major, must be multiples of
 * 8; N a multiple of 4. */
ee_status ee_test_gemm(int32_t a_kmajor, int32_t b_kmajor, const void* A, const void* B, float* C,
                       int32_t M, int32_t N, int32_t K, int32_t accumulate, void* stream);

/* ---- testing hook: the causal GQA attention kernels of the backbone / the
 * Layer exit (Llama-2 attention; head dim 128).  q [n x Hq*128],
 * k, v [n x Hkv*128], o [n x Hq*128] bf16 row-major (row = sequence * T + t,
 * no RoPE applied here); lse2 [n x Hq] fp32 out = log2-domain row statistics
 * (max + log2 sum of 2^(s/sqrt(d) * log2 e)).  If dout != NULL the backward
 * also runs: dq, dk, dv (shapes of q, k, v, bf16) and scratch fp32 [n x Hq].
 * seq_len a multiple of 64 dividing n; n_heads a multiple of n_kv_heads.
 * impl selects the forward and backward kernels: 0 = warp-level mma.sync,
 * 1 = tcgen05/TMEM with one query tile per CTA, 2 = tcgen05/TMEM with two
 * ping-ponged query tiles per CTA (the step's default forward); the backward
 * is tcgen05 for 1 and 2. */
ee_status ee_test_attention(const void* q, const void* k, const void* v, void* o, float* lse2,
                            const void* dout, void* dq, void* dk, void* dv, float* scratch,
                            int64_t n_tokens, int32_t seq_len, int32_t n_heads, int32_t n_kv_heads,
                            int32_t impl, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* EE_B200_H */
