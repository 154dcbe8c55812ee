/*
 * swiftspec.h -- C-ABI of the B200-native tensor-parallel tree-verification
 * step of SwiftSpec (arXiv 2506.11309).
 *
 * Citations: P:n = PAPER.md line n; S:n = SPEC.md line n (interfaces only);
 * Rn = reading n in DESIGN.md "Readings of the paper".
 *
 * The operation (Alg. 1 target branch P:288-298): the target worker
 * "gets the draft tokens from the draft tree and runs batch inferences to
 * calculate the logits. After that, it samples through the logits to generate
 * the tokens one by one and then sends the verified tokens back".  One call of
 * ss_verify_tree runs a T-node token tree (root first, parents[i] < i)
 * through an int4-AWQ group-128 Llama decoder sharded over tp_size
 * GPUs, with the square ancestor mask, the two
 * tensor-parallel all-reduces per layer fused into the O / down projection
 * epilogues, greedy acceptance (R6) and -- via
 * ss_commit_kv / ss_commit_accepted -- KV compaction of the accepted path.
 *
 * Conventions
 *  - Every function returns an ss_status; on a host-detected error nothing
 *    was launched and the shard state is unchanged; ss_last_error(shard)
 *    gives that shard's last message (ss_last_error(NULL): the calling
 *    thread's last message, e.g. after a failed ss_init_shard).
 *  - Call order: a verify without auto-commit leaves the tree
 *    rows pending; the next verify on the shard is refused with SS_ESTATE
 *    until they are committed (ss_commit_kv / ss_commit_accepted) or
 *    discarded (ss_set_committed_len).  Checks run in the order SS_EINVAL,
 *    SS_ESTATE, SS_ECAPACITY.
 *  - Collective semantics (NCCL-style): every rank of a TP group calls
 *    ss_verify_tree* / ss_commit_* with identical arguments, in the same order.
 *  - Ownership: the library owns every device allocation it makes (weights in
 *    kernel layout, KV cache, workspaces, peer buffers).  Host inputs are
 *    caller-owned and fully consumed before the call returns.  Device inputs
 *    of the *_dev variants are caller-owned and must stay valid until the
 *    stream reaches the enqueued work.
 *  - Streams are cudaStream_t passed as void* (NULL = legacy default stream).
 *  - No torch types appear here; the Python binding only marshals arguments.
 */
#ifndef SWIFTSPEC_H
#define SWIFTSPEC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SS_MAX_TREE 64   /* maximum T (tree nodes) per verify call */
#define SS_GROUP 128     /* AWQ group size */

typedef enum {
  SS_OK = 0,
  SS_EINVAL = -1,        /* bad argument: tree not root-first/topological, T out of range,
                            token out of vocab, chain not root-anchored, bad shape/kind/bytes */
  SS_ECAPACITY = -2,     /* L + T > max_ctx (no eviction) */
  SS_ECONSISTENCY = -3,  /* TP ranks were called with different trees (SS_DEBUG_CONSISTENCY checksum) */
  SS_ECUDA = -4,         /* a CUDA runtime error; message has cudaGetErrorString */
  SS_ETIMEOUT = -5,      /* a peer flag poll exceeded its budget */
  SS_ESTATE = -6         /* call order violated (commit without a verify, weights missing, ...) */
} ss_status;

/* Model shape (public Llama3 configs, R1).  head_dim must be 64 or 128;
 * hidden, n_heads*head_dim/tp and intermediate/tp must be multiples of 256;
 * n_kv_heads and intermediate must be divisible by tp_size. */
typedef struct {
  int32_t n_layers, hidden, intermediate, n_heads, n_kv_heads, head_dim, vocab;
  int32_t group_size;  /* must be 128 */
  int32_t max_ctx;     /* KV capacity per layer and kv head, committed + tree rows */
  int32_t max_tree;    /* largest T this shard will be called with, <= SS_MAX_TREE */
  float rms_eps;       /* 1e-5 (R1) */
  float rope_theta;    /* 500000 (R1) */
} ss_model_cfg;

typedef struct ss_shard ss_shard;

/* Result of one verify step (Fig. 4).
 *  n_accepted  = number of tree nodes on the accepted path INCLUDING the root
 *                (>= 1); these are the rows ss_commit_accepted commits (R9).
 *  accepted[k] = tree-node index of the k-th path node (accepted[0] == 0).
 *  bonus_token = the target's greedy token after the last accepted node; it is
 *                emitted but not committed (it is the next call's root, R9).
 *  argmax[i]   = the target's greedy token at tree node i (ties -> lowest id).
 *  status      = device-side result of the step: SS_OK, SS_EINVAL (tree
 *                invalid, e.g. a mailbox tree larger than the graph's
 *                capacity), SS_ETIMEOUT (a peer / inbox poll ran out of
 *                budget) or SS_ECONSISTENCY (ranks disagree, debug
 *                mode).  A step whose status is not SS_OK is never committed. */
typedef struct {
  int32_t n_accepted;
  int32_t accepted[SS_MAX_TREE];
  int32_t bonus_token;
  int32_t argmax[SS_MAX_TREE];
  int32_t status;
} ss_verify_result;

/* Weight kinds for ss_load_weights.  Linear layers W map x -> x @ W with
 * K = in-features, N = out-features (int4 AWQ g128, BF16 compute).
 * The caller passes the FULL unsharded canonical tensor; the library slices
 * its tensor-parallel shard (QKV / gate / up column-parallel by heads / I,
 * O / down row-parallel, LM head vocab-parallel, embedding replicated) and
 * repacks it into the kernel layout. */
typedef enum {
  SS_W_EMBED = 0,       /* uint16 bf16 bits [vocab][hidden]                       */
  SS_W_ATTN_NORM = 1,   /* uint16 bf16 bits [hidden]                               */
  SS_W_Q = 2,           /* linear, K = hidden, N = n_heads*head_dim                */
  SS_W_K = 3,           /* linear, K = hidden, N = n_kv_heads*head_dim             */
  SS_W_V = 4,           /* linear, K = hidden, N = n_kv_heads*head_dim             */
  SS_W_O = 5,           /* linear, K = n_heads*head_dim, N = hidden                */
  SS_W_MLP_NORM = 6,    /* uint16 bf16 bits [hidden]                               */
  SS_W_GATE = 7,        /* linear, K = hidden, N = intermediate                    */
  SS_W_UP = 8,          /* linear, K = hidden, N = intermediate                    */
  SS_W_DOWN = 9,        /* linear, K = intermediate, N = hidden                    */
  SS_W_FINAL_NORM = 10, /* uint16 bf16 bits [hidden]                               */
  SS_W_LM_HEAD = 11     /* uint16 bf16 bits [vocab][hidden]                        */
} ss_weight_kind;

/* Sub-tensors of a linear kind (the `sub` argument). */
typedef enum {
  SS_SUB_QWEIGHT = 0,   /* uint8 [K][N], one nibble value 0..15 per byte           */
  SS_SUB_QZEROS = 1,    /* uint8 [K/128][N], values 0..15                          */
  SS_SUB_SCALES = 2,    /* uint16 bf16 bits [K/128][N]                              */
  SS_SUB_DENSE = 0      /* for non-linear kinds                                     */
} ss_weight_sub;

/* ---- lifecycle ---------------------------------------------------------- */

/* Create the shard of TP rank tp_rank (0 <= tp_rank < tp_size, tp_size in
 * [1, 8]) on CUDA device `device`: allocates weights, the KV cache
 * [n_layers][ceil(n_kv_heads/tp)][max_ctx][head_dim] (fp16), workspaces and
 * the peer receive buffers.  *out receives the handle (owned by the caller,
 * free with ss_destroy).
 * Arbitrary TP: when tp_size does not divide n_kv_heads, the kv
 * heads (each with its n_heads/n_kv_heads query heads) are zero-padded to a
 * multiple of tp_size; when intermediate/tp_size is not a multiple of 256 the
 * intermediate size is zero-padded to a multiple of 256 tp_size.  Padded
 * weights and prefix K/V are zero (the loaders and generators fill them), so
 * results equal the unpadded model's; padded kv heads read back as zeros.
 * Errors: SS_EINVAL (shape rules above; padded n_heads*head_dim/tp must be a
 * multiple of 256), SS_ECUDA. */
ss_status ss_init_shard(const ss_model_cfg* cfg, int32_t tp_rank, int32_t tp_size,
                        int32_t device, ss_shard** out);

/* Peer setup for tp_size > 1 ("GPUs computing the same model are
 * connected tightly using NVLink"; P:413-420 fused all-reduce).
 * ss_export_handle writes this rank's cudaIpc handle blob (<= 4096 bytes) to
 * buf and its length to *len.  ss_import_peers takes all tp_size blobs in
 * rank order (own blob included) and maps the peers' receive buffers.
 * ss_import_local_peers is the single-process variant ("fake-peer" mode, or
 * one process driving several GPUs): it takes the other shard handles
 * directly.  Must be called before the first verify when tp_size > 1. */
ss_status ss_export_handle(ss_shard* s, void* buf, size_t* len);
ss_status ss_import_peers(ss_shard* s, const void* const* blobs, const size_t* lens);
ss_status ss_import_local_peers(ss_shard* s, ss_shard* const* shards);
/* Timing emulation of one rank of a tp_size group on a single GPU: the
 * fused all-reduce and the argmax exchange write this rank's partial into
 * every rank slot of its own receive buffer, so a rank's full step (its
 * weight shard, its KV heads, the LL traffic volume per step) runs without
 * peers.  Results are NOT the sharded model's (the sum is tp_size x this
 * rank's partial); bench.py --tp-emulate uses it to report per-GPU step
 * latency at TP 2/4/8 shapes on one B200.  Errors: SS_EINVAL if tp_size < 2. */
ss_status ss_import_loopback(ss_shard* s);

/* Launch-resource cap (fake-peer mode: several ranks share one GPU and every
 * rank's persistent kernels must be co-resident).  max_ctas_per_kernel <= 0
 * restores the default (all SMs). */
ss_status ss_set_launch_cap(ss_shard* s, int32_t max_ctas_per_kernel);

ss_status ss_destroy(ss_shard* s);
/* Last error message of shard s (s != NULL) or of the calling thread (s ==
 * NULL).  The pointer stays valid until the next failing call. */
const char* ss_last_error(const ss_shard* s);

/* Debug flags (SURVEY 8(b) "a debug mode checksums the arguments across
 * ranks"): with SS_DEBUG_CONSISTENCY every verify exchanges a checksum of
 * (T, tokens, parents) between the TP ranks over the peer buffers (one LL
 * round trip) and fails the step with result.status = SS_ECONSISTENCY on
 * every rank if any two disagree.  Set it identically on all ranks.
 * Errors: SS_EINVAL (unknown flag). */
#define SS_DEBUG_CONSISTENCY 1
/* SS_DEBUG_DETERMINISTIC: bit-identical results run to run (the
 * stream-K float reductions make logits vary by ~1e-3 between runs).  The
 * persistent step kernel (T <= 32) then gives every GEMM tile-group to one CTA
 * (no cross-CTA split-K: each accumulator element gets at most two flushes
 * onto zero, and fp32 addition of two terms commutes) and adds the RMSNorm
 * partial sums of squares as exact 2^-24 fixed point.  Slower (fewer CTAs
 * stream the short GEMMs); the per-phase path (T > 32) is not covered.
 * Results equal the default mode's to the logit tolerance. */
#define SS_DEBUG_DETERMINISTIC 2
ss_status ss_set_debug(ss_shard* s, int32_t flags);

/* Watchdog record (debugging aid): every wait of the persistent step kernel is
 * bounded (~10 s of SM clock); the first one that times out writes
 * out[0] = 1 + site (0 idle producer, 1 mbarrier, 2 global counter), out[1] =
 * the barrier's shared address or the counter's global address, out[2] =
 * parity / target, out[3] = the counter value seen, out[4] = blockIdx.x,
 * out[5] = threadIdx.x, then traps (the launch fails).  Process-wide, readable
 * after the failure (mapped host memory).  n <= 512. */
ss_status ss_watchdog_record(uint64_t* out, int32_t n);
/* Device address of the shard's per-layer phase counters ([n_layers][48] int32 +
 * globals), to decode a counter address of the watchdog record. */
uint64_t ss_debug_ctr_base(ss_shard* s);

/* ---- weights and KV ------------------------------------------------------ */

/* Copy one canonical host tensor (layer ignored for global kinds) into the
 * shard, slicing and repacking on the host.  `bytes` must equal the canonical
 * size.  Synchronous. */
ss_status ss_load_weights(ss_shard* s, int32_t layer, int32_t kind, int32_t sub,
                          const void* host, size_t bytes);

/* Device-side synthetic weights: the same counter-based generator as
 * synth/generators.py (DESIGN.md input recipe) evaluated on the GPU, written
 * straight into the kernel layout.  Used for 8B/70B shapes where a host copy
 * would be pointless.  Synchronous. */
ss_status ss_synth_weights(ss_shard* s, uint64_t seed);

/* Committed prefix rows [0, len) of one layer: k, v host uint16 bf16 bits
 * [len][n_kv_heads][head_dim] (FULL heads; the shard keeps its own).  Keys are
 * post-RoPE as cached.  Stored as fp16 (SS_EINVAL if a value exceeds the fp16
 * range).  Sets L = len when called for the last layer. */
ss_status ss_set_prefix_kv(ss_shard* s, int32_t layer, const void* k, const void* v, int32_t len);
/* Device-side synthetic prefix for all layers (synth.gen_prefix_kv), L = len. */
ss_status ss_synth_prefix_kv(ss_shard* s, uint64_t seed, int32_t len);
/* Read cache rows [row0, row0+n) of layer `layer` back to host as float32,
 * layout [n][n_kv_heads/tp][head_dim] (this shard's heads).  The cache stores
 * K/V as fp16 (exact for the bf16 prefix inputs).
 * Synchronises the device. */
ss_status ss_read_kv(ss_shard* s, int32_t layer, int32_t row0, int32_t n, float* k_out, float* v_out);
/* Set the committed length: truncate, or grow over rows that already hold
 * data (prefix rows, or tree rows written by an earlier verify: chain
 * prefill).  Discards a pending verify.  Synchronises the device.
 * Errors: SS_ECAPACITY (L + max_tree > max_ctx), SS_EINVAL (L beyond the
 * rows ever written). */
ss_status ss_set_committed_len(ss_shard* s, int32_t L);
/* Committed length L (synchronises with the device if the last commit was
 * device-driven).  Negative on error. */
int32_t ss_committed_len(ss_shard* s);

/* ---- the step ------------------------------------------------------------ */

/* Verify one tree (host buffers).  tokens/parents: int32[T], parents[0] = -1,
 * 0 <= parents[i] < i, tokens in [0, vocab).  Writes the tree's K/V into the
 * scratch rows [L, L+T) (node i at row L+i, R10) without committing.
 * out: filled before return (the call synchronises `stream`).
 * logits_out: nullable float[T][vocab_shard] (this rank's vocab slice
 * [rank*ceil(V/tp), ...)), for parity checks.
 * Errors: SS_EINVAL, SS_ESTATE (weights / peers missing, or a verify still
 * pending), SS_ECAPACITY (L + T > max_ctx), SS_ECUDA; a device-side failure
 * (out->status: SS_ETIMEOUT, SS_ECONSISTENCY) is returned as well, with out
 * filled and nothing pending. */
ss_status ss_verify_tree(ss_shard* s, const int32_t* tokens, const int32_t* parents, int32_t T,
                         ss_verify_result* out, float* logits_out, void* stream);

/* Same step, all-device and asynchronous (no host synchronisation): d_tokens,
 * d_parents are device int32[T]; the result is written to the device struct
 * d_result (nullable), logits to d_logits (nullable).  The tree is validated
 * on the device (result->status).  Replays a captured CUDA graph per
 * ceil(T/8).  If auto_commit != 0 the accepted path is committed on the
 * device in the same launch sequence (bit-identical to ss_commit_accepted). */
ss_status ss_verify_tree_dev(ss_shard* s, const int32_t* d_tokens, const int32_t* d_parents,
                             int32_t T, ss_verify_result* d_result, float* d_logits,
                             int32_t auto_commit, void* stream);

/* Non-square forward ("Non-square mask support"):
 * grow the pending tree by w new nodes and compute only them.  The pending
 * tree's first T0 nodes (from the last ss_verify_tree / ss_extend_tree since
 * the last commit; T0 <= its size, nodes >= T0 are discarded) keep their K/V
 * rows [L, L+T0) -- "the KV states of the tree are stored right after the
 * prefix".  New node T0+i (token tokens[i], parent parents[i] in
 * [0, T0+i), or -1 only when T0+i == 0) attends to the L prefix rows, its
 * cached ancestors and its new ancestors-or-self: a w x (T0+w) mask, e.g.
 * (4, 10) for a tree of 6 and 4 leaves.  Its K/V go to row L+T0+i;
 * cached rows enter as fp16 (like committed rows, R18).  T0 = 0 is
 * ss_verify_tree.  The step replays the graph of ceil(w/8) (graphs
 * per width; the tree offset is device state).
 * out: argmax[j] for every node j < T0+w (cached nodes keep the argmax of the
 * call that computed them) and the greedy accept walk over the whole grown
 * tree; logits_out: nullable float[w][vocab_shard], the new nodes only.
 * The tree stays pending: commit any root-anchored chain of its T0+w nodes
 * with ss_commit_kv / ss_commit_accepted, or discard it.
 * Errors: SS_EINVAL (w out of [1, 32], T0+w > max_tree, bad parents /
 * tokens, T0 > 0 with a tp_size whose step cannot run the persistent
 * kernel), SS_ESTATE (T0 > 0 without a pending tree of >= T0 nodes, T0 == 0
 * with one; weights / peers missing), SS_ECAPACITY (L+T0+w > max_ctx),
 * SS_ECUDA; device failures as ss_verify_tree. */
ss_status ss_extend_tree(ss_shard* s, const int32_t* tokens, const int32_t* parents, int32_t T0, int32_t w,
                         ss_verify_result* out, float* logits_out, void* stream);

/* Draft worker.  ss_extend_tree_topk: the same
 * non-square forward as ss_extend_tree, returning for each new node the K
 * (1..32) most probable tokens of this rank's vocab slice -- the children the
 * maximum-likelihood expansion adds -- as global token ids top_tok
 * [w][K] (-1 past the slice) with their logits top_logit[w][K] (larger first,
 * ties -> lower id), and the slice's log-sum-exp lse[w].  A node's value
 * log softmax = logit - log(sum over ranks of exp(lse_rank)).
 * Host outputs, filled before return.  Errors as ss_extend_tree, plus
 * SS_EINVAL for K out of range / null outputs. */
ss_status ss_extend_tree_topk(ss_shard* s, const int32_t* tokens, const int32_t* parents, int32_t T0, int32_t w,
                              int32_t K, int32_t* top_tok, float* top_logit, float* lse, ss_verify_result* out,
                              void* stream);

/* Re-root with KV reorganisation (draft side): commit the root-
 * anchored chain path[0..n) of the pending tree (rows L + path[k] -> L + k,
 * L += n, as ss_commit_kv) and keep the subtree keep[0..m) -- ascending node
 * indices, keep[0] a child of path[n-1] (or the root 0 when n == 0), every
 * other kept node's parent kept -- packed right after the new prefix (rows
 * L_old + keep[j] -> L_new + j): "reorganizes the remaining sub-tree ... into
 * the next positions available, discarding the KV states that are no longer
 * useful".  Kept node keep[j] becomes node j of the pending tree
 * (positions unchanged: pos = L + depth, both shift by n), which a later
 * ss_extend_tree(T0 <= m) grows; m == 0 leaves nothing pending.  Synchronises.
 * Errors: SS_ESTATE (no pending tree / its step failed), SS_EINVAL (not a
 * chain, keep not such a subtree, n + m out of [1, tree size]). */
ss_status ss_reroot(ss_shard* s, const int32_t* path, int32_t n, const int32_t* keep, int32_t m, void* stream);

/* Parallel tree generation (Alg. 1): greedy
 * speculative decoding of n_tokens tokens with a draft shard and a target
 * shard linked only by the a13 mailboxes.  Draft branch (calling thread):
 * expand the w most probable leaves d times (ss_extend_tree_topk, children =
 * top-K, K = w when 0, values = log softmax), get the verified path,
 * re-root and reorganise the draft KV (ss_reroot), expand while the
 * target root's subtree has < bs nodes, post the most probable bs-node
 * subgraph.  Target branch (its own thread): mailbox-driven verify
 * steps with auto-commit (ss_verify_tree_mailbox).  mode 0 = async (the draft
 * expands while the target verifies -- the paper's design); mode 1 = serial
 * (draft, then verify; the d expansions precede each post).  eos >= 0 stops
 * at that bonus token.  Both shards must hold the same committed prefix and
 * nothing pending; root_token = the last prompt token (in neither cache, R9).
 * out_tokens[n_tokens] receives the emitted tokens -- with greedy acceptance
 * exactly the target's greedy continuation of root_token.  Single-
 * rank shards on one device; run them concurrently by capping their grids
 * (ss_set_launch_cap) so both fit the SMs.  Afterwards the target has
 * committed at least the emitted tokens' prefix, the draft's tree is
 * discarded.  Errors: SS_EINVAL (arguments), SS_ESTATE (a pending verify),
 * SS_ETIMEOUT (mailbox), errors of the calls above. */
typedef struct {
  int32_t bs;        /* target batch: nodes per verified subgraph (paper: 8) */
  int32_t w;         /* leaves per draft expansion (paper: 8) */
  int32_t d;         /* expansions per round (t_target / t_draft) */
  int32_t K;         /* children per expanded node (0: w) */
  int32_t n_tokens;  /* tokens to generate */
  int32_t eos;       /* stop token (-1: none) */
  int32_t mode;      /* 0 async, 1 serial */
} ss_spec_cfg;
typedef struct {
  int32_t n_emitted;     /* tokens written to out_tokens */
  int32_t steps;         /* verify results received */
  int32_t target_steps;  /* verify steps the target ran (async: one more may run) */
  int32_t expansions;    /* draft forwards */
  int32_t accepted;      /* accepted draft tokens (emitted = accepted + one bonus per step) */
  double wall_ms;        /* host wall time of the loop */
} ss_spec_stats;
ss_status ss_speculative_decode(ss_shard* target, ss_shard* draft, int32_t root_token, const ss_spec_cfg* cfg,
                                int32_t* out_tokens, ss_spec_stats* stats, void* target_stream,
                                void* draft_stream);

/* Commit a root-anchored chain of tree nodes from the last verify:
 * accepted[0] == 0 and accepted[k] a child of accepted[k-1] (any such chain,
 * not only the accepted one: chain prefill, EOS truncation).  K/V rows
 * L + accepted[k] move to L + k in every layer; L += n.  Synchronises.
 * Errors: SS_ESTATE (no pending verify, or its device status was not SS_OK),
 * SS_EINVAL (not a chain / n out of range). */
ss_status ss_commit_kv(ss_shard* s, const int32_t* accepted, int32_t n, void* stream);
/* Commit the accepted path of the last verify, decided on the device. */
ss_status ss_commit_accepted(ss_shard* s, void* stream);

/* Number of kernels the verify (+ commit) launch sequence contains. */
int32_t ss_kernels_per_step(ss_shard* s, int32_t T, int32_t auto_commit);

/* Tensor-parallel all-reduce scheme of the persistent step kernel (SURVEY
 * 8(f) NEXT-2; the paper's fused one-shot design P:413-420 vs a two-shot
 * variant for large T x h).  mode 0 (default): one-shot LL -- each O / down
 * tile-group finaliser stores its fp32 partial to every rank, every rank sums
 * the P partials in rank order (one NVLink hop, (P-1) x T x h x 8 bytes of
 * LL egress per rank per all-reduce).  mode 1: two-shot LL -- the partial
 * goes only to the tile-group's home rank (tg mod P), which sums in rank order
 * and broadcasts the sum (two hops, ~2 (P-1)/P x T x h x 8 bytes).  Both give
 * bit-identical residuals on every rank; results equal to the logit
 * tolerance across modes (same rank-ordered sums: bit-identical).  Every rank
 * of a group must use the same mode.  Synchronises the device; drops the
 * shard's captured graphs.  The per-phase path (T > 32) is one-shot. */
ss_status ss_set_allreduce(ss_shard* s, int32_t mode);

/* Kernel organisation of the step.  on != 0 (the default): trees of T <= 32
 * run as ONE persistent kernel per step (every layer's GEMMs, attention,
 * all-reduces, the LM head and the accept walk; phases hand over through
 * device counters, weights stream ahead of their inputs).  on == 0: one
 * kernel per phase (QKV, attention, O, gate/up, down per layer, LM head) --
 * the path T > 32 always takes; kept selectable for A/B parity tests.
 * Results agree to the logit tolerance; both are bit-exact where the method
 * requires it.  ss_step_kernel_active returns 1 if a verify of T nodes uses
 * the persistent kernel, 0 if not, -1 on bad arguments. */
ss_status ss_set_step_kernel(ss_shard* s, int32_t on);
int32_t ss_step_kernel_active(ss_shard* s, int32_t T);

/* Measurement hook: on != 0 makes every later persistent-step launch record a
 * timeline -- per CTA (up to 512), per slot (layer * 5 + phase: 0 QKV,
 * 1 attention, 2 O, 3 gate/up, 4 down; slot n_layers * 5 = LM head), three
 * %globaltimer ns stamps (phase entry, first unit ready, phase exit; 0 = the
 * CTA had no work there).  ss_read_step_trace copies it to `host` (n >= 512 *
 * slots * 3 elements; *n_ctas = 512, *slots = n_layers * 5 + 1) after a device
 * synchronize.  on == 2 keeps the timeline in mapped host memory, read
 * without synchronising (diagnosis of a launch that does not finish).  Off by
 * default; toggling drops the captured graphs. */
ss_status ss_step_trace(ss_shard* s, int32_t on);
ss_status ss_read_step_trace(ss_shard* s, uint64_t* host, size_t n, int32_t* n_ctas, int32_t* slots);
/* The mapped host buffer of on == 2 (NULL otherwise): [512][slots][3] stamps,
 * then [512 CTAs][16 warps] progress words; readable with no CUDA call. */
void* ss_step_trace_host(ss_shard* s);

/* Measurement helper (bench.py's roofline): run one all-device step like
 * ss_verify_tree_dev(auto_commit=1) but launched eagerly with a CUDA event
 * pair around every kernel on `stream`; synchronises and writes the summed
 * device time (ms) and launch count per kernel kind to ms[SS_PROF_KINDS],
 * count[SS_PROF_KINDS].  Kinds: 0 embed+tree, 1 QKV, 2 attention, 3 O-proj,
 * 4 RMSNorm, 5 gate/up+SwiGLU, 6 down, 7 LM head+argmax+accept, 8 commit,
 * 9 the persistent step kernel (all of 1-7 in one launch, T <= 32). */
#define SS_PROF_KINDS 10
ss_status ss_profile_step(ss_shard* s, const int32_t* d_tokens, const int32_t* d_parents, int32_t T,
                          float* ms, int32_t* count, void* stream);

/* ---- a13: asynchronous draft -> target handoff ---------------------------
 * P:44 / P:228-234 / Alg. 1: the draft group sends the next tree,
 * the target group verifies it and sends back the verified tokens (or STOP),
 * with no host round trip.  Messages are 16-byte LL lines (data1, flag1,
 * data2, flag2; Alg. 2, R15) whose flags all equal the message
 * sequence number (1, 2, ...; 0 is the idle value), written with one
 * st.volatile.v4 into peer-mapped memory (NVLink) or local memory.
 *   inbox  (owned by the target shard): line 0 = (T, seq), line 1+i =
 *          (token_i, parent_i);
 *   outbox (owned by the draft side):   line 1+k = (accepted[k], token),
 *          then line 0 = (n_accepted | (-status & 0xFF) << 16 | stop << 31,
 *          bonus_token); a failed step posts n_accepted = 0 and its status;
 *          an inbox message that timed out (2 s of device time) gets no post
 *          and is polled again by the next step.
 * Sequence numbers are consecutive per shard, starting at 1. */

/* Device pointer of this shard's inbox ((1 + SS_MAX_TREE) lines x 16 B, a
 * separate cudaMalloc the draft side may map with cudaIpc). */
ss_status ss_mailbox_inbox(ss_shard* s, void** dev_ptr);
/* Where the verified path is posted (a device pointer valid in this shard's
 * context, e.g. a peer-mapped draft buffer of (1 + SS_MAX_TREE) lines); only
 * tp_rank 0 posts.  eos_token >= 0 sets the STOP bit when the bonus equals it. */
ss_status ss_attach_mailbox(ss_shard* s, void* outbox_dev, int32_t eos_token);
/* One verify step whose tree comes from the inbox (the kernels poll for
 * message mbox_seq + 1) and whose result is posted to the outbox after the
 * accept walk.  Asynchronous on `stream`; with auto_commit the accepted path
 * is committed in the same launch sequence.  Errors as ss_verify_tree_dev. */
ss_status ss_verify_tree_mailbox(ss_shard* s, int32_t auto_commit, void* stream);
/* Same, with the step captured for at most max_nodes (<= max_tree) nodes: the
 * graph of ceil(max_nodes / 8) token slots (a larger message is refused on the
 * device, status SS_EINVAL).  The draft side knows its batch size bs. */
ss_status ss_verify_tree_mailbox_n(ss_shard* s, int32_t max_nodes, int32_t auto_commit, void* stream);
/* Draft-side helpers: post a tree into an inbox / wait for a verified path in
 * an outbox and copy it to dev_out = [n, bonus, stop, status, (node, token)
 * x n] (int32, device; status != SS_OK -> n = 0; a message that never
 * arrives -> n = -1, status SS_ETIMEOUT).  The target refuses (status
 * SS_EINVAL) a tree larger than its max_tree.  Both enqueue one small
 * kernel on `stream`. */
ss_status ss_mailbox_post_tree(void* inbox_dev, const int32_t* tokens, const int32_t* parents, int32_t T,
                               uint32_t seq, void* stream);
ss_status ss_mailbox_recv_result(const void* outbox_dev, uint32_t seq, int32_t* dev_out, void* stream);

/* ---- inspection and test hooks (parity tests; not on the step's path) ---- */

/* Tree metadata of the last step as the device computed it (a0; P:321 square
 * ancestor mask, R8 positions): T, pos[64] = L + depth, anc[64] = ancestor-or-
 * self bitmask (bit j = node j), and optionally tokens[64] / parents[64] as
 * ingested.  Synchronises the device. */
ss_status ss_read_tree_meta(ss_shard* s, int32_t* T, int32_t* pos, uint64_t* anc, int32_t* tokens,
                            int32_t* parents);

/* Raw bytes of a device region in kernel layout: which = 0 QKV, 1 O, 2 gate/up,
 * 3 down (packed W4 units of `layer`), 4 LM head (bf16 units), 5 embedding,
 * 6 / 7 attention / MLP norm gain of `layer`, 8 final norm.  *total receives
 * the size; host may be NULL (size query), else bytes must equal *total.
 * Used to check the device generator against the host repack byte for byte. */
ss_status ss_read_packed(ss_shard* s, int32_t layer, int32_t which, void* host, size_t bytes, size_t* total);

/* One W4A16 GEMM of linear `which` (0 QKV, 1 O, 2 gate/up, 3 down) of `layer`
 * on caller activations: d_x device float [T][K_local] (rounded to fp16 like
 * the step's activations), d_y device float [T][N_pad] = the shard's output
 * rows in packed row order (QKV: local q | k | v heads; gate/up: per 128-row
 * tile-group 64 gate then 64 up columns; N_pad = N_local rounded up to 128).
 * allreduce != 0 (O / down): d_y = the fused tensor-parallel all-reduce of
 * every rank's partial (collective: all ranks call it; same T).  The same
 * kernel as the step (integer-valued inputs give bit-exact sums: SURVEY 8(c)).
 * Asynchronous on `stream`. */
ss_status ss_debug_gemm(ss_shard* s, int32_t layer, int32_t which, const float* d_x, int32_t T, float* d_y,
                        int32_t allreduce, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SWIFTSPEC_H */
