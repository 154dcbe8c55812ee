// internal.h -- shard state shared by the host C-ABI implementation and the
// kernel launchers.  Not part of the public ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <string>
#include <vector>
#include <map>

#include "../../include/swiftspec.h"
#include "host_logic.h"

namespace ss {

constexpr int kMaxPeers = 8;
constexpr int kCtrPerLayerH = 48;  // == kCtrPerLayer (step.h)
constexpr int kCtrGlobalH = 8;     // == kCtrGlobal

// Device-resident per-step state (read by every kernel through a pointer so
// that captured CUDA graphs replay with new trees).
struct DevState {
  int32_t L;                 // committed length
  int32_t T;                 // nodes of the current tree
  int32_t status;            // SS_OK / SS_EINVAL for the current tree
  int32_t have_verify;       // 1 after a verify, 0 after a commit
  int32_t tokens[SS_MAX_TREE];
  int32_t parents[SS_MAX_TREE];
  int32_t pos[SS_MAX_TREE];
  int32_t pad0;
  unsigned long long anc[SS_MAX_TREE];        // ancestor-or-self bitmask (bit j = node j)
  unsigned long long argmax_key[SS_MAX_TREE]; // packed (ordered logit, ~id) per node (this rank)
  ss_verify_result result;   // accept-walk result of the last verify
  int32_t commit_n;          // chain to commit (ss_commit_kv): length
  int32_t commit_chain[SS_MAX_TREE];
  int32_t lm_done;           // LM-head tile-groups finished (self-resetting)
  int32_t commit_done;       // commit CTAs finished (self-resetting)
  uint32_t epoch;            // LL flag epoch of the current step (TP)
  int32_t timeout;           // set when a peer poll exceeded its budget
  // a13 mailbox handoff (LL lines over NVLink / local memory)
  uint32_t mbox_seq;         // last message sequence number fully handled
  uint32_t mbox_cur;         // sequence number of the tree being verified
  int32_t mbox_mode;         // 1 while the current step came from the inbox
  int32_t mbox_post;         // 1 on the rank that posts the verified path
  int32_t eos;               // STOP when the bonus token equals eos (-1: never)
  int32_t max_written;       // highest KV row ever written + 1 (prefix, tree rows)
  uint4* mbox_out;           // draft group's outbox (peer-mapped), nullptr = none
  int32_t debug;             // SS_DEBUG_* flags (ss_set_debug)
  int32_t mbox_tmo;          // the current step's inbox message never (fully) arrived
  // non-square forward (ss_extend_tree): the step computes nodes
  // [T0, T0 + T) of a tree whose nodes [0, T0) are cached at rows [L, L + T0);
  // token slot t is node T0 + t.  0 for a square verify.
  int32_t T0;
  // ss_reroot (draft KV reorganisation): the kept subtree's nodes,
  // packed after the committed chain (commit_n / commit_chain)
  int32_t keep_n;
  int32_t keep[SS_MAX_TREE];
};

// One packed linear (W4 format, see common.cuh) or bf16 matrix.
struct PackedLinear {
  uint8_t* d = nullptr;      // device units
  size_t bytes = 0;
  int K = 0, N = 0;          // local (sharded) shape; N padded to 128 multiple
  int n_tg = 0, S = 0;       // tile-groups, K stages
};

struct LayerW {
  PackedLinear qkv, o, gu, down;
  uint16_t* attn_norm = nullptr;
  uint16_t* mlp_norm = nullptr;
};

// Host-side staging of canonical tensors until a linear's parts are complete.
struct CanonLinear {
  std::vector<uint8_t> q, z;
  std::vector<uint16_t> s;
  bool hq = false, hz = false, hs = false;
};

struct GemmScratch {
  float* accum = nullptr;    // [n_tg*128][8*NT_max] fp32, self-zeroing
  int* counters = nullptr;   // [n_tg + 2]
  float* ss = nullptr;       // [64] fused-norm sums of squares
  int* nbar = nullptr;       // fused-norm grid barrier
  size_t accum_elems = 0;
};

struct Graph {
  cudaGraphExec_t exec = nullptr;
  cudaGraphNode_t first = nullptr;
  int kernels = 0;
};

}  // namespace ss

struct ss_shard {
  ss_model_cfg cfg;
  int rank = 0, P = 1, device = 0;
  int n_sm = 148;
  int launch_cap = 0;
  // local shapes
  int Hq_l = 0, Hkv_l = 0, I_l = 0, G = 1, V_pad = 0, V_l = 0, V_off = 0, V_l_pad = 0;
  int max_ctx_pad = 0;

  // weights
  std::vector<ss::LayerW> layers;
  uint16_t* embed = nullptr;       // [V][h] bf16 (replicated)
  uint16_t* final_norm = nullptr;
  ss::PackedLinear lm_head;        // bf16 units
  std::map<long, ss::CanonLinear> staging;  // (layer, kind) -> canonical parts
  std::vector<uint32_t> loaded_mask;        // per layer bitmask of complete kinds
  uint32_t global_mask = 0;

  // KV cache [layer][kvh_l][max_ctx_pad][d] bf16, swizzled 64-row blocks
  uint16_t* kcache = nullptr;
  uint16_t* vcache = nullptr;
  float2* rope_cs = nullptr;       // [max_ctx_pad][d/2] (cos, sin)

  // activations / workspaces
  float* x = nullptr;              // residual [64][h] fp32
  uint8_t* act_h = nullptr;        // frag-ordered bf16, K = h, NT up to 8
  uint8_t* act_o = nullptr;        // K = Hq_l*d
  uint8_t* act_d = nullptr;        // K = I_l
  uint8_t* act_lm = nullptr;       // LM-head input, bf16 hi/lo, K = h, 2*NT tiles
  uint16_t* qbuf = nullptr;        // [Hkv_l][G*64][d] bf16 (post-RoPE q)
  float* attn_ws = nullptr;        // partial O [Hkv_l][Z][S][256][d]
  float* attn_ml = nullptr;        // partial (m, l)
  int* attn_bar = nullptr;         // [Hkv_l*Z*2] arrive/depart counters
  ss::GemmScratch sc_qkv, sc_o, sc_gu, sc_down, sc_lm;
  float* logits_dev = nullptr;     // optional [64][V_l_pad]

  // state
  ss::DevState* dstate = nullptr;  // device
  ss::DevState* hstate = nullptr;  // pinned host mirror for results
  int32_t* d_tree_in = nullptr;    // device staging for host trees [2*64]
  int32_t* d_topk = nullptr;       // draft top-K output: tokens [32][32], logits [32][32], lse [32]
  int32_t* h_tree_in = nullptr;    // pinned staging
  ss::host::CallState hs;          // host view: committed length, pending verify, rows written
  std::string err;                 // message of the last failed call on this shard
  int debug = 0;                   // SS_DEBUG_* flags

  // TP peers
  float* recv = nullptr;            // this rank's LL receive buffer
  size_t recv_bytes = 0;
  float* peer_recv[ss::kMaxPeers] = {nullptr};
  bool peers_ready = false;
  bool loopback = false;            // ss_import_loopback (timing emulation)
  int ar_mode = 0;                  // ss_set_allreduce: 0 one-shot, 1 two-shot (step kernel)
  bool ipc_opened[ss::kMaxPeers] = {false};

  // a13 mailbox: this shard's inbox (written by the draft group)
  uint4* mbox_in = nullptr;

  // persistent step kernel (step.cu) state
  int* step_ctr = nullptr;         // phase counters [n_layers][kCtrPerLayerH] + [kCtrGlobalH]
  float* step_ss = nullptr;        // [n_layers + 1][2][64]
  unsigned long long* step_ssx = nullptr;  // same shape, fixed point (SS_DEBUG_DETERMINISTIC)
  uint16_t* qf = nullptr;          // q fragments hi | lo
  uint16_t* klo = nullptr;         // tree K / V lo window [Hkv_l][128][d]
  uint16_t* vlo = nullptr;
  float* att_ws = nullptr;         // [max step CTAs][2][64][d]
  float2* att_ml = nullptr;
  void* layer_tab = nullptr;       // device LayerPtrs[n_layers]
  void* step_args_dev = nullptr;   // device StepArgs x 2 (without / with the logits output)
  int step_max_ctas = 0;
  unsigned long long* step_trace = nullptr;  // ss_step_trace timeline (null: off)
  int step_trace_slots = 0;
  unsigned long long* step_trace_host = nullptr;  // mapped host buffer (ss_step_trace(s, 2))
  bool use_step = true;            // NT <= 4: persistent step kernel; else per-phase kernels

  // graphs: key = NT*4 + auto_commit*2 + logits
  std::map<int, ss::Graph> graphs;
  cudaStream_t cap_stream = nullptr;
};

// LL line index of the cross-rank consistency area (SS_DEBUG_CONSISTENCY) in a
// receive buffer: after the two all-reduce parities and the argmax area.
inline size_t consistency_line_offset(const ss_shard* s) {
  return (size_t)2 * s->P * (s->cfg.hidden / 128) * 128 * 32 + (size_t)s->P * 64;
}
