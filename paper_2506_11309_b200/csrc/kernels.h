// kernels.h -- kernel argument structs and launchers (internal).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <algorithm>
#include <utility>
#include <cstdlib>
#include "internal.h"

namespace ss {

enum { EPI_QKV = 0, EPI_RESID = 1, EPI_SWIGLU = 2, EPI_ARGMAX = 3 };

// Tuning / debugging environment knobs exist only in experiment builds
// (`python -m paper_2506_11309_b200.build --variant x -D SS_EXPERIMENTS`): the
// product library reads no environment variable and can never skip work.
#ifdef SS_EXPERIMENTS
inline const char* exp_env(const char* name) { return getenv(name); }
#else
inline const char* exp_env(const char*) { return nullptr; }
#endif
inline int exp_env_int(const char* name, int dflt) {
  const char* v = exp_env(name);
  return v ? atoi(v) : dflt;
}

// Per-device launch caches (function attributes, occupancy): the dynamic
// shared-memory opt-in is per device, and one process may drive several GPUs
// (ss_import_local_peers).
constexpr int kMaxDevices = 16;
inline int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return (d >= 0 && d < kMaxDevices) ? d : 0;
}

// Launch with programmatic stream serialization (PDL): the kernel may begin
// while its predecessor drains; kernels call pdl_wait() before consuming
// their predecessors' outputs.  Works under stream capture (graph edges).
inline thread_local int ss_pdl_pos = 31;  // launch position in the layer body (debugging aid)
// Set while enqueueing a fake-peer shard (several TP ranks on one GPU, capped
// grids): an early-launched PDL grid holds SM slots while it waits, which can
// starve a peer rank's kernel that this rank's all-reduce is polling for.
inline thread_local bool ss_pdl_off = false;
template <typename... ExpT, typename... ActT>
inline cudaError_t launch_pdl(void (*k)(ExpT...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              ActT&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  static const bool no_pdl = exp_env("SS_NO_PDL") != nullptr;  // debugging aid
  // debugging aid: SS_NO_PDL_MASK bit i = no PDL for body launch position i (ss_pdl_pos)
  static const int no_pdl_mask = exp_env_int("SS_NO_PDL_MASK", 0);
  cfg.numAttrs = (no_pdl || ss_pdl_off || ((no_pdl_mask >> ss_pdl_pos) & 1)) ? 0 : 1;
  return cudaLaunchKernelEx(&cfg, k, std::forward<ActT>(args)...);
}

struct EpiArgs {
  int kind = 0;
  DevState* st = nullptr;
  int layer = 0;
  // QKV
  int d = 128, Hq_l = 0, Hkv_l = 0, G = 1, max_ctx_pad = 0;
  uint16_t* qbuf = nullptr;
  uint16_t* kc = nullptr;
  uint16_t* vc = nullptr;
  const float2* rope_cs = nullptr;
  // RESID (+ all-reduce)
  float* x = nullptr;
  int h = 0;
  int rank = 0, P = 1, n_tg_total = 0, ar_seq = 0;
  int loopback = 0;  // timing emulation of one TP rank on one GPU (ss_import_loopback)
  float* recv = nullptr;
  float* peer_recv[kMaxPeers] = {nullptr};
  // SWIGLU
  uint8_t* act_out = nullptr;
  // ARGMAX
  int V_l = 0, V_off = 0, logits_ld = 0;
  float* logits = nullptr;
};

struct GemmArgs {
  const uint8_t* W = nullptr;
  const uint8_t* act = nullptr;
  int n_tg = 0, S = 0;
  float* accum = nullptr;
  int* counters = nullptr;   // [n_tg] arrival counters + [2] (exit count in [1])
  int n_sm = 148;
  // optional: zero the X (group-sum) slots of a W4 activation buffer that a
  // later kernel fills with atomics (attention -> O input, SwiGLU -> down input)
  uint8_t* zero_x = nullptr;
  int zero_x_stages = 0, zero_x_nt = 1;
  // optional fused RMSNorm of the updated residual (EPI_RESID): output into
  // norm_out (fp16 + X, or bf16 hi/lo for the LM head when norm_split)
  const uint16_t* norm_gain = nullptr;
  uint8_t* norm_out = nullptr;
  int norm_split = 0;
  float eps = 1e-5f;
  float* ss = nullptr;       // [64] per-token sum of squares (self-cleaning)
  int* nbar = nullptr;       // grid barrier counter (self-cleaning)
  EpiArgs epi;
};

struct AttnArgs {
  DevState* st = nullptr;
  int layer = 0, Hkv_l = 0, G = 1, d = 128, max_ctx_pad = 0, NT = 1;
  int splits = 1, zchunks = 1;
  const uint16_t* qbuf = nullptr;
  const uint16_t* kc = nullptr;
  const uint16_t* vc = nullptr;
  float* ws = nullptr;     // [Hkv_l][Z][S][256][d]
  float* ml = nullptr;     // [Hkv_l][Z][S][256][2]
  int* bar = nullptr;      // [Hkv_l*Z][2]
  uint8_t* act_out = nullptr;  // O-proj input, frag order, K = Hq_l*d
};

int launch_gemm(const GemmArgs& g, int wfmt, int NT, int max_ctas, cudaStream_t st);
// persistent step kernel (step.cu, NT <= 4)
struct StepArgs;
int launch_step(const StepArgs& a, const StepArgs* dev_args, int NT, int max_ctas, cudaStream_t st);
int step_ctas(int NT, int d, int max_ctas);
void warm_step_kernels();
// watchdog panic record of the step kernel (mapped host memory; debugging aid)
void arm_watchdog_record();
const unsigned long long* watchdog_record();
// force-load every kernel (lazy module loading vs cross-kernel flag waits)
void warm_gemm_kernels();
void warm_attention_kernels();
void warm_misc_kernels();
void warm_draft_kernels();
// draft worker (draft.cu): top-K + log-sum-exp of the last step's logits rows,
// and the re-root KV reorganisation (DevState commit_chain / keep lists)
void launch_topk(ss_shard* s, int w, int K, int32_t* d_tok, float* d_val, float* d_lse, cudaStream_t st);
void launch_reroot(ss_shard* s, cudaStream_t st);
int launch_attention(const AttnArgs& a, int max_ctas, cudaStream_t st);

// embed + tree metadata (a0, a1) + first RMSNorm into the frag activation
void launch_embed_meta(ss_shard* s, const int32_t* tokens, const int32_t* parents, int T, int NT,
                       cudaStream_t st, bool from_mailbox = false, bool step_mode = false, int T0 = 0);
// a13 mailbox helpers for the draft side (and tests)
void launch_mailbox_post(void* inbox, const int32_t* tokens, const int32_t* parents, int T, uint32_t seq,
                         cudaStream_t st);
void launch_mailbox_recv(const void* outbox, uint32_t seq, int32_t* dev_out, cudaStream_t st);
// RMSNorm of the residual into frag activations (a2 / a7 / final)
void launch_prep_norm(ss_shard* s, const uint16_t* gain, int NT, int split, cudaStream_t st);
// ss_debug_gemm: caller fp32 activations -> W4 GEMM input layout
void launch_debug_act(ss_shard* s, const float* x, int T, int K, uint8_t* act, int NT, int bump_epoch,
                      cudaStream_t st);
// KV compaction + commit (a12); chain from the device result or commit list
void launch_commit(ss_shard* s, int from_result, cudaStream_t st);
// device synthetic generator (same counter-based hash as synth/generators.py)
struct LinMap {
  int mode;  // 0 QKV, 1 O, 2 GU, 3 DOWN
  int rank, Hq_l, Hkv_l, d, I_l, Kl, Nl_valid;
  // unpadded sizes (arbitrary TP by zero padding): global indices
  // at or beyond them are padding and map to zero weights
  int q_full, kv_full, I_full, K_full;
};
struct SynthLinArgs {
  uint64_t keys[3][3];  // [part][qweight, qzeros, scales] stream keys
  float scale_c[3];
  int N_full[3];
  LinMap m;
  int n_tg, S;
};
void launch_synth_linear_args(uint8_t* dst, const SynthLinArgs& a, cudaStream_t st);
void launch_synth_dense_key(uint16_t* dst, size_t n, uint64_t key, size_t idx0, int mode, float scale,
                            cudaStream_t st);
void launch_synth_lm_key(uint8_t* dst, int V_l, int V_off, int V_full, int h, int n_tg, uint64_t key, float scale,
                         cudaStream_t st);
void launch_synth_kv_key(uint16_t* cache, int layer, int Hkv_full, int Hkv_l, int kv0, int d, int L,
                         int max_ctx_pad, uint64_t key, cudaStream_t st);
void launch_rope_table(float2* cs, int max_pos, int d, double theta, cudaStream_t st);

}  // namespace ss
