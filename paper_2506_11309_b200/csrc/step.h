// step.h -- arguments and layouts of the persistent step kernel (step.cu),
// shared with the host (shard.cu).  Internal, not part of the C-ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.h"

namespace ss {

// Per-layer weight pointers (device table, one entry per layer).
struct LayerPtrs {
  const uint8_t* qkv;
  const uint8_t* o;
  const uint8_t* gu;
  const uint8_t* down;
  const uint16_t* attn_norm;
  const uint16_t* mlp_norm;
};

// Most layers the persistent step kernel runs (its per-layer pointer table is
// kept in shared memory; deeper models take the per-phase kernels).
constexpr int kStepMaxLayers = 128;

// Phase-completion counters, per layer (zeroed by the ingest kernel every step).
constexpr int kCtrPerLayer = kCtrPerLayerH;
enum { C_QKV = 0, C_ATT = 1, C_O = 2, C_GU = 3, C_DN = 4, C_MEET = 8 };  // C_MEET + kvh*Z + z (<= 32)
constexpr int kCtrGlobal = kCtrGlobalH;  // after the per-layer blocks: [0] LM tile-groups finalised

// W4 GEMM input of the step kernel: per 256-deep K stage, the tcgen05 B
// operand (K-major, no swizzle) of N = 16 NT columns -- fp16 hi of the 8 NT
// token slots, then fp16 lo (x - hi) -- followed by the per-(128-group,
// token) sums X of hi + lo in fp32 (DESIGN R18: hi + lo carries ~22 bits).
__host__ __device__ constexpr uint32_t a2_stage_bytes(int NT) { return (uint32_t)NT * 8192u + (uint32_t)NT * 64u; }
// Byte offset of element (token tt, k) (lo = 0 / 1: hi / lo part).  One K=16
// MMA step reads two 8-deep chunks, each [N rows][8 fp16] (16 B per row):
//   ((kstep * 2 + kap / 8) * N + lo * 8 NT + tt) * 16 + (kap % 8) * 2,
// where kap is the MMA's logical k of true k: pairs p = (k % 16) / 2 are
// permuted to kap / 2 = 2 (p % 4) + p / 4 -- the TMEM column order in which
// the dequantised A fragments land (tcgen05.st.16x256b of the mma.sync-order
// weight units, step.cu).  Both operands use the same permutation of k, so
// the MMA's sum over k is unchanged.  k and k + 1 (even k) are adjacent.
__host__ __device__ inline uint32_t a2_frag(int tt, int k, int NT, int lo) {
  const int kk = k & 15, p = kk >> 1;
  const int kap = ((((p & 3) << 1) | (p >> 2)) << 1) | (kk & 1);
  const int N = 16 * NT;
  return (uint32_t)(k >> 8) * a2_stage_bytes(NT) +
         (uint32_t)(((((k & 255) >> 4) * 2 + (kap >> 3)) * N + lo * 8 * NT + tt) * 16 + (kap & 7) * 2);
}
// X of (token tt, 128-group g): after the stage's B operand, [2 groups][8 NT] fp32.
__host__ __device__ inline uint32_t a2_xsum(int tt, int g, int NT) {
  return (uint32_t)(g >> 1) * a2_stage_bytes(NT) + (uint32_t)NT * 8192u + (uint32_t)(((g & 1) * 8 * NT + tt) * 4);
}

// Attention: keys per K/V tile (a 16 KB ring unit: K then V, 8 KB each).
__host__ __device__ constexpr int att_tile_keys(int d) { return 8192 / (2 * d); }

struct StepArgs {
  DevState* st = nullptr;
  const LayerPtrs* layers = nullptr;  // device [n_layers]
  int n_layers = 0, h = 0, d = 128, Hq_l = 0, Hkv_l = 0, G = 1, I_l = 0, max_ctx_pad = 0;
  int qkv_tg = 0, qkv_S = 0, o_tg = 0, o_S = 0, gu_tg = 0, gu_S = 0, dn_tg = 0, dn_S = 0, lm_tg = 0, lm_S = 0;
  const uint8_t* lm_w = nullptr;
  const uint16_t* final_norm = nullptr;
  float eps = 1e-5f;
  uint8_t* act_h = nullptr;   // QKV / gate-up input (a2 layout, K = h)
  uint8_t* act_o = nullptr;   // O input (K = Hq_l * d)
  uint8_t* act_d = nullptr;   // down input (K = I_l)
  uint8_t* act_lm = nullptr;  // LM head input (bf16 hi / lo fragments, K = h)
  uint16_t* qf = nullptr;     // q, mma A-fragment order: [hi|lo][Hkv_l][4G row blocks][d/16][32 lanes][8]
  uint16_t* kc = nullptr;     // KV cache [layer][Hkv_l][max_ctx_pad][d] fp16, swizzled 64-row blocks
  uint16_t* vc = nullptr;
  uint16_t* klo = nullptr;    // tree rows' lo parts, window of 128 rows from (L & ~63): [Hkv_l][128][d]
  uint16_t* vlo = nullptr;
  const float2* rope_cs = nullptr;
  float* x = nullptr;         // residual [64][h] fp32
  float* acc[5] = {nullptr};  // split-K accumulators: qkv, o, gu, down, lm  [n_tg][128][8 NT]
  int* arr[5] = {nullptr};    // arrival counters per tile-group (self-cleaning)
  int* ctr = nullptr;         // [n_layers][kCtrPerLayer] + [kCtrGlobal]
  float* ss = nullptr;        // [n_layers + 1][2][64] sums of squares (0: attn-norm input, 1: mlp-norm input)
  unsigned long long* ssx = nullptr;  // same shape, 2^-24 fixed point (deterministic mode)
  int det = 0;                // SS_DEBUG_DETERMINISTIC: whole tile-groups per CTA, fixed-point norm sums
  float* att_ws = nullptr;    // [n_ctas][2 key halves][64 rows][d] unnormalised partial outputs
  float2* att_ml = nullptr;   // [n_ctas][2][64] (running max, sum)
  int rank = 0, P = 1, loopback = 0;
  // all-reduce scheme: 0 one-shot LL (every finaliser
  // stores its partial to every rank), 1 two-shot LL (reduce-scatter to the
  // tile-group's home rank tg % P, which sums and broadcasts the sum)
  int ar_mode = 0;
  size_t bc_line0 = 0;        // first LL line of the two-shot broadcast area in every receive buffer
  float* recv = nullptr;
  float* peer_recv[kMaxPeers] = {nullptr};
  int V_l = 0, V_off = 0, logits_ld = 0;
  float* logits = nullptr;
  int n_ctas = 0;
  int att_min_tiles = 2;      // fewest K/V tiles per attention split
  // optional timeline (ss_step_trace): per CTA, per (layer, phase) slot, three
  // %globaltimer stamps: phase entry, first unit ready, phase exit
  unsigned long long* trace = nullptr;
  int trace_slots = 0;
  // hang diagnosis (ss_step_trace(s, 2), mapped host memory): per CTA and warp,
  // the last progress point reached: (code << 32) | low 32 bits of %globaltimer
  unsigned long long* where = nullptr;
  // unit timeline of CTA 0 (ss_step_trace): gate/up phase of layer n_layers / 2,
  // consumer warp 0: [unit 128][8] stamps; MMA warp: [4096 + k * 2 + {0, 1}]
  unsigned long long* utl = nullptr;
};

}  // namespace ss
