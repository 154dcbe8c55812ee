// shard.cu -- host implementation of the C-ABI in include/swiftspec.h:
// shard lifecycle and validation, host repack of canonical AWQ tensors into
// the kernel layout (TP slicing), device synthetic weights, the KV manager
// (committed length, scratch rows, capacity checks), CUDA-graph capture of
// the step per ceil(T/8), peer mapping for tensor parallelism, error state.
#include <cuda_runtime.h>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstddef>
#include <string>
#include <vector>

#include "common.cuh"
#include "internal.h"
#include "kernels.h"
#include "step.h"

using namespace ss;


// Error messages: the calling thread's last one (ss_last_error(NULL), e.g.
// after a failed ss_init_shard) and the last one per shard.  SCOPE(s) at the
// top of an entry point makes FAIL / CUDA_TRY record into that shard too.
static thread_local std::string g_err;
static thread_local ss_shard* g_scope = nullptr;
struct ScopeGuard {
  ss_shard* prev;
  explicit ScopeGuard(ss_shard* s) : prev(g_scope) { g_scope = s; }
  ~ScopeGuard() { g_scope = prev; }
};
#define SCOPE(s) ScopeGuard scope_guard_((s))
static void set_err(const std::string& m) {
  g_err = m;
  if (g_scope) g_scope->err = m;
}

#define FAIL(code, msg)  \
  do {                   \
    set_err(msg);        \
    return (code);       \
  } while (0)
#define CUDA_TRY(x)                                                            \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess) {                                                   \
      set_err(std::string(#x) + ": " + cudaGetErrorString(e_));                \
      return SS_ECUDA;                                                         \
    }                                                                          \
  } while (0)
// a host_logic.h check: propagate its status and message
#define HOST_CHECK(call, ...)                              \
  do {                                                     \
    std::string m_;                                        \
    ss_status r_ = ss::host::call(__VA_ARGS__, m_);        \
    if (r_ != SS_OK) FAIL(r_, m_);                         \
  } while (0)

extern "C" const char* ss_last_error(const ss_shard* s) { return s ? s->err.c_str() : g_err.c_str(); }

// ------------------------------------------------------------ generator keys
// Mirror of synth/generators.py stream_key / tensor_id.
static uint64_t fmix64_h(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}
static uint64_t tensor_id(int layer, int kind, int sub) {
  return ((uint64_t)(layer + 1) << 16) | ((uint64_t)kind << 4) | (uint64_t)sub;
}
static uint64_t stream_key(uint64_t seed, uint64_t tid) {
  return fmix64_h(fmix64_h(seed * 0x9E3779B97F4A7C15ull + 1) ^ (tid * 0xD1B54A32D192ED03ull));
}
static float scale_const(int K) { return (float)(1.0 / (4.64 * std::sqrt((double)K))); }

// ------------------------------------------------------------ helpers
// bf16 <-> fp16 <-> fp32 bit conversions for the fp16 KV cache (host side)
static float bits_f32(uint32_t b) {
  float f;
  std::memcpy(&f, &b, 4);
  return f;
}
static bool bf16_fits_f16(uint16_t b) {
  float f = bits_f32((uint32_t)b << 16);
  return std::isfinite(f) && std::fabs(f) <= 65504.0f;
}
static uint16_t bf16_to_f16(uint16_t b) {  // exact for normal-range values
  float f = bits_f32((uint32_t)b << 16);
  uint32_t x;
  std::memcpy(&x, &f, 4);
  uint32_t sign = (x >> 16) & 0x8000u;
  int e = (int)((x >> 23) & 0xFF) - 127 + 15;
  uint32_t mant = x & 0x7FFFFFu;
  if ((x & 0x7FFFFFFFu) == 0) return (uint16_t)sign;
  if (e >= 31) return (uint16_t)(sign | 0x7C00u);
  if (e <= 0) {  // fp16 subnormal: round to nearest even
    if (e < -10) return (uint16_t)sign;
    mant |= 0x800000u;
    int shift = 14 - e;
    uint32_t h = mant >> shift, rem = mant & ((1u << shift) - 1), half = 1u << (shift - 1);
    if (rem > half || (rem == half && (h & 1))) ++h;
    return (uint16_t)(sign | h);
  }
  uint32_t h = sign | ((uint32_t)e << 10) | (mant >> 13);
  uint32_t rem = mant & 0x1FFFu;
  if (rem > 0x1000u || (rem == 0x1000u && (h & 1))) ++h;
  return (uint16_t)h;
}
static float f16_to_f32(uint16_t h) {
  uint32_t sign = (uint32_t)(h & 0x8000u) << 16;
  int e = (h >> 10) & 0x1F;
  uint32_t mant = h & 0x3FFu;
  if (e == 0) {
    float f = std::ldexp((float)mant, -24);
    return sign ? -f : f;
  }
  if (e == 31) return bits_f32(sign | 0x7F800000u | (mant << 13));
  return bits_f32(sign | ((uint32_t)(e - 15 + 127) << 23) | (mant << 13));
}
static int round_up(int a, int b) { return (a + b - 1) / b * b; }
static int nt_of(int T) {
  int nt = (T + 7) / 8;
  return nt <= 1 ? 1 : nt <= 2 ? 2 : nt <= 4 ? 4 : 8;
}

template <class T>
static cudaError_t dalloc(T** p, size_t bytes) {
  cudaError_t e = cudaMalloc((void**)p, bytes ? bytes : 16);
  if (e == cudaSuccess) e = cudaMemset(*p, 0, bytes ? bytes : 16);
  return e;
}

static void setup_linear(PackedLinear& pl, int K, int N) {
  pl.K = K;
  pl.N = round_up(N, 128);
  pl.n_tg = pl.N / 128;
  pl.S = K / kW4KS;
  pl.bytes = (size_t)pl.n_tg * pl.S * kW4UnitBytes;
}

// mapping of packed local rows / k to canonical parts (same as misc.cu lin_map)
static bool lin_map_h(const LinMap& m, int row, int k, int& part, int& n, int& kk) {
  kk = k;
  if (m.mode == 0) {
    int nq = m.Hq_l * m.d, nk = m.Hkv_l * m.d;
    if (row < nq) { part = 0; n = m.rank * nq + row; }
    else if (row < nq + nk) { part = 1; n = m.rank * nk + row - nq; }
    else if (row < nq + 2 * nk) { part = 2; n = m.rank * nk + row - nq - nk; }
    else return false;
    if (n >= (part == 0 ? m.q_full : m.kv_full)) return false;  // zero-padded head
  } else if (m.mode == 1 || m.mode == 3) {
    part = 0; n = row; kk = m.rank * m.Kl + k;
    if (kk >= m.K_full) return false;  // zero-padded input rows
  } else {
    int tg = row >> 7, r = row & 127;
    part = r < 64 ? 0 : 1;
    if (tg * 64 + (r & 63) >= m.I_l) return false;
    n = m.rank * m.I_l + tg * 64 + (r & 63);
    if (n >= m.I_full) return false;  // zero-padded intermediate columns
  }
  return true;
}

static LinMap make_map(const ss_shard* s, int mode, int Kl) {
  LinMap m{};
  m.mode = mode;
  m.rank = s->rank;
  m.Hq_l = s->Hq_l;
  m.Hkv_l = s->Hkv_l;
  m.d = s->cfg.head_dim;
  m.I_l = s->I_l;
  m.Kl = Kl;
  const ss_model_cfg& c = s->cfg;
  m.q_full = c.n_heads * c.head_dim;
  m.kv_full = c.n_kv_heads * c.head_dim;
  m.I_full = c.intermediate;
  m.K_full = mode == 1 ? m.q_full : mode == 3 ? m.I_full : 1 << 30;
  return m;
}

// Host repack of canonical parts into W4 units (mirror of synth_linear_kernel).
static void pack_w4_host(const PackedLinear& pl, const LinMap& m, const CanonLinear* parts[3], const int Nfull[3],
                         std::vector<uint8_t>& out) {
  out.assign(pl.bytes, 0);
  for (int tg = 0; tg < pl.n_tg; ++tg)
    for (int s = 0; s < pl.S; ++s) {
      uint8_t* ub = out.data() + ((size_t)tg * pl.S + s) * kW4UnitBytes;
      uint32_t* words = reinterpret_cast<uint32_t*>(ub);
      for (int warp = 0; warp < 8; ++warp)
        for (int kb = 0; kb < 4; ++kb)
          for (int lane = 0; lane < 32; ++lane)
            for (int j = 0; j < 4; ++j) {
              int gq = lane >> 2, tq = lane & 3;
              uint32_t word = 0;
              for (int p = 0; p < 8; ++p) {
                int row = tg * 128 + warp * 16 + gq + 8 * (p & 1);
                int k = s * 256 + kb * 64 + j * 16 + 2 * tq + (p >> 2) + 8 * ((p >> 1) & 1);
                int part, n, kk;
                uint32_t q = 8;
                if (lin_map_h(m, row, k, part, n, kk)) q = parts[part]->q[(size_t)kk * Nfull[part] + n];
                word |= (q & 15u) << (4 * p);
              }
              words[((warp * 4 + kb) * 32 + lane) * 4 + j] = word;
            }
      for (int warp = 0; warp < 8; ++warp)
        for (int grp = 0; grp < 2; ++grp) {
          uint16_t sv[16];
          uint32_t zv[16];
          for (int i = 0; i < 16; ++i) {
            int row = tg * 128 + warp * 16 + i;
            int part, n, kk;
            sv[i] = 0;
            zv[i] = 8;
            if (lin_map_h(m, row, (s * 2 + grp) * 128, part, n, kk)) {
              size_t gi = (size_t)(kk / 128) * Nfull[part] + n;
              sv[i] = parts[part]->s[gi];
              zv[i] = parts[part]->z[gi] & 15u;
            }
          }
          // lane-indexed pairs (rows gq, gq+8): see common.cuh
          uint32_t* sc = reinterpret_cast<uint32_t*>(ub + kW4Bytes) + (warp * 2 + grp) * 8;
          uint8_t* zb = ub + kW4Bytes + 512 + (warp * 2 + grp) * 8;
          for (int gq = 0; gq < 8; ++gq) {
            sc[gq] = (uint32_t)sv[gq] | ((uint32_t)sv[gq + 8] << 16);
            zb[gq] = (uint8_t)(zv[gq] | (zv[gq + 8] << 4));
          }
        }
    }
}

static void pack_lm_host(const std::vector<uint16_t>& W, int V_full, int V_l, int V_off, int h, int n_tg,
                         std::vector<uint8_t>& out) {
  const int S = h / 64;
  out.assign((size_t)n_tg * S * kBFUnitBytes, 0);
  uint32_t* words = reinterpret_cast<uint32_t*>(out.data());
  size_t nw = out.size() / 4;
  for (size_t i = 0; i < nw; ++i) {
    size_t u = i / 4096;
    int w_in = (int)(i % 4096);
    int tg = (int)(u / S), s = (int)(u % S);
    int warp = w_in >> 9, j = (w_in >> 7) & 3, lane = (w_in >> 2) & 31, r = w_in & 3;
    int gq = lane >> 2, tq = lane & 3;
    int row = tg * 128 + warp * 16 + gq + 8 * (r & 1);
    int k = s * 64 + j * 16 + 2 * tq + 8 * (r >> 1);
    int v = V_off + row;
    uint32_t word = 0;
    if (row < V_l && v < V_full) word = (uint32_t)W[(size_t)v * h + k] | ((uint32_t)W[(size_t)v * h + k + 1] << 16);
    words[i] = word;
  }
}

// ------------------------------------------------------------ lifecycle
extern "C" ss_status ss_init_shard(const ss_model_cfg* cfg, int32_t tp_rank, int32_t tp_size, int32_t device,
                                   ss_shard** out) {
  if (!cfg || !out) FAIL(SS_EINVAL, "null argument");
  *out = nullptr;
  const ss_model_cfg& c = *cfg;
  if (tp_size < 1 || tp_size > kMaxPeers) FAIL(SS_EINVAL, "tp_size must be in [1, 8]");
  if (tp_rank < 0 || tp_rank >= tp_size) FAIL(SS_EINVAL, "tp_rank out of range");
  if (c.group_size != SS_GROUP) FAIL(SS_EINVAL, "group_size must be 128");
  if (c.head_dim != 64 && c.head_dim != 128) FAIL(SS_EINVAL, "head_dim must be 64 or 128");
  if (c.n_layers < 1 || c.hidden < 256 || c.vocab < 2 || c.n_heads < 1 || c.n_kv_heads < 1)
    FAIL(SS_EINVAL, "bad model shape");
  if (c.n_heads % c.n_kv_heads) FAIL(SS_EINVAL, "n_heads must be a multiple of n_kv_heads");
  if (c.hidden % kW4KS) FAIL(SS_EINVAL, "hidden must be a multiple of 256");
  // Arbitrary TP by zero padding: kv heads (with their query
  // heads) padded to a multiple of tp_size, the intermediate size to a
  // multiple of 256 tp_size when tp_size does not split it into 256-multiples;
  // padded weights are zero, so the padded model equals the unpadded one.
  const int Hkv_pad = (c.n_kv_heads + tp_size - 1) / tp_size * tp_size;
  const int Hq_pad = Hkv_pad * (c.n_heads / c.n_kv_heads);
  const int I_pad = (c.intermediate % tp_size || (c.intermediate / tp_size) % kW4KS)
                        ? (c.intermediate + kW4KS * tp_size - 1) / (kW4KS * tp_size) * (kW4KS * tp_size)
                        : c.intermediate;
  if ((Hq_pad / tp_size * c.head_dim) % kW4KS)
    FAIL(SS_EINVAL, "padded n_heads*head_dim/tp must be a multiple of 256");
  if (c.hidden > 8192) FAIL(SS_EINVAL, "hidden must be <= 8192");
  if (c.max_tree < 1 || c.max_tree > SS_MAX_TREE) FAIL(SS_EINVAL, "max_tree must be in [1, 64]");
  if (c.max_ctx < c.max_tree) FAIL(SS_EINVAL, "max_ctx too small");
  int G = c.n_heads / c.n_kv_heads;
  if (G * nt_of(c.max_tree) * 8 > 512) FAIL(SS_EINVAL, "(n_heads/n_kv_heads) * max_tree too large (<= 512 rows)");

  CUDA_TRY(cudaSetDevice(device));
  warm_gemm_kernels();
  warm_attention_kernels();
  warm_misc_kernels();
  warm_draft_kernels();
  arm_watchdog_record();
  warm_step_kernels();
  ss_shard* s = new ss_shard();
  s->cfg = c;
  s->rank = tp_rank;
  s->P = tp_size;
  s->device = device;
  cudaDeviceGetAttribute(&s->n_sm, cudaDevAttrMultiProcessorCount, device);
  s->Hq_l = Hq_pad / tp_size;
  s->Hkv_l = Hkv_pad / tp_size;
  s->I_l = I_pad / tp_size;
  s->G = G;
  int vp = (c.vocab + tp_size - 1) / tp_size;
  s->V_off = tp_rank * vp;
  s->V_l = std::max(0, std::min(c.vocab, (tp_rank + 1) * vp) - s->V_off);
  s->V_l_pad = round_up(std::max(s->V_l, 1), 128);
  s->max_ctx_pad = round_up(c.max_ctx, 64);
  s->hs.max_ctx = c.max_ctx;
  s->hs.max_tree = c.max_tree;
  s->hs.vocab = c.vocab;
  s->hs.peers_ready = tp_size == 1;
  const int h = c.hidden, d = c.head_dim;

  auto fail = [&](ss_status st) {
    ss_destroy(s);
    return st;
  };
#define A(ptr, bytes)                                                        \
  do {                                                                       \
    cudaError_t e_ = dalloc(&(ptr), (bytes));                                \
    if (e_ != cudaSuccess) {                                                 \
      set_err(std::string("cudaMalloc ") + #ptr + ": " + cudaGetErrorString(e_)); \
      return fail(SS_ECUDA);                                                 \
    }                                                                        \
  } while (0)

  s->layers.resize(c.n_layers);
  s->loaded_mask.assign(c.n_layers, 0);
  for (auto& lw : s->layers) {
    setup_linear(lw.qkv, h, (s->Hq_l + 2 * s->Hkv_l) * d);
    setup_linear(lw.o, s->Hq_l * d, h);
    setup_linear(lw.gu, h, 2 * s->I_l);
    setup_linear(lw.down, s->I_l, h);
    A(lw.qkv.d, lw.qkv.bytes);
    A(lw.o.d, lw.o.bytes);
    A(lw.gu.d, lw.gu.bytes);
    A(lw.down.d, lw.down.bytes);
    A(lw.attn_norm, h * 2);
    A(lw.mlp_norm, h * 2);
  }
  A(s->embed, (size_t)c.vocab * h * 2);
  A(s->final_norm, h * 2);
  s->lm_head.K = h;
  s->lm_head.N = s->V_l_pad;
  s->lm_head.n_tg = s->V_l_pad / 128;
  s->lm_head.S = h / kBFKS;
  s->lm_head.bytes = (size_t)s->lm_head.n_tg * s->lm_head.S * kBFUnitBytes;
  A(s->lm_head.d, s->lm_head.bytes);

  size_t kv_elems = (size_t)c.n_layers * s->Hkv_l * s->max_ctx_pad * d;
  A(s->kcache, kv_elems * 2);
  A(s->vcache, kv_elems * 2);
  A(s->rope_cs, (size_t)s->max_ctx_pad * (d / 2) * sizeof(float2));
  launch_rope_table(s->rope_cs, s->max_ctx_pad, d, (double)c.rope_theta, 0);

  A(s->x, (size_t)SS_MAX_TREE * h * 4);
  // W4 activations: K/256 stages x (NT=8: 32 KB fragments + 512 B group sums)
  A(s->act_h, (size_t)(h / 256) * 8 * 4160);
  A(s->act_o, (size_t)(s->Hq_l * d / 256) * 8 * 4160);
  A(s->act_d, (size_t)(s->I_l / 256) * 8 * 4160);
  A(s->act_lm, (size_t)h * 256);
  A(s->qbuf, (size_t)s->Hkv_l * G * SS_MAX_TREE * d * 2);  // fp16, swizzled rows
  A(s->attn_ws, (size_t)s->Hkv_l * 2 * 64 * 256 * d * 4);
  A(s->attn_ml, (size_t)s->Hkv_l * 2 * 64 * 256 * 2 * 4);
  A(s->attn_bar, (size_t)s->Hkv_l * 2 * 2 * 4);
  auto mk_scratch = [&](GemmScratch& g, int n_tg) -> bool {
    g.accum_elems = (size_t)n_tg * 128 * 64;
    if (dalloc(&g.accum, g.accum_elems * 4) != cudaSuccess) return false;
    if (dalloc(&g.counters, (size_t)(n_tg + 2) * 4) != cudaSuccess) return false;
    if (dalloc(&g.ss, (size_t)SS_MAX_TREE * 4) != cudaSuccess) return false;
    if (dalloc(&g.nbar, 16) != cudaSuccess) return false;
    return true;
  };
  if (!mk_scratch(s->sc_qkv, s->layers[0].qkv.n_tg) || !mk_scratch(s->sc_o, s->layers[0].o.n_tg) ||
      !mk_scratch(s->sc_gu, s->layers[0].gu.n_tg) || !mk_scratch(s->sc_down, s->layers[0].down.n_tg) ||
      !mk_scratch(s->sc_lm, s->lm_head.n_tg)) {
    set_err("cudaMalloc scratch failed");
    return fail(SS_ECUDA);
  }
  A(s->logits_dev, (size_t)SS_MAX_TREE * s->V_l_pad * 4);
  // persistent step kernel (step.cu)
  s->step_max_ctas = s->n_sm * 2;
  A(s->step_ctr, ((size_t)c.n_layers * kCtrPerLayer + kCtrGlobal) * 4);
  A(s->step_ss, (size_t)(c.n_layers + 1) * 2 * 64 * 4);
  A(s->step_ssx, (size_t)(c.n_layers + 1) * 2 * 64 * 8);
  A(s->qf, (size_t)2 * s->Hkv_l * G * 64 * d * 2);
  A(s->klo, (size_t)s->Hkv_l * 128 * d * 2);
  A(s->vlo, (size_t)s->Hkv_l * 128 * d * 2);
  A(s->att_ws, (size_t)s->step_max_ctas * 2 * 64 * d * 4);
  A(s->att_ml, (size_t)s->step_max_ctas * 2 * 64 * sizeof(float2));
  A(s->layer_tab, (size_t)c.n_layers * sizeof(LayerPtrs));
  A(s->step_args_dev, 6 * sizeof(StepArgs));  // [NT = 1, 2, 4][logits off / on]
  {
    std::vector<LayerPtrs> tab(c.n_layers);
    for (int l = 0; l < c.n_layers; ++l)
      tab[l] = LayerPtrs{s->layers[l].qkv.d, s->layers[l].o.d, s->layers[l].gu.d, s->layers[l].down.d,
                         s->layers[l].attn_norm, s->layers[l].mlp_norm};
    if (cudaMemcpy(s->layer_tab, tab.data(), tab.size() * sizeof(LayerPtrs), cudaMemcpyHostToDevice) != cudaSuccess) {
      set_err("layer table copy failed");
      return fail(SS_ECUDA);
    }
  }
  A(s->dstate, sizeof(DevState));
  A(s->d_tree_in, 2 * SS_MAX_TREE * 4);
  A(s->d_topk, (32 * 32 * 2 + 32) * 4);
  if (cudaMallocHost((void**)&s->hstate, sizeof(DevState)) != cudaSuccess ||
      cudaMallocHost((void**)&s->h_tree_in, 2 * SS_MAX_TREE * 4) != cudaSuccess) {
    set_err("cudaMallocHost failed");
    return fail(SS_ECUDA);
  }
  {
    DevState init{};
    init.epoch = 1;
    init.eos = -1;
    init.mbox_post = tp_rank == 0 ? 1 : 0;
    if (cudaMemcpy(s->dstate, &init, sizeof(DevState), cudaMemcpyHostToDevice) != cudaSuccess) {
      set_err("init state copy failed");
      return fail(SS_ECUDA);
    }
  }
  // LL receive buffer: [2 parities][P][n_tg_total][128 rows][32 lines] x 16 B
  // (fp32 pairs + flags), then the argmax area [P][64] and the debug
  // consistency area [P] (consistency_line_offset)
  A(s->mbox_in, (size_t)(1 + SS_MAX_TREE) * 16);
  if (tp_size > 1) {
    // + the two-shot broadcast area [2 parities][n_tg_total][128 rows][32 lines]
    s->recv_bytes = ((size_t)2 * tp_size * (h / 128) * 128 * 32 + (size_t)tp_size * 64 + (size_t)tp_size +
                     (size_t)2 * (h / 128) * 128 * 32) * 16;
    A(s->recv, s->recv_bytes);
  }
  if (cudaStreamCreateWithFlags(&s->cap_stream, cudaStreamNonBlocking) != cudaSuccess) {
    set_err("stream create failed");
    return fail(SS_ECUDA);
  }
  if (cudaDeviceSynchronize() != cudaSuccess) {
    set_err(std::string("init: ") + cudaGetErrorString(cudaGetLastError()));
    return fail(SS_ECUDA);
  }
#undef A
  *out = s;
  return SS_OK;
}

extern "C" ss_status ss_destroy(ss_shard* s) {
  if (!s) return SS_OK;
  cudaSetDevice(s->device);
  cudaDeviceSynchronize();
  for (auto& kv : s->graphs)
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
  for (auto& lw : s->layers) {
    cudaFree(lw.qkv.d); cudaFree(lw.o.d); cudaFree(lw.gu.d); cudaFree(lw.down.d);
    cudaFree(lw.attn_norm); cudaFree(lw.mlp_norm);
  }
  for (int p = 0; p < s->P; ++p)
    if (s->ipc_opened[p] && s->peer_recv[p]) cudaIpcCloseMemHandle(s->peer_recv[p]);
  void* ptrs[] = {s->embed, s->final_norm, s->lm_head.d, s->kcache, s->vcache, s->rope_cs, s->x, s->act_h,
                  s->act_o, s->act_d, s->act_lm, s->qbuf, s->attn_ws, s->attn_ml, s->attn_bar, s->logits_dev, s->dstate,
                  s->d_tree_in, s->recv, s->mbox_in, s->sc_qkv.accum, s->sc_qkv.counters, s->sc_o.accum, s->sc_o.counters,
                  s->sc_gu.accum, s->sc_gu.counters, s->sc_down.accum, s->sc_down.counters, s->sc_lm.accum,
                  s->sc_lm.counters, s->sc_o.ss, s->sc_o.nbar, s->sc_down.ss, s->sc_down.nbar, s->step_ctr,
                  s->step_ss, s->qf, s->klo, s->vlo, s->att_ws, s->att_ml, s->layer_tab, s->sc_qkv.ss,
                  s->sc_qkv.nbar, s->sc_gu.ss, s->sc_gu.nbar, s->sc_lm.ss, s->sc_lm.nbar, s->step_args_dev,
                  s->d_topk, s->step_ssx};
  if (s->step_trace_host) cudaFreeHost(s->step_trace_host);
  else if (s->step_trace) cudaFree(s->step_trace);
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (s->hstate) cudaFreeHost(s->hstate);
  if (s->h_tree_in) cudaFreeHost(s->h_tree_in);
  if (s->cap_stream) cudaStreamDestroy(s->cap_stream);
  delete s;
  return SS_OK;
}

extern "C" ss_status ss_set_launch_cap(ss_shard* s, int32_t cap) {
  SCOPE(s);
  if (!s) FAIL(SS_EINVAL, "null shard");
  s->launch_cap = cap > 0 ? cap : 0;
  for (auto& kv : s->graphs)
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
  s->graphs.clear();
  return SS_OK;
}

extern "C" ss_status ss_set_allreduce(ss_shard* s, int32_t mode) {
  SCOPE(s);
  if (!s) FAIL(SS_EINVAL, "null shard");
  if (mode != 0 && mode != 1) FAIL(SS_EINVAL, "mode must be 0 (one-shot) or 1 (two-shot)");
  cudaSetDevice(s->device);
  CUDA_TRY(cudaDeviceSynchronize());
  s->ar_mode = mode;
  for (auto& kv : s->graphs)
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
  s->graphs.clear();
  return SS_OK;
}

// ------------------------------------------------------------ weights
static const int kLinearKinds[] = {SS_W_Q, SS_W_K, SS_W_V, SS_W_O, SS_W_GATE, SS_W_UP, SS_W_DOWN};
static bool is_linear(int kind) {
  for (int k : kLinearKinds)
    if (k == kind) return true;
  return false;
}

static void linear_shape(const ss_model_cfg& c, int kind, int& K, int& N) {
  const int h = c.hidden, d = c.head_dim;
  switch (kind) {
    case SS_W_Q: K = h; N = c.n_heads * d; break;
    case SS_W_K: case SS_W_V: K = h; N = c.n_kv_heads * d; break;
    case SS_W_O: K = c.n_heads * d; N = h; break;
    case SS_W_GATE: case SS_W_UP: K = h; N = c.intermediate; break;
    default: K = c.intermediate; N = h; break;
  }
}

static ss_status try_pack_layer(ss_shard* s, int layer, int group_kind) {
  // group_kind: 0 = qkv (Q,K,V), 1 = o, 2 = gu (GATE,UP), 3 = down
  static const int members[4][3] = {{SS_W_Q, SS_W_K, SS_W_V}, {SS_W_O, -1, -1}, {SS_W_GATE, SS_W_UP, -1},
                                    {SS_W_DOWN, -1, -1}};
  const CanonLinear* parts[3] = {nullptr, nullptr, nullptr};
  int Nfull[3] = {0, 0, 0};
  for (int i = 0; i < 3; ++i) {
    int k = members[group_kind][i];
    if (k < 0) continue;
    auto it = s->staging.find((long)layer * 64 + k);
    if (it == s->staging.end() || !(it->second.hq && it->second.hz && it->second.hs)) return SS_OK;  // not yet
    parts[i] = &it->second;
    int K, N;
    linear_shape(s->cfg, k, K, N);
    Nfull[i] = N;
  }
  LayerW& lw = s->layers[layer];
  PackedLinear* pl = group_kind == 0 ? &lw.qkv : group_kind == 1 ? &lw.o : group_kind == 2 ? &lw.gu : &lw.down;
  int mode = group_kind;  // 0 QKV, 1 O, 2 GU, 3 DOWN
  LinMap m = make_map(s, mode, pl->K);
  std::vector<uint8_t> packed;
  pack_w4_host(*pl, m, parts, Nfull, packed);
  CUDA_TRY(cudaMemcpy(pl->d, packed.data(), packed.size(), cudaMemcpyHostToDevice));
  for (int i = 0; i < 3; ++i) {
    int k = members[group_kind][i];
    if (k >= 0) {
      s->staging.erase((long)layer * 64 + k);
      s->loaded_mask[layer] |= 1u << k;
    }
  }
  return SS_OK;
}

extern "C" ss_status ss_load_weights(ss_shard* s, int32_t layer, int32_t kind, int32_t sub, const void* host,
                                     size_t bytes) {
  SCOPE(s);
  if (!s || !host) FAIL(SS_EINVAL, "null argument");
  const ss_model_cfg& c = s->cfg;
  const int h = c.hidden;
  cudaSetDevice(s->device);
  if (is_linear(kind)) {
    if (layer < 0 || layer >= c.n_layers) FAIL(SS_EINVAL, "layer out of range");
    int K, N;
    linear_shape(c, kind, K, N);
    size_t want = sub == SS_SUB_QWEIGHT ? (size_t)K * N : sub == SS_SUB_QZEROS ? (size_t)(K / 128) * N
                                                                               : (size_t)(K / 128) * N * 2;
    if (sub < 0 || sub > 2) FAIL(SS_EINVAL, "bad sub-tensor");
    if (bytes != want) FAIL(SS_EINVAL, "byte count does not match the canonical shape");
    CanonLinear& cl = s->staging[(long)layer * 64 + kind];
    if (sub == SS_SUB_QWEIGHT) {
      cl.q.assign((const uint8_t*)host, (const uint8_t*)host + bytes);
      cl.hq = true;
    } else if (sub == SS_SUB_QZEROS) {
      cl.z.assign((const uint8_t*)host, (const uint8_t*)host + bytes);
      cl.hz = true;
    } else {
      cl.s.assign((const uint16_t*)host, (const uint16_t*)host + bytes / 2);
      cl.hs = true;
    }
    int grp = (kind == SS_W_Q || kind == SS_W_K || kind == SS_W_V) ? 0 : kind == SS_W_O ? 1
              : (kind == SS_W_GATE || kind == SS_W_UP) ? 2 : 3;
    return try_pack_layer(s, layer, grp);
  }
  switch (kind) {
    case SS_W_ATTN_NORM:
    case SS_W_MLP_NORM: {
      if (layer < 0 || layer >= c.n_layers) FAIL(SS_EINVAL, "layer out of range");
      if (bytes != (size_t)h * 2) FAIL(SS_EINVAL, "norm must be hidden bf16 values");
      uint16_t* dst = kind == SS_W_ATTN_NORM ? s->layers[layer].attn_norm : s->layers[layer].mlp_norm;
      CUDA_TRY(cudaMemcpy(dst, host, bytes, cudaMemcpyHostToDevice));
      s->loaded_mask[layer] |= 1u << kind;
      return SS_OK;
    }
    case SS_W_FINAL_NORM:
      if (bytes != (size_t)h * 2) FAIL(SS_EINVAL, "norm must be hidden bf16 values");
      CUDA_TRY(cudaMemcpy(s->final_norm, host, bytes, cudaMemcpyHostToDevice));
      s->global_mask |= 1u << kind;
      return SS_OK;
    case SS_W_EMBED:
      if (bytes != (size_t)c.vocab * h * 2) FAIL(SS_EINVAL, "embed must be [vocab][hidden] bf16");
      CUDA_TRY(cudaMemcpy(s->embed, host, bytes, cudaMemcpyHostToDevice));
      s->global_mask |= 1u << kind;
      return SS_OK;
    case SS_W_LM_HEAD: {
      if (bytes != (size_t)c.vocab * h * 2) FAIL(SS_EINVAL, "lm_head must be [vocab][hidden] bf16");
      std::vector<uint16_t> W((const uint16_t*)host, (const uint16_t*)host + bytes / 2);
      std::vector<uint8_t> packed;
      pack_lm_host(W, c.vocab, s->V_l, s->V_off, h, s->lm_head.n_tg, packed);
      CUDA_TRY(cudaMemcpy(s->lm_head.d, packed.data(), packed.size(), cudaMemcpyHostToDevice));
      s->global_mask |= 1u << kind;
      return SS_OK;
    }
    default:
      FAIL(SS_EINVAL, "unknown weight kind");
  }
}

extern "C" ss_status ss_synth_weights(ss_shard* s, uint64_t seed) {
  SCOPE(s);
  if (!s) FAIL(SS_EINVAL, "null shard");
  cudaSetDevice(s->device);
  const ss_model_cfg& c = s->cfg;
  const int h = c.hidden, d = c.head_dim;
  for (int l = 0; l < c.n_layers; ++l) {
    LayerW& lw = s->layers[l];
    struct G {
      PackedLinear* pl;
      int mode;
      int kinds[3];
    } groups[4] = {{&lw.qkv, 0, {SS_W_Q, SS_W_K, SS_W_V}},
                   {&lw.o, 1, {SS_W_O, -1, -1}},
                   {&lw.gu, 2, {SS_W_GATE, SS_W_UP, -1}},
                   {&lw.down, 3, {SS_W_DOWN, -1, -1}}};
    for (auto& g : groups) {
      SynthLinArgs a{};
      for (int i = 0; i < 3; ++i) {
        int k = g.kinds[i];
        if (k < 0) continue;
        for (int sub = 0; sub < 3; ++sub) a.keys[i][sub] = stream_key(seed, tensor_id(l, k, sub));
        int K, N;
        linear_shape(c, k, K, N);
        a.scale_c[i] = scale_const(K);
        a.N_full[i] = N;
      }
      a.m = make_map(s, g.mode, g.pl->K);
      a.n_tg = g.pl->n_tg;
      a.S = g.pl->S;
      launch_synth_linear_args(g.pl->d, a, 0);
    }
    launch_synth_dense_key(lw.attn_norm, h, stream_key(seed, tensor_id(l, SS_W_ATTN_NORM, 0)), 0, 1, 0.f, 0);
    launch_synth_dense_key(lw.mlp_norm, h, stream_key(seed, tensor_id(l, SS_W_MLP_NORM, 0)), 0, 1, 0.f, 0);
    s->loaded_mask[l] = 0xFFFFFFFFu;
  }
  launch_synth_dense_key(s->embed, (size_t)c.vocab * h, stream_key(seed, tensor_id(-1, SS_W_EMBED, 0)), 0, 0, 1.0f, 0);
  launch_synth_dense_key(s->final_norm, h, stream_key(seed, tensor_id(-1, SS_W_FINAL_NORM, 0)), 0, 1, 0.f, 0);
  float lm_scale = (float)(4.0 / std::sqrt((double)h));
  launch_synth_lm_key(s->lm_head.d, s->V_l, s->V_off, c.vocab, h, s->lm_head.n_tg,
                      stream_key(seed, tensor_id(-1, SS_W_LM_HEAD, 0)), lm_scale, 0);
  s->global_mask = 0xFFFFFFFFu;
  CUDA_TRY(cudaDeviceSynchronize());
  (void)d;
  return SS_OK;
}

static bool weights_complete(const ss_shard* s) {
  const uint32_t need = (1u << SS_W_ATTN_NORM) | (1u << SS_W_Q) | (1u << SS_W_K) | (1u << SS_W_V) | (1u << SS_W_O) |
                        (1u << SS_W_MLP_NORM) | (1u << SS_W_GATE) | (1u << SS_W_UP) | (1u << SS_W_DOWN);
  for (uint32_t m : s->loaded_mask)
    if ((m & need) != need) return false;
  const uint32_t gneed = (1u << SS_W_EMBED) | (1u << SS_W_FINAL_NORM) | (1u << SS_W_LM_HEAD);
  return (s->global_mask & gneed) == gneed;
}

// ------------------------------------------------------------ KV
// Set the committed length on the device and the host view; rows [0, rows)
// now hold data (prefix) -- DevState::max_written mirrors hs.max_written.
static ss_status write_L(ss_shard* s, int L, int rows_written) {
  s->hs.max_written = std::max(s->hs.max_written, rows_written);
  int32_t v[2] = {L, 0};
  CUDA_TRY(cudaMemcpy(&s->dstate->L, &v[0], 4, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(&s->dstate->max_written, &s->hs.max_written, 4, cudaMemcpyHostToDevice));
  ss::host::on_set_len(s->hs, L);
  int zero = 0;
  CUDA_TRY(cudaMemcpy(&s->dstate->have_verify, &zero, 4, cudaMemcpyHostToDevice));
  return SS_OK;
}

extern "C" ss_status ss_set_prefix_kv(ss_shard* s, int32_t layer, const void* k, const void* v, int32_t len) {
  SCOPE(s);
  if (!s || (!k && len) || (!v && len)) FAIL(SS_EINVAL, "null argument");
  const ss_model_cfg& c = s->cfg;
  if (layer < 0 || layer >= c.n_layers) FAIL(SS_EINVAL, "layer out of range");
  if (len < 0 || len + c.max_tree > c.max_ctx) FAIL(SS_ECAPACITY, "prefix + max_tree exceeds max_ctx");
  cudaSetDevice(s->device);
  const int d = c.head_dim, Hf = c.n_kv_heads, kv0 = s->rank * s->Hkv_l;
  const int rows = round_up(std::max(len, 1), 64);
  std::vector<uint16_t> buf((size_t)rows * d);
  // the cache is fp16: every bf16 input value must be representable
  for (int which = 0; which < 2; ++which) {
    const uint16_t* src = (const uint16_t*)(which ? v : k);
    for (size_t i = 0; i < (size_t)len * Hf * d; ++i)
      if (!bf16_fits_f16(src[i])) FAIL(SS_EINVAL, "prefix K/V value outside the fp16 range of the cache");
  }
  for (int which = 0; which < 2; ++which) {
    const uint16_t* src = (const uint16_t*)(which ? v : k);
    uint16_t* cache = which ? s->vcache : s->kcache;
    for (int kh = 0; kh < s->Hkv_l; ++kh) {
      std::fill(buf.begin(), buf.end(), 0);
      for (int pos = 0; pos < len; ++pos)
        for (int j = 0; j < d; ++j) {
          int r = pos & 63, cidx = (j >> 3) ^ (r & 7);
          buf[(size_t)(pos - r) * d + r * d + cidx * 8 + (j & 7)] =
              kv0 + kh < Hf ? bf16_to_f16(src[((size_t)pos * Hf + kv0 + kh) * d + j]) : (uint16_t)0;  // padded head
        }
      size_t base = ((size_t)layer * s->Hkv_l + kh) * s->max_ctx_pad * d;
      CUDA_TRY(cudaMemcpy(cache + base, buf.data(), (size_t)rows * d * 2, cudaMemcpyHostToDevice));
    }
  }
  if (layer == c.n_layers - 1) return write_L(s, len, len);
  return SS_OK;
}

extern "C" ss_status ss_synth_prefix_kv(ss_shard* s, uint64_t seed, int32_t len) {
  SCOPE(s);
  if (!s) FAIL(SS_EINVAL, "null shard");
  const ss_model_cfg& c = s->cfg;
  if (len < 0 || len + c.max_tree > c.max_ctx) FAIL(SS_ECAPACITY, "prefix + max_tree exceeds max_ctx");
  cudaSetDevice(s->device);
  for (int l = 0; l < c.n_layers; ++l) {
    if (len == 0) break;
    launch_synth_kv_key(s->kcache, l, c.n_kv_heads, s->Hkv_l, s->rank * s->Hkv_l, c.head_dim, len, s->max_ctx_pad,
                        stream_key(seed, tensor_id(l, 12, 0)), 0);
    launch_synth_kv_key(s->vcache, l, c.n_kv_heads, s->Hkv_l, s->rank * s->Hkv_l, c.head_dim, len, s->max_ctx_pad,
                        stream_key(seed, tensor_id(l, 13, 0)), 0);
  }
  CUDA_TRY(cudaDeviceSynchronize());
  return write_L(s, len, len);
}

extern "C" ss_status ss_read_kv(ss_shard* s, int32_t layer, int32_t row0, int32_t n, float* k_out, float* v_out) {
  SCOPE(s);
  if (!s || !k_out || !v_out) FAIL(SS_EINVAL, "null argument");
  const ss_model_cfg& c = s->cfg;
  if (layer < 0 || layer >= c.n_layers || row0 < 0 || n < 0 || row0 + n > s->max_ctx_pad)
    FAIL(SS_EINVAL, "row range out of bounds");
  cudaSetDevice(s->device);
  CUDA_TRY(cudaDeviceSynchronize());
  const int d = c.head_dim;
  int b0 = row0 / 64 * 64, b1 = round_up(row0 + n, 64);
  std::vector<uint16_t> buf((size_t)(b1 - b0) * d);
  for (int which = 0; which < 2; ++which) {
    float* dst = which ? v_out : k_out;
    const uint16_t* cache = which ? s->vcache : s->kcache;
    for (int kh = 0; kh < s->Hkv_l; ++kh) {
      size_t base = ((size_t)layer * s->Hkv_l + kh) * s->max_ctx_pad * d + (size_t)b0 * d;
      CUDA_TRY(cudaMemcpy(buf.data(), cache + base, buf.size() * 2, cudaMemcpyDeviceToHost));
      for (int i = 0; i < n; ++i) {
        int pos = row0 + i, r = pos & 63;
        for (int j = 0; j < d; ++j) {
          int cidx = (j >> 3) ^ (r & 7);
          dst[((size_t)i * s->Hkv_l + kh) * d + j] = f16_to_f32(buf[(size_t)(pos - r - b0) * d + r * d + cidx * 8 + (j & 7)]);
        }
      }
    }
  }
  return SS_OK;
}

// Read the device-side committed length and rows-written bound back (after
// device-driven commits the host only knows an upper bound).
static ss_status sync_L(ss_shard* s) {
  if (s->hs.L_known) return SS_OK;
  cudaSetDevice(s->device);
  CUDA_TRY(cudaDeviceSynchronize());
  int32_t L = -1, mw = 0;
  CUDA_TRY(cudaMemcpy(&L, &s->dstate->L, 4, cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemcpy(&mw, &s->dstate->max_written, 4, cudaMemcpyDeviceToHost));
  s->hs.L = L;
  s->hs.L_known = true;
  s->hs.max_written = std::max(s->hs.max_written, std::max(mw, L));
  return SS_OK;
}

extern "C" ss_status ss_set_committed_len(ss_shard* s, int32_t L) {
  SCOPE(s);
  if (!s) FAIL(SS_EINVAL, "null shard");
  cudaSetDevice(s->device);
  CUDA_TRY(cudaDeviceSynchronize());
  ss_status r = sync_L(s);
  if (r != SS_OK) return r;
  int32_t mw = 0;
  CUDA_TRY(cudaMemcpy(&mw, &s->dstate->max_written, 4, cudaMemcpyDeviceToHost));
  s->hs.max_written = std::max(s->hs.max_written, mw);
  HOST_CHECK(check_set_len, s->hs, L);
  return write_L(s, L, 0);
}

extern "C" int32_t ss_committed_len(ss_shard* s) {
  SCOPE(s);
  if (!s) return -1;
  if (sync_L(s) != SS_OK) return -1;
  return s->hs.L;
}

// ------------------------------------------------------------ the step
static GemmArgs gemm_args(ss_shard* s, const PackedLinear& pl, const uint8_t* act, GemmScratch& sc, int kind,
                          int layer) {
  GemmArgs g;
  g.W = pl.d;
  g.act = act;
  g.n_tg = pl.n_tg;
  g.S = pl.S;
  g.accum = sc.accum;
  g.counters = sc.counters;
  g.ss = sc.ss;
  g.nbar = sc.nbar;
  g.eps = s->cfg.rms_eps;
  g.n_sm = s->n_sm;
  EpiArgs& e = g.epi;
  e.kind = kind;
  e.st = s->dstate;
  e.layer = layer;
  e.d = s->cfg.head_dim;
  e.Hq_l = s->Hq_l;
  e.Hkv_l = s->Hkv_l;
  e.G = s->G;
  e.max_ctx_pad = s->max_ctx_pad;
  e.qbuf = s->qbuf;
  e.kc = s->kcache;
  e.vc = s->vcache;
  e.rope_cs = s->rope_cs;
  e.x = s->x;
  e.h = s->cfg.hidden;
  e.rank = s->rank;
  e.P = s->P;
  e.n_tg_total = s->cfg.hidden / 128;
  e.recv = s->recv;
  for (int p = 0; p < s->P; ++p) e.peer_recv[p] = s->peer_recv[p];
  e.loopback = s->loopback ? 1 : 0;
  e.act_out = s->act_d;
  e.V_l = s->V_l;
  e.V_off = s->V_off;
  e.logits_ld = s->V_l_pad;
  return g;
}

// Optional per-kernel event bracketing (ss_profile_step, eager launches only).
struct Prof {
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> ev;
  size_t next = 0;
  cudaStream_t st = nullptr;
  void begin(int kind) {
    if (next == ev.size()) {
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      ev.push_back({kind, {a, b}});
    }
    ev[next].first = kind;
    cudaEventRecord(ev[next].second.first, st);
  }
  void end() { cudaEventRecord(ev[next++].second.second, st); }
};
static Prof* g_prof = nullptr;
#define PROF_BEGIN(k) \
  if (g_prof) g_prof->begin(k)
#define PROF_END() \
  if (g_prof) g_prof->end()

// Whether the persistent step kernel runs this tree width: T <= 32 (NT <= 4)
// and every attention (kv head, 64-row chunk) group fits the grid.
static bool step_path(const ss_shard* s, int NT) {
  if (!s->use_step || NT > 4 || s->cfg.n_layers > kStepMaxLayers) return false;
  const int groups = s->Hkv_l * ((s->G * 8 * NT + 63) / 64);
  return groups <= step_ctas(NT, s->cfg.head_dim, s->launch_cap);
}

static StepArgs step_args(ss_shard* s, int want_logits) {
  const ss_model_cfg& c = s->cfg;
  StepArgs a;
  a.st = s->dstate;
  a.layers = (const LayerPtrs*)s->layer_tab;
  a.n_layers = c.n_layers;
  a.h = c.hidden;
  a.d = c.head_dim;
  a.Hq_l = s->Hq_l;
  a.Hkv_l = s->Hkv_l;
  a.G = s->G;
  a.I_l = s->I_l;
  a.max_ctx_pad = s->max_ctx_pad;
  const LayerW& l0 = s->layers[0];
  a.qkv_tg = l0.qkv.n_tg; a.qkv_S = l0.qkv.S;
  a.o_tg = l0.o.n_tg; a.o_S = l0.o.S;
  a.gu_tg = l0.gu.n_tg; a.gu_S = l0.gu.S;
  a.dn_tg = l0.down.n_tg; a.dn_S = l0.down.S;
  a.lm_tg = s->lm_head.n_tg; a.lm_S = s->lm_head.S;
  a.lm_w = s->lm_head.d;
  a.final_norm = s->final_norm;
  a.eps = c.rms_eps;
  a.act_h = s->act_h;
  a.act_o = s->act_o;
  a.act_d = s->act_d;
  a.act_lm = s->act_lm;
  a.qf = s->qf;
  a.kc = s->kcache;
  a.vc = s->vcache;
  a.klo = s->klo;
  a.vlo = s->vlo;
  a.rope_cs = s->rope_cs;
  a.x = s->x;
  GemmScratch* sc[5] = {&s->sc_qkv, &s->sc_o, &s->sc_gu, &s->sc_down, &s->sc_lm};
  for (int i = 0; i < 5; ++i) {
    a.acc[i] = sc[i]->accum;
    a.arr[i] = sc[i]->counters;
  }
  a.ctr = s->step_ctr;
  a.ss = s->step_ss;
  a.ssx = s->step_ssx;
  a.det = (s->debug & SS_DEBUG_DETERMINISTIC) ? 1 : 0;
  a.att_ws = s->att_ws;
  a.att_ml = s->att_ml;
  a.rank = s->rank;
  a.P = s->P;
  a.loopback = s->loopback ? 1 : 0;
  a.ar_mode = s->ar_mode;
  a.bc_line0 = consistency_line_offset(s) + (size_t)s->P;
  a.recv = s->recv;
  for (int p = 0; p < s->P; ++p) a.peer_recv[p] = s->peer_recv[p];
  a.V_l = s->V_l;
  a.V_off = s->V_off;
  a.logits_ld = s->V_l_pad;
  a.logits = want_logits ? s->logits_dev : nullptr;
  a.trace = s->step_trace;
  a.trace_slots = s->step_trace_slots;
  a.where = s->step_trace_host ? s->step_trace + (size_t)512 * s->step_trace_slots * 3 : nullptr;
  a.utl = s->step_trace ? s->step_trace + (size_t)512 * s->step_trace_slots * 3 + 512 * 16 : nullptr;
  return a;
}

// The step kernel reads its arguments from device memory (one copy per
// logits mode): written before graph capture / an eager profile launch.
static int step_args_slot(int NT, int want_logits) { return (NT == 1 ? 0 : NT == 2 ? 1 : 2) * 2 + want_logits; }
static ss_status write_step_args(ss_shard* s, int NT) {
  if (!step_path(s, NT)) return SS_OK;
  StepArgs h[2];
  for (int w = 0; w < 2; ++w) {
    h[w] = step_args(s, w);
    h[w].n_ctas = step_ctas(NT, s->cfg.head_dim, s->launch_cap);
  }
  CUDA_TRY(cudaMemcpy(reinterpret_cast<StepArgs*>(s->step_args_dev) + step_args_slot(NT, 0), h, sizeof(h),
                      cudaMemcpyHostToDevice));
  return SS_OK;
}

// Enqueue everything after a0/a1 (the graph body).  Returns the kernel count.
static int enqueue_body(ss_shard* s, int NT, int auto_commit, int want_logits, cudaStream_t st) {
  const ss_model_cfg& c = s->cfg;
  int n = 0;
  if (step_path(s, NT)) {
    ss_pdl_off = s->launch_cap > 0 && !s->loopback;  // capped: shares the GPU (fake peers, async split)
    StepArgs a = step_args(s, want_logits);
    a.n_ctas = step_ctas(NT, c.head_dim, s->launch_cap);
    PROF_BEGIN(9);
    n += launch_step(a, reinterpret_cast<const StepArgs*>(s->step_args_dev) + step_args_slot(NT, want_logits), NT,
                     s->launch_cap, st);
    PROF_END();
    if (auto_commit) {
      // fake-peer shards: no PDL here either -- an early-launched commit grid
      // holds an SM the next shard's persistent grid needs
      PROF_BEGIN(8);
      launch_commit(s, 1, st);
      PROF_END();
      ++n;
    }
    ss_pdl_off = false;
    return n;
  }
  // timing experiments only (results are wrong; experiment builds only, the
  // product library always runs every launch): SS_EXP_SKIP = bitmask of
  // launches to leave out, 1 qkv, 2 attention, 4 o, 8 gate/up, 16 down
#ifdef SS_EXPERIMENTS
  static const int skip = exp_env_int("SS_EXP_SKIP", 0);
#else
  constexpr int skip = 0;
#endif
  const int cap = s->launch_cap;
  // capped grids share this GPU (fake-peer TP ranks, the two groups of the
  // async split): no PDL, see ss_pdl_off
  ss_pdl_off = cap > 0 && !s->loopback;
  for (int l = 0; l < c.n_layers; ++l) {
    LayerW& lw = s->layers[l];
    GemmArgs g = gemm_args(s, lw.qkv, s->act_h, s->sc_qkv, EPI_QKV, l);
    g.zero_x = s->act_o;  // attention accumulates the O-input group sums
    g.zero_x_stages = lw.o.S;
    g.zero_x_nt = NT;
    PROF_BEGIN(1);
    ss_pdl_pos = 0;
    if (!(skip & 1)) n += launch_gemm(g, 0, NT, cap, st);
    PROF_END();
    AttnArgs a;
    a.st = s->dstate;
    a.layer = l;
    a.Hkv_l = s->Hkv_l;
    a.G = s->G;
    a.d = c.head_dim;
    a.max_ctx_pad = s->max_ctx_pad;
    a.NT = NT;
    a.qbuf = s->qbuf;
    a.kc = s->kcache;
    a.vc = s->vcache;
    a.ws = s->attn_ws;
    a.ml = s->attn_ml;
    a.bar = s->attn_bar;
    a.act_out = s->act_o;
    PROF_BEGIN(2);
    ss_pdl_pos = 1;
    if (!(skip & 2)) n += launch_attention(a, cap, st);
    PROF_END();
    g = gemm_args(s, lw.o, s->act_o, s->sc_o, EPI_RESID, l);
    g.epi.ar_seq = 2 * l;
    g.zero_x = s->act_d;  // the SwiGLU epilogue accumulates the down-input group sums
    g.zero_x_stages = lw.down.S;
    g.zero_x_nt = NT;
    g.norm_gain = lw.mlp_norm;  // a7 fused: RMSNorm into the gate/up input
    g.norm_out = s->act_h;
    g.norm_split = 0;
    PROF_BEGIN(3);
    ss_pdl_pos = 2;
    if (!(skip & 4)) n += launch_gemm(g, 0, NT, cap, st);
    PROF_END();
    g = gemm_args(s, lw.gu, s->act_h, s->sc_gu, EPI_SWIGLU, l);
    PROF_BEGIN(5);
    ss_pdl_pos = 3;
    if (!(skip & 8)) n += launch_gemm(g, 0, NT, cap, st);
    PROF_END();
    g = gemm_args(s, lw.down, s->act_d, s->sc_down, EPI_RESID, l);
    g.epi.ar_seq = 2 * l + 1;
    // a2 of the next layer (or the final norm before the LM head) fused
    g.norm_gain = l + 1 < c.n_layers ? s->layers[l + 1].attn_norm : s->final_norm;
    g.norm_out = l + 1 < c.n_layers ? s->act_h : s->act_lm;
    g.norm_split = l + 1 < c.n_layers ? 0 : 1;
    PROF_BEGIN(6);
    ss_pdl_pos = 4;
    if (!(skip & 16)) n += launch_gemm(g, 0, NT, cap, st);
    PROF_END();
  }
  GemmArgs g = gemm_args(s, s->lm_head, s->act_lm, s->sc_lm, EPI_ARGMAX, 0);
  g.epi.logits = want_logits ? s->logits_dev : nullptr;
  g.epi.ar_seq = 2 * c.n_layers;
  PROF_BEGIN(7);
  ss_pdl_pos = 5;
  n += launch_gemm(g, 1, NT, cap, st);
  PROF_END();
  ss_pdl_pos = 31;
  ss_pdl_off = false;
  if (auto_commit) {
    PROF_BEGIN(8);
    launch_commit(s, 1, st);
    PROF_END();
    ++n;
  }
  return n;
}

static ss_status get_graph(ss_shard* s, int NT, int auto_commit, int want_logits, Graph** out) {
  int key = NT * 4 + auto_commit * 2 + want_logits;
  auto it = s->graphs.find(key);
  if (it != s->graphs.end()) {
    *out = &it->second;
    return SS_OK;
  }
  // warm the launch helpers (function attributes, occupancy) outside capture
  ss_status ra = write_step_args(s, NT);
  if (ra != SS_OK) return ra;
  Graph gr;
  cudaGraph_t graph;
  CUDA_TRY(cudaStreamBeginCapture(s->cap_stream, cudaStreamCaptureModeThreadLocal));
  gr.kernels = enqueue_body(s, NT, auto_commit, want_logits, s->cap_stream);
  cudaError_t e = cudaStreamEndCapture(s->cap_stream, &graph);
  if (e != cudaSuccess) FAIL(SS_ECUDA, std::string("graph capture: ") + cudaGetErrorString(e));
  e = cudaGraphInstantiate(&gr.exec, graph, 0);
  cudaGraphDestroy(graph);
  if (e != cudaSuccess) FAIL(SS_ECUDA, std::string("graph instantiate: ") + cudaGetErrorString(e));
  s->graphs[key] = gr;
  *out = &s->graphs[key];
  return SS_OK;
}

static ss_status check_ready(ss_shard* s, int T) {
  s->hs.weights_ready = weights_complete(s);
  s->hs.peers_ready = s->P == 1 || s->peers_ready;
  if (!s->hs.L_known && (int64_t)s->hs.L + T > s->cfg.max_ctx) {  // upper bound too loose: read L back
    ss_status r = sync_L(s);
    if (r != SS_OK) return r;
  }
  HOST_CHECK(check_verify, s->hs, T);
  return SS_OK;
}

static ss_status run_step(ss_shard* s, const int32_t* d_tokens, const int32_t* d_parents, int T, int auto_commit,
                          int want_logits, cudaStream_t st, bool from_mailbox = false, int T0 = 0) {
  const int NT = nt_of(T);
  Graph* gr;
  ss_status r = get_graph(s, NT, auto_commit, want_logits, &gr);
  if (r != SS_OK) return r;
  launch_embed_meta(s, d_tokens, d_parents, T, NT, st, from_mailbox, step_path(s, NT), T0);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaGraphLaunch(gr->exec, st));
  return SS_OK;
}

static const char* status_msg(int st) {
  switch (st) {
    case SS_EINVAL: return "device-side tree validation failed";
    case SS_ETIMEOUT: return "a peer / mailbox flag poll exceeded its budget";
    case SS_ECONSISTENCY: return "TP ranks were called with different trees (debug checksum)";
    default: return "verify failed";
  }
}

extern "C" ss_status ss_verify_tree(ss_shard* s, const int32_t* tokens, const int32_t* parents, int32_t T,
                                    ss_verify_result* out, float* logits_out, void* stream) {
  SCOPE(s);
  if (!s || !out) FAIL(SS_EINVAL, "null argument");
  HOST_CHECK(check_tree, s->hs, tokens, parents, T);
  cudaSetDevice(s->device);
  ss_status r = check_ready(s, T);
  if (r != SS_OK) return r;
  cudaStream_t st = (cudaStream_t)stream;
  std::memcpy(s->h_tree_in, tokens, T * 4);
  std::memcpy(s->h_tree_in + SS_MAX_TREE, parents, T * 4);
  CUDA_TRY(cudaMemcpyAsync(s->d_tree_in, s->h_tree_in, 2 * SS_MAX_TREE * 4, cudaMemcpyHostToDevice, st));
  r = run_step(s, s->d_tree_in, s->d_tree_in + SS_MAX_TREE, T, 0, logits_out != nullptr, st);
  if (r != SS_OK) return r;
  CUDA_TRY(cudaMemcpyAsync(&s->hstate->result, &s->dstate->result, sizeof(ss_verify_result), cudaMemcpyDeviceToHost,
                           st));
  if (logits_out)
    CUDA_TRY(cudaMemcpy2DAsync(logits_out, (size_t)s->V_l * 4, s->logits_dev, (size_t)s->V_l_pad * 4,
                               (size_t)s->V_l * 4, T, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  std::memcpy(out, &s->hstate->result, sizeof(ss_verify_result));
  if (out->status != SS_OK) {  // device-detected failure: nothing to commit (out is still filled)
    s->hs.max_written = std::max(s->hs.max_written, s->hs.L + T);
    FAIL((ss_status)out->status, status_msg(out->status));
  }
  ss::host::on_verify(s->hs, T, parents, false);
  return SS_OK;
}

static ss_status read_last_tree(ss_shard* s, cudaStream_t st, int32_t* status);

static ss_status extend_impl(ss_shard* s, const int32_t* tokens, const int32_t* parents, int32_t T0, int32_t w,
                             ss_verify_result* out, float* logits_out, int32_t K, int32_t* top_tok,
                             float* top_logit, float* lse, void* stream) {
  if (!s || !out) FAIL(SS_EINVAL, "null argument");
  if (K != 0 && (K < 1 || K > 32 || !top_tok || !top_logit || !lse)) FAIL(SS_EINVAL, "K out of [1, 32] / null top-K output");
  s->hs.weights_ready = weights_complete(s);
  s->hs.peers_ready = s->P == 1 || s->peers_ready;
  if (!s->hs.L_known) {
    ss_status r = sync_L(s);
    if (r != SS_OK) return r;
  }
  HOST_CHECK(check_extend, s->hs, tokens, parents, T0, w);
  // the cached-tree offset is handled by the persistent step kernel only
  if (T0 > 0 && !step_path(s, nt_of(w))) FAIL(SS_EINVAL, "T0 > 0 needs the persistent step kernel (w <= 32)");
  cudaSetDevice(s->device);
  cudaStream_t st = (cudaStream_t)stream;
  std::memcpy(s->h_tree_in, tokens, w * 4);
  std::memcpy(s->h_tree_in + SS_MAX_TREE, parents, w * 4);
  CUDA_TRY(cudaMemcpyAsync(s->d_tree_in, s->h_tree_in, 2 * SS_MAX_TREE * 4, cudaMemcpyHostToDevice, st));
  const bool want = logits_out != nullptr || K > 0;
  ss_status r = run_step(s, s->d_tree_in, s->d_tree_in + SS_MAX_TREE, w, 0, want, st, false, T0);
  if (r != SS_OK) return r;
  CUDA_TRY(cudaMemcpyAsync(&s->hstate->result, &s->dstate->result, sizeof(ss_verify_result), cudaMemcpyDeviceToHost,
                           st));
  if (K > 0) {
    // top-K tokens / logits + log-sum-exp per new node, in the tree-input staging's tail
    int32_t* d_tok = s->d_topk;
    float* d_val = reinterpret_cast<float*>(d_tok + 32 * 32);
    float* d_lse = d_val + 32 * 32;
    launch_topk(s, w, K, d_tok, d_val, d_lse, st);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpyAsync(top_tok, d_tok, (size_t)w * K * 4, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(top_logit, d_val, (size_t)w * K * 4, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(lse, d_lse, (size_t)w * 4, cudaMemcpyDeviceToHost, st));
  }
  if (logits_out)
    CUDA_TRY(cudaMemcpy2DAsync(logits_out, (size_t)s->V_l * 4, s->logits_dev, (size_t)s->V_l_pad * 4,
                               (size_t)s->V_l * 4, w, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  std::memcpy(out, &s->hstate->result, sizeof(ss_verify_result));
  if (out->status != SS_OK) {
    s->hs.max_written = std::max(s->hs.max_written, s->hs.L + T0 + w);
    s->hs.have_verify = false;  // the tree is no longer usable
    FAIL((ss_status)out->status, status_msg(out->status));
  }
  ss::host::on_extend(s->hs, T0, w, parents);
  return SS_OK;
}

extern "C" ss_status ss_extend_tree(ss_shard* s, const int32_t* tokens, const int32_t* parents, int32_t T0,
                                    int32_t w, ss_verify_result* out, float* logits_out, void* stream) {
  SCOPE(s);
  return extend_impl(s, tokens, parents, T0, w, out, logits_out, 0, nullptr, nullptr, nullptr, stream);
}

extern "C" ss_status ss_extend_tree_topk(ss_shard* s, const int32_t* tokens, const int32_t* parents, int32_t T0,
                                         int32_t w, int32_t K, int32_t* top_tok, float* top_logit, float* lse,
                                         ss_verify_result* out, void* stream) {
  SCOPE(s);
  return extend_impl(s, tokens, parents, T0, w, out, nullptr, K, top_tok, top_logit, lse, stream);
}

extern "C" ss_status ss_reroot(ss_shard* s, const int32_t* path, int32_t n, const int32_t* keep, int32_t m,
                               void* stream) {
  SCOPE(s);
  if (!s) FAIL(SS_EINVAL, "null shard");
  if (!s->hs.have_verify) FAIL(SS_ESTATE, "re-root without a pending tree");
  cudaSetDevice(s->device);
  cudaStream_t st = (cudaStream_t)stream;
  int32_t vstatus = 0;
  ss_status r = read_last_tree(s, st, &vstatus);
  if (r != SS_OK) return r;
  if (vstatus != SS_OK) FAIL(SS_ESTATE, "the last step failed on the device; nothing to re-root");
  HOST_CHECK(check_reroot, s->hs, path, n, keep, m);
  r = sync_L(s);
  if (r != SS_OK) return r;
  std::vector<int32_t> buf(1 + SS_MAX_TREE, 0);
  buf[0] = n;
  for (int k = 0; k < n; ++k) buf[1 + k] = path[k];
  CUDA_TRY(cudaMemcpyAsync(&s->dstate->commit_n, buf.data(), (1 + SS_MAX_TREE) * 4, cudaMemcpyHostToDevice, st));
  std::vector<int32_t> kb(1 + SS_MAX_TREE, 0);
  kb[0] = m;
  for (int j = 0; j < m; ++j) kb[1 + j] = keep[j];
  static_assert(offsetof(DevState, keep) == offsetof(DevState, keep_n) + 4, "layout");
  CUDA_TRY(cudaMemcpyAsync(&s->dstate->keep_n, kb.data(), (1 + SS_MAX_TREE) * 4, cudaMemcpyHostToDevice, st));
  launch_reroot(s, st);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaStreamSynchronize(st));
  ss::host::on_reroot(s->hs, path, n, keep, m);
  return SS_OK;
}

extern "C" ss_status ss_verify_tree_dev(ss_shard* s, const int32_t* d_tokens, const int32_t* d_parents, int32_t T,
                                        ss_verify_result* d_result, float* d_logits, int32_t auto_commit,
                                        void* stream) {
  SCOPE(s);
  if (!s || !d_tokens || !d_parents) FAIL(SS_EINVAL, "null argument");
  if (T < 1 || T > s->cfg.max_tree) FAIL(SS_EINVAL, "T out of [1, max_tree]");
  cudaSetDevice(s->device);
  ss_status r = check_ready(s, T);
  if (r != SS_OK) return r;
  cudaStream_t st = (cudaStream_t)stream;
  r = run_step(s, d_tokens, d_parents, T, auto_commit ? 1 : 0, d_logits != nullptr, st);
  if (r != SS_OK) return r;
  if (d_result)
    CUDA_TRY(cudaMemcpyAsync(d_result, &s->dstate->result, sizeof(ss_verify_result), cudaMemcpyDeviceToDevice, st));
  if (d_logits)
    CUDA_TRY(cudaMemcpy2DAsync(d_logits, (size_t)s->V_l * 4, s->logits_dev, (size_t)s->V_l_pad * 4,
                               (size_t)s->V_l * 4, T, cudaMemcpyDeviceToDevice, st));
  ss::host::on_verify(s->hs, T, nullptr, auto_commit != 0);  // parents live on the device
  return SS_OK;
}

// Parents of the last verified tree and its device status (device truth:
// the tree of a *_dev / mailbox verify never passed through the host).
static ss_status read_last_tree(ss_shard* s, cudaStream_t st, int32_t* status) {
  CUDA_TRY(cudaMemcpyAsync(s->hs.last_parents, s->dstate->parents, sizeof(s->hs.last_parents),
                           cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(&s->hstate->result.status, &s->dstate->result.status, 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(&s->hstate->T, &s->dstate->T, 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(&s->hstate->T0, &s->dstate->T0, 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  *status = s->hstate->result.status;
  s->hs.last_T = s->hstate->T0 + s->hstate->T;  // nodes of the pending tree
  return SS_OK;
}

extern "C" ss_status ss_commit_kv(ss_shard* s, const int32_t* accepted, int32_t n, void* stream) {
  SCOPE(s);
  if (!s || !accepted) FAIL(SS_EINVAL, "null argument");
  if (!s->hs.have_verify) FAIL(SS_ESTATE, "commit without a preceding verify");
  cudaSetDevice(s->device);
  cudaStream_t st = (cudaStream_t)stream;
  int32_t vstatus = 0;
  ss_status r = read_last_tree(s, st, &vstatus);
  if (r != SS_OK) return r;
  if (vstatus != SS_OK) FAIL(SS_ESTATE, "the last verify failed on the device; nothing to commit");
  HOST_CHECK(check_commit, s->hs, accepted, n);
  r = sync_L(s);
  if (r != SS_OK) return r;
  std::vector<int32_t> buf(1 + SS_MAX_TREE, 0);
  buf[0] = n;
  for (int k = 0; k < n; ++k) buf[1 + k] = accepted[k];
  static_assert(offsetof(DevState, commit_chain) == offsetof(DevState, commit_n) + 4, "layout");
  CUDA_TRY(cudaMemcpyAsync(&s->dstate->commit_n, buf.data(), (1 + SS_MAX_TREE) * 4, cudaMemcpyHostToDevice, st));
  launch_commit(s, 0, st);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaStreamSynchronize(st));
  ss::host::on_commit(s->hs, n);
  return SS_OK;
}

extern "C" ss_status ss_commit_accepted(ss_shard* s, void* stream) {
  SCOPE(s);
  if (!s) FAIL(SS_EINVAL, "null shard");
  if (!s->hs.have_verify) FAIL(SS_ESTATE, "commit without a preceding verify");
  cudaSetDevice(s->device);
  cudaStream_t st = (cudaStream_t)stream;
  launch_commit(s, 1, st);  // the device commits only a verify whose status is SS_OK
  CUDA_TRY(cudaGetLastError());
  s->hs.L_known = false;
  s->hs.L += s->hs.last_T;  // upper bound until read back
  s->hs.have_verify = false;
  return SS_OK;
}

extern "C" ss_status ss_set_step_kernel(ss_shard* s, int32_t on) {
  SCOPE(s);
  if (!s) FAIL(SS_EINVAL, "null shard");
  cudaSetDevice(s->device);
  CUDA_TRY(cudaDeviceSynchronize());
  s->use_step = on != 0;
  for (auto& kv : s->graphs)
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
  s->graphs.clear();
  return SS_OK;
}

extern "C" ss_status ss_step_trace(ss_shard* s, int32_t on) {
  SCOPE(s);
  if (!s) FAIL(SS_EINVAL, "null shard");
  cudaSetDevice(s->device);
  CUDA_TRY(cudaDeviceSynchronize());
  if (s->step_trace) {
    if (s->step_trace_host) cudaFreeHost(s->step_trace_host);
    else cudaFree(s->step_trace);
  }
  s->step_trace = nullptr;
  s->step_trace_host = nullptr;
  s->step_trace_slots = 0;
  if (on) {
    s->step_trace_slots = s->cfg.n_layers * 5 + 1;
    const size_t n = (size_t)512 * s->step_trace_slots * 3 + 512 * 16 + 65536;
    if (on == 2) {  // mapped host memory: readable while a launch is still running (hang diagnosis)
      CUDA_TRY(cudaHostAlloc(&s->step_trace_host, n * 8, cudaHostAllocMapped));
      memset(s->step_trace_host, 0, n * 8);
      CUDA_TRY(cudaHostGetDevicePointer((void**)&s->step_trace, s->step_trace_host, 0));
    } else {
      CUDA_TRY(cudaMalloc(&s->step_trace, n * 8));
      CUDA_TRY(cudaMemset(s->step_trace, 0, n * 8));
    }
  }
  for (auto& kv : s->graphs)
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
  s->graphs.clear();
  return SS_OK;
}

extern "C" void* ss_step_trace_host(ss_shard* s) { return s ? (void*)s->step_trace_host : nullptr; }

extern "C" ss_status ss_read_step_trace(ss_shard* s, uint64_t* host, size_t n, int32_t* n_ctas, int32_t* slots) {
  SCOPE(s);
  if (!s || !host) FAIL(SS_EINVAL, "null argument");
  if (!s->step_trace) FAIL(SS_ESTATE, "trace not enabled");
  const size_t need = (size_t)512 * s->step_trace_slots * 3 + 512 * 16 + 65536;
  if (n < need) FAIL(SS_EINVAL, "buffer too small");
  cudaSetDevice(s->device);
  if (s->step_trace_host) {
    memcpy(host, s->step_trace_host, need * 8);  // no synchronisation (on == 2)
  } else {
    CUDA_TRY(cudaDeviceSynchronize());
    CUDA_TRY(cudaMemcpy(host, s->step_trace, need * 8, cudaMemcpyDeviceToHost));
  }
  if (n_ctas) *n_ctas = 512;
  if (slots) *slots = s->step_trace_slots;
  return SS_OK;
}

extern "C" int32_t ss_step_kernel_active(ss_shard* s, int32_t T) {
  if (!s || T < 1 || T > SS_MAX_TREE) return -1;
  return step_path(s, nt_of(T)) ? 1 : 0;
}

extern "C" uint64_t ss_debug_ctr_base(ss_shard* s) { return s ? (uint64_t)(uintptr_t)s->step_ctr : 0; }

extern "C" ss_status ss_watchdog_record(uint64_t* out, int32_t n) {
  const unsigned long long* r = watchdog_record();
  if (!out || n < 0 || n > 64 * 1024) return SS_EINVAL;
  for (int i = 0; i < n; ++i) out[i] = r ? r[i] : 0;
  return SS_OK;
}

extern "C" ss_status ss_set_debug(ss_shard* s, int32_t flags) {
  SCOPE(s);
  if (!s) FAIL(SS_EINVAL, "null shard");
  if (flags & ~(SS_DEBUG_CONSISTENCY | SS_DEBUG_DETERMINISTIC)) FAIL(SS_EINVAL, "unknown debug flag");
  cudaSetDevice(s->device);
  CUDA_TRY(cudaDeviceSynchronize());
  CUDA_TRY(cudaMemcpy(&s->dstate->debug, &flags, 4, cudaMemcpyHostToDevice));
  if ((flags ^ s->debug) & SS_DEBUG_DETERMINISTIC) {  // the step kernel's schedule changes
    for (auto& kv : s->graphs)
      if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
    s->graphs.clear();
  }
  s->debug = flags;
  return SS_OK;
}

extern "C" int32_t ss_kernels_per_step(ss_shard* s, int32_t T, int32_t auto_commit) {
  if (!s || T < 1 || T > SS_MAX_TREE) return -1;
  Graph* gr;
  if (get_graph(s, nt_of(T), auto_commit ? 1 : 0, 0, &gr) != SS_OK) return -1;
  return gr->kernels + 1;  // + the a0/a1 ingest kernel launched outside the graph
}

// ------------------------------------------------------------ peers (TP)
extern "C" ss_status ss_export_handle(ss_shard* s, void* buf, size_t* len) {
  SCOPE(s);
  if (!s || !buf || !len) FAIL(SS_EINVAL, "null argument");
  if (s->P == 1) {
    *len = 0;
    return SS_OK;
  }
  cudaSetDevice(s->device);
  cudaIpcMemHandle_t hnd;
  CUDA_TRY(cudaIpcGetMemHandle(&hnd, s->recv));
  std::memcpy(buf, &hnd, sizeof(hnd));
  *len = sizeof(hnd);
  return SS_OK;
}

extern "C" ss_status ss_import_peers(ss_shard* s, const void* const* blobs, const size_t* lens) {
  SCOPE(s);
  if (!s || !blobs || !lens) FAIL(SS_EINVAL, "null argument");
  cudaSetDevice(s->device);
  for (int p = 0; p < s->P; ++p) {
    if (p == s->rank) {
      s->peer_recv[p] = s->recv;
      continue;
    }
    if (lens[p] != sizeof(cudaIpcMemHandle_t)) FAIL(SS_EINVAL, "bad handle blob");
    cudaIpcMemHandle_t hnd;
    std::memcpy(&hnd, blobs[p], sizeof(hnd));
    void* ptr = nullptr;
    CUDA_TRY(cudaIpcOpenMemHandle(&ptr, hnd, cudaIpcMemLazyEnablePeerAccess));
    s->peer_recv[p] = (float*)ptr;
    s->ipc_opened[p] = true;
  }
  s->peers_ready = true;
  for (auto& kv : s->graphs)
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
  s->graphs.clear();
  return SS_OK;
}

extern "C" ss_status ss_import_local_peers(ss_shard* s, ss_shard* const* shards) {
  SCOPE(s);
  if (!s || !shards) FAIL(SS_EINVAL, "null argument");
  cudaSetDevice(s->device);
  for (int p = 0; p < s->P; ++p) {
    if (!shards[p] || shards[p]->P != s->P || shards[p]->rank != p) FAIL(SS_EINVAL, "shards must be given in rank order");
    if (shards[p]->device != s->device) {
      cudaError_t e = cudaDeviceEnablePeerAccess(shards[p]->device, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) FAIL(SS_ECUDA, "peer access not available");
      cudaGetLastError();
    }
    s->peer_recv[p] = shards[p]->recv;
  }
  s->peers_ready = true;
  for (auto& kv : s->graphs)
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
  s->graphs.clear();
  return SS_OK;
}

extern "C" ss_status ss_import_loopback(ss_shard* s) {
  SCOPE(s);
  if (!s) FAIL(SS_EINVAL, "null argument");
  if (s->P < 2) FAIL(SS_EINVAL, "loopback needs tp_size > 1");
  for (int p = 0; p < s->P; ++p) s->peer_recv[p] = s->recv;
  s->loopback = true;
  s->peers_ready = true;
  for (auto& kv : s->graphs)
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
  s->graphs.clear();
  return SS_OK;
}

extern "C" ss_status ss_profile_step(ss_shard* s, const int32_t* d_tokens, const int32_t* d_parents, int32_t T,
                                     float* ms, int32_t* count, void* stream) {
  SCOPE(s);
  if (!s || !d_tokens || !d_parents || !ms || !count) FAIL(SS_EINVAL, "null argument");
  if (T < 1 || T > s->cfg.max_tree) FAIL(SS_EINVAL, "T out of [1, max_tree]");
  cudaSetDevice(s->device);
  ss_status r = check_ready(s, T);
  if (r != SS_OK) return r;
  cudaStream_t st = (cudaStream_t)stream;
  static Prof prof;
  prof.next = 0;
  prof.st = st;
  const int NT = nt_of(T);
  // make sure function attributes are set before timing
  Graph* gr;
  r = get_graph(s, NT, 1, 0, &gr);
  if (r != SS_OK) return r;
  g_prof = &prof;
  prof.begin(0);
  launch_embed_meta(s, d_tokens, d_parents, T, NT, st, false, step_path(s, NT));
  prof.end();
  enqueue_body(s, NT, 1, 0, st);
  g_prof = nullptr;
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaStreamSynchronize(st));
  for (int k = 0; k < SS_PROF_KINDS; ++k) {
    ms[k] = 0.f;
    count[k] = 0;
  }
  for (size_t i = 0; i < prof.next; ++i) {
    float t = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&t, prof.ev[i].second.first, prof.ev[i].second.second));
    ms[prof.ev[i].first] += t;
    count[prof.ev[i].first] += 1;
  }
  ss::host::on_verify(s->hs, T, nullptr, true);
  return SS_OK;
}

// ------------------------------------------------------------ a13 mailbox
extern "C" ss_status ss_mailbox_inbox(ss_shard* s, void** dev_ptr) {
  SCOPE(s);
  if (!s || !dev_ptr) FAIL(SS_EINVAL, "null argument");
  *dev_ptr = s->mbox_in;
  return SS_OK;
}

extern "C" ss_status ss_attach_mailbox(ss_shard* s, void* outbox_dev, int32_t eos_token) {
  SCOPE(s);
  if (!s) FAIL(SS_EINVAL, "null shard");
  cudaSetDevice(s->device);
  CUDA_TRY(cudaDeviceSynchronize());
  uint4* p = (uint4*)outbox_dev;
  CUDA_TRY(cudaMemcpy(&s->dstate->mbox_out, &p, sizeof(p), cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(&s->dstate->eos, &eos_token, 4, cudaMemcpyHostToDevice));
  return SS_OK;
}

extern "C" ss_status ss_verify_tree_mailbox(ss_shard* s, int32_t auto_commit, void* stream) {
  SCOPE(s);
  if (!s) FAIL(SS_EINVAL, "null shard");
  return ss_verify_tree_mailbox_n(s, s->cfg.max_tree, auto_commit, stream);
}

extern "C" ss_status ss_verify_tree_mailbox_n(ss_shard* s, int32_t max_nodes, int32_t auto_commit, void* stream) {
  SCOPE(s);
  if (!s) FAIL(SS_EINVAL, "null shard");
  if (max_nodes < 1 || max_nodes > s->cfg.max_tree) FAIL(SS_EINVAL, "max_nodes out of [1, max_tree]");
  cudaSetDevice(s->device);
  const int T = max_nodes;  // the tree size arrives with the message; the step's graph holds ceil(T/8)*8 slots
  ss_status r = check_ready(s, T);
  if (r != SS_OK) return r;
  cudaStream_t st = (cudaStream_t)stream;
  r = run_step(s, nullptr, nullptr, T, auto_commit ? 1 : 0, 0, st, true);
  if (r != SS_OK) return r;
  ss::host::on_verify(s->hs, T, nullptr, auto_commit != 0);  // T: upper bound (the message carries it)
  return SS_OK;
}

extern "C" ss_status ss_mailbox_post_tree(void* inbox_dev, const int32_t* tokens, const int32_t* parents, int32_t T,
                                          uint32_t seq, void* stream) {
  if (!inbox_dev || !tokens || !parents) FAIL(SS_EINVAL, "null argument");
  if (T < 1 || T > SS_MAX_TREE) FAIL(SS_EINVAL, "T out of [1, 64]");
  if (seq == 0) FAIL(SS_EINVAL, "sequence number 0 is reserved (idle lines)");
  launch_mailbox_post(inbox_dev, tokens, parents, T, seq, (cudaStream_t)stream);
  CUDA_TRY(cudaGetLastError());
  return SS_OK;
}

extern "C" ss_status ss_mailbox_recv_result(const void* outbox_dev, uint32_t seq, int32_t* dev_out, void* stream) {
  if (!outbox_dev || !dev_out) FAIL(SS_EINVAL, "null argument");
  if (seq == 0) FAIL(SS_EINVAL, "sequence number 0 is reserved (idle lines)");
  launch_mailbox_recv(outbox_dev, seq, dev_out, (cudaStream_t)stream);
  CUDA_TRY(cudaGetLastError());
  return SS_OK;
}

// ------------------------------------------------------------ test / inspection hooks
extern "C" ss_status ss_read_tree_meta(ss_shard* s, int32_t* T, int32_t* pos, uint64_t* anc, int32_t* tokens,
                                       int32_t* parents) {
  SCOPE(s);
  if (!s || !T || !pos || !anc) FAIL(SS_EINVAL, "null argument");
  cudaSetDevice(s->device);
  CUDA_TRY(cudaDeviceSynchronize());
  CUDA_TRY(cudaMemcpy(s->hstate, s->dstate, sizeof(DevState), cudaMemcpyDeviceToHost));
  *T = s->hstate->T0 + s->hstate->T;  // nodes of the tree (cached + this step's)
  std::memcpy(pos, s->hstate->pos, sizeof(s->hstate->pos));
  std::memcpy(anc, s->hstate->anc, sizeof(s->hstate->anc));
  if (tokens) std::memcpy(tokens, s->hstate->tokens, sizeof(s->hstate->tokens));
  if (parents) std::memcpy(parents, s->hstate->parents, sizeof(s->hstate->parents));
  return SS_OK;
}

static ss_status packed_region(ss_shard* s, int32_t layer, int32_t which, const void** ptr, size_t* bytes) {
  const ss_model_cfg& c = s->cfg;
  if (which <= 3 || which == 6 || which == 7) {
    if (layer < 0 || layer >= c.n_layers) FAIL(SS_EINVAL, "layer out of range");
    LayerW& lw = s->layers[layer];
    if (which <= 3) {
      const PackedLinear& pl = which == 0 ? lw.qkv : which == 1 ? lw.o : which == 2 ? lw.gu : lw.down;
      *ptr = pl.d;
      *bytes = pl.bytes;
    } else {
      *ptr = which == 6 ? lw.attn_norm : lw.mlp_norm;
      *bytes = (size_t)c.hidden * 2;
    }
    return SS_OK;
  }
  switch (which) {
    case 4: *ptr = s->lm_head.d; *bytes = s->lm_head.bytes; return SS_OK;
    case 5: *ptr = s->embed; *bytes = (size_t)c.vocab * c.hidden * 2; return SS_OK;
    case 8: *ptr = s->final_norm; *bytes = (size_t)c.hidden * 2; return SS_OK;
    default: FAIL(SS_EINVAL, "unknown packed region");
  }
}

extern "C" ss_status ss_read_packed(ss_shard* s, int32_t layer, int32_t which, void* host, size_t bytes,
                                    size_t* total) {
  SCOPE(s);
  if (!s || !total) FAIL(SS_EINVAL, "null argument");
  const void* p = nullptr;
  size_t n = 0;
  ss_status r = packed_region(s, layer, which, &p, &n);
  if (r != SS_OK) return r;
  *total = n;
  if (!host) return SS_OK;
  if (bytes != n) FAIL(SS_EINVAL, "bytes must equal the region size (*total)");
  cudaSetDevice(s->device);
  CUDA_TRY(cudaDeviceSynchronize());
  CUDA_TRY(cudaMemcpy(host, p, n, cudaMemcpyDeviceToHost));
  return SS_OK;
}

extern "C" ss_status ss_debug_gemm(ss_shard* s, int32_t layer, int32_t which, const float* d_x, int32_t T, float* d_y,
                                   int32_t allreduce, void* stream) {
  SCOPE(s);
  if (!s || !d_x || !d_y) FAIL(SS_EINVAL, "null argument");
  if (layer < 0 || layer >= s->cfg.n_layers || which < 0 || which > 3) FAIL(SS_EINVAL, "layer / linear out of range");
  if (T < 1 || T > SS_MAX_TREE) FAIL(SS_EINVAL, "T out of [1, 64]");
  if (allreduce && (which == 0 || which == 2)) FAIL(SS_EINVAL, "all-reduce applies to the O / down projections");
  if (allreduce && s->P > 1 && !s->peers_ready) FAIL(SS_ESTATE, "peers not imported (tp_size > 1)");
  if (!weights_complete(s)) FAIL(SS_ESTATE, "weights not fully loaded");
  cudaSetDevice(s->device);
  cudaStream_t st = (cudaStream_t)stream;
  LayerW& lw = s->layers[layer];
  PackedLinear& pl = which == 0 ? lw.qkv : which == 1 ? lw.o : which == 2 ? lw.gu : lw.down;
  GemmScratch& sc = which == 0 ? s->sc_qkv : which == 1 ? s->sc_o : which == 2 ? s->sc_gu : s->sc_down;
  uint8_t* act = which == 1 ? s->act_o : which == 3 ? s->act_d : s->act_h;
  const int NT = nt_of(T);
  CUDA_TRY(cudaMemsetAsync(d_y, 0, (size_t)T * pl.N * 4, st));
  launch_debug_act(s, d_x, T, pl.K, act, NT, allreduce ? 1 : 0, st);
  GemmArgs g = gemm_args(s, pl, act, sc, EPI_RESID, layer);
  g.epi.x = d_y;           // x += y with x = 0: the raw GEMM rows (or the all-reduced sum)
  g.epi.h = pl.N;
  g.epi.P = allreduce ? s->P : 1;
  g.epi.ar_seq = 0;
  ss_pdl_off = s->launch_cap > 0 && !s->loopback;  // capped: shares the GPU (fake peers, async split)
  launch_gemm(g, 0, NT, s->launch_cap, st);
  ss_pdl_off = false;
  CUDA_TRY(cudaGetLastError());
  return SS_OK;
}
