// misc.cu -- small kernels of the step: tree ingest + embedding (a0, a1),
// RMSNorm into fragment-ordered bf16 activations (a2, a7, final), KV
// compaction + commit (a12), the RoPE table, and the device-side synthetic
// input generator (same counter-based hash as synth/generators.py).
#include "common.cuh"
#include "internal.h"
#include "kernels.h"
#include "step.h"

namespace ss {

// ---------------------------------------------------------------- a0 + a1
// One CTA per token slot (8*NT of them).  Every CTA validates the tree the
// same way (root first, 0 <= parents[i] < i, token in vocab: S:45-47); CTA 0
// publishes T, status, depth-derived positions pos = L + depth (R8) and the
// ancestor-or-self bitmasks.  CTA t < T gathers E[token] (P:501 bf16
// embedding) into the fp32 residual and writes RMSNorm(x) * g (layer 0 attn
// norm) into the fragment-ordered activation; slots t >= T are zeroed.
constexpr int kNormSplit = 4;   // CTAs per token for the row kernels
constexpr int kMaxVec = 8;      // h <= 256 threads * 4 * kMaxVec = 8192

// Block reduction of one float across 256 threads (result in every thread).
SS_DEV float block_sum_256(float v, float* s_red) {
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = v;
  __syncthreads();
  float r = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) r += s_red[i];
  return r;
}

// a13 inbox poll: spin on one LL line until its flag equals seq, for at most
// kMailboxPollNs of device time (%globaltimer), then report a timeout.
constexpr unsigned long long kMailboxPollNs = 2000000000ull;  // 2 s
SS_DEV unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
SS_DEV bool ll_wait(const uint4* line, uint32_t seq, uint32_t& d1, uint32_t& d2) {
  if (ll_try_load(line, seq, d1, d2)) return true;
  const unsigned long long t0 = global_ns();
  while (global_ns() - t0 < kMailboxPollNs)
    for (int i = 0; i < 64; ++i)
      if (ll_try_load(line, seq, d1, d2)) return true;
  return false;
}

// Cross-rank consistency check (debug mode, SS_DEBUG_CONSISTENCY; SURVEY 8(b)
// "a debug mode checksums the arguments across ranks"): every rank posts a
// checksum of (T, tokens, parents) to every peer's receive buffer as an LL
// line flagged with this step's epoch, then compares all P lines.
// Step-kernel mode of the ingest kernel (step.cu): the first layer's QKV input
// is x * g in fp16 hi + lo with group sums X (the RMSNorm scale is deferred to
// the QKV epilogue, which reads the token's sum of squares ss[0][t]); every
// per-step counter and sum is zeroed and the padded token slots [T, 8 NT) of
// every activation buffer are cleared.
struct StepIngest {
  int on = 0;
  int* ctr = nullptr;
  int n_ctr = 0;
  float* ss = nullptr;      // [n_layers + 1][2][64]
  unsigned long long* ssx = nullptr;  // same shape, fixed point (deterministic mode)
  int n_ss = 0;
  uint8_t* act_o = nullptr;
  uint8_t* act_d = nullptr;
  uint8_t* act_lm = nullptr;
  int K_o = 0, K_d = 0;
};
// zero token slot t of an a2-layout buffer with K columns (columns split over kNormSplit CTAs)
SS_DEV void zero_a2_slot(uint8_t* act, int t, int K, int NT, int part) {
  for (int f = threadIdx.x; f < K / 4; f += 256)
    if ((f % 4) == part)
      for (int lo = 0; lo < 2; ++lo) {
        *reinterpret_cast<uint32_t*>(act + a2_frag(t, 4 * f, NT, lo)) = 0u;
        *reinterpret_cast<uint32_t*>(act + a2_frag(t, 4 * f + 2, NT, lo)) = 0u;
      }
  for (int g = threadIdx.x; g < K / 128; g += 256)
    if ((g % 4) == part) *reinterpret_cast<float*>(act + a2_xsum(t, g, NT)) = 0.f;
}

struct ConsistencyArgs {
  uint4* recv = nullptr;                  // own receive buffer (consistency area)
  uint4* peer_recv[kMaxPeers] = {nullptr};  // every rank's consistency area
  int rank = 0, P = 1, loopback = 0, flag_ofs = 0;
};

__global__ void __launch_bounds__(256) embed_meta_kernel(DevState* st, const int32_t* tokens,
                                                         const int32_t* parents, int T_in, const uint16_t* E,
                                                         int V, int h, float* x, const uint16_t* gain,
                                                         uint8_t* act, int NT, float eps, int epoch_stride,
                                                         const uint4* mbox_in, int max_tree, ConsistencyArgs ca,
                                                         StepIngest si, int T0) {
  __shared__ int s_tok[SS_MAX_TREE], s_par[SS_MAX_TREE];
  __shared__ int s_bad;
  __shared__ int s_T;
  __shared__ int s_tmo;
  __shared__ float s_red[8];
  pdl_wait();
  pdl_trigger();
  const int tid = threadIdx.x;
  // graph capacity: the step was captured for 8*NT token slots (and the KV /
  // RoPE capacity checks assumed max_tree): larger trees are refused
  // non-square forward (ss_extend_tree): slots are nodes [T0, T0 + T)
  // of a tree whose nodes [0, T0) are cached; the mailbox carries whole trees
  if (mbox_in) T0 = 0;
  const int cap = max(0, min(8 * NT, max_tree - T0));
  if (tid == 0) s_tmo = 0;
  // a13: the tree arrives in the inbox as LL lines ("sends a
  // sub-graph ... to the target worker"): line 0 = (T, seq), line 1+i =
  // (token_i, parent_i), every line flagged with the message sequence number.
  uint32_t mtok = 0, mpar = 0;
  if (mbox_in) {
    const uint32_t seq = st->mbox_seq + 1;
    if (tid == 0) {
      uint32_t d1 = 0, d2 = 0;
      const bool ok = ll_wait(mbox_in, seq, d1, d2);
      s_T = ok ? (int)d1 : 0;
      if (!ok) s_tmo = 1;
      if (blockIdx.x == 0 && blockIdx.y == 0) {
        st->mbox_cur = seq;
        st->mbox_mode = 1;
      }
    }
    __syncthreads();
    T_in = s_T;
    if (tid < min(max(T_in, 0), cap)) {
      // a line that never arrives is a timeout of the whole message (never a
      // silently substituted node)
      if (!ll_wait(mbox_in + 1 + tid, seq, mtok, mpar)) { mtok = 0; mpar = 0; s_tmo = 1; }
    }
  } else if (blockIdx.x == 0 && blockIdx.y == 0 && tid == 0) {
    st->mbox_mode = 0;
  }
  const int T = min(max(T_in, 1), cap);
  if (tid == 0) s_bad = (T_in < 1 || T_in > cap) ? 1 : 0;
  __syncthreads();
  if (blockIdx.x == 0 && blockIdx.y == 0 && tid == 0) {
    st->mbox_tmo = s_tmo;
    if (s_tmo) st->timeout = 1;
  }
  if (tid < T) {
    int p = mbox_in ? (int)mpar : parents[tid], tk = mbox_in ? (int)mtok : tokens[tid];
    const int node = T0 + tid;  // parents index the whole tree
    bool bad = (node == 0) ? (p != -1) : (p < 0 || p >= node);
    bad = bad || tk < 0 || tk >= V;
    if (bad) atomicOr(&s_bad, 1);
    s_par[tid] = (node == 0) ? -1 : ((p < 0 || p >= node) ? 0 : p);
    s_tok[tid] = (tk < 0 || tk >= V) ? 0 : tk;
  }
  __syncthreads();
  const int t = blockIdx.x, part = blockIdx.y;
  if (t == 0 && part == 0 && tid < SS_MAX_TREE) {
    if (tid >= T0 && tid < T0 + T) {
      // walk the new nodes' parents; a cached ancestor contributes its stored
      // ancestor mask and depth (pos - L)
      unsigned long long anc = 0;
      int dep = 0, j = tid;
      while (j >= T0) {
        anc |= 1ull << j;
        j = s_par[j - T0];
        ++dep;
      }
      if (j >= 0) {
        anc |= st->anc[j];
        dep += st->pos[j] - st->L;
      } else {
        dep -= 1;
      }
      st->anc[tid] = anc;
      st->pos[tid] = st->L + dep;
      st->tokens[tid] = s_tok[tid - T0];
      st->parents[tid] = s_par[tid - T0];
    } else if (tid >= T0) {
      st->anc[tid] = 0ull;
      st->pos[tid] = st->L;
      st->tokens[tid] = -1;
      st->parents[tid] = -2;
    }
    if (tid == 0) {
      st->T = T;
      st->T0 = T0;
      int status = s_bad ? SS_EINVAL : SS_OK;
      // LL flag epoch of this step: flags epoch + [0, epoch_stride) are used
      // by the all-reduces and the argmax exchange; 0 is never a live flag.
      uint32_t e = st->epoch + (uint32_t)epoch_stride;
      if (e < st->epoch || e + (uint32_t)epoch_stride < e) e = 1;
      st->epoch = e;
      st->max_written = max(st->max_written, st->L + T0 + T);
      if ((st->debug & SS_DEBUG_CONSISTENCY) && ca.P > 1) {
        uint32_t hsh = (2166136261u ^ (uint32_t)T_in) * 16777619u ^ (uint32_t)T0;
        for (int i = 0; i < T; ++i) {
          hsh = (hsh ^ (uint32_t)s_tok[i]) * 16777619u;
          hsh = (hsh ^ (uint32_t)s_par[i]) * 16777619u;
        }
        hsh ^= (uint32_t)s_bad << 31;
        const uint32_t flag = e + (uint32_t)ca.flag_ofs;
        for (int p = 0; p < ca.P; ++p)
          ll_store(ca.peer_recv[p] + (ca.loopback ? p : ca.rank), hsh, (uint32_t)T, flag);
        for (int p = 0; p < ca.P; ++p) {
          uint32_t d1 = 0, d2 = 0;
          long spins = 0;
          while (!ll_try_load(ca.recv + p, flag, d1, d2))
            if (++spins > (1L << 26)) { st->timeout = 1; break; }
          if (d1 != hsh) status = SS_ECONSISTENCY;
        }
      }
      st->status = status;
    }
  }
  const int nv = h / 4;  // 4-element vectors per row
  if (si.on) {
    // per-step counters and sums of squares (ss[0][t < T] is written below)
    const int nb = gridDim.x * gridDim.y, bi = blockIdx.y * gridDim.x + blockIdx.x;
    for (int i = bi * 256 + tid; i < si.n_ctr; i += nb * 256) si.ctr[i] = 0;
    for (int i = bi * 256 + tid; i < si.n_ss; i += nb * 256) {
      if (i >= 64 || i >= T) si.ss[i] = 0.f;
      if (si.ssx) si.ssx[i] = 0ull;
    }
  }
  if (t >= T && si.on) {  // padded token slot of every step-kernel input
    zero_a2_slot(act, t, h, NT, part);
    zero_a2_slot(si.act_o, t, si.K_o, NT, part);
    zero_a2_slot(si.act_d, t, si.K_d, NT, part);
    for (int f = tid; f < nv; f += 256)
      if ((f % kNormSplit) == part)
        for (int hl = 0; hl < 2; ++hl) {
          *reinterpret_cast<uint32_t*>(si.act_lm + frag_offset(t + hl * 8 * NT, 4 * f, 2 * NT)) = 0u;
          *reinterpret_cast<uint32_t*>(si.act_lm + frag_offset(t + hl * 8 * NT, 4 * f + 2, 2 * NT)) = 0u;
        }
    return;
  }
  if (t >= T) {          // padded token slot: zero its activation column and group sums
    for (int f = tid; f < nv; f += 256)
      if ((f % kNormSplit) == part) {
        *reinterpret_cast<uint32_t*>(act + act_frag_offset(t, 4 * f, NT)) = 0u;
        *reinterpret_cast<uint32_t*>(act + act_frag_offset(t, 4 * f + 2, NT)) = 0u;
      }
    for (int g = tid; g < h / 128; g += 256)
      if ((g % kNormSplit) == part) *reinterpret_cast<float*>(act + act_xsum_offset(t, g, NT)) = 0.f;
    return;
  }
  const uint2* e = reinterpret_cast<const uint2*>(E + (size_t)s_tok[t] * h);
  float4 v[kMaxVec];
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < kMaxVec; ++i) {
    int f = tid + 256 * i;
    if (f < nv) {
      uint2 w = e[f];
      v[i] = make_float4(bf16_lo(w.x), bf16_hi(w.x), bf16_lo(w.y), bf16_hi(w.y));
      ss += v[i].x * v[i].x + v[i].y * v[i].y + v[i].z * v[i].z + v[i].w * v[i].w;
    }
  }
  ss = block_sum_256(ss, s_red);
  if (si.on) {
    // x * g (fp16 hi + lo, X of hi + lo); the QKV epilogue applies rsqrt(ss / h + eps)
    if (part == 0 && tid == 0) si.ss[t] = ss;
    float4* xs4 = reinterpret_cast<float4*>(x + (size_t)t * h);
#pragma unroll
    for (int i = 0; i < kMaxVec; ++i) {
      const int f = tid + 256 * i;
      if (256 * i >= nv) continue;  // warp-uniform
      float xs = 0.f;
      if (f < nv) {
        const uint2 gw = reinterpret_cast<const uint2*>(gain)[f];
        const float y0 = v[i].x * bf16_lo(gw.x), y1 = v[i].y * bf16_hi(gw.x);
        const float y2 = v[i].z * bf16_lo(gw.y), y3 = v[i].w * bf16_hi(gw.y);
        const uint32_t h01 = pack_half2(y0, y1), h23 = pack_half2(y2, y3);
        const __half2 a01 = *reinterpret_cast<const __half2*>(&h01), a23 = *reinterpret_cast<const __half2*>(&h23);
        const uint32_t l01 = pack_half2(y0 - __low2float(a01), y1 - __high2float(a01));
        const uint32_t l23 = pack_half2(y2 - __low2float(a23), y3 - __high2float(a23));
        xs = (half2_sum(h01) + half2_sum(l01)) + (half2_sum(h23) + half2_sum(l23));
        if ((f % kNormSplit) == part) {
          xs4[f] = v[i];
          *reinterpret_cast<uint32_t*>(act + a2_frag(t, 4 * f, NT, 0)) = h01;
          *reinterpret_cast<uint32_t*>(act + a2_frag(t, 4 * f + 2, NT, 0)) = h23;
          *reinterpret_cast<uint32_t*>(act + a2_frag(t, 4 * f, NT, 1)) = l01;
          *reinterpret_cast<uint32_t*>(act + a2_frag(t, 4 * f + 2, NT, 1)) = l23;
        }
      }
      xs = warp_sum(xs);  // the warp's 32 vectors are exactly one 128-group
      const int g = f >> 5;
      if ((tid & 31) == 0 && f < nv && (g % kNormSplit) == part) *reinterpret_cast<float*>(act + a2_xsum(t, g, NT)) = xs;
    }
    return;
  }
  const float r = rsqrtf(ss / (float)h + eps);
  float4* xr = reinterpret_cast<float4*>(x + (size_t)t * h);
#pragma unroll
  for (int i = 0; i < kMaxVec; ++i) {
    const int f = tid + 256 * i;
    if (256 * i < nv) {  // warp-uniform: nv is a multiple of 32
      float xs = 0.f;
      if (f < nv) {
        const uint2 gw = reinterpret_cast<const uint2*>(gain)[f];
        const uint32_t p01 = pack_half2(v[i].x * r * bf16_lo(gw.x), v[i].y * r * bf16_hi(gw.x));
        const uint32_t p23 = pack_half2(v[i].z * r * bf16_lo(gw.y), v[i].w * r * bf16_hi(gw.y));
        xs = half2_sum(p01) + half2_sum(p23);
        if ((f % kNormSplit) == part) {
          xr[f] = v[i];
          *reinterpret_cast<uint32_t*>(act + act_frag_offset(t, 4 * f, NT)) = p01;
          *reinterpret_cast<uint32_t*>(act + act_frag_offset(t, 4 * f + 2, NT)) = p23;
        }
      }
      xs = warp_sum(xs);  // the warp's 32 vectors are exactly one 128-group
      const int g = f >> 5;
      if ((tid & 31) == 0 && f < nv && (g % kNormSplit) == part)
        *reinterpret_cast<float*>(act + act_xsum_offset(t, g, NT)) = xs;
    }
  }
}

void launch_embed_meta(ss_shard* s, const int32_t* tokens, const int32_t* parents, int T, int NT,
                       cudaStream_t st, bool from_mailbox, bool step_mode, int T0) {
  const uint16_t* g0 = s->layers[0].attn_norm;
  ConsistencyArgs ca;
  ca.rank = s->rank;
  ca.P = s->P;
  ca.loopback = s->loopback ? 1 : 0;
  ca.flag_ofs = 2 * s->cfg.n_layers + 1;  // inside the step's epoch stride, unused by the all-reduces
  if (s->P > 1 && s->recv) {
    const size_t ofs = consistency_line_offset(s);
    ca.recv = reinterpret_cast<uint4*>(s->recv) + ofs;
    for (int p = 0; p < s->P; ++p)
      ca.peer_recv[p] = s->peer_recv[p] ? reinterpret_cast<uint4*>(s->peer_recv[p]) + ofs : nullptr;
  }
  StepIngest si;
  if (step_mode) {
    si.on = 1;
    si.ctr = s->step_ctr;
    si.n_ctr = s->cfg.n_layers * kCtrPerLayerH + kCtrGlobalH;
    si.ss = s->step_ss;
    si.ssx = s->step_ssx;
    si.n_ss = (s->cfg.n_layers + 1) * 2 * 64;
    si.act_o = s->act_o;
    si.act_d = s->act_d;
    si.act_lm = s->act_lm;
    si.K_o = s->Hq_l * s->cfg.head_dim;
    si.K_d = s->I_l;
  }
  ss_pdl_off = s->launch_cap > 0 && !s->loopback;  // capped grids share the GPU (kernels.h)
  launch_pdl(embed_meta_kernel, dim3(8 * NT, kNormSplit), dim3(256), 0, st, s->dstate, tokens, parents, T,
             (const uint16_t*)s->embed, s->cfg.vocab, s->cfg.hidden, s->x, g0, s->act_h, NT, s->cfg.rms_eps,
             2 * s->cfg.n_layers + 2, from_mailbox ? (const uint4*)s->mbox_in : (const uint4*)nullptr,
             s->cfg.max_tree, ca, si, T0);
  ss_pdl_off = false;
}

// ---------------------------------------------------------------- a13 draft-side helpers
// Post one tree into a target inbox as LL lines (the draft group's send,
// Alg. 1 P:286 "Send it to the target worker to verify").
struct MboxTree {
  int32_t tokens[SS_MAX_TREE];
  int32_t parents[SS_MAX_TREE];
};
__global__ void mailbox_post_kernel(uint4* inbox, MboxTree tree, int T, uint32_t seq) {
  const int i = threadIdx.x;
  if (i < T) ll_store(inbox + 1 + i, (uint32_t)tree.tokens[i], (uint32_t)tree.parents[i], seq);
  if (i == 0) ll_store(inbox, (uint32_t)T, seq, seq);
}
void launch_mailbox_post(void* inbox, const int32_t* tokens, const int32_t* parents, int T, uint32_t seq,
                         cudaStream_t st) {
  MboxTree t{};
  for (int i = 0; i < T && i < SS_MAX_TREE; ++i) {
    t.tokens[i] = tokens[i];
    t.parents[i] = parents[i];
  }
  mailbox_post_kernel<<<1, SS_MAX_TREE, 0, st>>>((uint4*)inbox, t, T, seq);
}
// Wait for the verified path with sequence number seq in an outbox and copy
// it out: out[0] = n_accepted, out[1] = bonus, out[2] = stop, out[3] = the
// step's status (SS_OK, or SS_EINVAL / SS_ETIMEOUT / SS_ECONSISTENCY: then
// n = 0 and no path follows), then n (node index, token) pairs.  A message
// that never arrives gives n = -1, status SS_ETIMEOUT.
__global__ void mailbox_recv_kernel(const uint4* outbox, uint32_t seq, int32_t* out) {
  __shared__ int s_n;
  uint32_t d1 = 0, d2 = 0;
  if (threadIdx.x == 0) {
    const bool ok = ll_wait(outbox, seq, d1, d2);
    s_n = ok ? (int)(d1 & 0xFFFFu) : -1;
    out[0] = s_n;
    out[1] = ok ? (int)d2 : 0;
    out[2] = ok ? (int)(d1 >> 31) : 0;
    out[3] = ok ? -(int)((d1 >> 16) & 0xFFu) : SS_ETIMEOUT;
  }
  __syncthreads();
  const int i = threadIdx.x;
  if (i < s_n && ll_wait(outbox + 1 + i, seq, d1, d2)) {
    out[4 + 2 * i] = (int)d1;
    out[5 + 2 * i] = (int)d2;
  }
}
void launch_mailbox_recv(const void* outbox, uint32_t seq, int32_t* dev_out, cudaStream_t st) {
  mailbox_recv_kernel<<<1, SS_MAX_TREE, 0, st>>>((const uint4*)outbox, seq, dev_out);
}

// ---------------------------------------------------------------- RMSNorm
// xn = x * rsqrt(mean(x^2) + eps) * g (R5).  split == 0: fp16 fragment-ordered
// input of a W4 GEMM.  split == 1: the LM-head input as bf16 hi = bf16(xn) in
// n-tiles [0, NT) and lo = bf16(xn - hi) in [NT, 2NT) (the LM head is bf16,
// P:501; hi + lo carries ~16 mantissa bits).
SS_DEV uint32_t split_pack(float a, float b, int lo) {
  uint32_t hi = pack_bf16x2(a, b);
  if (!lo) return hi;
  return pack_bf16x2(a - bf16_lo(hi), b - bf16_hi(hi));
}

__global__ void __launch_bounds__(256) prep_norm_kernel(const DevState* st, const float* x, int h,
                                                        const uint16_t* gain, uint8_t* act, int NT, float eps,
                                                        int split) {
  __shared__ float s_red[8];
  pdl_wait();
  pdl_trigger();
  const int t = blockIdx.x, part = blockIdx.y, tid = threadIdx.x;
  if (t >= st->T) return;
  const int nv = h / 4;
  const float4* xr = reinterpret_cast<const float4*>(x + (size_t)t * h);
  float4 v[kMaxVec];
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < kMaxVec; ++i) {
    int f = tid + 256 * i;
    if (f < nv) {
      v[i] = __ldcg(xr + f);
      ss += v[i].x * v[i].x + v[i].y * v[i].y + v[i].z * v[i].z + v[i].w * v[i].w;
    }
  }
  ss = block_sum_256(ss, s_red);
  const float r = rsqrtf(ss / (float)h + eps);
#pragma unroll
  for (int i = 0; i < kMaxVec; ++i) {
    const int f = tid + 256 * i;
    if (256 * i >= nv) continue;  // warp-uniform
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
    if (f < nv) {
      const uint2 gw = reinterpret_cast<const uint2*>(gain)[f];
      a0 = v[i].x * r * bf16_lo(gw.x);
      a1 = v[i].y * r * bf16_hi(gw.x);
      a2 = v[i].z * r * bf16_lo(gw.y);
      a3 = v[i].w * r * bf16_hi(gw.y);
    }
    const int k = 4 * f;
    if (!split) {
      const uint32_t p01 = pack_half2(a0, a1), p23 = pack_half2(a2, a3);
      if (f < nv && (f % kNormSplit) == part) {
        *reinterpret_cast<uint32_t*>(act + act_frag_offset(t, k, NT)) = p01;
        *reinterpret_cast<uint32_t*>(act + act_frag_offset(t, k + 2, NT)) = p23;
      }
      float xs = f < nv ? half2_sum(p01) + half2_sum(p23) : 0.f;
      xs = warp_sum(xs);  // the warp's 32 vectors are exactly one 128-group
      const int g = f >> 5;
      if ((tid & 31) == 0 && f < nv && (g % kNormSplit) == part)
        *reinterpret_cast<float*>(act + act_xsum_offset(t, g, NT)) = xs;
    } else if (f < nv && (f % kNormSplit) == part) {
      // LM head input: 2*NT n-tiles, token t in tile t/8 (bf16 hi) and NT + t/8 (lo)
      *reinterpret_cast<uint32_t*>(act + frag_offset(t, k, 2 * NT)) = split_pack(a0, a1, 0);
      *reinterpret_cast<uint32_t*>(act + frag_offset(t, k + 2, 2 * NT)) = split_pack(a2, a3, 0);
      *reinterpret_cast<uint32_t*>(act + frag_offset(t + 8 * NT, k, 2 * NT)) = split_pack(a0, a1, 1);
      *reinterpret_cast<uint32_t*>(act + frag_offset(t + 8 * NT, k + 2, 2 * NT)) = split_pack(a2, a3, 1);
    }
  }
}

void launch_prep_norm(ss_shard* s, const uint16_t* gain, int NT, int split, cudaStream_t st) {
  launch_pdl(prep_norm_kernel, dim3(8 * NT, kNormSplit), dim3(256), 0, st, (const DevState*)s->dstate,
             (const float*)s->x, s->cfg.hidden, gain, split ? s->act_lm : s->act_h, NT, s->cfg.rms_eps, split);
}

// ---------------------------------------------------------------- a12 commit
// For every (layer, local kv head): K/V[L + k] <- K/V[L + chain[k]], k < n
// (BASELINE north_star "KV-cache compaction that keeps only the accepted
// path").  Two-phase (all loads, barrier, all stores) because the
// source and destination row ranges overlap.  The CTA that finishes last
// advances L by n (root + accepted, never the bonus: R9).
__global__ void __launch_bounds__(256) commit_kernel(DevState* st, uint16_t* kc, uint16_t* vc, int Hkv_l, int d,
                                                     int max_ctx_pad, int from_result) {
  pdl_wait();
  pdl_trigger();
  const int kvh = blockIdx.x, layer = blockIdx.y;
  int n;
  const int* chain;
  if (from_result) {
    bool ok = st->have_verify && st->result.status == SS_OK;
    n = ok ? st->result.n_accepted : 0;
    chain = st->result.accepted;
  } else {
    n = st->commit_n;
    chain = st->commit_chain;
  }
  const int L = st->L;
  const int cpr = d / 8;  // 16-byte chunks per row
  const size_t base = ((size_t)layer * Hkv_l + kvh) * max_ctx_pad * d;
  uint4 buf[2][8];
  const int total = n * cpr;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    int idx = threadIdx.x + i * 256;
    if (idx < total) {
      int k = idx / cpr, c = idx % cpr;
      int src = L + chain[k];
      size_t off = base + (size_t)(src - (src & 63)) * d + (src & 63) * d + ((c ^ (src & 7)) << 3);
      buf[0][i] = *reinterpret_cast<const uint4*>(kc + off);
      buf[1][i] = *reinterpret_cast<const uint4*>(vc + off);
    }
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    int idx = threadIdx.x + i * 256;
    if (idx < total) {
      int k = idx / cpr, c = idx % cpr;
      int dst = L + k;
      size_t off = base + (size_t)(dst - (dst & 63)) * d + (dst & 63) * d + ((c ^ (dst & 7)) << 3);
      *reinterpret_cast<uint4*>(kc + off) = buf[0][i];
      *reinterpret_cast<uint4*>(vc + off) = buf[1][i];
    }
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    int old = atomicAdd(&st->commit_done, 1);
    if (old == (int)(gridDim.x * gridDim.y) - 1) {
      st->commit_done = 0;
      st->L = L + n;
      st->have_verify = 0;
    }
  }
}

void launch_commit(ss_shard* s, int from_result, cudaStream_t st) {
  dim3 grid(s->Hkv_l, s->cfg.n_layers);
  launch_pdl(commit_kernel, grid, dim3(256), 0, st, s->dstate, s->kcache, s->vcache, s->Hkv_l, s->cfg.head_dim,
             s->max_ctx_pad, from_result);
}

// ---------------------------------------------------------------- RoPE table
// cos/sin(pos * theta^(-2j/d)) evaluated in fp64 (R2), stored fp32.
__global__ void rope_table_kernel(float2* cs, int max_pos, int d, double theta) {
  int half = d / 2;
  size_t n = (size_t)max_pos * half;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    int pos = (int)(i / half), j = (int)(i % half);
    double ang = (double)pos * pow(theta, -2.0 * j / d);
    double s, c;
    sincos(ang, &s, &c);
    cs[i] = make_float2((float)c, (float)s);
  }
}

void launch_rope_table(float2* cs, int max_pos, int d, double theta, cudaStream_t st) {
  rope_table_kernel<<<592, 256, 0, st>>>(cs, max_pos, d, theta);
}

// ---------------------------------------------------------------- synthetic inputs
// Device re-implementation of synth/generators.py (counter-based SplitMix64
// finaliser; exactly-rounded fp32 conversions in the same order).
constexpr uint64_t GOLDEN = 0x9E3779B97F4A7C15ull;
constexpr uint64_t C1 = 0xBF58476D1CE4E5B9ull;
constexpr uint64_t C2 = 0x94D049BB133111EBull;

SS_DEV uint64_t fmix64(uint64_t z) {
  z ^= z >> 30;
  z *= C1;
  z ^= z >> 27;
  z *= C2;
  z ^= z >> 31;
  return z;
}
SS_DEV uint64_t hash_u64(uint64_t key, uint64_t idx) { return fmix64(key + (idx + 1) * GOLDEN); }
SS_DEV float approx_normal(uint64_t hv) {
  const float inv16 = 1.0f / 65536.0f;
  float u0 = __fmul_rn((float)(uint32_t)(hv & 0xFFFF), inv16);
  float u1 = __fmul_rn((float)(uint32_t)((hv >> 16) & 0xFFFF), inv16);
  float u2 = __fmul_rn((float)(uint32_t)((hv >> 32) & 0xFFFF), inv16);
  float u3 = __fmul_rn((float)(uint32_t)((hv >> 48) & 0xFFFF), inv16);
  float s = __fadd_rn(__fadd_rn(__fadd_rn(u0, u1), u2), u3);
  return __fmul_rn(__fsub_rn(s, 2.0f), 1.7320508075688772f);
}
SS_DEV uint16_t bf16_rne_bits(float f) {
  uint32_t b = __float_as_uint(f);
  return (uint16_t)((b + 0x7FFFu + ((b >> 16) & 1u)) >> 16);
}

__constant__ uint64_t c_keys[3];  // qweight, qzeros, scales stream keys of the current tensor

// canonical coordinates (part = which of the fused canonical tensors, n, k)
SS_DEV bool lin_map(const LinMap& m, int row, int k, int& part, int& n, int& kk) {
  kk = k;
  if (m.mode == 0) {
    int nq = m.Hq_l * m.d, nk = m.Hkv_l * m.d;
    if (row < nq) { part = 0; n = m.rank * nq + row; }
    else if (row < nq + nk) { part = 1; n = m.rank * nk + row - nq; }
    else if (row < nq + 2 * nk) { part = 2; n = m.rank * nk + row - nq - nk; }
    else return false;
    if (n >= (part == 0 ? m.q_full : m.kv_full)) return false;  // zero-padded head
  } else if (m.mode == 1) {
    part = 0; n = row; kk = m.rank * m.Kl + k;
    if (kk >= m.K_full) return false;
  } else if (m.mode == 2) {
    int tg = row >> 7, r = row & 127;
    part = r < 64 ? 0 : 1;
    n = m.rank * m.I_l + tg * 64 + (r & 63);
    if (tg * 64 + (r & 63) >= m.I_l || n >= m.I_full) return false;
  } else {
    part = 0; n = row; kk = m.rank * m.Kl + k;
    if (kk >= m.K_full) return false;
  }
  return true;
}

// One thread per 32-bit nibble word of the packed W4 layout + metadata.
__global__ void synth_linear_kernel(uint8_t* dst, SynthLinArgs a) {
  const size_t units = (size_t)a.n_tg * a.S;
  const size_t words_per_unit = kW4Bytes / 4;      // 4096
  const size_t total = units * (words_per_unit + 32);  // + 32 meta "slots" (16 rows x 2 groups) per warp... see below
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    size_t u = i / (words_per_unit + 32);
    int w_in = (int)(i % (words_per_unit + 32));
    int tg = (int)(u / a.S), s = (int)(u % a.S);
    uint8_t* ub = dst + u * kW4UnitBytes;
    if (w_in < (int)words_per_unit) {
      int warp = w_in >> 9, rem = w_in & 511;
      int kb = rem >> 7, lane = (rem >> 2) & 31, j = rem & 3;
      int gq = lane >> 2, tq = lane & 3;
      uint32_t word = 0;
      for (int p = 0; p < 8; ++p) {
        int row = tg * 128 + warp * 16 + gq + 8 * (p & 1);
        int k = s * 256 + kb * 64 + j * 16 + 2 * tq + (p >> 2) + 8 * ((p >> 1) & 1);
        int part, n, kk;
        uint32_t q = 0;
        if (lin_map(a.m, row, k, part, n, kk)) {
          q = (uint32_t)(hash_u64(a.keys[part][0], (uint64_t)kk * a.N_full[part] + n) & 15u);
        } else {
          q = 8;  // padding rows: q == z == 8 -> weight 0
        }
        word |= q << (4 * p);
      }
      reinterpret_cast<uint32_t*>(ub)[w_in] = word;
    } else {
      // metadata: 32 slots per unit = 8 warps x 2 groups x (scales, zeros),
      // stored as lane-indexed (row gq, row gq+8) pairs (common.cuh)
      int slot = w_in - (int)words_per_unit;
      int warp = slot >> 2, grp = (slot >> 1) & 1, which = slot & 1;
      int g = s * 2 + grp;
      uint16_t sv[16];
      uint32_t zv[16];
      for (int i2 = 0; i2 < 16; ++i2) {
        int row = tg * 128 + warp * 16 + i2;
        int part, n, kk;
        sv[i2] = 0;
        zv[i2] = 8;
        if (lin_map(a.m, row, g * 128, part, n, kk)) {
          int gg = kk / 128;
          if (which == 0) {
            uint64_t hs = hash_u64(a.keys[part][2], (uint64_t)gg * a.N_full[part] + n);
            float u = __fmul_rn((float)(uint32_t)((hs >> 41) + (1u << 22)), 1.1920928955078125e-07f);
            sv[i2] = bf16_rne_bits(__fmul_rn(u, a.scale_c[part]));
          } else {
            zv[i2] = 6u + (uint32_t)(hash_u64(a.keys[part][1], (uint64_t)gg * a.N_full[part] + n) & 3u);
          }
        }
      }
      if (which == 0) {
        uint32_t* sc = reinterpret_cast<uint32_t*>(ub + kW4Bytes) + (warp * 2 + grp) * 8;
        for (int gq = 0; gq < 8; ++gq) sc[gq] = (uint32_t)sv[gq] | ((uint32_t)sv[gq + 8] << 16);
      } else {
        uint8_t* zb = ub + kW4Bytes + 512 + (warp * 2 + grp) * 8;
        for (int gq = 0; gq < 8; ++gq) zb[gq] = (uint8_t)(zv[gq] | (zv[gq + 8] << 4));
      }
    }
  }
}

void launch_synth_linear_args(uint8_t* dst, const SynthLinArgs& a, cudaStream_t st) {
  synth_linear_kernel<<<148 * 8, 256, 0, st>>>(dst, a);
}

// dense bf16 tensors: mode 0 = N(0,1)-like * scale, mode 1 = 1 + 0.1 * N(0,1)-like
__global__ void synth_dense_kernel(uint16_t* dst, size_t n, uint64_t key, size_t idx0, int mode, float scale) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    float v = approx_normal(hash_u64(key, idx0 + i));
    if (mode == 0) v = scale == 1.0f ? v : __fmul_rn(v, scale);
    else v = __fadd_rn(1.0f, __fmul_rn(v, 0.1f));
    dst[i] = bf16_rne_bits(v);
  }
}

void launch_synth_dense_key(uint16_t* dst, size_t n, uint64_t key, size_t idx0, int mode, float scale,
                            cudaStream_t st) {
  synth_dense_kernel<<<148 * 8, 256, 0, st>>>(dst, n, key, idx0, mode, scale);
}

// LM head, bf16 A-fragment units: [tg][s][warp][j][lane][4 words]
__global__ void synth_lm_kernel(uint8_t* dst, int V_l, int V_off, int V_full, int h, int n_tg, uint64_t key,
                                float scale) {
  const int S = h / 64;
  const size_t words = (size_t)n_tg * S * (kBFUnitBytes / 4);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < words; i += (size_t)gridDim.x * blockDim.x) {
    size_t u = i / 4096;
    int w_in = (int)(i % 4096);
    int tg = (int)(u / S), s = (int)(u % S);
    int warp = w_in >> 9, j = (w_in >> 7) & 3, lane = (w_in >> 2) & 31, r = w_in & 3;
    int gq = lane >> 2, tq = lane & 3;
    int row = tg * 128 + warp * 16 + gq + 8 * (r & 1);
    int k = s * 64 + j * 16 + 2 * tq + 8 * (r >> 1);
    uint32_t word = 0;
    int v = V_off + row;
    if (row < V_l && v < V_full) {
      uint16_t lo = bf16_rne_bits(__fmul_rn(approx_normal(hash_u64(key, (uint64_t)v * h + k)), scale));
      uint16_t hi = bf16_rne_bits(__fmul_rn(approx_normal(hash_u64(key, (uint64_t)v * h + k + 1)), scale));
      word = (uint32_t)lo | ((uint32_t)hi << 16);
    }
    reinterpret_cast<uint32_t*>(dst)[i] = word;
  }
}

void launch_synth_lm_key(uint8_t* dst, int V_l, int V_off, int V_full, int h, int n_tg, uint64_t key, float scale,
                         cudaStream_t st) {
  synth_lm_kernel<<<148 * 8, 256, 0, st>>>(dst, V_l, V_off, V_full, h, n_tg, key, scale);
}

// prefix KV rows [0, L) of one layer: canonical idx (pos*Hkv + kvh)*d + j
__global__ void synth_kv_kernel(uint16_t* cache, int layer, int Hkv_full, int Hkv_l, int kv0, int d, int L,
                                int max_ctx_pad, uint64_t key) {
  size_t n = (size_t)Hkv_l * L * d;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    int j = (int)(i % d);
    size_t r = i / d;
    int pos = (int)(r % L);
    int kvh = (int)(r / L);
    uint64_t idx = ((uint64_t)pos * Hkv_full + kv0 + kvh) * d + j;
    // canonical value = bf16(normal) (synth/generators.py); the cache holds it
    // exactly as fp16.  Zero-padded heads (arbitrary TP) hold 0.
    const float v = kv0 + kvh < Hkv_full
                        ? __uint_as_float((uint32_t)bf16_rne_bits(approx_normal(hash_u64(key, idx))) << 16)
                        : 0.f;
    size_t base = ((size_t)layer * Hkv_l + kvh) * max_ctx_pad * d;
    cache[base + kv_elem_offset(pos, j, d)] = f32_to_f16_bits(v);
  }
}

void launch_synth_kv_key(uint16_t* cache, int layer, int Hkv_full, int Hkv_l, int kv0, int d, int L,
                         int max_ctx_pad, uint64_t key, cudaStream_t st) {
  synth_kv_kernel<<<148 * 8, 256, 0, st>>>(cache, layer, Hkv_full, Hkv_l, kv0, d, L, max_ctx_pad, key);
}

}  // namespace ss

namespace ss {
// ---------------------------------------------------------------- test hook
// ss_debug_gemm: caller activations x[T][K] (fp32, rounded to fp16 like the
// step's own activations) -> the W4 GEMM input layout (fp16 fragments + the
// per-(group, token) sums X); token slots [T, 8 NT) are zeroed.  Thread-block
// t handles token t; block 0 also publishes T and (all-reduce mode) advances
// the LL flag epoch exactly like the step's ingest kernel.
__global__ void debug_act_kernel(DevState* st, const float* x, int T, int K, uint8_t* act, int NT, int bump_epoch,
                                 int epoch_stride) {
  const int t = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (t == 0 && threadIdx.x == 0) {
    st->T = T;
    if (bump_epoch) {
      uint32_t e = st->epoch + (uint32_t)epoch_stride;
      if (e < st->epoch || e + (uint32_t)epoch_stride < e) e = 1;
      st->epoch = e;
    }
  }
  // one warp per 128-column group: 4 columns per lane
  for (int g = warp; g < K / 128; g += blockDim.x / 32) {
    const int k = g * 128 + lane * 4;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (t < T) v = *reinterpret_cast<const float4*>(x + (size_t)t * K + k);
    const uint32_t p01 = pack_half2(v.x, v.y), p23 = pack_half2(v.z, v.w);
    *reinterpret_cast<uint32_t*>(act + act_frag_offset(t, k, NT)) = p01;
    *reinterpret_cast<uint32_t*>(act + act_frag_offset(t, k + 2, NT)) = p23;
    const float xs = warp_sum(half2_sum(p01) + half2_sum(p23));
    if (lane == 0) *reinterpret_cast<float*>(act + act_xsum_offset(t, g, NT)) = xs;
  }
}
void launch_debug_act(ss_shard* s, const float* x, int T, int K, uint8_t* act, int NT, int bump_epoch,
                      cudaStream_t st) {
  debug_act_kernel<<<8 * NT, 256, 0, st>>>(s->dstate, x, T, K, act, NT, bump_epoch, 2 * s->cfg.n_layers + 2);
}

// Lazy module loading (the CUDA 12 default) loads a kernel at its first
// launch, which can wait for running kernels: a producer whose kernel is
// loaded only after a consumer already spins on its flags would deadlock.
// Every kernel that takes part in a cross-kernel wait is loaded up front.
void warm_misc_kernels() {
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, embed_meta_kernel);
  cudaFuncGetAttributes(&a, prep_norm_kernel);
  cudaFuncGetAttributes(&a, commit_kernel);
  cudaFuncGetAttributes(&a, mailbox_post_kernel);
  cudaFuncGetAttributes(&a, mailbox_recv_kernel);
  cudaFuncGetAttributes(&a, debug_act_kernel);
}
}  // namespace ss
