// gemm.cu -- skinny W4A16 / BF16 GEMM for T-token trees (SURVEY 8(a) a3, a6,
// a8, a9, a10) with fused epilogues:
//   EPI_QKV    : RoPE ("fuse the position embedding") + q store + tree
//                K/V write into the cache at rows L+i (R10)
//   EPI_RESID  : residual add x += y; for tp > 1 the tensor-parallel
//                all-reduce is fused here as flagged peer stores
//   EPI_SWIGLU : silu(x W) * (x V) on the same tile (R4)
//   EPI_ARGMAX : per-node argmax over the vocab shard (R6), then the greedy
//                accept walk (a11) in the CTA that finishes last.
//
// Design (B200): weights stream HBM -> SMEM through the TMA bulk engine
// (cp.async.bulk + mbarrier ring, one producer warp), 8 consumer warps
// dequantise int4 -> bf16 in registers ((128+q) via lop3, minus (128+z) with
// one bf16x2 subtract: exact integers) and issue mma.sync m16n8k16 with the
// weights as the M=16 operand and the T tree tokens as N=8 columns.  The
// group scale is applied in fp32 after each 128-deep group, so no weight is
// ever rounded (R3).  Work = (tile-group of 128 rows) x (K stage) units split
// evenly over a persistent grid (stream-K); partial tiles are reduced with
// red.global.add.v2.f32 and a per-tile-group arrival counter picks the CTA
// that runs the epilogue (no extra kernel, no grid barrier).
#include "common.cuh"
#include "internal.h"
#include "kernels.h"

namespace ss {

template <int WFMT, int NT>
struct GemmCfg {
  static constexpr int KS = WFMT == 0 ? kW4KS : kBFKS;
  static constexpr int WBYTES = WFMT == 0 ? kW4UnitBytes : kBFUnitBytes;
  static constexpr int ANT = WFMT == 0 ? NT : 2 * NT;  // LM head: bf16 hi + lo tiles
  static constexpr int ABYTES = (KS / 16) * ANT * 256;
  static constexpr int UBYTES = WBYTES + ABYTES;
  // NT <= 2: 3 stages (~63-76 KB) -> 3 CTAs / SM; larger NT: 4 stages, 1-2 CTAs / SM
#ifdef SS_EXP_STAGES
  static constexpr int STAGES = SS_EXP_STAGES;
#else
  static constexpr int STAGES = (UBYTES <= 26 * 1024) ? 3 : 4;
#endif
  static constexpr int SMEM = STAGES * UBYTES + 1024;
  static constexpr int THREADS = 288;  // 8 consumer warps + 1 producer warp
};

// ---------------------------------------------------------------- epilogues
template <int NT>
__device__ void epi_qkv(const EpiArgs& e, int tg, const float* acc, int T) {
  const int TP = NT * 8;
  const int d = e.d, half = d >> 1;
  const int nq = e.Hq_l * d, nk = e.Hkv_l * d;
  const int L = e.st->L;
  for (int idx = threadIdx.x; idx < 128 * T; idx += 256) {
    int r = idx / T, t = idx - r * T;
    int row = tg * 128 + r;
    float v = __ldcg(acc + (size_t)r * TP + t);
    int j = row % d;
    int pos = e.st->pos[t];
    if (row < nq + nk) {  // q or k: rotate-half RoPE (R2)
      int pr = (j < half) ? r + half : r - half;
      float pv = __ldcg(acc + (size_t)pr * TP + t);
      float2 cs = e.rope_cs[(size_t)pos * half + (j % half)];
      v = (j < half) ? (v * cs.x - pv * cs.y) : (v * cs.x + pv * cs.y);
    }
    uint16_t b = f32_to_bf16_bits(v);
    if (row < nq) {  // q as bf16 hi + lo planes (attention.cu)
      int hq = row / d, kvh = hq / e.G, jj = hq - kvh * e.G;
      size_t qi = ((size_t)kvh * (e.G * SS_MAX_TREE) + t * e.G + jj) * d + j;
      e.qbuf[qi] = b;
      e.qbuf[qi + (size_t)e.Hkv_l * e.G * SS_MAX_TREE * d] = f32_to_bf16_bits(v - bf16_bits_to_f32(b));
    } else {
      int kvh = (row < nq + nk) ? (row - nq) / d : (row - nq - nk) / d;
      uint16_t* c = (row < nq + nk) ? e.kc : e.vc;
      size_t base = ((size_t)e.layer * e.Hkv_l + kvh) * e.max_ctx_pad * d;
      c[base + kv_elem_offset(L + t, j, d)] = b;
    }
  }
}

template <int NT>
__device__ void epi_swiglu(const EpiArgs& e, int tg, const float* acc, int T) {
  const int TP = NT * 8;
  // tile-group rows: [0,64) gate, [64,128) up for intermediate columns tg*64..+64
  for (int idx = threadIdx.x; idx < 32 * T; idx += 256) {
    int cp = idx / T, t = idx - cp * T;
    float g0 = __ldcg(acc + (size_t)(2 * cp) * TP + t);
    float g1 = __ldcg(acc + (size_t)(2 * cp + 1) * TP + t);
    float u0 = __ldcg(acc + (size_t)(64 + 2 * cp) * TP + t);
    float u1 = __ldcg(acc + (size_t)(64 + 2 * cp + 1) * TP + t);
    float h0 = g0 / (1.f + __expf(-g0)) * u0;
    float h1 = g1 / (1.f + __expf(-g1)) * u1;
    int k = tg * 64 + 2 * cp;
    *reinterpret_cast<uint32_t*>(e.act_out + act_frag_offset(t, k, NT)) = pack_half2(h0, h1);
  }
}

template <int NT>
__device__ void epi_resid_local(const EpiArgs& e, int tg, const float* acc, int T) {
  const int TP = NT * 8;
  for (int idx = threadIdx.x; idx < 128 * T; idx += 256) {
    int t = idx >> 7, r = idx & 127;
    e.x[(size_t)t * e.h + tg * 128 + r] += __ldcg(acc + (size_t)r * TP + t);
  }
}

// tp > 1, phase 1 (right after the tile-group completes): push this rank's
// fp32 partial of the tile-group to every peer as LL lines (2 floats + 2
// flags per 16 B).  Line index = ((tg * 128 + r) * T64 + t/2) for rank slot.
template <int NT>
__device__ void epi_ar_send(const EpiArgs& e, int tg, const float* acc, int T) {
  const int TP = NT * 8;
  const uint32_t flag = e.st->epoch + e.ar_seq;
  const int pairs = (T + 1) >> 1;
  for (int idx = threadIdx.x; idx < 128 * pairs; idx += 256) {
    int r = idx / pairs, tp = idx - r * pairs;
    float a = __ldcg(acc + (size_t)r * TP + 2 * tp);
    float b = __ldcg(acc + (size_t)r * TP + 2 * tp + 1);
    size_t line = (((size_t)(e.ar_seq & 1) * e.P + e.rank) * e.n_tg_total + tg) * 128 * 32 + (size_t)r * 32 + tp;
    for (int p = 0; p < e.P; ++p)
      ll_store(reinterpret_cast<uint4*>(e.peer_recv[p]) + line, __float_as_uint(a), __float_as_uint(b), flag);
  }
}

// tp > 1, phase 2 (after the CTA's compute loop): wait for every rank's
// partial of the tile-group, sum in rank order (identical on all ranks), add.
template <int NT>
__device__ void epi_ar_recv(const EpiArgs& e, int tg, int T) {
  const uint32_t flag = e.st->epoch + e.ar_seq;
  const int pairs = (T + 1) >> 1;
  for (int idx = threadIdx.x; idx < 128 * pairs; idx += 256) {
    int r = idx / pairs, tp = idx - r * pairs;
    float s0 = 0.f, s1 = 0.f;
    for (int p = 0; p < e.P; ++p) {
      const uint4* src = reinterpret_cast<const uint4*>(e.recv) +
                         (((size_t)(e.ar_seq & 1) * e.P + p) * e.n_tg_total + tg) * 128 * 32 + (size_t)r * 32 + tp;
      uint32_t d1, d2;
      long spins = 0;
      while (!ll_try_load(src, flag, d1, d2)) {
        if (++spins > (1L << 26)) { e.st->timeout = 1; break; }
      }
      s0 += __uint_as_float(d1);
      s1 += __uint_as_float(d2);
    }
    int t0 = 2 * tp;
    e.x[(size_t)t0 * e.h + tg * 128 + r] += s0;
    if (t0 + 1 < T) e.x[(size_t)(t0 + 1) * e.h + tg * 128 + r] += s1;
  }
}

template <int NT>
__device__ void epi_argmax(const EpiArgs& e, int tg, const float* acc, int T) {
  const int TP = NT * 8;
  int r = threadIdx.x & 127;
  int v = tg * 128 + r;
  bool valid = v < e.V_l;
  for (int t = threadIdx.x >> 7; t < T; t += 2) {
    float val = valid ? __ldcg(acc + (size_t)r * TP + t) : -INFINITY;
    if (valid && e.logits) e.logits[(size_t)t * e.logits_ld + v] = val;
    unsigned long long key = valid ? argmax_key(val, (uint32_t)(e.V_off + v)) : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      unsigned long long other = __shfl_xor_sync(0xffffffffu, key, o);
      key = other > key ? other : key;
    }
    if ((threadIdx.x & 31) == 0 && key) atomicMax(&e.st->argmax_key[t], key);
  }
}

// tp > 1: all-gather the per-rank (logit, id) keys of every node through LL
// lines (one 8-byte key per 16-byte line) and keep the max (ties -> lowest id);
// every rank then walks the same accepted path.
__device__ void argmax_exchange(const EpiArgs& e, DevState* st) {
  const uint32_t flag = st->epoch + e.ar_seq;
  const size_t base = (size_t)2 * e.P * e.n_tg_total * 128 * 32;
  const int T = st->T;
  for (int t = 0; t < T; ++t) {
    unsigned long long k = __ldcg(&st->argmax_key[t]);
    for (int p = 0; p < e.P; ++p)
      ll_store(reinterpret_cast<uint4*>(e.peer_recv[p]) + base + (size_t)e.rank * 64 + t, (uint32_t)k,
               (uint32_t)(k >> 32), flag);
  }
  for (int t = 0; t < T; ++t) {
    unsigned long long best = 0;
    for (int p = 0; p < e.P; ++p) {
      const uint4* src = reinterpret_cast<const uint4*>(e.recv) + base + (size_t)p * 64 + t;
      uint32_t d1, d2;
      long spins = 0;
      while (!ll_try_load(src, flag, d1, d2)) {
        if (++spins > (1L << 26)) { st->timeout = 1; break; }
      }
      unsigned long long k = ((unsigned long long)d2 << 32) | d1;
      best = k > best ? k : best;
    }
    st->argmax_key[t] = best;
  }
}

// Greedy accept walk (a11; R6, R7) on the device.
__device__ void accept_walk_dev(DevState* st) {
  int T = st->T;
  ss_verify_result& res = st->result;
  for (int i = 0; i < SS_MAX_TREE; ++i) {
    unsigned long long k = i < T ? __ldcg(&st->argmax_key[i]) : 0ull;
    res.argmax[i] = i < T ? (int)argmax_key_index(k) : 0;
    st->argmax_key[i] = 0ull;
  }
  int cur = 0, n = 1;
  res.accepted[0] = 0;
  while (true) {
    int tok = res.argmax[cur];
    int nxt = -1;
    for (int c = cur + 1; c < T; ++c)
      if (st->parents[c] == cur && st->tokens[c] == tok) { nxt = c; break; }
    if (nxt < 0) { res.bonus_token = tok; break; }
    res.accepted[n++] = nxt;
    cur = nxt;
  }
  for (int i = n; i < SS_MAX_TREE; ++i) res.accepted[i] = -1;
  res.n_accepted = n;
  res.status = st->status;
  st->have_verify = 1;
}

// ---------------------------------------------------------------- kernel
template <int WFMT, int NT, int EPI>
__global__ void __launch_bounds__(288) gemm_kernel(GemmArgs g) {
  using C = GemmCfg<WFMT, NT>;
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[C::STAGES], empty[C::STAGES];
  __shared__ int s_last;
  __shared__ int s_done_list[16];
  __shared__ int s_ndone;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long U = (long)g.n_tg * g.S;
  const long u0 = (long)blockIdx.x * U / gridDim.x, u1 = (long)(blockIdx.x + 1) * U / gridDim.x;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
#ifdef SS_EXP_ALLARRIVE
      mbar_init(&empty[s], 256);
#else
      mbar_init(&empty[s], 8);
#endif
    }
    fence_mbar_init();
    s_ndone = 0;
  }
  __syncthreads();

  if (warp == 8) {
    // ---------------- producer: TMA bulk copies into the stage ring.  The
    // weights do not depend on earlier kernels, so the first STAGES units'
    // weights are requested before the PDL wait (overlapping the previous
    // kernel's tail); activations only after it.
    if (lane == 0) {
      uint64_t pol = policy_evict_first();
      const long npre = min((long)C::STAGES, u1 - u0);
      for (long i = 0; i < npre; ++i) {
        uint8_t* dst = smem + i * C::UBYTES;
        mbar_expect_tx(&full[i], C::UBYTES);
        bulk_g2s(dst, g.W + (size_t)(u0 + i) * C::WBYTES, C::WBYTES, &full[i], pol);
      }
      pdl_wait();
      for (long i = 0; i < npre; ++i) {
        int ks = (int)((u0 + i) % g.S);
        bulk_g2s_nohint(smem + i * C::UBYTES + C::WBYTES, g.act + (size_t)ks * C::ABYTES, C::ABYTES, &full[i]);
      }
      int s = (int)(npre % C::STAGES);
      uint32_t ph = (npre == C::STAGES) ? 1u : 0u;
      for (long u = u0 + npre; u < u1; ++u) {
        mbar_wait(&empty[s], ph ^ 1);
        // the consumers' generic-proxy reads of this stage must be ordered
        // before the async-proxy (TMA) overwrite: without this fence a stage
        // can be refilled under a slow reader (observed as whole-tile-group
        // errors at 3-4 CTAs/SM).
        fence_proxy_async_smem();
        uint8_t* dst = smem + s * C::UBYTES;
        mbar_expect_tx(&full[s], C::UBYTES);
        bulk_g2s(dst, g.W + (size_t)u * C::WBYTES, C::WBYTES, &full[s], pol);
        int ks = (int)(u % g.S);
        bulk_g2s_nohint(dst + C::WBYTES, g.act + (size_t)ks * C::ABYTES, C::ABYTES, &full[s]);
        if (++s == C::STAGES) { s = 0; ph ^= 1; }
      }
    }
    return;  // producer warp does not take part in epilogues
  }
  pdl_wait();
  pdl_trigger();
  const int T = g.epi.st->T;

  // ---------------- consumers
  const int gq = lane >> 2, tq = lane & 3;
  float acc[NT][4];
#pragma unroll
  for (int n = 0; n < NT; ++n) acc[n][0] = acc[n][1] = acc[n][2] = acc[n][3] = 0.f;
  int s = 0;
  uint32_t ph = 0;
  long u = u0;
  while (u < u1) {
    const int tg = (int)(u / g.S);
    const long tg_end = min((long)(tg + 1) * g.S, u1);
    const int nst = (int)(tg_end - u);
    for (; u < tg_end; ++u) {
      mbar_wait(&full[s], ph);
      const uint8_t* stw = smem + s * C::UBYTES;
      if constexpr (WFMT == 0) {
        const uint4* wl = reinterpret_cast<const uint4*>(stw) + warp * 128;
        const uint16_t* sc = reinterpret_cast<const uint16_t*>(stw + kW4Bytes) + warp * 32;
        const uint2* zp = reinterpret_cast<const uint2*>(stw + kW4Bytes + 512) + warp * 2;
        const uint4* sa = reinterpret_cast<const uint4*>(stw + C::WBYTES);
#pragma unroll
        for (int grp = 0; grp < 2; ++grp) {
          uint2 zz = zp[grp];
          uint64_t z64 = ((uint64_t)zz.y << 32) | zz.x;
          uint32_t z0 = (uint32_t)(z64 >> (4 * gq)) & 15u, z8 = (uint32_t)(z64 >> (4 * (gq + 8))) & 15u;
          // rows g: subtract fp16(1024 + z); rows g+8: (1024 + 16 q) / 16 - fp16(64 + z)
          const uint32_t zA = (0x6400u + z0) * 0x10001u;
          const uint32_t zB = (0xD400u + (z8 << 4)) * 0x10001u;  // -(64 + z) in fp16
          const uint32_t sixteenth = 0x2C002C00u;                 // 1/16 in fp16
          float cg[NT][4];
#pragma unroll
          for (int n = 0; n < NT; ++n) cg[n][0] = cg[n][1] = cg[n][2] = cg[n][3] = 0.f;
#pragma unroll
          for (int kb2 = 0; kb2 < 2; ++kb2) {
            const int kb = grp * 2 + kb2;
            uint4 wv = wl[kb * 32 + lane];
            uint32_t wa[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
            for (int jp = 0; jp < 2; ++jp) {
              uint4 bb[NT];
#pragma unroll
              for (int n = 0; n < NT; ++n) bb[n] = sa[((kb * 2 + jp) * NT + n) * 32 + lane];
#pragma unroll
              for (int js = 0; js < 2; ++js) {
                uint32_t a[4];
#ifdef SS_EXP_NODEQ
                a[0] = wa[jp * 2 + js]; a[1] = a[0] ^ 0x1111u; a[2] = a[0] ^ 0x2222u; a[3] = a[0] ^ 0x3333u;
#else
                dequant8(wa[jp * 2 + js], a);
#endif
#ifndef SS_EXP_NOZERO
                a[0] = f16x2_sub(a[0], zA);
                a[1] = f16x2_fma(a[1], sixteenth, zB);
                a[2] = f16x2_sub(a[2], zA);
                a[3] = f16x2_fma(a[3], sixteenth, zB);
#endif
#pragma unroll
                for (int n = 0; n < NT; ++n)
                  mma_f16_16816(cg[n], a, js ? bb[n].z : bb[n].x, js ? bb[n].w : bb[n].y);
              }
            }
          }
          float s0 = bf16_bits_to_f32(sc[grp * 16 + gq]), s8 = bf16_bits_to_f32(sc[grp * 16 + gq + 8]);
#pragma unroll
          for (int n = 0; n < NT; ++n) {
            acc[n][0] = fmaf(s0, cg[n][0], acc[n][0]);
            acc[n][1] = fmaf(s0, cg[n][1], acc[n][1]);
            acc[n][2] = fmaf(s8, cg[n][2], acc[n][2]);
            acc[n][3] = fmaf(s8, cg[n][3], acc[n][3]);
          }
        }
      } else {
        const uint4* wl = reinterpret_cast<const uint4*>(stw) + warp * 128;
        const uint4* sa = reinterpret_cast<const uint4*>(stw + C::WBYTES);
#pragma unroll
        for (int jp = 0; jp < 2; ++jp) {
#pragma unroll
          for (int js = 0; js < 2; ++js) {
            uint4 wv = wl[(jp * 2 + js) * 32 + lane];
            uint32_t a[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
            for (int n = 0; n < NT; ++n) {
              uint4 bh = sa[(jp * 2 * NT + n) * 32 + lane];
              uint4 bl = sa[(jp * 2 * NT + NT + n) * 32 + lane];
              mma_bf16_16816(acc[n], a, js ? bh.z : bh.x, js ? bh.w : bh.y);
              mma_bf16_16816(acc[n], a, js ? bl.z : bl.x, js ? bl.w : bl.y);
            }
          }
        }
      }
#ifdef SS_EXP_ALLARRIVE
      mbar_arrive(&empty[s]);
#else
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
#endif
      if (++s == C::STAGES) { s = 0; ph ^= 1; }
    }
    // ---- flush this tile-group's partial
    {
      const int TP = NT * 8;
      float* base = g.accum + ((size_t)tg * 128 + warp * 16 + gq) * TP;
#pragma unroll
      for (int n = 0; n < NT; ++n) {
        red_add_v2(base + n * 8 + 2 * tq, acc[n][0], acc[n][1]);
        red_add_v2(base + 8 * TP + n * 8 + 2 * tq, acc[n][2], acc[n][3]);
        acc[n][0] = acc[n][1] = acc[n][2] = acc[n][3] = 0.f;
      }
    }
    // every thread's reductions must be performed (device scope) before the
    // arrival is counted: a fence by thread 0 alone does not cover the other
    // threads' in-flight red.global ops.
    __threadfence();
    named_bar_sync(1, 256);
    if (threadIdx.x == 0) {
      int old = atomicAdd(&g.counters[tg], nst);
      s_last = (old + nst == g.S);
      if (s_last) __threadfence();
    }
    named_bar_sync(1, 256);
    if (s_last) {
      const float* accp = g.accum + (size_t)tg * 128 * NT * 8;
      if constexpr (EPI == EPI_QKV) epi_qkv<NT>(g.epi, tg, accp, T);
      else if constexpr (EPI == EPI_SWIGLU) epi_swiglu<NT>(g.epi, tg, accp, T);
      else if constexpr (EPI == EPI_ARGMAX) epi_argmax<NT>(g.epi, tg, accp, T);
      else {
        if (g.epi.P == 1) epi_resid_local<NT>(g.epi, tg, accp, T);
        else {
          epi_ar_send<NT>(g.epi, tg, accp, T);
          if (threadIdx.x == 0) s_done_list[s_ndone++] = tg;
        }
      }
      named_bar_sync(1, 256);
      // self-clean the accumulator + counter for the next launch
      float* accw = g.accum + (size_t)tg * 128 * NT * 8;
      for (int i = threadIdx.x; i < 128 * NT * 8; i += 256) accw[i] = 0.f;
      if (threadIdx.x == 0) g.counters[tg] = 0;
      if constexpr (EPI == EPI_ARGMAX) {
        __threadfence();  // this CTA's argmax atomics (all threads) before the arrival
        named_bar_sync(1, 256);
        if (threadIdx.x == 0) {
          int old = atomicAdd(&g.epi.st->lm_done, 1);
          if (old == g.n_tg - 1) {
            __threadfence();
            if (g.epi.P > 1) argmax_exchange(g.epi, g.epi.st);
            accept_walk_dev(g.epi.st);
            g.epi.st->lm_done = 0;
          }
        }
      }
    }
  }
  if constexpr (EPI == EPI_RESID) {
    if (g.epi.P > 1) {
      named_bar_sync(1, 256);
      for (int i = 0; i < s_ndone; ++i) epi_ar_recv<NT>(g.epi, s_done_list[i], T);
    }
  }
}

// ---------------------------------------------------------------- launch
template <int WFMT, int NT, int EPI>
static int launch_t(const GemmArgs& g, int max_ctas, cudaStream_t st) {
  using C = GemmCfg<WFMT, NT>;
  auto k = gemm_kernel<WFMT, NT, EPI>;
  static bool attr_set = false;
  static int occ = 1;
  if (!attr_set) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, C::THREADS, C::SMEM);
    if (occ < 1) occ = 1;
    attr_set = true;
  }
  long U = (long)g.n_tg * g.S;
  static const int occ_cap = getenv("SS_GEMM_OCC") ? atoi(getenv("SS_GEMM_OCC")) : 0;  // debugging aid
  int o = (occ_cap > 0 && occ_cap < occ) ? occ_cap : occ;
  int grid = (int)std::min<long>(U, (long)g.n_sm * o);
  if (max_ctas > 0 && grid > max_ctas) grid = max_ctas;
  launch_pdl(k, dim3(grid), dim3(C::THREADS), C::SMEM, st, g);
  return 1;
}

template <int WFMT, int EPI>
static int launch_nt(const GemmArgs& g, int NT, int max_ctas, cudaStream_t st) {
  switch (NT) {
    case 1: return launch_t<WFMT, 1, EPI>(g, max_ctas, st);
    case 2: return launch_t<WFMT, 2, EPI>(g, max_ctas, st);
    case 4: return launch_t<WFMT, 4, EPI>(g, max_ctas, st);
    default: return launch_t<WFMT, 8, EPI>(g, max_ctas, st);
  }
}

int launch_gemm(const GemmArgs& g, int wfmt, int NT, int max_ctas, cudaStream_t st) {
  if (wfmt == 1) return launch_nt<1, EPI_ARGMAX>(g, NT, max_ctas, st);
  switch (g.epi.kind) {
    case EPI_QKV: return launch_nt<0, EPI_QKV>(g, NT, max_ctas, st);
    case EPI_SWIGLU: return launch_nt<0, EPI_SWIGLU>(g, NT, max_ctas, st);
    default: return launch_nt<0, EPI_RESID>(g, NT, max_ctas, st);
  }
}

}  // namespace ss
