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
// (cp.async.bulk + mbarrier ring; producer warp lane 0), 8 consumer warps --
// each owns two 16-row tiles x one 128-deep AWQ group of every 128 x 256
// unit, so one load of B fragments feeds two MMAs -- turn int4 nibbles into
// fp16 (1024 + q) / (1024 + 16 q) with mul.hi + lop3 (exact integers) and
// issue mma.sync m16n8k16 with the weights as the M=16 operand and the T tree
// tokens as the N=8 columns.  Per group, s (acc - (1024 + z) X) in fp32 (X =
// the group's activation sum from the producer): no weight is ever rounded
// (R3, R19, R20).  Work = (tile-group of 128 rows) x (K stage) units in
// contiguous static ranges over a persistent grid (stream-K); partial tiles
// are reduced with red.global.add.v2.f32; the producer warp's lane 1 (flush
// signaler) publishes a CTA's share of a tile-group with one GPU-scope fence
// + arrival count, and the last arriver runs the epilogue (no extra kernel).
// The tcgen05 (TMEM A operand) variant of this kernel lives on the
// `tcgen05-w4` branch.
#include <cstdio>

#include "common.cuh"
#include "internal.h"
#include "kernels.h"
#include "accept.cuh"

namespace ss {

template <int WFMT, int NT>
struct GemmCfg {
  static constexpr int KS = WFMT == 0 ? kW4KS : kBFKS;
  static constexpr int WBYTES = WFMT == 0 ? kW4UnitBytes : kBFUnitBytes;
  static constexpr int ANT = WFMT == 0 ? NT : 2 * NT;  // LM head: bf16 hi + lo tiles
  // W4: fragments + X (group sums, 2 groups x 8NT fp32); LM head: fragments only
  static constexpr int ABYTES = (KS / 16) * ANT * 256 + (WFMT == 0 ? NT * 64 : 0);
  static constexpr int UBYTES = WBYTES + ABYTES;
  // NT <= 2: 3 stages (~63-76 KB) -> 3 CTAs / SM; larger NT: 4 stages, 1-2 CTAs / SM
#ifdef SS_EXP_NCW
  static constexpr int NCW = SS_EXP_NCW;
#else
  static constexpr int NCW = 8;  // consumer warps: one per 16-row tile (measured best at T <= 16)
#endif
  // ring depth: NT <= 2 -> 3 stages (~63-76 KB, 3 CTAs/SM); larger NT -> 4
#ifdef SS_EXP_STAGES
  static constexpr int STAGES = SS_EXP_STAGES;
#elif defined(SS_EXP_STAGES_WIDE)
  static constexpr int STAGES = (UBYTES <= 26 * 1024) ? 3 : SS_EXP_STAGES_WIDE;
#else
  static constexpr int STAGES = (UBYTES <= 26 * 1024) ? 3 : 4;
#endif
  // no slack: 3 CTAs of the T <= 16 configurations must fit one SM's 228 KB
  static constexpr int SMEM = STAGES * UBYTES;
  static constexpr int KPARTS = NCW / 8;
  // W4: a warp owns two 16-row tiles x one 128-deep group of each unit, so the
  // B fragments it loads serve two MMAs (half the activation reads of the
  // one-tile-per-warp mapping)
#ifdef SS_EXP_NOPAIR
  static constexpr bool PAIR = false;
#elif defined(SS_EXP_PAIRMAXNT)
  static constexpr bool PAIR = WFMT == 0 && NCW == 8 && NT <= SS_EXP_PAIRMAXNT;
#else
  static constexpr bool PAIR = WFMT == 0 && NCW == 8;
#endif
#ifdef SS_EXP_NACC
  static constexpr int NACC = SS_EXP_NACC;
#else
  static constexpr int NACC = 1;  // one accumulator set per warp (a 2-set split measured slower: 8 more FADDs)
#endif
  static constexpr int THREADS = 32 * (NCW + 1);  // + 1 producer warp
  // resident CTAs per SM the register budget is sized for (3 at T <= 16)
#ifdef SS_EXP_MINB
  static constexpr int MINB = SS_EXP_MINB;
#else
  static constexpr int MINB = SMEM <= 75 * 1024 ? 3 : (SMEM <= 112 * 1024 ? 2 : 1);
#endif
};

// ---------------------------------------------------------------- epilogues
// The epilogues run after the main loop on the CTA that completed the
// tile-group: their accumulator reads are L2 round trips, so each thread
// issues the loads of EB items before using any of them.
constexpr int EB = 4;

template <int NT>
__device__ void epi_qkv(const EpiArgs& e, int tg, const float* acc, int T) {
  const int TP = NT * 8;
  const int d = e.d, half = d >> 1;
  const int nq = e.Hq_l * d, nk = e.Hkv_l * d;
  const int L = e.st->L;
  const int n = 128 * T;
  for (int i0 = threadIdx.x; i0 < n; i0 += 256 * EB) {
    float v[EB], pv[EB];
    float2 cs[EB];
#pragma unroll
    for (int b = 0; b < EB; ++b) {
      const int idx = i0 + 256 * b;
      v[b] = pv[b] = 0.f;
      cs[b] = make_float2(1.f, 0.f);
      if (idx < n) {
        const int r = idx / T, t = idx - r * T;
        const int row = tg * 128 + r, j = row % d;
        v[b] = __ldcg(acc + (size_t)r * TP + t);
        if (row < nq + nk) {
          const int pr = (j < half) ? r + half : r - half;
          pv[b] = __ldcg(acc + (size_t)pr * TP + t);
          cs[b] = e.rope_cs[(size_t)e.st->pos[t] * half + (j % half)];
        }
      }
    }
#pragma unroll
    for (int b = 0; b < EB; ++b) {
      const int idx = i0 + 256 * b;
      if (idx >= n) break;
      const int r = idx / T, t = idx - r * T;
      const int row = tg * 128 + r, j = row % d;
      float x = v[b];
      if (row < nq + nk)  // q or k: rotate-half RoPE (R2)
        x = (j < half) ? (x * cs[b].x - pv[b] * cs[b].y) : (x * cs[b].x + pv[b] * cs[b].y);
      const uint16_t h16 = f32_to_f16_bits(x);  // q and the KV cache are fp16
      if (row < nq) {
        const int hq = row / d, kvh = hq / e.G, jj = hq - kvh * e.G;
        const int m = t * e.G + jj;  // attention row; 16-byte chunks swizzled by m % 8
        e.qbuf[((size_t)kvh * (e.G * SS_MAX_TREE) + m) * d + ((((j >> 3) ^ (m & 7))) << 3) + (j & 7)] = h16;
      } else {
        const int kvh = (row < nq + nk) ? (row - nq) / d : (row - nq - nk) / d;
        uint16_t* c = (row < nq + nk) ? e.kc : e.vc;
        const size_t base = ((size_t)e.layer * e.Hkv_l + kvh) * e.max_ctx_pad * d;
        c[base + kv_elem_offset(L + t, j, d)] = h16;
      }
    }
  }
}

template <int NT>
__device__ void epi_swiglu(const EpiArgs& e, int tg, const float* acc, int T) {
  const int TP = NT * 8;
  // tile-group rows: [0,64) gate, [64,128) up for intermediate columns tg*64..+64.
  // One warp per token: lane cp owns columns (2cp, 2cp+1); the fp16 outputs'
  // sum over the 64 columns is half of the down-proj group sum X (atomic).
  const int warp = threadIdx.x >> 5, cp = threadIdx.x & 31;
  for (int t = warp; t < T; t += 8) {
    const float g0 = __ldcg(acc + (size_t)(2 * cp) * TP + t);
    const float g1 = __ldcg(acc + (size_t)(2 * cp + 1) * TP + t);
    const float u0 = __ldcg(acc + (size_t)(64 + 2 * cp) * TP + t);
    const float u1 = __ldcg(acc + (size_t)(64 + 2 * cp + 1) * TP + t);
    const float h0 = g0 / (1.f + __expf(-g0)) * u0;
    const float h1 = g1 / (1.f + __expf(-g1)) * u1;
    const int k = tg * 64 + 2 * cp;
    const uint32_t hv = pack_half2(h0, h1);
    *reinterpret_cast<uint32_t*>(e.act_out + act_frag_offset(t, k, NT)) = hv;
    float xsum = __low2float(*reinterpret_cast<const __half2*>(&hv)) + __high2float(*reinterpret_cast<const __half2*>(&hv));
    xsum = warp_sum(xsum);
    if (cp == 0) atomicAdd(reinterpret_cast<float*>(e.act_out + act_xsum_offset(t, k >> 7, NT)), xsum);
  }
}

template <int NT>
__device__ void epi_resid_local(const EpiArgs& e, int tg, const float* acc, int T, float* ss) {
  const int TP = NT * 8;
  // warp = 32 columns of one token: the new residual's squares reduce per
  // warp into the per-token sum the fused RMSNorm needs
  const int n = 128 * T;
  for (int i0 = threadIdx.x; i0 < n; i0 += 256 * EB) {
    float xv[EB], av[EB];
#pragma unroll
    for (int b = 0; b < EB; ++b) {
      const int idx = i0 + 256 * b;
      xv[b] = av[b] = 0.f;
      if (idx < n) {
        const int t = idx >> 7, r = idx & 127;
        xv[b] = e.x[(size_t)t * e.h + tg * 128 + r];
        av[b] = __ldcg(acc + (size_t)r * TP + t);
      }
    }
#pragma unroll
    for (int b = 0; b < EB; ++b) {
      const int idx = i0 + 256 * b;
      if (idx >= n) break;  // warp-uniform (n is a multiple of 128)
      const int t = idx >> 7, r = idx & 127;
      const float nx = xv[b] + av[b];
      e.x[(size_t)t * e.h + tg * 128 + r] = nx;
      if (ss) {
        const float q = warp_sum(nx * nx);
        if ((threadIdx.x & 31) == 0) atomicAdd(ss + t, q);
      }
    }
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
  const int n = 128 * pairs;
  for (int i0 = threadIdx.x; i0 < n; i0 += 256 * EB) {
    float2 v[EB];
#pragma unroll
    for (int q = 0; q < EB; ++q) {
      const int idx = i0 + 256 * q;
      v[q] = make_float2(0.f, 0.f);
      if (idx < n) {
        const int r = idx / pairs, tp = idx - r * pairs;
        v[q] = __ldcg(reinterpret_cast<const float2*>(acc + (size_t)r * TP + 2 * tp));
      }
    }
#pragma unroll
    for (int q = 0; q < EB; ++q) {
      const int idx = i0 + 256 * q;
      if (idx >= n) break;
      const int r = idx / pairs, tp = idx - r * pairs;
      for (int p = 0; p < e.P; ++p) {
        // loopback emulation (one rank on one GPU, timing only): every rank
        // slot of the own buffer receives this rank's partial
        const int slot = e.loopback ? p : e.rank;
        // dense line layout: PP = 4 NT token pairs per row (the launch's width)
        const size_t line = (((size_t)(e.ar_seq & 1) * e.P + slot) * e.n_tg_total + tg) * 128 * (4 * NT) +
                            (size_t)r * (4 * NT) + tp;
        ll_store(reinterpret_cast<uint4*>(e.peer_recv[p]) + line, __float_as_uint(v[q].x), __float_as_uint(v[q].y),
                 flag);
      }
    }
  }
}

// tp > 1, phase 2 (after the CTA's compute loop): wait for every rank's
// partial of the tile-group, sum in rank order (identical on all ranks), add.
// The P lines of an item are loaded together (independent L2 / NVLink round
// trips in flight) and only lines whose flags are not there yet are re-polled.
template <int NT>
__device__ void epi_ar_recv(const EpiArgs& e, int tg, int T, float* ss) {
  constexpr int PP = 4 * NT;  // token pairs per row in the LL line layout (epi_ar_send)
  const uint32_t flag = e.st->epoch + e.ar_seq;
  const int pairs = (T + 1) >> 1;
  for (int idx = threadIdx.x; idx < 128 * pairs; idx += 256) {
    const int tp = idx >> 7, r = idx & 127;  // warp = 32 rows of one token pair
    const uint4* src0 = reinterpret_cast<const uint4*>(e.recv) +
                        (((size_t)(e.ar_seq & 1) * e.P) * e.n_tg_total + tg) * 128 * PP + (size_t)r * PP + tp;
    const size_t pstride = (size_t)e.n_tg_total * 128 * PP;
    uint32_t d1[kMaxPeers], d2[kMaxPeers];
    unsigned ready = 0;
#pragma unroll
    for (int p = 0; p < kMaxPeers; ++p)
      if (p < e.P && ll_try_load(src0 + p * pstride, flag, d1[p], d2[p])) ready |= 1u << p;
    const unsigned all = (1u << e.P) - 1u;
    long spins = 0;
#ifdef SS_EXP_NOPOLL
    ready = all;  // timing experiment: take whatever the first loads returned
#endif
    while (ready != all) {
#pragma unroll
      for (int p = 0; p < kMaxPeers; ++p)
        if (p < e.P && !(ready & (1u << p)) && ll_try_load(src0 + p * pstride, flag, d1[p], d2[p])) ready |= 1u << p;
      if (++spins > (1L << 24)) { e.st->timeout = 1; break; }
    }
    float s0 = 0.f, s1 = 0.f;
#pragma unroll
    for (int p = 0; p < kMaxPeers; ++p)
      if (p < e.P) {
        s0 += __uint_as_float(d1[p]);
        s1 += __uint_as_float(d2[p]);
      }
    const int t0 = 2 * tp;
    float* x0 = e.x + (size_t)t0 * e.h + tg * 128 + r;
    const float n0 = *x0 + s0;
    *x0 = n0;
    float n1 = 0.f;
    if (t0 + 1 < T) {
      float* x1 = x0 + e.h;
      n1 = *x1 + s1;
      *x1 = n1;
    }
    if (ss) {
      const float q0 = warp_sum(n0 * n0), q1 = warp_sum(n1 * n1);
      if ((threadIdx.x & 31) == 0) {
        atomicAdd(ss + t0, q0);
        if (t0 + 1 < T) atomicAdd(ss + t0 + 1, q1);
      }
    }
  }
}

// Fused RMSNorm of the updated residual (R5) into the next GEMM's input, for
// one 128-column group of every token, after all tile-groups of the launch
// are added (see the EPI_RESID tail of gemm_kernel): warp = token, 4 columns
// per lane -- fp16 fragments + group sum X for a W4 GEMM, or bf16 hi/lo
// fragments for the LM head (split).
template <int NT>
__device__ void norm_group(const GemmArgs& g, int T, int grp) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int h = g.epi.h;
  for (int t = warp; t < T; t += 8) {
    const int k = grp * 128 + lane * 4;
    const float4 v = __ldcg(reinterpret_cast<const float4*>(g.epi.x + (size_t)t * h + k));
    const uint2 gw = *reinterpret_cast<const uint2*>(g.norm_gain + k);
    const float r = rsqrtf(__ldcg(g.ss + t) / (float)h + g.eps);
    const float a0 = v.x * r * bf16_lo(gw.x), a1 = v.y * r * bf16_hi(gw.x);
    const float a2 = v.z * r * bf16_lo(gw.y), a3 = v.w * r * bf16_hi(gw.y);
    if (!g.norm_split) {
      const uint32_t p01 = pack_half2(a0, a1), p23 = pack_half2(a2, a3);
      *reinterpret_cast<uint32_t*>(g.norm_out + act_frag_offset(t, k, NT)) = p01;
      *reinterpret_cast<uint32_t*>(g.norm_out + act_frag_offset(t, k + 2, NT)) = p23;
      const float xs = warp_sum(half2_sum(p01) + half2_sum(p23));
      if (lane == 0) *reinterpret_cast<float*>(g.norm_out + act_xsum_offset(t, grp, NT)) = xs;
    } else {
      uint32_t h01 = pack_bf16x2(a0, a1), h23 = pack_bf16x2(a2, a3);
      *reinterpret_cast<uint32_t*>(g.norm_out + frag_offset(t, k, 2 * NT)) = h01;
      *reinterpret_cast<uint32_t*>(g.norm_out + frag_offset(t, k + 2, 2 * NT)) = h23;
      *reinterpret_cast<uint32_t*>(g.norm_out + frag_offset(t + 8 * NT, k, 2 * NT)) =
          pack_bf16x2(a0 - bf16_lo(h01), a1 - bf16_hi(h01));
      *reinterpret_cast<uint32_t*>(g.norm_out + frag_offset(t + 8 * NT, k + 2, 2 * NT)) =
          pack_bf16x2(a2 - bf16_lo(h23), a3 - bf16_hi(h23));
    }
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

// ---------------------------------------------------------------- kernel
// CTA = NCW consumer warps + 1 producer warp.  Consumer warp cw works on tile
// (16 output rows) cw % 8 of the tile-group and on K-part cw / 8 of each unit:
// for W4 one 128-deep group (2 kblocks), for the bf16 LM head two k16 steps.
// Two warps per tile double the warps available to hide the dequant / MMA
// latency chains (the kernel is latency-, not issue-bound at T=8).
#ifdef SS_EXP_TIMING
__device__ unsigned long long g_ts[1 << 16];
__device__ unsigned int g_ts_launch;
SS_DEV unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ int g_ts_kind = -1;
__device__ int g_ts_par = -1;  // RESID: 0 = O-proj, 1 = down, -1 = any
#define TS(slot) do { if (threadIdx.x == 0 && blockIdx.x < 1024 && g.epi.kind == g_ts_kind && (WFMT == 1 || g.epi.layer == 0) && (g_ts_par < 0 || (g.epi.ar_seq & 1) == g_ts_par)) g_ts[(blockIdx.x * 8 + (slot)) & 0xFFFF] = gtimer(); } while (0)
#else
#define TS(slot) do {} while (0)
#endif

template <int WFMT, int NT, int EPI>
__global__ void __launch_bounds__(GemmCfg<WFMT, NT>::THREADS, GemmCfg<WFMT, NT>::MINB) gemm_kernel(GemmArgs g) {
  using C = GemmCfg<WFMT, NT>;
  constexpr int NCW = C::NCW, NCT = NCW * 32;
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[C::STAGES], empty[C::STAGES];
  __shared__ int s_done_list[64];  // tile-groups this CTA finalises (<= tile-groups its range touches)
  __shared__ int s_ndone;
  __shared__ int s_flushed;          // consumer-warp flushes so far (signaler)
  __shared__ int s_unit[C::STAGES];  // tile-group of each ring slot (-1 = no more work)

  TS(0);
#ifdef SS_EXP_TIMING
  if (threadIdx.x == 0 && blockIdx.x < 1024 && g.epi.kind == g_ts_kind && (WFMT == 1 || g.epi.layer == 0)) {
    unsigned int sm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    g_ts[(blockIdx.x * 8 + 6) & 0xFFFF] = sm;
  }
#endif
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // Static stream-K schedule: units (tile-group, K-stage) are numbered
  // tile-group major and split into equal contiguous ranges, one per CTA
  // (one or two tile-groups per CTA: few partial flushes, a spread-out HBM
  // access pattern).  A dynamic work queue and a static + pool hybrid were
  // both measured slower (profiles/r01_experiments.md).
  const int U = g.n_tg * g.S;
  const int u0 = (int)((long)blockIdx.x * U / gridDim.x), u1 = (int)((long)(blockIdx.x + 1) * U / gridDim.x);

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    fence_mbar_init();
    s_ndone = 0;
    s_flushed = 0;
  }
  __syncthreads();

  if (warp == NCW) {
    // ---------------- producer (lane 0): TMA bulk copies of the CTA's static
    // unit range into the ring.  The weights do not depend on earlier
    // kernels, so the first STAGES units' weights are requested before the
    // PDL wait (overlapping the previous kernel's tail); activations only
    // after it.
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      int s = 0;
      uint32_t ph = 0;
      int pre_u[C::STAGES], npre = 0;
      bool waited = false;
      for (int u = u0;; ++u) {
        const bool have = u < u1;
        const int utg = have ? u / g.S : -1, uks = have ? u - utg * g.S : 0;
        if (!waited && (npre == C::STAGES || !have)) {
          pdl_wait();
          waited = true;
          for (int i = 0; i < npre; ++i)
            bulk_g2s_nohint(smem + i * C::UBYTES + C::WBYTES, g.act + (size_t)pre_u[i] * C::ABYTES, C::ABYTES,
                            &full[i]);
        }
        mbar_wait(&empty[s], ph ^ 1);
        // the consumers' generic-proxy reads of this slot must be ordered
        // before the async-proxy (TMA) overwrite (observed as whole-tile-group
        // errors at 3-4 CTAs/SM without it)
        fence_proxy_async_smem();
        s_unit[s] = utg;
        if (!have) {
          mbar_arrive(&full[s]);  // publishes s_unit[s] = -1: no more work
          break;
        }
        uint8_t* dst = smem + s * C::UBYTES;
        mbar_expect_tx(&full[s], C::UBYTES);
        bulk_g2s(dst, g.W + (size_t)u * C::WBYTES, C::WBYTES, &full[s], pol);
        if (waited) bulk_g2s_nohint(dst + C::WBYTES, g.act + (size_t)uks * C::ABYTES, C::ABYTES, &full[s]);
        else pre_u[npre++] = uks;
        if (++s == C::STAGES) { s = 0; ph ^= 1; }
      }
      if (!waited) pdl_wait();
    } else if (lane == 1 && u1 > u0) {
      // ---------------- flush signaler: once all consumer warps have pushed
      // a tile-group's partial sums (red.add), one GPU-scope fence + arrival
      // count for the CTA, off the consumers' critical path
      int k = 0;
      for (int tg = u0 / g.S; tg <= (u1 - 1) / g.S; ++tg) {
        const int nst = min(u1, (tg + 1) * g.S) - max(u0, tg * g.S);
        ++k;
        int v;
        do {
          asm volatile("ld.acquire.cta.shared.b32 %0, [%1];" : "=r"(v) : "r"(smem_u32(&s_flushed)) : "memory");
          if (v < NCW * k) __nanosleep(100);
        } while (v < NCW * k);
        fence_acq_rel_gpu();
        const int old = atomicAdd(&g.counters[tg], nst);
        if (old + nst == g.S && s_ndone < 64) s_done_list[s_ndone++] = tg;
      }
    }
    __syncwarp();
    named_bar_sync(3, NCT + 32);  // s_done_list is complete for the epilogue threads
    return;  // producer warp does not take part in epilogues
  }
  pdl_wait();
  pdl_trigger();
  TS(1);
  const int T = g.epi.st->T;
  if (blockIdx.x == 0 && g.zero_x) {  // X slots a later kernel accumulates into atomically
    const int n = g.zero_x_stages * 16 * g.zero_x_nt;
    for (int i = threadIdx.x; i < n; i += NCT) {
      const int stg = i / (16 * g.zero_x_nt), j = i % (16 * g.zero_x_nt);
      reinterpret_cast<float*>(g.zero_x + (size_t)stg * w4_act_stage_bytes(g.zero_x_nt) + g.zero_x_nt * 4096)[j] = 0.f;
    }
  }

  // ---------------- consumers
  // tile = 16-row tile of this warp (pair mode: first of its two tiles)
  const int tile = C::PAIR ? 2 * (warp & 3) : (warp & 7), part = C::PAIR ? 0 : (warp >> 3);
  const int pgrp = warp >> 2;  // pair mode: the warp's 128-deep group of each unit
  const int gq = lane >> 2, tq = lane & 3;
  float acc[NT][4], acc1[NT][4];
#pragma unroll
  for (int n = 0; n < NT; ++n) {
    acc[n][0] = acc[n][1] = acc[n][2] = acc[n][3] = 0.f;
    acc1[n][0] = acc1[n][1] = acc1[n][2] = acc1[n][3] = 0.f;
  }
  int s = 0;
  uint32_t ph = 0;
  int cur_tg = -1, nst = 0;
  bool done = false;
  // shared-window addresses, computed once: stage base + per-warp offsets
  const uint32_t sm0 = opaque(smem_u32(smem)), full0 = opaque(smem_u32(full)), empty0 = opaque(smem_u32(empty));
  int uc = u0;  // next unit to consume
  const uint32_t o_w = opaque((uint32_t)(tile * 128 + lane) * 16);            // weight chunks
  const uint32_t o_sc = opaque((uint32_t)(kW4Bytes + tile * 64 + gq * 4));     // [grp][gq] scale pairs
  const uint32_t o_z = opaque((uint32_t)(kW4Bytes + 512 + tile * 16 + gq));    // [grp][gq] zero pairs
  const uint32_t o_b = opaque((uint32_t)(C::WBYTES + lane * 16));              // B fragments
  const uint32_t o_x = opaque((uint32_t)(C::WBYTES + NT * 4096 + 8 * tq));     // group sums X
  while (!done) {
    int tg = -1;
    // consume consecutive units of one tile-group; stop at a tile-group change
    // (the new unit stays in its slot for the next round) or at end of work
    while (true) {
      // the unit sequence is the static range [u0, u1): computed here, not
      // read back from the producer's slot tags (no generic smem hand-off
      // beside the TMA-completed barrier)
      if (uc >= u1) { done = true; break; }
      mbar_wait_a(full0 + 8 * s, ph);
      tg = uc / g.S;
      if (cur_tg >= 0 && tg != cur_tg) break;
      cur_tg = tg;
      ++nst;
#ifdef SS_EXP_TIMING
      if (nst == 1 && cur_tg == tg && s_ndone == 0) { TS(2); }
#endif
      const uint8_t* stw = smem + s * C::UBYTES;
      const uint32_t sst = sm0 + s * C::UBYTES;
#ifdef SS_EXP_NOCOMPUTE
      if (false) {
#else
      if constexpr (WFMT == 0) {
#endif
        // MMA on A = (1024 + q) for rows g and (1024 + 16 q) for rows g+8 (what
        // lop3 yields, dequant8), then per 128-group, with X = sum_k x_k:
        //   rows g  : s * (acc - (1024 + z) X)          = s * sum (q - z) x
        //   rows g+8: s/16 * (acc - (1024 + 16 z) X)    = s * sum (q - z) x
        // exact integer weights, no per-weight subtract (R3, DESIGN "W4 GEMM").
        if constexpr (C::PAIR) {
          const int grp = pgrp;
          uint32_t wa[2][8];
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const uint4 w0 = lds128(sst + o_w + i * 2048 + (grp * 2) * 512);
            const uint4 w1 = lds128(sst + o_w + i * 2048 + (grp * 2 + 1) * 512);
            wa[i][0] = w0.x; wa[i][1] = w0.y; wa[i][2] = w0.z; wa[i][3] = w0.w;
            wa[i][4] = w1.x; wa[i][5] = w1.y; wa[i][6] = w1.z; wa[i][7] = w1.w;
          }
          float cg[2][NT][4];
#pragma unroll
          for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int n = 0; n < NT; ++n) cg[i][n][0] = cg[i][n][1] = cg[i][n][2] = cg[i][n][3] = 0.f;
#pragma unroll
          for (int jp = 0; jp < 4; ++jp) {  // pairs of k16 steps inside the group
            uint4 bb[NT];
#pragma unroll
            for (int n = 0; n < NT; ++n) bb[n] = lds128(sst + o_b + ((grp * 4 + jp) * NT + n) * 512);
#pragma unroll
            for (int js = 0; js < 2; ++js)
#pragma unroll
              for (int i = 0; i < 2; ++i) {
                uint32_t a[4];
                dequant8(wa[i][jp * 2 + js], a);
#pragma unroll
                for (int n = 0; n < NT; ++n)
                  mma_f16_16816(cg[i][n], a, js ? bb[n].z : bb[n].x, js ? bb[n].w : bb[n].y);
              }
          }
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const uint32_t zb = lds8(sst + o_z + i * 16 + grp * 8), sp = lds32(sst + o_sc + i * 64 + grp * 32);
            const float c0 = __uint_as_float(0x44800000u | ((zb & 15u) << 13));
            const float c8 = __uint_as_float(0x44800000u | ((zb >> 4) << 17));
            const float s0 = __uint_as_float(sp << 16);
            const float s8 = __uint_as_float(sp & 0xFFFF0000u) * 0.0625f;
#pragma unroll
            for (int n = 0; n < NT; ++n) {
              const float2 X = lds64f(sst + o_x + (grp * 8 * NT + n * 8) * 4);
              float* ac = i ? acc1[n] : acc[n];
              ac[0] = fmaf(s0, fmaf(-c0, X.x, cg[i][n][0]), ac[0]);
              ac[1] = fmaf(s0, fmaf(-c0, X.y, cg[i][n][1]), ac[1]);
              ac[2] = fmaf(s8, fmaf(-c8, X.x, cg[i][n][2]), ac[2]);
              ac[3] = fmaf(s8, fmaf(-c8, X.y, cg[i][n][3]), ac[3]);
            }
          }
        } else {
#pragma unroll
        for (int gi = 0; gi < 2 / C::KPARTS; ++gi) {
        const int grp = part + gi;  // this warp's 128-deep group(s) of the unit
        const uint4 w0 = lds128(sst + o_w + (grp * 2) * 512), w1 = lds128(sst + o_w + (grp * 2 + 1) * 512);
        const uint32_t wa[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
        // NACC accumulator sets (even / odd k16 steps) -- 1 in the product (see GemmCfg)
        float cg[C::NACC][NT][4];
#pragma unroll
        for (int h = 0; h < C::NACC; ++h)
#pragma unroll
          for (int n = 0; n < NT; ++n) cg[h][n][0] = cg[h][n][1] = cg[h][n][2] = cg[h][n][3] = 0.f;
#pragma unroll
        for (int jp = 0; jp < 4; ++jp) {  // pairs of k16 steps inside the group
          uint4 bb[NT];
#pragma unroll
          for (int n = 0; n < NT; ++n) bb[n] = lds128(sst + o_b + ((grp * 4 + jp) * NT + n) * 512);
#pragma unroll
          for (int js = 0; js < 2; ++js) {
            uint32_t a[4];
#ifdef SS_EXP_NODEQ
            a[0] = wa[jp * 2 + js]; a[1] = a[0] ^ 0x1111u; a[2] = a[0] ^ 0x2222u; a[3] = a[0] ^ 0x3333u;
#else
            dequant8(wa[jp * 2 + js], a);
#endif
#pragma unroll
            for (int n = 0; n < NT; ++n)
              mma_f16_16816(cg[js % C::NACC][n], a, js ? bb[n].z : bb[n].x, js ? bb[n].w : bb[n].y);
          }
        }
        // c0 = 1024 + z, c8 = 1024 + 16 z built directly as fp32 bits (1024 = 0x44800000,
        // one ulp = 2^-13 there); scales are the bf16 halves of one word
        const uint32_t zb = lds8(sst + o_z + grp * 8), sp = lds32(sst + o_sc + grp * 32);
        const float c0 = __uint_as_float(0x44800000u | ((zb & 15u) << 13));
        const float c8 = __uint_as_float(0x44800000u | ((zb >> 4) << 17));
        const float s0 = __uint_as_float(sp << 16);
        const float s8 = __uint_as_float(sp & 0xFFFF0000u) * 0.0625f;
#pragma unroll
        for (int n = 0; n < NT; ++n) {
          const float2 X = lds64f(sst + o_x + (grp * 8 * NT + n * 8) * 4);
          float c[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) c[e] = C::NACC == 2 ? cg[0][n][e] + cg[C::NACC - 1][n][e] : cg[0][n][e];
          acc[n][0] = fmaf(s0, fmaf(-c0, X.x, c[0]), acc[n][0]);
          acc[n][1] = fmaf(s0, fmaf(-c0, X.y, c[1]), acc[n][1]);
          acc[n][2] = fmaf(s8, fmaf(-c8, X.x, c[2]), acc[n][2]);
          acc[n][3] = fmaf(s8, fmaf(-c8, X.y, c[3]), acc[n][3]);
        }
        }  // gi
        }  // !PAIR
      } else if (WFMT == 1) {
        // bf16 LM head: this warp's k16 pair jp = part of the 64-deep unit
        const uint4* wl = reinterpret_cast<const uint4*>(stw) + tile * 128;
        const uint4* sa = reinterpret_cast<const uint4*>(stw + C::WBYTES);
#pragma unroll
        for (int ji = 0; ji < 2 / C::KPARTS; ++ji) {
        const int jp = part + ji;
#pragma unroll
        for (int js = 0; js < 2; ++js) {
          const uint4 wv = wl[(jp * 2 + js) * 32 + lane];
          const uint32_t a[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
          for (int n = 0; n < NT; ++n) {
            const uint4 bh = sa[(jp * 2 * NT + n) * 32 + lane];
            const uint4 bl = sa[(jp * 2 * NT + NT + n) * 32 + lane];
            mma_bf16_16816(acc[n], a, js ? bh.z : bh.x, js ? bh.w : bh.y);
            mma_bf16_16816(acc[n], a, js ? bl.z : bl.x, js ? bl.w : bl.y);
          }
        }
        }  // ji
      }
      __syncwarp();
      if (lane == 0) mbar_arrive_a(empty0 + 8 * s);
      if (++s == C::STAGES) { s = 0; ph ^= 1; }
      ++uc;
    }
    if (cur_tg < 0) break;  // no work at all
    TS(3);
    const int ftg = cur_tg;
    // ---- flush this tile-group's partial (both K-part warps of a tile add)
    {
      const int TP = NT * 8;
      float* base = g.accum + ((size_t)ftg * 128 + tile * 16 + gq) * TP;
#pragma unroll
      for (int n = 0; n < NT; ++n) {
        red_add_v2(base + n * 8 + 2 * tq, acc[n][0], acc[n][1]);
        red_add_v2(base + 8 * TP + n * 8 + 2 * tq, acc[n][2], acc[n][3]);
        acc[n][0] = acc[n][1] = acc[n][2] = acc[n][3] = 0.f;
        if constexpr (C::PAIR) {  // the warp's second tile
          red_add_v2(base + 16 * TP + n * 8 + 2 * tq, acc1[n][0], acc1[n][1]);
          red_add_v2(base + 24 * TP + n * 8 + 2 * tq, acc1[n][2], acc1[n][3]);
          acc1[n][0] = acc1[n][1] = acc1[n][2] = acc1[n][3] = 0.f;
        }
      }
    }
    // hand the flush to the signaler lane: the block-scope release orders this
    // warp's reductions before its fence (cumulative) and arrival count
    __syncwarp();
    if (lane == 0) {
      __threadfence_block();
      atomicAdd_block(&s_flushed, 1);
    }
    cur_tg = done ? -1 : tg;  // the unit waiting in the current slot starts the next group
    nst = 0;
    TS(4);
  }
  // ---- epilogues of the tile-groups this CTA completed (last arriver)
  named_bar_sync(3, NCT + 32);  // with the signaler: s_done_list is complete
  if (s_ndone) fence_acq_rel_gpu();  // acquire side of the arrival counts
  const int ndone = s_ndone;
  for (int i = 0; i < ndone; ++i) {
    const int tg = s_done_list[i];
    const float* accp = g.accum + (size_t)tg * 128 * NT * 8;
    if (threadIdx.x < 256) {  // epilogues are written for 256 threads
      if constexpr (EPI == EPI_QKV) epi_qkv<NT>(g.epi, tg, accp, T);
      else if constexpr (EPI == EPI_SWIGLU) epi_swiglu<NT>(g.epi, tg, accp, T);
      else if constexpr (EPI == EPI_ARGMAX) epi_argmax<NT>(g.epi, tg, accp, T);
      else {
        if (g.epi.P == 1) epi_resid_local<NT>(g.epi, tg, accp, T, g.norm_out ? g.ss : nullptr);
        else epi_ar_send<NT>(g.epi, tg, accp, T);
      }
    }
    named_bar_sync(1, NCT);
    // self-clean the accumulator + counter for the next launch
    float* accw = g.accum + (size_t)tg * 128 * NT * 8;
    for (int j = threadIdx.x; j < 128 * NT * 8; j += NCT) accw[j] = 0.f;
    if (threadIdx.x == 0) g.counters[tg] = 0;
  }
  if constexpr (EPI == EPI_ARGMAX) {
    named_bar_sync(1, NCT);
    if (threadIdx.x == 0 && ndone) {
      fence_acq_rel_gpu();  // the CTA's argmax atomics (ordered by bar.sync) before the arrival
      const int old = atomicAdd(&g.epi.st->lm_done, ndone);
      if (old + ndone == g.n_tg) {
        fence_acq_rel_gpu();
        if (g.epi.P > 1) {
          const ArgmaxXArgs x{g.epi.P, g.epi.rank, g.epi.loopback, g.epi.ar_seq, g.epi.n_tg_total, g.epi.recv,
                              g.epi.peer_recv};
          argmax_exchange(x, g.epi.st);
        }
        accept_walk_dev(g.epi.st);
        g.epi.st->lm_done = 0;
      }
    }
  }
  if constexpr (EPI == EPI_RESID) {
    if (g.epi.P > 1) {  // all sends are out: now wait for the peers' partials
#ifdef SS_EXP_TIMING
      if (threadIdx.x == 0 && blockIdx.x < 1024 && g.epi.kind == g_ts_kind && g.epi.layer == 0)
        g_ts[(blockIdx.x * 8 + 6) & 0xFFFF] = (unsigned long long)ndone;
#endif
#ifdef SS_EXP_TIMING
      if (threadIdx.x == 0 && blockIdx.x < 1024 && g.epi.kind == g_ts_kind && g.epi.layer == 0)
        g_ts[(blockIdx.x * 8 + 2) & 0xFFFF] = gtimer();
#endif
      named_bar_sync(1, NCT);
#ifdef SS_EXP_TIMING
      if (threadIdx.x == 0 && blockIdx.x < 1024 && g.epi.kind == g_ts_kind && g.epi.layer == 0)
        g_ts[(blockIdx.x * 8 + 3) & 0xFFFF] = gtimer();
#endif
      if (threadIdx.x < 256)
        for (int i = 0; i < ndone; ++i) epi_ar_recv<NT>(g.epi, s_done_list[i], T, g.norm_out ? g.ss : nullptr);
    }
    TS(5);
    if (g.norm_out && ndone > 0) {
      // fused RMSNorm: only the CTAs that finalised tile-groups take part
      // (the others have left already); they meet once every tile-group of
      // the residual is added (per-token sums complete), then each
      // normalises the 128-column groups of its own tile-groups
      named_bar_sync(1, NCT);
      if (threadIdx.x == 0) {
        fence_acq_rel_gpu();
        atomicAdd(&g.nbar[0], ndone);
#ifndef SS_EXP_NONORMMEET  // timing experiment only: norm without waiting for the other tile-groups
        while (*reinterpret_cast<volatile int*>(&g.nbar[0]) < g.n_tg) spin_pause();
#endif
        fence_acq_rel_gpu();
      }
      named_bar_sync(1, NCT);
      if (threadIdx.x < 256)
        for (int i = 0; i < ndone; ++i) norm_group<NT>(g, T, s_done_list[i]);
      // the last finaliser out resets the barrier and the per-token sums
      named_bar_sync(1, NCT);
      if (threadIdx.x == 0) {
        fence_acq_rel_gpu();
        if (atomicAdd(&g.nbar[1], ndone) + ndone == g.n_tg) {
          g.nbar[0] = 0;
          g.nbar[1] = 0;
          for (int t = 0; t < SS_MAX_TREE; ++t) g.ss[t] = 0.f;
        }
      }
    }
  }
  TS(7);
}

// ---------------------------------------------------------------- launch
template <int WFMT, int NT, int EPI>
static int launch_t(const GemmArgs& g, int max_ctas, cudaStream_t st) {
  using C = GemmCfg<WFMT, NT>;
  auto k = gemm_kernel<WFMT, NT, EPI>;
  static int occ_dev[kMaxDevices] = {0};  // 0 = attributes not yet set on that device
  const int dev = current_device();
  if (!occ_dev[dev]) {
    int occ = 1;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, C::THREADS, C::SMEM);
    if (occ < 1) occ = 1;
    if (exp_env("SS_DEBUG_OCC")) {
      cudaFuncAttributes fa;
      cudaFuncGetAttributes(&fa, k);
      fprintf(stderr, "gemm WFMT=%d NT=%d EPI=%d: stages %d, dyn smem %d, static smem %zu, regs %d, CTAs/SM %d\n",
              WFMT, NT, EPI, C::STAGES, C::SMEM, fa.sharedSizeBytes, fa.numRegs, occ);
    }
    occ_dev[dev] = occ;
  }
  const int occ = occ_dev[dev];
  long U = (long)g.n_tg * g.S;
  static const int occ_cap = exp_env_int("SS_GEMM_OCC", 0);  // debugging aid
  int o = (occ_cap > 0 && occ_cap < occ) ? occ_cap : occ;
  // minimum stream-K units per CTA: at T <= 8 (NT = 1) two units per CTA
  // (fewer, longer ranges: fewer partial flushes per tile-group) make the
  // small per-rank GEMMs of TP 4 / 8 faster (TP4-rank emulation 6.86 -> 6.61
  // ms) at no cost at TP 1-2; at T >= 16 a unit is longer and spreading wins.
  // SS_GEMM_MINU overrides (tuning aid).
  static const int minu_env = std::max(0, exp_env_int("SS_GEMM_MINU", 0));
  // A GEMM whose whole K fits in <= 4 units (the O projection at TP 8) gives
  // every CTA whole tile-groups: no partial flush, no shared arrival counts
  // (TP8-rank step 5.97 -> 5.87 ms).  The residual (+ all-reduce) GEMMs take
  // >= 4 units per CTA while that still leaves >= 200 CTAs (TP 8 down, TP 2
  // O): fewer partial flushes ahead of the all-reduce tail.
  int min_units = NT == 1 ? 2 : 1;
  if (g.S <= 4) min_units = std::max(min_units, g.S);
  if (EPI == EPI_RESID && U >= 800) min_units = std::max(min_units, 4);
  if (minu_env) min_units = minu_env;
  int grid = (int)std::min<long>((U + min_units - 1) / min_units, (long)g.n_sm * o);
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

template <int WFMT, int EPI>
static void warm_nt() {
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, gemm_kernel<WFMT, 1, EPI>);
  cudaFuncGetAttributes(&a, gemm_kernel<WFMT, 2, EPI>);
  cudaFuncGetAttributes(&a, gemm_kernel<WFMT, 4, EPI>);
  cudaFuncGetAttributes(&a, gemm_kernel<WFMT, 8, EPI>);
}
// see warm_misc_kernels (misc.cu): load every GEMM variant before any launch
void warm_gemm_kernels() {
  warm_nt<0, EPI_QKV>();
  warm_nt<0, EPI_RESID>();
  warm_nt<0, EPI_SWIGLU>();
  warm_nt<1, EPI_ARGMAX>();
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

#ifdef SS_EXP_TIMING
extern "C" int ss_debug_gemm_set_kind(int kind) {
  const int par = kind >= 10 ? kind / 10 - 1 : -1;  // 11 = O-proj (RESID, parity 0), 21 = down
  const int k = kind % 10;
  if (cudaMemcpyToSymbol(ss::g_ts_par, &par, 4) != cudaSuccess) return -1;
  return cudaMemcpyToSymbol(ss::g_ts_kind, &k, 4) == cudaSuccess ? 0 : -1;
}
extern "C" int ss_debug_gemm_timestamps(unsigned long long* out, int n) {
  if (n > (1 << 16)) n = 1 << 16;
  cudaDeviceSynchronize();
  return cudaMemcpyFromSymbol(out, ss::g_ts, (size_t)n * 8) == cudaSuccess ? n : -1;
}
#endif
