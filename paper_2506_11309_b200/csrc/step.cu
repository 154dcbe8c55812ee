// step.cu -- the persistent tree-verify step kernel (SURVEY 8(a) a1..a11 for
// T <= 32): ONE launch runs every layer's QKV GEMM + RoPE + tree-KV write,
// tree attention, O GEMM + all-reduce + residual, gate/up + SwiGLU, down +
// all-reduce + residual, then the LM head + argmax and the accept walk.
//
// Why one kernel (B200): at TP 8 a 70B layer streams only ~55 MB per GPU
// (~8.5 us at HBM speed), while the per-phase kernels of the first build spent
// ~70 us per layer in launch ramp, tails and grid-wide meets.
// Here every CTA stays resident (grid = SMs x CTAs/SM) and walks a static
// schedule; phases hand over through per-layer completion counters in global
// memory instead of kernel boundaries, and -- the point -- weights never wait
// for activations: each CTA's producer warp streams the NEXT units' weights
// into its shared-memory ring while the consumer warps wait for the current
// phase's inputs (TMA bulk copies, mbarrier ring).  A unit's bytes arrive in
// two parts: part 1 (weights, or prefix K/V tiles) is independent of the step
// and issued as soon as a ring slot frees; part 2 (activations, or tree K/V
// rows) is issued once the producing phase's counter reaches its target.
//
// Numerics (R18, tools/err_budget.py): W4 GEMM activations and q
// are fp16 hi + lo pairs (two MMAs per fragment), the tree rows' K and V carry
// a lo part next to the fp16 cache; the RMSNorm scale is deferred: the GEMMs
// consume x * g and the epilogue multiplies by rsqrt(mean x^2 + eps) (a
// per-token scalar commutes with the GEMM), so a residual tile-group's
// next-GEMM input is written as soon as its all-reduce lands -- no grid-wide
// norm meet.
#include "accept.cuh"
#include "common.cuh"
#include "internal.h"
#include "kernels.h"
#include "step.h"

namespace ss {

template <int NT>
struct StepCfg {
  static constexpr int ABYTES = (int)a2_stage_bytes(NT);           // W4 input per unit (hi, lo, X)
  static constexpr int LM_ABYTES = (kBFKS / 16) * 2 * NT * 256;     // LM input per unit (bf16 hi, lo)
  static constexpr int SLOT = kW4UnitBytes + ABYTES;                // >= LM unit, >= one 16 KB K/V tile
  static constexpr int CTAS_PER_SM = NT <= 2 ? 2 : 1;
  static constexpr int STAGES = (CTAS_PER_SM == 2 ? 102400 : 204800) / SLOT;
  static constexpr int SMEM = STAGES * SLOT;
  static constexpr int THREADS = 288;  // 8 consumer warps + 1 producer warp
  static constexpr int NCT = 256;
  static_assert(SLOT >= kBFUnitBytes + LM_ABYTES && SLOT >= 16384 && STAGES >= 3, "slot");
};

enum { PH_QKV = 0, PH_ATT = 1, PH_O = 2, PH_GU = 3, PH_DN = 4, PH_LM = 5, PH_END = 6 };
enum { ACC_QKV = 0, ACC_O = 1, ACC_GU = 2, ACC_DN = 3, ACC_LM = 4 };

SS_DEV uint32_t a2_frag(int tt, int k, int NT, int lo) {
  return (uint32_t)(k >> 8) * a2_stage_bytes(NT) + (lo ? (uint32_t)NT * 4096u : 0u) + frag_offset(tt, k & 255, NT);
}
SS_DEV uint32_t a2_xsum(int tt, int g, int NT) {
  return (uint32_t)(g >> 1) * a2_stage_bytes(NT) + (uint32_t)NT * 8192u + (uint32_t)(((g & 1) * 8 * NT + tt) * 4);
}
// fp16 hi + lo of a pair of values; returns (hi + lo) summed as floats
SS_DEV float split16(float a, float b, uint32_t& hi, uint32_t& lo) {
  hi = pack_half2(a, b);
  const __half2 h = *reinterpret_cast<const __half2*>(&hi);
  const float ha = __low2float(h), hb = __high2float(h);
  lo = pack_half2(a - ha, b - hb);
  const __half2 l = *reinterpret_cast<const __half2*>(&lo);
  return (ha + __low2float(l)) + (hb + __high2float(l));
}

// Watchdog: every wait of the persistent kernel is bounded; a protocol bug
// traps (the launch fails with an error) instead of hanging the GPU.
constexpr unsigned long long kWatchdogNs = 10000000000ull;  // 10 s
SS_DEV unsigned long long now_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
SS_DEV void watchdog(unsigned long long t0) {
  if (now_ns() - t0 > kWatchdogNs) asm volatile("trap;");
}
SS_DEV bool mbar_try_a(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
SS_DEV void mbar_wait_wd(uint32_t bar, uint32_t parity) {
  if (mbar_try_a(bar, parity)) return;
  const unsigned long long t0 = now_ns();
  while (!mbar_try_a(bar, parity)) watchdog(t0);
}
SS_DEV void spin_until_geq(const int* p, int target) {
  if (ld_acquire_gpu(p) >= target) return;
  const unsigned long long t0 = now_ns();
  while (ld_acquire_gpu(p) < target) {
    __nanosleep(64);
    watchdog(t0);
  }
}

// Static schedule ------------------------------------------------------------
// GEMM phases: the U units (tile-group major) are split in equal contiguous
// ranges over min(n_ctas, U) CTAs.
SS_DEV void gemm_range(int U, int n_ctas, int b, int& u0, int& u1) {
  const int parts = U < n_ctas ? U : n_ctas;
  if (b >= parts) { u0 = u1 = 0; return; }
  u0 = (int)((long)b * U / parts);
  u1 = (int)((long)(b + 1) * U / parts);
}

struct Sched {
  int qkv0, qkv1, o0, o1, gu0, gu1, dn0, dn1, lm0, lm1;
  // attention: item of this CTA (grp = kvh * Z + z, split), tiles [t0, t1)
  int att_item, att_S, att_Z, att_A, att_t0, att_t1, att_KT;
  int L, T;
};

SS_DEV void make_sched(const StepArgs& a, int b, int L, int T, int NT, Sched& s) {
  gemm_range(a.qkv_tg * a.qkv_S, a.n_ctas, b, s.qkv0, s.qkv1);
  gemm_range(a.o_tg * a.o_S, a.n_ctas, b, s.o0, s.o1);
  gemm_range(a.gu_tg * a.gu_S, a.n_ctas, b, s.gu0, s.gu1);
  gemm_range(a.dn_tg * a.dn_S, a.n_ctas, b, s.dn0, s.dn1);
  gemm_range(a.lm_tg * a.lm_S, a.n_ctas, b, s.lm0, s.lm1);
  const int KT = att_tile_keys(a.d);
  const int ntiles = (L + T + KT - 1) / KT;
  const int Z = (a.G * 8 * NT + 63) / 64;           // 64-row chunks of the G x T rows per kv head
  const int groups = a.Hkv_l * Z;
  int S = a.n_ctas / groups;
  const int smax = (ntiles + a.att_min_tiles - 1) / a.att_min_tiles;
  if (S > smax) S = smax;
  if (S < 1) S = 1;
  const int per = (ntiles + S - 1) / S;
  S = (ntiles + per - 1) / per;                     // fewest splits with the same longest split
  s.att_S = S;
  s.att_Z = Z;
  s.att_A = groups * S;
  s.att_KT = KT;
  s.att_item = b < s.att_A ? b : -1;
  if (s.att_item >= 0) {
    const int split = b % S;
    s.att_t0 = split * per;
    s.att_t1 = min(ntiles, s.att_t0 + per);
  } else {
    s.att_t0 = s.att_t1 = 0;
  }
  s.L = L;
  s.T = T;
}

// A tile whose rows reach the tree rows [L, L+T) waits for the QKV epilogue
// and is followed by a second ring unit with its lo parts (K_lo, V_lo).
SS_DEV bool tile_is_tree(const Sched& s, int tile) { return (tile + 1) * s.att_KT > s.L; }

// Producer iterator over this CTA's unit sequence ---------------------------
struct UnitIt {
  int layer, ph, i, lo;
};

SS_DEV void range_of(const Sched& s, int ph, int& i0, int& i1) {
  switch (ph) {
    case PH_QKV: i0 = s.qkv0; i1 = s.qkv1; return;
    case PH_ATT: i0 = s.att_t0; i1 = s.att_t1; return;
    case PH_O: i0 = s.o0; i1 = s.o1; return;
    case PH_GU: i0 = s.gu0; i1 = s.gu1; return;
    case PH_DN: i0 = s.dn0; i1 = s.dn1; return;
    case PH_LM: i0 = s.lm0; i1 = s.lm1; return;
    default: i0 = i1 = 0; return;
  }
}

// Move to the first unit at or after (layer, ph, i).
SS_DEV void it_settle(const Sched& s, int n_layers, UnitIt& it) {
  while (it.ph != PH_END) {
    int i0, i1;
    range_of(s, it.ph, i0, i1);
    if (it.i < i0) it.i = i0;
    if (it.i < i1) return;
    it.lo = 0;
    if (it.ph == PH_LM) { it.ph = PH_END; return; }
    if (it.ph == PH_DN) {
      if (++it.layer == n_layers) it.ph = PH_LM;
      else it.ph = PH_QKV;
    } else {
      ++it.ph;
    }
    it.i = -1;
  }
}

SS_DEV void it_next(const Sched& s, int n_layers, UnitIt& it) {
  if (it.ph == PH_ATT && !it.lo && tile_is_tree(s, it.i)) {
    it.lo = 1;
    return;
  }
  it.lo = 0;
  ++it.i;
  it_settle(s, n_layers, it);
}

// Bytes and sources of one unit.
struct UnitSrc {
  const void* w; uint32_t wbytes;        // part 1
  const void* a; uint32_t abytes;        // part 2 (after the dependency)
  const void* a2; uint32_t a2bytes;      // part 2, second copy (V of a K/V tile)
  uint32_t a_off, a2_off;                // slot offsets of the part-2 copies
  const int* dep; int target;            // part-2 dependency (nullptr: none beyond the PDL wait)
  const void* w2; uint32_t w2bytes; uint32_t w2_off;  // part 1, second copy (V of a prefix tile)
};

template <int NT>
SS_DEV void unit_src(const StepArgs& a, const Sched& s, const UnitIt& it, UnitSrc& u) {
  using C = StepCfg<NT>;
  u.w = u.a = u.a2 = u.w2 = nullptr;
  u.wbytes = u.abytes = u.a2bytes = u.w2bytes = 0;
  u.a_off = u.a2_off = u.w2_off = 0;
  u.dep = nullptr;
  u.target = 0;
  const int l = it.layer;
  const int* ctr = a.ctr + (size_t)l * kCtrPerLayer;
  if (it.ph == PH_ATT) {
    const int KT = s.att_KT, d = a.d;
    const int grp = s.att_item / s.att_S, kvh = grp / s.att_Z;
    const uint32_t half = (uint32_t)KT * d * 2;  // 8 KB
    if (!it.lo) {
      const size_t base = (((size_t)l * a.Hkv_l + kvh) * a.max_ctx_pad + (size_t)it.i * KT) * d;
      if (tile_is_tree(s, it.i)) {
        u.a = a.kc + base; u.abytes = half; u.a_off = 0;
        u.a2 = a.vc + base; u.a2bytes = half; u.a2_off = half;
        u.dep = ctr + C_QKV; u.target = a.qkv_tg;
      } else {
        u.w = a.kc + base; u.wbytes = half;
        u.w2 = a.vc + base; u.w2bytes = half; u.w2_off = half;
      }
    } else {
      const int wb = s.L & ~63;
      const size_t base = ((size_t)kvh * 128 + (size_t)(it.i * KT - wb)) * d;
      u.a = a.klo + base; u.abytes = half; u.a_off = 0;
      u.a2 = a.vlo + base; u.a2bytes = half; u.a2_off = half;
      u.dep = ctr + C_QKV; u.target = a.qkv_tg;
    }
    return;
  }
  if (it.ph == PH_LM) {
    u.w = a.lm_w + (size_t)it.i * kBFUnitBytes; u.wbytes = kBFUnitBytes;
    u.a = a.act_lm + (size_t)(it.i % a.lm_S) * C::LM_ABYTES; u.abytes = C::LM_ABYTES; u.a_off = kBFUnitBytes;
    u.dep = a.ctr + (size_t)(a.n_layers - 1) * kCtrPerLayer + C_DN; u.target = a.dn_tg;
    return;
  }
  const LayerPtrs& lp = a.layers[l];
  const uint8_t* W;
  const uint8_t* act;
  int S;
  switch (it.ph) {
    case PH_QKV:
      W = lp.qkv; act = a.act_h; S = a.qkv_S;
      if (l > 0) { u.dep = ctr - kCtrPerLayer + C_DN; u.target = a.dn_tg; }
      break;
    case PH_O: W = lp.o; act = a.act_o; S = a.o_S; u.dep = ctr + C_ATT; u.target = s.att_A; break;
    case PH_GU: W = lp.gu; act = a.act_h; S = a.gu_S; u.dep = ctr + C_O; u.target = a.o_tg; break;
    default: W = lp.down; act = a.act_d; S = a.dn_S; u.dep = ctr + C_GU; u.target = a.gu_tg; break;
  }
  u.w = W + (size_t)it.i * kW4UnitBytes; u.wbytes = kW4UnitBytes;
  u.a = act + (size_t)(it.i % S) * C::ABYTES; u.abytes = C::ABYTES; u.a_off = kW4UnitBytes;
}

// The producer: lane 0 of warp 8.  Issues part 1 of unit w whenever its ring
// slot is free and part 2 of the oldest unit still missing it whenever that
// unit's dependency is met -- never blocking on one while the other could
// make progress.
template <int NT>
__device__ __noinline__ void producer(const StepArgs* __restrict__ ap, const Sched* __restrict__ sp, uint32_t sm0,
                                      uint32_t full0, uint32_t empty0) {
  using C = StepCfg<NT>;
  const StepArgs& a = *ap;
  const Sched s = *sp;
  const uint64_t pol = policy_evict_first();
  UnitIt wi{0, PH_QKV, -1, 0}, ai;
  it_settle(s, a.n_layers, wi);
  ai = wi;
  int wk = 0, ak = 0;        // units issued (part 1 / part 2)
  const int* ok_dep = nullptr;
  int ok_target = 0;
  unsigned long long t_idle = now_ns();
  while (ai.ph != PH_END) {
    bool prog = false;
    if (wi.ph != PH_END) {
      const int slot = wk % C::STAGES;
      const uint32_t par = (uint32_t)((wk / C::STAGES) & 1);
      if (mbar_test_a(empty0 + 8 * slot, par ^ 1)) {
        fence_proxy_async_smem();  // consumers' reads of the slot before the TMA overwrite
        UnitSrc u;
        unit_src<NT>(a, s, wi, u);
        const uint32_t dst = sm0 + slot * C::SLOT, bar = full0 + 8 * slot;
        if (u.wbytes) {
          const uint32_t tot = u.wbytes + u.w2bytes;
          if (u.abytes) mbar_expect_tx_noarrive_a(bar, tot);
          else mbar_arrive_expect_tx_a(bar, tot);
          bulk_g2s_a(dst, u.w, u.wbytes, bar, pol);
          if (u.w2bytes) bulk_g2s_a(dst + u.w2_off, u.w2, u.w2bytes, bar, pol);
        }
        ++wk;
        it_next(s, a.n_layers, wi);
        prog = true;
      }
    }
    if (ak < wk) {
      UnitSrc u;
      unit_src<NT>(a, s, ai, u);
      bool go = true;
      if (u.abytes && u.dep && !(u.dep == ok_dep && u.target <= ok_target)) {
        const int v = ld_acquire_gpu(u.dep);
        go = v >= u.target;
        if (go) {
          ok_dep = u.dep;
          ok_target = u.target;
          fence_proxy_async_global();  // the producers' generic stores before our async-proxy reads
        }
      }
      if (go) {
        if (u.abytes) {
          const int slot = ak % C::STAGES;
          const uint32_t dst = sm0 + slot * C::SLOT, bar = full0 + 8 * slot;
          mbar_arrive_expect_tx_a(bar, u.abytes + u.a2bytes);
          bulk_g2s_nohint_a(dst + u.a_off, u.a, u.abytes, bar);
          if (u.a2bytes) bulk_g2s_nohint_a(dst + u.a2_off, u.a2, u.a2bytes, bar);
        }
        ++ak;
        it_next(s, a.n_layers, ai);
        prog = true;
      }
    }
    if (!prog) {
      __nanosleep(32);
      watchdog(t_idle);
    } else {
      t_idle = now_ns();
    }
  }
}

// Consumers -------------------------------------------------------------------
struct Ring {
  uint32_t sm0, full0, empty0;
  int k;  // units consumed so far
};

template <int NT>
SS_DEV uint32_t ring_wait(const Ring& r) {
  using C = StepCfg<NT>;
  const int slot = r.k % C::STAGES;
  mbar_wait_wd(r.full0 + 8 * slot, (uint32_t)((r.k / C::STAGES) & 1));
  return r.sm0 + slot * C::SLOT;
}
template <int NT>
SS_DEV void ring_release(Ring& r) {
  using C = StepCfg<NT>;
  __syncwarp();
  if ((threadIdx.x & 31) == 0) mbar_arrive_a(r.empty0 + 8 * (r.k % C::STAGES));
  ++r.k;
}

SS_DEV void cbar() { named_bar_sync(1, 256); }  // the 8 consumer warps

SS_DEV void wait_counter(const int* p, int target) {
  if (threadIdx.x == 0) spin_until_geq(p, target);
  cbar();
}

// One W4 unit, PAIR mapping (gemm.cu): warp = two 16-row tiles x one 128-deep
// group; B fragments (fp16 hi and lo) feed two MMAs each.
template <int NT>
SS_DEV void w4_unit(uint32_t sst, int warp, int lane, float (&acc)[NT][4], float (&acc1)[NT][4]) {
  const int tile = 2 * (warp & 3), grp = warp >> 2;
  const int gq = lane >> 2, tq = lane & 3;
  const uint32_t o_w = (uint32_t)(tile * 128 + lane) * 16;
  const uint32_t o_sc = (uint32_t)(kW4Bytes + tile * 64 + gq * 4);
  const uint32_t o_z = (uint32_t)(kW4Bytes + 512 + tile * 16 + gq);
  const uint32_t o_b = (uint32_t)(kW4UnitBytes + lane * 16);
  const uint32_t o_x = (uint32_t)(kW4UnitBytes + NT * 8192 + 8 * tq);
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
  for (int jp = 0; jp < 4; ++jp) {
    uint4 bh[NT], bl[NT];
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      bh[n] = lds128(sst + o_b + ((grp * 4 + jp) * NT + n) * 512);
      bl[n] = lds128(sst + o_b + NT * 4096 + ((grp * 4 + jp) * NT + n) * 512);
    }
#pragma unroll
    for (int js = 0; js < 2; ++js)
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        uint32_t af[4];
        dequant8(wa[i][jp * 2 + js], af);
#pragma unroll
        for (int n = 0; n < NT; ++n) {
          mma_f16_16816(cg[i][n], af, js ? bh[n].z : bh[n].x, js ? bh[n].w : bh[n].y);
          mma_f16_16816(cg[i][n], af, js ? bl[n].z : bl[n].x, js ? bl[n].w : bl[n].y);
        }
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
}

// One bf16 LM-head unit (128 vocab rows x 64 k): warp = one 16-row tile.
template <int NT>
SS_DEV void lm_unit(uint32_t sst, int warp, int lane, float (&acc)[NT][4]) {
  const int tile = warp;
#pragma unroll
  for (int jp = 0; jp < 2; ++jp)
#pragma unroll
    for (int js = 0; js < 2; ++js) {
      const uint4 wv = lds128(sst + (uint32_t)((tile * 128 + (jp * 2 + js) * 32 + lane) * 16));
      const uint32_t af[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
      for (int n = 0; n < NT; ++n) {
        const uint4 bh = lds128(sst + kBFUnitBytes + (uint32_t)(((jp * 2 * NT + n) * 32 + lane) * 16));
        const uint4 bl = lds128(sst + kBFUnitBytes + (uint32_t)(((jp * 2 * NT + NT + n) * 32 + lane) * 16));
        mma_bf16_16816(acc[n], af, js ? bh.z : bh.x, js ? bh.w : bh.y);
        mma_bf16_16816(acc[n], af, js ? bl.z : bl.x, js ? bl.w : bl.y);
      }
    }
}

// Epilogues (256 consumer threads) --------------------------------------------
SS_DEV float norm_scale(const float* ss, int t, int h, float eps) { return rsqrtf(__ldcg(ss + t) / (float)h + eps); }

SS_DEV uint32_t q_frag_index(int m, int j, int d, int rbmax, int kvh) {
  const int rb = m >> 4, r = m & 15, kk = j >> 4, c = j & 15;
  const int lane = ((r & 7) << 2) | ((c & 7) >> 1);
  const int reg = (r >> 3) + 2 * (c >> 3);
  return ((((uint32_t)kvh * rbmax + rb) * (d / 16) + kk) * 32 + lane) * 8 + reg * 2 + (c & 1);
}

// a4: deferred attn-norm scale, RoPE (R2), q hi/lo in fragment order,
// tree K/V rows: fp16 hi into the cache at L + t (R10), lo into the window.
template <int NT>
SS_DEV void epi_qkv(const StepArgs& a, int layer, int tg, const float* acc, const Sched& s) {
  const int TP = NT * 8, T = s.T, L = s.L, d = a.d, half = d >> 1;
  const int nq = a.Hq_l * d, nk = a.Hkv_l * d;
  const float* ssa = a.ss + (size_t)layer * 2 * 64;
  const int wb = L & ~63;
  const int rbmax = 4 * a.G;
  const size_t qlo = (size_t)a.Hkv_l * rbmax * (d / 16) * 32 * 8;
  const int n = 128 * T;
  for (int idx = threadIdx.x; idx < n; idx += 256) {
    const int r = idx / T, t = idx - r * T;
    const int row = tg * 128 + r, j = row % d;
    const float rs = norm_scale(ssa, t, a.h, a.eps);
    float x = __ldcg(acc + (size_t)r * TP + t) * rs;
    if (row < nq + nk) {
      const int pr = (j < half) ? r + half : r - half;
      const float pv = __ldcg(acc + (size_t)pr * TP + t) * rs;
      const float2 cs = a.rope_cs[(size_t)a.st->pos[t] * half + (j % half)];
      x = (j < half) ? (x * cs.x - pv * cs.y) : (x * cs.x + pv * cs.y);
    }
    const __half hh = __float2half_rn(x);
    const __half hl = __float2half_rn(x - __half2float(hh));
    if (row < nq) {
      const int hq = row / d, kvh = hq / a.G, jj = hq - kvh * a.G;
      const uint32_t fi = q_frag_index(t * a.G + jj, j, d, rbmax, kvh);
      a.qf[fi] = __half_as_ushort(hh);
      a.qf[qlo + fi] = __half_as_ushort(hl);
    } else if (row < nq + 2 * nk) {
      const bool isk = row < nq + nk;
      const int kvh = (isk ? row - nq : row - nq - nk) / d;
      uint16_t* c = isk ? a.kc : a.vc;
      uint16_t* lo = isk ? a.klo : a.vlo;
      const size_t base = ((size_t)layer * a.Hkv_l + kvh) * a.max_ctx_pad * d;
      c[base + kv_elem_offset(L + t, j, d)] = __half_as_ushort(hh);
      lo[(size_t)kvh * 128 * d + kv_elem_offset(L + t - wb, j, d)] = __half_as_ushort(hl);
    }
  }
  // zero the lo window rows outside the tree of this tile-group's K / V heads
  // (a tree tile's prefix rows add q . 0)
  const int row0 = tg * 128;
  if (row0 + 127 >= nq && row0 < nq + 2 * nk) {
    for (int hd = 0; hd < 128 / d; ++hd) {
      const int row = row0 + hd * d;
      if (row < nq || row >= nq + 2 * nk) continue;
      const bool isk = row < nq + nk;
      const int kvh = (isk ? row - nq : row - nq - nk) / d;
      uint16_t* lo = (isk ? a.klo : a.vlo) + (size_t)kvh * 128 * d;
      for (int i = threadIdx.x; i < 128 * d / 8; i += 256) {
        const int w = i / (d / 8);
        const int pos = wb + w;
        if (pos >= L && pos < L + T) continue;
        *reinterpret_cast<uint4*>(lo + (size_t)w * d + (i % (d / 8)) * 8) = make_uint4(0, 0, 0, 0);
      }
    }
  }
}

// a8: deferred mlp-norm scale + SwiGLU (R4) -> down input (hi/lo, X)
template <int NT>
SS_DEV void epi_swiglu(const StepArgs& a, int layer, int tg, const float* acc, int T) {
  const int TP = NT * 8;
  const float* ssm = a.ss + (size_t)layer * 2 * 64 + 64;
  const int warp = threadIdx.x >> 5, cp = threadIdx.x & 31;
  for (int t = warp; t < T; t += 8) {
    const float rs = norm_scale(ssm, t, a.h, a.eps);
    const float g0 = __ldcg(acc + (size_t)(2 * cp) * TP + t) * rs;
    const float g1 = __ldcg(acc + (size_t)(2 * cp + 1) * TP + t) * rs;
    const float u0 = __ldcg(acc + (size_t)(64 + 2 * cp) * TP + t) * rs;
    const float u1 = __ldcg(acc + (size_t)(64 + 2 * cp + 1) * TP + t) * rs;
    const float h0 = g0 / (1.f + __expf(-g0)) * u0;
    const float h1 = g1 / (1.f + __expf(-g1)) * u1;
    const int k = tg * 64 + 2 * cp;
    uint32_t hi, lo;
    float xs = split16(h0, h1, hi, lo);
    *reinterpret_cast<uint32_t*>(a.act_d + a2_frag(t, k, NT, 0)) = hi;
    *reinterpret_cast<uint32_t*>(a.act_d + a2_frag(t, k, NT, 1)) = lo;
    xs = warp_sum(xs);
    if (cp == 0) atomicAdd(reinterpret_cast<float*>(a.act_d + a2_xsum(t, k >> 7, NT)), xs);
  }
}

// TP > 1: this rank's fp32 partial of tile-group tg to every peer as LL lines
// (data1, flag1, data2, flag2, R15), same layout as gemm.cu.
template <int NT>
SS_DEV void ar_send(const StepArgs& a, int tg, const float* acc, int T, int ar_seq) {
  const int TP = NT * 8;
  const uint32_t flag = a.st->epoch + ar_seq;
  const int pairs = (T + 1) >> 1;
  const int ntg = a.h / 128;
  for (int idx = threadIdx.x; idx < 128 * pairs; idx += 256) {
    const int r = idx / pairs, tp = idx - r * pairs;
    const float2 v = __ldcg(reinterpret_cast<const float2*>(acc + (size_t)r * TP + 2 * tp));
    for (int p = 0; p < a.P; ++p) {
      const int slot = a.loopback ? p : a.rank;
      const size_t line = (((size_t)(ar_seq & 1) * a.P + slot) * ntg + tg) * 128 * (4 * NT) + (size_t)r * (4 * NT) + tp;
      ll_store(reinterpret_cast<uint4*>(a.peer_recv[p]) + line, __float_as_uint(v.x), __float_as_uint(v.y), flag);
    }
  }
}

// Residual update of tile-group tg: x += acc (P == 1) or the rank-ordered sum
// of every rank's partial (TP all-reduce receive).
template <int NT>
SS_DEV void resid_update(const StepArgs& a, int tg, const float* acc, int T, int ar_seq) {
  const int TP = NT * 8;
  if (a.P == 1) {
    for (int idx = threadIdx.x; idx < 128 * T; idx += 256) {
      const int t = idx >> 7, r = idx & 127;
      float* xp = a.x + (size_t)t * a.h + tg * 128 + r;
      *xp = __ldcg(xp) + __ldcg(acc + (size_t)r * TP + t);
    }
    return;
  }
  constexpr int PP = 4 * NT;
  const uint32_t flag = a.st->epoch + ar_seq;
  const int pairs = (T + 1) >> 1;
  const int ntg = a.h / 128;
  for (int idx = threadIdx.x; idx < 128 * pairs; idx += 256) {
    const int tp = idx >> 7, r = idx & 127;
    const uint4* src0 = reinterpret_cast<const uint4*>(a.recv) +
                        (((size_t)(ar_seq & 1) * a.P) * ntg + tg) * 128 * PP + (size_t)r * PP + tp;
    const size_t pstride = (size_t)ntg * 128 * PP;
    uint32_t d1[kMaxPeers], d2[kMaxPeers];
    unsigned ready = 0;
    const unsigned all = (1u << a.P) - 1u;
    long spins = 0;
    while (ready != all) {
#pragma unroll
      for (int p = 0; p < kMaxPeers; ++p)
        if (p < a.P && !(ready & (1u << p)) && ll_try_load(src0 + p * pstride, flag, d1[p], d2[p])) ready |= 1u << p;
      if (++spins > (1L << 24)) { a.st->timeout = 1; break; }
    }
    float s0 = 0.f, s1 = 0.f;
#pragma unroll
    for (int p = 0; p < kMaxPeers; ++p)
      if (p < a.P) {
        s0 += __uint_as_float(d1[p]);
        s1 += __uint_as_float(d2[p]);
      }
    const int t0 = 2 * tp;
    float* x0 = a.x + (size_t)t0 * a.h + tg * 128 + r;
    *x0 = __ldcg(x0) + s0;
    if (t0 + 1 < T) x0[a.h] = __ldcg(x0 + a.h) + s1;
  }
}

// After the residual of tile-group tg is final: the next GEMM's input for its
// 128 columns (x * g, fp16 hi/lo + X; or bf16 hi/lo for the LM head) and the
// token's sum of squares (the deferred RMSNorm scale, R5).
template <int NT>
SS_DEV void next_input(const StepArgs& a, int tg, int T, const uint16_t* gain, float* ss, uint8_t* act, int lm) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int k = tg * 128 + lane * 4;
  const uint2 gw = *reinterpret_cast<const uint2*>(gain + k);
  for (int t = warp; t < T; t += 8) {
    const float4 v = __ldcg(reinterpret_cast<const float4*>(a.x + (size_t)t * a.h + k));
    const float q = warp_sum(v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w);
    if (lane == 0) atomicAdd(ss + t, q);
    const float y0 = v.x * bf16_lo(gw.x), y1 = v.y * bf16_hi(gw.x), y2 = v.z * bf16_lo(gw.y), y3 = v.w * bf16_hi(gw.y);
    if (lm) {
      const uint32_t h01 = pack_bf16x2(y0, y1), h23 = pack_bf16x2(y2, y3);
      *reinterpret_cast<uint32_t*>(act + frag_offset(t, k, 2 * NT)) = h01;
      *reinterpret_cast<uint32_t*>(act + frag_offset(t, k + 2, 2 * NT)) = h23;
      *reinterpret_cast<uint32_t*>(act + frag_offset(t + 8 * NT, k, 2 * NT)) =
          pack_bf16x2(y0 - bf16_lo(h01), y1 - bf16_hi(h01));
      *reinterpret_cast<uint32_t*>(act + frag_offset(t + 8 * NT, k + 2, 2 * NT)) =
          pack_bf16x2(y2 - bf16_lo(h23), y3 - bf16_hi(h23));
    } else {
      uint32_t h01, l01, h23, l23;
      float xs = split16(y0, y1, h01, l01) + split16(y2, y3, h23, l23);
      *reinterpret_cast<uint32_t*>(act + a2_frag(t, k, NT, 0)) = h01;
      *reinterpret_cast<uint32_t*>(act + a2_frag(t, k + 2, NT, 0)) = h23;
      *reinterpret_cast<uint32_t*>(act + a2_frag(t, k, NT, 1)) = l01;
      *reinterpret_cast<uint32_t*>(act + a2_frag(t, k + 2, NT, 1)) = l23;
      xs = warp_sum(xs);
      if (lane == 0) *reinterpret_cast<float*>(act + a2_xsum(t, tg, NT)) = xs;
    }
  }
}

template <int NT>
SS_DEV void epi_argmax(const StepArgs& a, int tg, const float* acc, int T) {
  const int TP = NT * 8;
  const float* ssf = a.ss + (size_t)a.n_layers * 2 * 64;
  const int r = threadIdx.x & 127;
  const int v = tg * 128 + r;
  const bool valid = v < a.V_l;
  for (int t = threadIdx.x >> 7; t < T; t += 2) {
    const float rs = norm_scale(ssf, t, a.h, a.eps);
    const float val = valid ? __ldcg(acc + (size_t)r * TP + t) * rs : -INFINITY;
    if (valid && a.logits) a.logits[(size_t)t * a.logits_ld + v] = val;
    unsigned long long key = valid ? argmax_key(val, (uint32_t)(a.V_off + v)) : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long other = __shfl_xor_sync(0xffffffffu, key, o);
      key = other > key ? other : key;
    }
    if ((threadIdx.x & 31) == 0 && key) atomicMax(&a.st->argmax_key[t], key);
  }
}

// A GEMM phase: consume this CTA's units [u0, u1), flush partial tile-groups
// (red.add), count arrivals, run the epilogues of the tile-groups completed
// here.  Returns the number of tile-groups this CTA finalised.
template <int NT, int PH>
__device__ __noinline__ int gemm_phase(const StepArgs* __restrict__ ap, const Sched* __restrict__ sp, int layer,
                                       int u0, int u1, Ring ring, int* s_done, int* s_nd) {
  const StepArgs& a = *ap;
  const Sched& s = *sp;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gq = lane >> 2, tq = lane & 3;
  const int TP = NT * 8;
  const int S = PH == PH_QKV ? a.qkv_S : PH == PH_O ? a.o_S : PH == PH_GU ? a.gu_S : PH == PH_DN ? a.dn_S : a.lm_S;
  const int ai = PH == PH_QKV ? ACC_QKV : PH == PH_O ? ACC_O : PH == PH_GU ? ACC_GU : PH == PH_DN ? ACC_DN : ACC_LM;
  float* accb = a.acc[ai];
  int* arr = a.arr[ai];
  const int T = s.T;
  float acc[NT][4], acc1[NT][4];
#pragma unroll
  for (int n = 0; n < NT; ++n)
#pragma unroll
    for (int e = 0; e < 4; ++e) acc[n][e] = acc1[n][e] = 0.f;
  for (int u = u0; u < u1; ++u) {
    const uint32_t sst = ring_wait<NT>(ring);
    if constexpr (PH == PH_LM) lm_unit<NT>(sst, warp, lane, acc);
    else w4_unit<NT>(sst, warp, lane, acc, acc1);
    ring_release<NT>(ring);
    const int tg = u / S;
    if (u + 1 == u1 || (u + 1) / S != tg) {  // flush this tile-group's partial
      if constexpr (PH == PH_LM) {
        float* base = accb + ((size_t)tg * 128 + warp * 16 + gq) * TP;
#pragma unroll
        for (int n = 0; n < NT; ++n) {
          red_add_v2(base + n * 8 + 2 * tq, acc[n][0], acc[n][1]);
          red_add_v2(base + 8 * TP + n * 8 + 2 * tq, acc[n][2], acc[n][3]);
          acc[n][0] = acc[n][1] = acc[n][2] = acc[n][3] = 0.f;
        }
      } else {
        float* base = accb + ((size_t)tg * 128 + 2 * (warp & 3) * 16 + gq) * TP;
#pragma unroll
        for (int n = 0; n < NT; ++n) {
          red_add_v2(base + n * 8 + 2 * tq, acc[n][0], acc[n][1]);
          red_add_v2(base + 8 * TP + n * 8 + 2 * tq, acc[n][2], acc[n][3]);
          red_add_v2(base + 16 * TP + n * 8 + 2 * tq, acc1[n][0], acc1[n][1]);
          red_add_v2(base + 24 * TP + n * 8 + 2 * tq, acc1[n][2], acc1[n][3]);
#pragma unroll
          for (int e = 0; e < 4; ++e) acc[n][e] = acc1[n][e] = 0.f;
        }
      }
    }
  }
  // arrivals: the barrier orders every warp's reductions before thread 0's
  // GPU-scope fence (cumulative) and arrival counts
  cbar();
  if (threadIdx.x == 0) {
    int nd = 0;
    if (u1 > u0) {
      fence_acq_rel_gpu();
      for (int tg = u0 / S; tg <= (u1 - 1) / S; ++tg) {
        const int nst = min(u1, (tg + 1) * S) - max(u0, tg * S);
        if (atomicAdd(&arr[tg], nst) + nst == S) s_done[nd++] = tg;
      }
      if (nd) fence_acq_rel_gpu();  // acquire side: the other CTAs' partials
    }
    *s_nd = nd;
  }
  cbar();
  const int nd = *s_nd;
  if (nd == 0) return ring.k;
  int* ctr = a.ctr + (size_t)layer * kCtrPerLayer;
  if constexpr (PH == PH_QKV || PH == PH_GU || PH == PH_LM) {
    for (int i = 0; i < nd; ++i) {
      const int tg = s_done[i];
      const float* accp = accb + (size_t)tg * 128 * TP;
      if constexpr (PH == PH_QKV) epi_qkv<NT>(a, layer, tg, accp, s);
      else if constexpr (PH == PH_GU) epi_swiglu<NT>(a, layer, tg, accp, T);
      else epi_argmax<NT>(a, tg, accp, T);
    }
  } else {
    // residual phases: sends of every completed tile-group first, then the
    // receives (no rank waits on a tile-group it has not sent yet)
    const int ar_seq = 2 * layer + (PH == PH_DN ? 1 : 0);
    if (a.P > 1)
      for (int i = 0; i < nd; ++i) ar_send<NT>(a, s_done[i], accb + (size_t)s_done[i] * 128 * TP, T, ar_seq);
    for (int i = 0; i < nd; ++i) resid_update<NT>(a, s_done[i], accb + (size_t)s_done[i] * 128 * TP, T, ar_seq);
    cbar();
    const bool last = PH == PH_DN && layer + 1 == a.n_layers;
    const uint16_t* gain = PH == PH_O ? a.layers[layer].mlp_norm
                                      : (last ? a.final_norm : a.layers[layer + 1].attn_norm);
    float* ssn = a.ss + (size_t)(PH == PH_O ? layer * 2 + 1 : (layer + 1) * 2) * 64;
    uint8_t* act = last ? a.act_lm : a.act_h;
    for (int i = 0; i < nd; ++i) next_input<NT>(a, s_done[i], T, gain, ssn, act, last ? 1 : 0);
    if constexpr (PH == PH_O) {
      // zero the down input's X slots (the SwiGLU epilogues of this layer add into them)
      const int ngrp = a.I_l / 128;
      for (int i = 0; i < nd; ++i)
        for (int g = s_done[i]; g < ngrp; g += a.o_tg)
          for (int t = threadIdx.x; t < 8 * NT; t += 256)
            *reinterpret_cast<float*>(a.act_d + a2_xsum(t, g, NT)) = 0.f;
    }
  }
  cbar();
  // self-clean the accumulators and arrival counters for the next layer
  for (int i = 0; i < nd; ++i) {
    float* accw = accb + (size_t)s_done[i] * 128 * TP;
    for (int j = threadIdx.x; j < 128 * TP; j += 256) accw[j] = 0.f;
    if (threadIdx.x == 0) arr[s_done[i]] = 0;
  }
  cbar();
  if (threadIdx.x == 0) {
    fence_acq_rel_gpu();  // epilogue outputs (and the cleaning) before the completion count
    if constexpr (PH == PH_LM) {
      int* lmc = a.ctr + (size_t)a.n_layers * kCtrPerLayer;
      if (atomicAdd(lmc, nd) + nd == a.lm_tg) {
        fence_acq_rel_gpu();
        if (a.P > 1) {
          const ArgmaxXArgs x{a.P, a.rank, a.loopback, 2 * a.n_layers, a.h / 128, a.recv, a.peer_recv};
          argmax_exchange(x, a.st);
        }
        accept_walk_dev(a.st);
      }
    } else {
      const int ci = PH == PH_QKV ? C_QKV : PH == PH_O ? C_O : PH == PH_GU ? C_GU : C_DN;
      red_release_gpu_add(ctr + ci, nd);
    }
  }
  return ring.k;
}

// Tree-masked attention (a5, R11) of one work item: (kv head,
// 64-row chunk z, key split).  Warp w = (row block rb = w % 4, half h = w / 4):
// it computes the scores of its 16 query rows against key half h of every
// tile (q hi + lo fragments from global memory -- written by the QKV epilogue,
// L1-resident -- times the K tile in the ring; tree tiles add q_hi K_lo),
// the warp pair (rb, 0) / (rb, 1) exchanges row maxima and the fp16
// probabilities P through shared memory, then each warp accumulates O for
// d-half h over ALL keys of the tile (P V_hi + P V_lo on tree tiles): no
// duplicated MMAs and a 16 x d/2 fp32 accumulator per warp.  The split's
// unnormalised partial goes to the workspace; after the splits of the group
// meet, each merges a slice of the rows by log-sum-exp into the O input.
template <int NT, int D>
__device__ __noinline__ int attn_item(const StepArgs* __restrict__ ap, const Sched* __restrict__ sp, int layer,
                                      Ring ring, float* s_rmax, uint16_t* s_p) {
  const StepArgs& a = *ap;
  const Sched& s = *sp;
  constexpr int KT = 4096 / D, KH = KT / 2, NTK = KH / 8, DH = D / 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rb = warp & 3, kh = warp >> 2;
  const int gq = lane >> 2, tq = lane & 3;
  const int b = s.att_item;
  const int grp = b / s.att_S, split = b % s.att_S;
  const int kvh = grp / s.att_Z, z = grp % s.att_Z;
  const int G = a.G, T = s.T, L = s.L;
  const int Mrows = G * T;
  const int rbmax = 4 * G;
  const size_t qlo = (size_t)a.Hkv_l * rbmax * (D / 16) * 32 * 8;
  int* ctr = a.ctr + (size_t)layer * kCtrPerLayer;
  wait_counter(ctr + C_QKV, a.qkv_tg);  // q, tree rows and their lo parts are written
  const DevState* st = a.st;
  const int rbg = z * 4 + rb;
  const int ra = rb * 16 + gq, rbr = ra + 8;  // rows within the chunk
  const int rowA = z * 64 + ra, rowB = z * 64 + rbr;
  const int tokA = min(rowA / G, SS_MAX_TREE - 1), tokB = min(rowB / G, SS_MAX_TREE - 1);
  const unsigned long long ancA = st->anc[tokA], ancB = st->anc[tokB];
  const bool okA = rowA < Mrows, okB = rowB < Mrows;
  const float sl2 = rsqrtf((float)D) * 1.4426950408889634f;
  const uint4* qh = reinterpret_cast<const uint4*>(a.qf) + (((size_t)kvh * rbmax + rbg) * (D / 16)) * 32 + lane;
  const uint4* ql = reinterpret_cast<const uint4*>(a.qf + qlo) + (((size_t)kvh * rbmax + rbg) * (D / 16)) * 32 + lane;
  const int pair_bar = 2 + rb;                 // named barrier of warps rb and rb + 4
  const uint32_t spb = smem_u32(s_p);           // P [64 rows][KT keys] fp16, 16-byte chunks swizzled by row
  float mA = -INFINITY, mB = -INFINITY, lA = 0.f, lB = 0.f;
  float o[DH / 8][4];
#pragma unroll
  for (int n = 0; n < DH / 8; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
  const int kofs = kh * KH;
  for (int it = s.att_t0; it < s.att_t1; ++it) {
    const bool tree = tile_is_tree(s, it);
    const uint32_t shi = ring_wait<NT>(ring);
    Ring r2 = ring;
    ++r2.k;
    const uint32_t slo = tree ? ring_wait<NT>(r2) : shi;
    float sc[NTK][4];
#pragma unroll
    for (int n = 0; n < NTK; ++n) sc[n][0] = sc[n][1] = sc[n][2] = sc[n][3] = 0.f;
#pragma unroll 2
    for (int kk = 0; kk < D / 16; ++kk) {
      const uint4 fh = qh[kk * 32], fl = ql[kk * 32];
      const uint32_t ah[4] = {fh.x, fh.y, fh.z, fh.w}, al[4] = {fl.x, fl.y, fl.z, fl.w};
#pragma unroll
      for (int np = 0; np < NTK / 2; ++np) {
        const int key = kofs + np * 16 + (lane & 7) + ((lane >> 4) << 3);
        const int ch = kk * 2 + ((lane >> 3) & 1);
        const uint32_t koff = (uint32_t)(key * D + ((ch ^ (key & 7)) << 3)) * 2;
        uint32_t kb[4];
        asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                     : "=r"(kb[0]), "=r"(kb[1]), "=r"(kb[2]), "=r"(kb[3]) : "r"(shi + koff));
        mma_f16_16816(sc[2 * np], ah, kb[0], kb[1]);
        mma_f16_16816(sc[2 * np + 1], ah, kb[2], kb[3]);
        mma_f16_16816(sc[2 * np], al, kb[0], kb[1]);
        mma_f16_16816(sc[2 * np + 1], al, kb[2], kb[3]);
        if (tree) {
          asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                       : "=r"(kb[0]), "=r"(kb[1]), "=r"(kb[2]), "=r"(kb[3]) : "r"(slo + koff));
          mma_f16_16816(sc[2 * np], ah, kb[0], kb[1]);
          mma_f16_16816(sc[2 * np + 1], ah, kb[2], kb[3]);
        }
      }
    }
    // mask: prefix always visible; tree rows by ancestor bit; beyond L+T never
    const int kbase = it * KT + kofs;
    float mxA = -INFINITY, mxB = -INFINITY;
#pragma unroll
    for (int n = 0; n < NTK; ++n)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int key = kbase + n * 8 + 2 * tq + (e & 1);
        const unsigned long long anc = (e < 2) ? ancA : ancB;
        const bool ok = (e < 2) ? okA : okB;
        const bool vis = ok && (key < L || (key < L + T && ((anc >> (key - L)) & 1ull)));
        const float v = vis ? sc[n][e] * sl2 : -INFINITY;
        sc[n][e] = v;
        if (e < 2) mxA = fmaxf(mxA, v); else mxB = fmaxf(mxB, v);
      }
    mxA = fmaxf(mxA, __shfl_xor_sync(0xffffffffu, mxA, 1));
    mxA = fmaxf(mxA, __shfl_xor_sync(0xffffffffu, mxA, 2));
    mxB = fmaxf(mxB, __shfl_xor_sync(0xffffffffu, mxB, 1));
    mxB = fmaxf(mxB, __shfl_xor_sync(0xffffffffu, mxB, 2));
    // the pair's row maxima over the whole tile (both warps then hold the same running max)
    if (tq == 0) {
      s_rmax[kh * 64 + ra] = mxA;
      s_rmax[kh * 64 + rbr] = mxB;
    }
    named_bar_sync(pair_bar, 64);
    mxA = fmaxf(mxA, s_rmax[(kh ^ 1) * 64 + ra]);
    mxB = fmaxf(mxB, s_rmax[(kh ^ 1) * 64 + rbr]);
    const float mnA = fmaxf(mA, mxA), mnB = fmaxf(mB, mxB);
    const float uA = (mnA == -INFINITY) ? 0.f : mnA, uB = (mnB == -INFINITY) ? 0.f : mnB;
    const float alA = exp2f(mA - uA), alB = exp2f(mB - uB);
    float sumA = 0.f, sumB = 0.f;
#pragma unroll
    for (int n = 0; n < NTK; ++n) {
      const float p0 = exp2f(sc[n][0] - uA), p1 = exp2f(sc[n][1] - uA);
      const float p2 = exp2f(sc[n][2] - uB), p3 = exp2f(sc[n][3] - uB);
      sumA += p0 + p1;
      sumB += p2 + p3;
      // P[row][key] fp16: row-major KT keys, 16-byte chunk index XOR row % 8
      const int key = kofs + n * 8 + 2 * tq;
      const uint32_t offA = (uint32_t)(ra * KT + ((((key >> 3) ^ (ra & 7))) << 3) + (key & 7)) * 2;
      const uint32_t offB = (uint32_t)(rbr * KT + ((((key >> 3) ^ (rbr & 7))) << 3) + (key & 7)) * 2;
      asm volatile("st.shared.b32 [%0], %1;" ::"r"(spb + offA), "r"(pack_half2(p0, p1)) : "memory");
      asm volatile("st.shared.b32 [%0], %1;" ::"r"(spb + offB), "r"(pack_half2(p2, p3)) : "memory");
    }
    sumA += __shfl_xor_sync(0xffffffffu, sumA, 1);
    sumA += __shfl_xor_sync(0xffffffffu, sumA, 2);
    sumB += __shfl_xor_sync(0xffffffffu, sumB, 1);
    sumB += __shfl_xor_sync(0xffffffffu, sumB, 2);
    lA = lA * alA + sumA;  // this warp's keys only; the two halves are added at the end
    lB = lB * alB + sumB;
    mA = mnA;
    mB = mnB;
    if (__any_sync(0xffffffffu, alA != 1.f || alB != 1.f)) {
#pragma unroll
      for (int n = 0; n < DH / 8; ++n) {
        o[n][0] *= alA; o[n][1] *= alA; o[n][2] *= alB; o[n][3] *= alB;
      }
    }
    named_bar_sync(pair_bar, 64);  // P of both key halves is in shared memory
    const uint32_t vh = shi + KT * D * 2, vl = slo + KT * D * 2;
#pragma unroll
    for (int kk = 0; kk < KT / 16; ++kk) {
      uint32_t pa[4];
      {  // A fragment of P: rows rb*16.., keys kk*16..
        const int prow = rb * 16 + (lane & 15);
        const int ch = kk * 2 + (lane >> 4);
        asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                     : "=r"(pa[0]), "=r"(pa[1]), "=r"(pa[2]), "=r"(pa[3])
                     
                     : "r"(spb + (uint32_t)(prow * KT + ((ch ^ (prow & 7)) << 3)) * 2));
      }
#pragma unroll
      for (int dp = 0; dp < DH / 16; ++dp) {
        const int key = kk * 16 + (lane & 7) + (((lane >> 3) & 1) << 3);
        const int ch = (kh * DH) / 8 + dp * 2 + (lane >> 4);
        const uint32_t voff = (uint32_t)(key * D + ((ch ^ (key & 7)) << 3)) * 2;
        uint32_t vb[4];
        asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                     : "=r"(vb[0]), "=r"(vb[1]), "=r"(vb[2]), "=r"(vb[3]) : "r"(vh + voff));
        mma_f16_16816(o[2 * dp], pa, vb[0], vb[1]);
        mma_f16_16816(o[2 * dp + 1], pa, vb[2], vb[3]);
        if (tree) {
          asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                       : "=r"(vb[0]), "=r"(vb[1]), "=r"(vb[2]), "=r"(vb[3]) : "r"(vl + voff));
          mma_f16_16816(o[2 * dp], pa, vb[0], vb[1]);
          mma_f16_16816(o[2 * dp + 1], pa, vb[2], vb[3]);
        }
      }
    }
    ring_release<NT>(ring);
    if (tree) ring_release<NT>(ring);
    named_bar_sync(pair_bar, 64);  // P reads done before the next tile's P writes
  }
  // the split's partial -> workspace: O (this warp's rows x d-half) and (m, l)
  // with l summed over the two key halves
  {
    float* ws = a.att_ws + (size_t)b * 64 * D;
#pragma unroll
    for (int n = 0; n < DH / 8; ++n) {
      const int c = kh * DH + n * 8 + 2 * tq;
      *reinterpret_cast<float2*>(ws + (size_t)ra * D + c) = make_float2(o[n][0], o[n][1]);
      *reinterpret_cast<float2*>(ws + (size_t)rbr * D + c) = make_float2(o[n][2], o[n][3]);
    }
    if (kh == 1 && tq == 0) {
      s_rmax[ra] = lA;
      s_rmax[rbr] = lB;
    }
    named_bar_sync(pair_bar, 64);
    if (kh == 0 && tq == 0) {
      a.att_ml[(size_t)b * 64 + ra] = make_float2(mA, lA + s_rmax[ra]);
      a.att_ml[(size_t)b * 64 + rbr] = make_float2(mB, lB + s_rmax[rbr]);
    }
  }
  // meet the other splits of this (kv head, row chunk)
  cbar();
  if (threadIdx.x == 0) {
    fence_acq_rel_gpu();
    atomicAdd(ctr + C_MEET + grp, 1);
    spin_until_geq(ctr + C_MEET + grp, s.att_S);
  }
  cbar();
  // merge a slice of the row groups (one 128-wide group of the O input: one
  // head at d = 128, two at d = 64) across the S partials, R11 log-sum-exp
  constexpr int RPG = 128 / D;             // rows per group
  constexpr int NRG = 64 / RPG;
  const int rg0 = split * NRG / s.att_S, rg1 = (split + 1) * NRG / s.att_S;
  for (int rg = rg0 + warp; rg < rg1; rg += 8) {
    const int rr = rg * RPG + (RPG == 2 ? (lane >> 4) : 0);  // row within the chunk
    const int c4 = (RPG == 2 ? (lane & 15) : lane) * 4;       // 4 columns
    const int m = z * 64 + rr;
    const bool valid = m < Mrows;
    float mx = -INFINITY;
    for (int p = 0; p < s.att_S; ++p)
      mx = fmaxf(mx, __ldcg(&a.att_ml[((size_t)grp * s.att_S + p) * 64 + rr].x));
    float l = 0.f;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int p = 0; p < s.att_S; ++p) {
      const size_t pb = (size_t)grp * s.att_S + p;
      const float2 v = __ldcg(&a.att_ml[pb * 64 + rr]);
      const float w = (v.x == -INFINITY) ? 0.f : exp2f(v.x - mx);
      l += w * v.y;
      const float4 ov = __ldcg(reinterpret_cast<const float4*>(a.att_ws + (pb * 64 + rr) * D + c4));
      acc.x += w * ov.x;
      acc.y += w * ov.y;
      acc.z += w * ov.z;
      acc.w += w * ov.w;
    }
    const float inv = l > 0.f ? 1.f / l : 0.f;
    acc.x *= inv; acc.y *= inv; acc.z *= inv; acc.w *= inv;
    const int t = m / G, hq = kvh * G + (m % G);
    const int k = hq * D + c4;
    uint32_t h01, l01, h23, l23;
    float xs = split16(acc.x, acc.y, h01, l01) + split16(acc.z, acc.w, h23, l23);
    if (valid) {
      *reinterpret_cast<uint32_t*>(a.act_o + a2_frag(t, k, NT, 0)) = h01;
      *reinterpret_cast<uint32_t*>(a.act_o + a2_frag(t, k + 2, NT, 0)) = h23;
      *reinterpret_cast<uint32_t*>(a.act_o + a2_frag(t, k, NT, 1)) = l01;
      *reinterpret_cast<uint32_t*>(a.act_o + a2_frag(t, k + 2, NT, 1)) = l23;
    }
    xs = warp_sum(valid ? xs : 0.f);
    if (lane == 0 && valid) *reinterpret_cast<float*>(a.act_o + a2_xsum(t, k >> 7, NT)) = xs;
  }
  cbar();
  if (threadIdx.x == 0) {
    fence_acq_rel_gpu();
    red_release_gpu_add(ctr + C_ATT, 1);
  }
  return ring.k;
}

template <int NT, int D>
__global__ void __launch_bounds__(StepCfg<NT>::THREADS, StepCfg<NT>::CTAS_PER_SM)
    step_kernel(const StepArgs* __restrict__ ap) {
  using C = StepCfg<NT>;
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[C::STAGES], empty[C::STAGES];
  __shared__ int s_done[128];
  __shared__ int s_nd;
  __shared__ float s_rmax[2 * 64];
  __shared__ Sched s_sched;
  __shared__ __align__(16) uint16_t s_p[64 * (4096 / D)];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < C::STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 8);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const uint32_t sm0 = smem_u32(smem), full0 = smem_u32(full), empty0 = smem_u32(empty);
  // everything below reads the ingest kernel's outputs (T, L, tree, counters)
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x == 0) make_sched(*ap, blockIdx.x, ap->st->L, ap->st->T, NT, s_sched);
  __syncthreads();
  if (warp == 8) {
    if (lane == 0) producer<NT>(ap, &s_sched, sm0, full0, empty0);
    return;
  }
  Ring ring{sm0, full0, empty0, 0};
  const int n_layers = ap->n_layers;
  const bool att = s_sched.att_item >= 0;
  for (int l = 0; l < n_layers; ++l) {
    ring.k = gemm_phase<NT, PH_QKV>(ap, &s_sched, l, s_sched.qkv0, s_sched.qkv1, ring, s_done, &s_nd);
    if (att) ring.k = attn_item<NT, D>(ap, &s_sched, l, ring, s_rmax, s_p);
    ring.k = gemm_phase<NT, PH_O>(ap, &s_sched, l, s_sched.o0, s_sched.o1, ring, s_done, &s_nd);
    ring.k = gemm_phase<NT, PH_GU>(ap, &s_sched, l, s_sched.gu0, s_sched.gu1, ring, s_done, &s_nd);
    ring.k = gemm_phase<NT, PH_DN>(ap, &s_sched, l, s_sched.dn0, s_sched.dn1, ring, s_done, &s_nd);
  }
  gemm_phase<NT, PH_LM>(ap, &s_sched, 0, s_sched.lm0, s_sched.lm1, ring, s_done, &s_nd);
}

template <int NT, int D>
static int ctas_t(int max_ctas) {
  using C = StepCfg<NT>;
  static int occ_dev[kMaxDevices] = {0};
  const int dev = current_device();
  if (!occ_dev[dev]) {
    int occ = 1;
    cudaFuncSetAttribute(step_kernel<NT, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, step_kernel<NT, D>, C::THREADS, C::SMEM);
    occ_dev[dev] = occ < 1 ? 1 : occ;
  }
  int n_sm = 148;
  cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
  int n = n_sm * std::min(occ_dev[dev], C::CTAS_PER_SM);
  return (max_ctas > 0 && n > max_ctas) ? max_ctas : n;
}

template <int NT, int D>
static int launch_step_t(const StepArgs& a0, const StepArgs* dev_args, int max_ctas, cudaStream_t st) {
  using C = StepCfg<NT>;
  const int n = ctas_t<NT, D>(max_ctas);  // every CTA co-resident (flag waits)
  if (n != a0.n_ctas) return 0;           // the device copy of the arguments was written for another grid
  launch_pdl(step_kernel<NT, D>, dim3(n), dim3(C::THREADS), C::SMEM, st, dev_args);
  return 1;
}

// Grid of the step kernel (all CTAs co-resident): SMs x resident CTAs per SM,
// capped by max_ctas (fake-peer TP shards share one GPU).
int step_ctas(int NT, int d, int max_ctas) {
  if (d == 64) return NT == 1 ? ctas_t<1, 64>(max_ctas) : NT == 2 ? ctas_t<2, 64>(max_ctas) : ctas_t<4, 64>(max_ctas);
  return NT == 1 ? ctas_t<1, 128>(max_ctas) : NT == 2 ? ctas_t<2, 128>(max_ctas) : ctas_t<4, 128>(max_ctas);
}

// dev_args: a device copy of a (written by the host before graph capture).
int launch_step(const StepArgs& a, const StepArgs* dev_args, int NT, int max_ctas, cudaStream_t st) {
  if (a.d == 64) {
    switch (NT) {
      case 1: return launch_step_t<1, 64>(a, dev_args, max_ctas, st);
      case 2: return launch_step_t<2, 64>(a, dev_args, max_ctas, st);
      default: return launch_step_t<4, 64>(a, dev_args, max_ctas, st);
    }
  }
  switch (NT) {
    case 1: return launch_step_t<1, 128>(a, dev_args, max_ctas, st);
    case 2: return launch_step_t<2, 128>(a, dev_args, max_ctas, st);
    default: return launch_step_t<4, 128>(a, dev_args, max_ctas, st);
  }
}

void warm_step_kernels() {
  cudaFuncAttributes at;
  cudaFuncGetAttributes(&at, step_kernel<1, 64>);
  cudaFuncGetAttributes(&at, step_kernel<2, 64>);
  cudaFuncGetAttributes(&at, step_kernel<4, 64>);
  cudaFuncGetAttributes(&at, step_kernel<1, 128>);
  cudaFuncGetAttributes(&at, step_kernel<2, 128>);
  cudaFuncGetAttributes(&at, step_kernel<4, 128>);
}

}  // namespace ss
