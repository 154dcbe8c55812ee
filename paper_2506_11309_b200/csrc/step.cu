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
  static constexpr int CTAS_PER_SM = 1;  // owns the SM's 512 TMEM columns
  // attention: the item's q fragments (64 rows x d <= 128, hi + lo, 32 KB);
  // GEMM tails: the tile-group's accumulator block and new residual rows
  static constexpr int QBYTES = 34816;
  static constexpr int STAGES = (218112 - QBYTES) / SLOT;
  static constexpr int SMEM = STAGES * SLOT + QBYTES;
  // 8 consumer warps (warpgroups 0, 1) + warpgroup 2: producer warp, two MMA
  // warps (one per AWQ group of a unit), one idle warp.  Launched at 168 registers (3 warps per SMSP); warpgroup 2
  // gives registers back (setmaxnreg) so the consumers run with 208.
  static constexpr int THREADS = 384;
  static constexpr int REG_CONSUMER = 208, REG_AUX = 80;  // 8 x 208 + 4 x 80 <= 12 x 168 (the CTA pool)
  static constexpr int TP = 8 * NT;    // token slots
  static constexpr int N = 2 * TP;     // MMA N: hi and lo columns of every token slot
  static constexpr int NCT = 256;
  static_assert(SLOT >= kBFUnitBytes + LM_ABYTES && SLOT >= 16384 && STAGES >= 3, "slot");
};

enum { PH_QKV = 0, PH_ATT = 1, PH_O = 2, PH_GU = 3, PH_DN = 4, PH_LM = 5, PH_END = 6 };
enum { ACC_QKV = 0, ACC_O = 1, ACC_GU = 2, ACC_DN = 3, ACC_LM = 4 };

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
// (clock64 based: %globaltimer reads are slow and sit on the producer's and
// the waits' critical paths; 2e10 cycles = 10 s at 1.965 GHz)
constexpr unsigned long long kWatchdogClk = 20000000000ull;
SS_DEV unsigned long long now_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
SS_DEV unsigned long long clk64() {
  unsigned long long c;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
  return c;
}
// Panic record of the first wait that times out (mapped host memory, read by
// ss_watchdog_record after the failed launch): [0] = 1 + site, [1] = address
// (shared-memory barrier or global counter), [2] = parity / target, [3] =
// value seen, [4] = blockIdx.x, [5] = threadIdx.x, [6] = ring / unit info.
__device__ unsigned long long* g_panic = nullptr;
__device__ int g_panic_map = 0;
// Every timed-out waiter also fills its warp's slot [64 + (block * 16 + warp) * 4]
// (site + 1, address, parity / target, seen) and lingers ~1 s before trapping,
// so the other waiters of a deadlock record themselves too.
SS_DEV void panic_trap(int site, unsigned long long addr, unsigned long long want, unsigned long long seen) {
#ifdef SS_WATCHDOG_RECORD  // debugging builds (tools/wd70.py): record every timed-out waiter
  unsigned long long* p = g_panic;
  if (p) {
    if (atomicCAS(p, 0ull, (unsigned long long)(1 + site)) == 0ull) {
      p[1] = addr;
      p[2] = want;
      p[3] = seen;
      p[4] = blockIdx.x;
      p[5] = threadIdx.x;
    }
    unsigned long long* q = p + 64 + ((size_t)blockIdx.x * 16 + (threadIdx.x >> 5)) * 4;
    q[0] = 1 + site;
    q[1] = addr;
    q[2] = want;
    q[3] = seen;
    __threadfence_system();
    const unsigned long long t = clk64();
    while (clk64() - t < 2000000000ull) __nanosleep(1000);
  }
#else
  (void)site; (void)addr; (void)want; (void)seen;
#endif
  asm volatile("trap;");
}
SS_DEV void watchdog(unsigned long long t0) {
  // the producer's idle wait: twice the bound, so the wait that starved it is recorded first
  if (clk64() - t0 > 2 * kWatchdogClk) panic_trap(0, 0, 0, 0);
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
  const unsigned long long t0 = clk64();
  while (!mbar_try_a(bar, parity))
    if (clk64() - t0 > kWatchdogClk) panic_trap(1, bar, parity, 0);
}
SS_DEV int ld_relaxed_gpu(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Poll relaxed (ld.acquire.gpu invalidates the SM's L1 on every poll, hurting
// every warp that reads cached global data), acquire once when satisfied.
SS_DEV void spin_until_geq(const int* p, int target) {
  if (ld_acquire_gpu(p) >= target) return;
  const unsigned long long t0 = clk64();
  while (ld_relaxed_gpu(p) < target) {
    __nanosleep(64);
    if (clk64() - t0 > kWatchdogClk) panic_trap(2, (unsigned long long)p, target, ld_relaxed_gpu(p));
  }
  (void)ld_acquire_gpu(p);
}

// GPU-scope atomics with release / acquire semantics: the release is
// cumulative over the CTA's writes ordered before it by a CTA barrier, so no
// separate fence.acq_rel.gpu is needed around the arrival counts.
SS_DEV int atom_add_acqrel_gpu(int* p, int v) {
  int old;
  asm volatile("atom.add.acq_rel.gpu.global.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
SS_DEV void atom_add_release_gpu(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

SS_DEV void tmark(const StepArgs& a, int slot, int which) {
  if (a.trace && threadIdx.x == 0) a.trace[((size_t)blockIdx.x * a.trace_slots + slot) * 3 + which] = now_ns();
}

// tcgen05 (5th-gen tensor cores, TMEM accumulators) ------------------------
// TMEM map of the CTA (512 columns, lane = output row of the 128-row tile):
//   [0, 128 kNbuf)   A operand, kNbuf buffers of one W4 unit (256 k = 128 fp16x2 columns)
//   [128 kNbuf, 512) fp32 accumulators, [slot kNacc][AWQ group 2][N columns]
// T <= 8: three A buffers (the dequant of unit k waits for unit k - 3's MMAs,
// one unit more slack than two buffers); the accumulators fill the rest.
constexpr uint32_t kTmemCols = 512;
template <int NT> constexpr int kNbuf = 2;  // a third buffer at T <= 8 measured neutral (DESIGN 6b)
template <int NT> constexpr uint32_t kAccColT = 128u * kNbuf<NT>;
// accumulator slots [kNacc][AWQ group 2][N]: 4 at T <= 16 (the two warp sets
// alternate two each, so a unit's MMAs never write the accumulator the
// previous unit's epilogue is reading), 2 at T <= 32
template <int NT> constexpr int kNacc = NT <= 2 ? 4 : 2;
SS_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
SS_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
SS_DEV void tc_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
SS_DEV void tc_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
// 16 TMEM lanes x 32 columns; register 4j + (0..3) of thread (g, q) = (lane g,
// col 8j + 2q), (g, 8j + 2q + 1), (g + 8, 8j + 2q), (g + 8, 8j + 2q + 1)
// (the mma.m16n8 fragment pattern, CuTe SM100_TMEM_STORE_16dp256b).
SS_DEV void tc_st_16x256b_x4(uint32_t ta, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.16x256b.x4.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(ta),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
// thread i <- TMEM lane (base lane + i), 16 consecutive columns
SS_DEV void tc_ld_32x32b_x16(uint32_t ta, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(ta)
      : "memory");
}
// Shared-memory matrix descriptor, K-major, no swizzle (sm100 version 1):
// lbo = bytes between the two 8-deep k chunks, sbo = bytes between 8-row groups.
SS_DEV uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
// Instruction descriptor kind::f16: D f32, A / B f16, both K-major, N, M.
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) {
  return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

SS_DEV void where(const StepArgs& a, uint32_t code) {
  if (a.where && (threadIdx.x & 31) == 0)
    *reinterpret_cast<volatile unsigned long long*>(a.where + blockIdx.x * 16 + (threadIdx.x >> 5)) =
        ((unsigned long long)code << 32) | (now_ns() & 0xFFFFFFFFull);
}
SS_DEV int lane_id() { return threadIdx.x & 31; }
#define WCODE(layer, ph, pt) (((uint32_t)(layer) << 16) | ((uint32_t)(ph) << 8) | (uint32_t)(pt))

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
  int L, T, T0;  // committed length, token slots, cached tree nodes (slot t = node T0 + t)
};

// Tile-group-aligned split: c = n_ctas / n_tg CTAs per tile-group, each a
// contiguous chunk of one tile-group, so no CTA finalises two tile-groups
// (their tails -- all-reduce, RoPE / KV writes -- would run back to back).
// Used when it does not lengthen the longest range by more than one unit.
SS_DEV void gemm_range_tg(int n_tg, int S, int n_ctas, int b, int& u0, int& u1) {
  const int U = n_tg * S;
  const int c = n_ctas / n_tg;
  if (c >= 2 && (S + c - 1) / c <= (U + n_ctas - 1) / n_ctas + 1) {
    if (b >= n_tg * c) { u0 = u1 = 0; return; }
    const int tg = b / c, j = b % c;
    u0 = tg * S + j * S / c;
    u1 = tg * S + (j + 1) * S / c;
    return;
  }
  gemm_range(U, n_ctas, b, u0, u1);
}

// Deterministic mode: whole tile-groups per CTA (no cross-CTA split-K, so each
// accumulator element receives one flush per warp set, in a fixed place).
SS_DEV void gemm_range_whole(int n_tg, int S, int n_ctas, int b, int& u0, int& u1) {
  int t0, t1;
  gemm_range(n_tg, n_ctas, b, t0, t1);
  u0 = t0 * S;
  u1 = t1 * S;
}

SS_DEV void make_sched(const StepArgs& a, int b, int L, int T, int T0, int NT, Sched& s) {
  if (a.det) {
    gemm_range_whole(a.qkv_tg, a.qkv_S, a.n_ctas, b, s.qkv0, s.qkv1);
    gemm_range_whole(a.o_tg, a.o_S, a.n_ctas, b, s.o0, s.o1);
    gemm_range_whole(a.gu_tg, a.gu_S, a.n_ctas, b, s.gu0, s.gu1);
    gemm_range_whole(a.dn_tg, a.dn_S, a.n_ctas, b, s.dn0, s.dn1);
    gemm_range_whole(a.lm_tg, a.lm_S, a.n_ctas, b, s.lm0, s.lm1);
  } else {
    gemm_range_tg(a.qkv_tg, a.qkv_S, a.n_ctas, b, s.qkv0, s.qkv1);
    gemm_range_tg(a.o_tg, a.o_S, a.n_ctas, b, s.o0, s.o1);
    gemm_range_tg(a.gu_tg, a.gu_S, a.n_ctas, b, s.gu0, s.gu1);
    gemm_range_tg(a.dn_tg, a.dn_S, a.n_ctas, b, s.dn0, s.dn1);
    gemm_range(a.lm_tg * a.lm_S, a.n_ctas, b, s.lm0, s.lm1);
  }
  const int KT = att_tile_keys(a.d);
  const int ntiles = (L + T0 + T + KT - 1) / KT;  // prefix + cached tree rows + new rows
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
  s.T0 = T0;
}

// A tile whose rows reach the tree rows [L, L+T) waits for the QKV epilogue
// and is followed by a second ring unit with its lo parts (K_lo, V_lo).
SS_DEV bool tile_is_tree(const Sched& s, int tile) { return (tile + 1) * s.att_KT > s.L; }

// Producer iterator over this CTA's unit sequence ---------------------------
// Per-phase data (unit range, weight / activation bases, dependency) is cached
// at each phase change, so advancing over a GEMM / LM-head unit is a handful
// of integer ops: the single producer thread shares its SMSP with two busy
// consumer warps, and its per-unit instruction count bounds the stream rate.
struct UnitIt {
  int layer, ph, i, lo;
  int i1, st, S;             // range end, stage i % S, stages per tile-group
  const uint8_t* w;          // GEMM / LM head: unit 0's weights of this phase
  const uint8_t* act;        // stage 0's activations
  const int* dep;            // part-2 dependency
  int target;
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

// Cache the per-phase fields of it (it.ph, it.layer, it.i set).
SS_DEV void it_cache(const StepArgs& a, const Sched& s, UnitIt& it) {
  const int l = it.layer;
  const int* ctr = a.ctr + (size_t)l * kCtrPerLayer;
  it.dep = nullptr;
  it.target = 0;
  it.S = 1;
  it.w = it.act = nullptr;
  if (it.ph == PH_ATT || it.ph == PH_END) return;
  if (it.ph == PH_LM) {
    it.w = a.lm_w; it.act = a.act_lm; it.S = a.lm_S;
    it.dep = a.ctr + (size_t)(a.n_layers - 1) * kCtrPerLayer + C_DN; it.target = a.dn_tg;
  } else {
    const LayerPtrs& lp = a.layers[l];
    switch (it.ph) {
      case PH_QKV:
        it.w = lp.qkv; it.act = a.act_h; it.S = a.qkv_S;
        if (l > 0) { it.dep = ctr - kCtrPerLayer + C_DN; it.target = a.dn_tg; }
        break;
      case PH_O: it.w = lp.o; it.act = a.act_o; it.S = a.o_S; it.dep = ctr + C_ATT; it.target = s.att_A; break;
      case PH_GU: it.w = lp.gu; it.act = a.act_h; it.S = a.gu_S; it.dep = ctr + C_O; it.target = a.o_tg; break;
      default: it.w = lp.down; it.act = a.act_d; it.S = a.dn_S; it.dep = ctr + C_GU; it.target = a.gu_tg; break;
    }
  }
  it.st = it.i % it.S;
}

// Move to the first unit at or after (layer, ph, i).
SS_DEV void it_settle(const StepArgs& a, const Sched& s, UnitIt& it) {
  while (it.ph != PH_END) {
    int i0, i1;
    range_of(s, it.ph, i0, i1);
    if (it.i < i0) it.i = i0;
    if (it.i < i1) {
      it.i1 = i1;
      it_cache(a, s, it);
      return;
    }
    it.lo = 0;
    if (it.ph == PH_LM) { it.ph = PH_END; return; }
    if (it.ph == PH_DN) {
      if (++it.layer == a.n_layers) it.ph = PH_LM;
      else it.ph = PH_QKV;
    } else {
      ++it.ph;
    }
    it.i = -1;
  }
}

SS_DEV void it_next(const StepArgs& a, const Sched& s, UnitIt& it) {
  if (it.ph == PH_ATT && !it.lo && tile_is_tree(s, it.i)) {
    it.lo = 1;
    return;
  }
  it.lo = 0;
  ++it.i;
  if (++it.st == it.S) it.st = 0;
  if (it.i >= it.i1) it_settle(a, s, it);
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

// The producer: lane 0 of warp 8.  Issues part 1 of every unit whose ring
// slot is free and part 2 of every unit (in order) whose dependency is met --
// as many as possible per pass, never blocking on one while the other could
// make progress.
template <int NT>
__device__ __noinline__ void producer(const StepArgs* __restrict__ ap, const Sched* __restrict__ sp, uint32_t sm0,
                                      uint32_t full0, uint32_t empty0) {
  using C = StepCfg<NT>;
  const StepArgs& a = *ap;
  const Sched s = *sp;
  const uint64_t pol = policy_evict_first();
  UnitIt wi;
  wi.layer = 0; wi.ph = PH_QKV; wi.i = -1; wi.lo = 0;
  it_settle(a, s, wi);
  UnitIt ai = wi;
  int wk = 0, ak = 0;        // units issued (part 1 / part 2)
  const int* ok_dep = nullptr;
  int ok_target = 0;
  unsigned long long t_idle = clk64();
  while (ai.ph != PH_END) {
    bool prog = false;
    // part 1: weights (or prefix K/V tiles) into every free slot; one proxy
    // fence per batch orders the consumers' generic reads of the freed slots
    // before the TMA overwrites
    bool fenced = false;
    while (wi.ph != PH_END && wk - ak < C::STAGES) {
      const int slot = wk % C::STAGES;
      if (!mbar_test_a(empty0 + 8 * slot, (uint32_t)(((wk / C::STAGES) & 1) ^ 1))) break;
      if (!fenced) {
        fence_proxy_async_smem();
        fenced = true;
      }
      const uint32_t dst = sm0 + slot * C::SLOT, bar = full0 + 8 * slot;
      if (wi.ph != PH_ATT) {
        const uint32_t ub = wi.ph == PH_LM ? (uint32_t)kBFUnitBytes : (uint32_t)kW4UnitBytes;
        mbar_expect_tx_noarrive_a(bar, ub);
        bulk_g2s_a(dst, wi.w + (size_t)wi.i * ub, ub, bar, pol);
      } else {
        UnitSrc u;
        unit_src<NT>(a, s, wi, u);
        if (u.wbytes) {
          const uint32_t tot = u.wbytes + u.w2bytes;
          if (u.abytes) mbar_expect_tx_noarrive_a(bar, tot);
          else mbar_arrive_expect_tx_a(bar, tot);
          bulk_g2s_a(dst, u.w, u.wbytes, bar, pol);
          if (u.w2bytes) bulk_g2s_a(dst + u.w2_off, u.w2, u.w2bytes, bar, pol);
        }
      }
      ++wk;
      it_next(a, s, wi);
      prog = true;
    }
    // part 2: activations (or tree K/V rows) once their producing phase is done
    while (ak < wk) {
      const int* dep;
      int target;
      UnitSrc u;
      const bool att = ai.ph == PH_ATT;
      if (att) {
        unit_src<NT>(a, s, ai, u);
        dep = u.dep;
        target = u.target;
      } else {
        dep = ai.dep;
        target = ai.target;
      }
      if (dep && !(dep == ok_dep && target <= ok_target)) {
        if (ld_relaxed_gpu(dep) < target) break;
        (void)ld_acquire_gpu(dep);
        ok_dep = dep;
        ok_target = target;
        fence_proxy_async_global();  // the producers' generic stores before our async-proxy reads
      }
      const int slot = ak % C::STAGES;
      const uint32_t dst = sm0 + slot * C::SLOT, bar = full0 + 8 * slot;
      if (!att) {
        const uint32_t abytes = ai.ph == PH_LM ? (uint32_t)C::LM_ABYTES : (uint32_t)C::ABYTES;
        const uint32_t aoff = ai.ph == PH_LM ? (uint32_t)kBFUnitBytes : (uint32_t)kW4UnitBytes;
        mbar_arrive_expect_tx_a(bar, abytes);
        bulk_g2s_nohint_a(dst + aoff, ai.act + (size_t)ai.st * abytes, abytes, bar);
      } else if (u.abytes) {
        mbar_arrive_expect_tx_a(bar, u.abytes + u.a2bytes);
        bulk_g2s_nohint_a(dst + u.a_off, u.a, u.abytes, bar);
        if (u.a2bytes) bulk_g2s_nohint_a(dst + u.a2_off, u.a2, u.a2bytes, bar);
      }
      ++ak;
      it_next(a, s, ai);
      prog = true;
    }
    if (!prog) {
      where(a, WCODE(ai.layer, 0x40 + ai.ph, wi.ph == PH_END ? 0xEE : 0x01));
      __nanosleep(32);
      watchdog(t_idle);
    } else {
      t_idle = clk64();
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

template <int NT>
SS_DEV uint32_t ring_wait_at(const Ring& r, int k) {
  using C = StepCfg<NT>;
  const int slot = k % C::STAGES;
  mbar_wait_wd(r.full0 + 8 * slot, (uint32_t)((k / C::STAGES) & 1));
  return r.sm0 + slot * C::SLOT;
}
template <int NT>
SS_DEV void ring_release_at(const Ring& r, int k) {
  using C = StepCfg<NT>;
  __syncwarp();
  if ((threadIdx.x & 31) == 0) mbar_arrive_a(r.empty0 + 8 * (k % C::STAGES));
}
SS_DEV void red_add_v4(float* p, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}

// the 8 consumer warps; each warp converges first (a thread-0-only block
// before a barrier must not let the warp's other lanes arrive without it)
SS_DEV void cbar() {
  __syncwarp();
  named_bar_sync(1, 256);
}

SS_DEV void wait_counter(const int* p, int target) {
  if (threadIdx.x == 0) spin_until_geq(p, target);
  cbar();
}

// W4 units on tcgen05 -----------------------------------------------------------
// A unit = 128 output rows x 256 k (gemm.cu layout: [16-row tile 8][64-deep
// k block 4][lane 32][4 nibble words], each word one m16n8k16 A fragment).
// Consumer warp w (quadrant qd = w % 4, half hh = w / 4) dequantises tile
// 2 qd + hh -- TMEM lanes 32 qd + 16 hh .. + 15, the lanes its quadrant may
// access -- with the lop3 trick into fp16 (1024 + q, or 1024 + 16 q on the
// tile's rows 8..15) and stores the fragments with tcgen05.st.16x256b, whose
// register pattern is the fragment pattern: column pair order within each k16
// step becomes (0 4 1 5 2 6 3 7), matched by the activation layout (a2_frag).
// The MMA warp runs the unit's 16 MMAs (M 128, N = 2 TP hi + lo columns, K 16)
// into one fresh accumulator per AWQ group; then warp w reads group hh of
// rows 32 qd + lane and applies the exact zero point / scale (R3, R19, R20):
//   y[t] += s * ((acc_hi[t] + acc_lo[t]) - (1024 + z) * X[t]).
struct Tc {
  uint32_t tbase;    // TMEM base address
  uint32_t ardy0;    // mbarrier[kNbuf]: the unit's A operand is in TMEM (8 warp arrivals)
  uint32_t mdone0;   // mbarrier[kNbuf buffers][2 groups]: MMAs reading the A buffer completed
  uint32_t* slot;    // shared [kNbuf]: smem address of the unit's ring slot (0 = stop)
};
// The epilogue of unit k waits for its MMAs on the A buffer's barrier (phase
// parity (k / kNbuf) & 1).  The barrier cannot complete again before: the next
// user of the buffer, unit k + kNbuf, belongs to the same warp set (kNbuf = 2,
// sets on alternating units) and is dequantised after this epilogue.
template <int NT>
SS_DEV void tc_wait_acc(const Tc& tc, int k) {
  constexpr int NB = kNbuf<NT>;
  const int b = k % NB;
  mbar_wait_wd(tc.mdone0 + 8 * (2 * b), (uint32_t)((k / NB) & 1));
  mbar_wait_wd(tc.mdone0 + 8 * (2 * b + 1), (uint32_t)((k / NB) & 1));
}
// Before unit k's dequant overwrites A buffer k % kNbuf: unit k - kNbuf's MMAs.
template <int NT>
SS_DEV void tc_wait_buf(const Tc& tc, int k) {
  constexpr int NB = kNbuf<NT>;
  if (k < NB) return;
  const int kp = k - NB, b = kp % NB;
  mbar_wait_wd(tc.mdone0 + 8 * (2 * b), (uint32_t)((kp / NB) & 1));
  mbar_wait_wd(tc.mdone0 + 8 * (2 * b + 1), (uint32_t)((kp / NB) & 1));
}

template <int NT>
SS_DEV void tc_dequant(const Tc& tc, uint32_t sst, int b, int warp, int lane) {
  const int qd = warp & 3, hh = warp >> 2;
  const uint32_t wbase = sst + (uint32_t)(((2 * qd + hh) * 4) * 512 + lane * 16);
  const uint32_t ta = tc.tbase + ((uint32_t)(32 * qd + 16 * hh) << 16) + (uint32_t)(b * 128);
  __syncwarp();  // tcgen05 .sync.aligned: the warp must be converged (lanes leave the ring wait apart)
#pragma unroll
  for (int kb = 0; kb < 4; ++kb) {
    const uint4 w = lds128(wbase + kb * 512);
    uint32_t r[16], af[4];
    const uint32_t wv[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      dequant8(wv[j], af);
      r[4 * j + 0] = af[0];
      r[4 * j + 1] = af[2];
      r[4 * j + 2] = af[1];
      r[4 * j + 3] = af[3];
    }
    tc_st_16x256b_x4(ta + kb * 32, r);
  }
}
// The unit's A operand is complete in TMEM: hand it to the MMA warp.
SS_DEV void tc_signal(const Tc& tc, uint32_t sst, int b, int warp, int lane) {
  tc_wait_st();
  tc_fence_before();
  __syncwarp();
  if (warp == 0 && lane == 0) tc.slot[b] = sst;
  if (lane == 0) mbar_arrive_a(tc.ardy0 + 8 * b);
}

// Two-set variant (T <= 16): warps 4 s .. 4 s + 3 (set s) take every other
// unit; warp (quadrant qd, set s) dequantises BOTH 16-row tiles of its
// quadrant (rows 32 qd .. 32 qd + 31) -- so each unit is handled by one set
// while the other set's dequant / store drain / epilogue overlap it.
SS_DEV void tc_dequant_q(const Tc& tc, uint32_t sst, int b, int qd, int lane) {
  __syncwarp();  // tcgen05 .sync.aligned: the warp must be converged
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const uint32_t wbase = sst + (uint32_t)(((2 * qd + h) * 4) * 512 + lane * 16);
    const uint32_t ta = tc.tbase + ((uint32_t)(32 * qd + 16 * h) << 16) + (uint32_t)(b * 128);
#pragma unroll
    for (int kb = 0; kb < 4; ++kb) {
      const uint4 w = lds128(wbase + kb * 512);
      uint32_t r[16], af[4];
      const uint32_t wv[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        dequant8(wv[j], af);
        r[4 * j + 0] = af[0];
        r[4 * j + 1] = af[2];
        r[4 * j + 2] = af[1];
        r[4 * j + 3] = af[3];
      }
      tc_st_16x256b_x4(ta + kb * 32, r);
    }
  }
}
// The set's 4 warps arrive with count 2 each (ardy count 8); the set's
// quadrant-0 warp publishes the slot address first.
SS_DEV void tc_signal_q(const Tc& tc, uint32_t sst, int b, int qd, int lane) {
  tc_wait_st();
  tc_fence_before();
  __syncwarp();
  if (qd == 0 && lane == 0) tc.slot[b] = sst;
  if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], 2;" ::"r"(tc.ardy0 + 8 * b) : "memory");
}
// Epilogue of unit k for rows 32 qd + lane, both AWQ groups.
template <int NT>
// waited: the set already observed unit k's MMA completion (its tc_wait_buf
// for unit k + 2).  The epilogue must not wait on the buffer's barrier after
// unit k + 2 was handed to the MMA warps: if k + 2's MMAs completed first, the
// barrier's phase parity would read as k's phase still pending (two phases
// later) and the set would wait for unit k + 4, which only it can produce --
// the intermittent deadlock (watchdog trap) of round 2's T = 1 decode steps.
SS_DEV void tc_epilogue_q(const Tc& tc, uint32_t sst, int k, int qd, int lane, float (&y)[8 * NT], bool waited) {
  constexpr int TP = 8 * NT, N = 16 * NT;
  if (!waited) tc_wait_acc<NT>(tc, k);
  __syncwarp();
  tc_fence_after();
  const int m = 32 * qd + lane, tile = m >> 4, r16 = m & 15, g8 = r16 & 7, up = r16 >> 3;
#pragma unroll
  for (int hh = 0; hh < 2; ++hh) {
    const uint32_t zb = lds8(sst + kW4Bytes + 512 + tile * 16 + hh * 8 + g8);
    const uint32_t sp = lds32(sst + kW4Bytes + tile * 64 + hh * 32 + g8 * 4);
    const float sc = up ? __uint_as_float(sp & 0xFFFF0000u) * 0.0625f : __uint_as_float(sp << 16);
    const float cz = up ? 1024.f + 16.f * (float)(zb >> 4) : 1024.f + (float)(zb & 15u);
    float X[TP];
    const uint32_t xo = sst + kW4UnitBytes + NT * 8192 + hh * TP * 4;
#pragma unroll
    for (int t = 0; t < TP; t += 4) {
      const uint4 v = lds128(xo + t * 4);
      X[t] = __uint_as_float(v.x); X[t + 1] = __uint_as_float(v.y);
      X[t + 2] = __uint_as_float(v.z); X[t + 3] = __uint_as_float(v.w);
    }
    const uint32_t ta = tc.tbase + ((uint32_t)(32 * qd) << 16) + kAccColT<NT> + (uint32_t)(((k & (kNacc<NT> - 1)) * 2 + hh) * N);
#pragma unroll
    for (int j = 0; j < (TP + 15) / 16; ++j) {
      uint32_t rh[16], rl[16];
      if constexpr (TP == 8) {
        tc_ld_32x32b_x16(ta, rh);
      } else {
        tc_ld_32x32b_x16(ta + 16 * j, rh);
        tc_ld_32x32b_x16(ta + TP + 16 * j, rl);
      }
      tc_wait_ld();
#pragma unroll
      for (int t = 0; t < (TP == 8 ? 8 : 16); ++t) {
        const float hi = __uint_as_float(rh[t]), lo = __uint_as_float(TP == 8 ? rh[8 + t] : rl[t]);
        y[16 * j + t] = fmaf(sc, fmaf(-cz, X[16 * j + t], hi + lo), y[16 * j + t]);
      }
    }
  }
  tc_fence_before();
}

template <int NT>
SS_DEV void tc_epilogue(const Tc& tc, uint32_t sst, int k, int warp, int lane, float (&y)[8 * NT]) {
  constexpr int TP = 8 * NT, N = 16 * NT;
  const int qd = warp & 3, hh = warp >> 2;
  // both groups' MMAs (two issuers; the same completion also frees the A
  // buffer this warp's next-but-one dequant overwrites)
  tc_wait_acc<NT>(tc, k);
  __syncwarp();
  tc_fence_after();
  // metadata of row m = 32 qd + lane (tile m / 16, fragment row m % 16) in group hh
  const int m = 32 * qd + lane, tile = m >> 4, r16 = m & 15, g8 = r16 & 7, up = r16 >> 3;
  const uint32_t zb = lds8(sst + kW4Bytes + 512 + tile * 16 + hh * 8 + g8);
  const uint32_t sp = lds32(sst + kW4Bytes + tile * 64 + hh * 32 + g8 * 4);
  const float sc = up ? __uint_as_float(sp & 0xFFFF0000u) * 0.0625f : __uint_as_float(sp << 16);
  const float cz = up ? 1024.f + 16.f * (float)(zb >> 4) : 1024.f + (float)(zb & 15u);
  float X[TP];
  const uint32_t xo = sst + kW4UnitBytes + NT * 8192 + hh * TP * 4;
#pragma unroll
  for (int t = 0; t < TP; t += 4) {
    const uint4 v = lds128(xo + t * 4);
    X[t] = __uint_as_float(v.x); X[t + 1] = __uint_as_float(v.y);
    X[t + 2] = __uint_as_float(v.z); X[t + 3] = __uint_as_float(v.w);
  }
  const uint32_t ta = tc.tbase + ((uint32_t)(32 * qd) << 16) + kAccColT<NT> + (uint32_t)(((k & (kNacc<NT> - 1)) * 2 + hh) * N);
  if constexpr (TP == 8) {
    uint32_t r[16];
    tc_ld_32x32b_x16(ta, r);
    tc_wait_ld();
#pragma unroll
    for (int t = 0; t < 8; ++t)
      y[t] = fmaf(sc, fmaf(-cz, X[t], __uint_as_float(r[t]) + __uint_as_float(r[8 + t])), y[t]);
  } else {
#pragma unroll
    for (int j = 0; j < TP / 16; ++j) {
      uint32_t rh[16], rl[16];
      tc_ld_32x32b_x16(ta + 16 * j, rh);
      tc_ld_32x32b_x16(ta + TP + 16 * j, rl);
      tc_wait_ld();
#pragma unroll
      for (int t = 0; t < 16; ++t)
        y[16 * j + t] = fmaf(sc, fmaf(-cz, X[16 * j + t], __uint_as_float(rh[t]) + __uint_as_float(rl[t])), y[16 * j + t]);
    }
  }
  tc_fence_before();  // the TMEM reads before the next MMA into this accumulator
}

// The MMA warps (one per AWQ group g of the unit: a single issuing thread
// sustains only one 128 x N x 16 MMA per ~70 cycles): for every W4 unit of the
// CTA (in the consumers' order), wait for its A operand, issue the group's
// 8 MMAs (K 16 each; the first overwrites the accumulator), commit to
// mdone[b][g].  Stop on slot == 0.
template <int NT>
__device__ __noinline__ void mma_warp(const StepArgs* __restrict__ ap, Tc tc, int g) {
  const StepArgs& a = *ap;
  constexpr int N = 16 * NT;
  constexpr uint32_t idesc = idesc_f16(128, N);
  for (int k = 0;; ++k) {
    const int b = k % kNbuf<NT>;
    where(a, WCODE(k & 0xFFFF, 0x20, 1));
    mbar_wait_wd(tc.ardy0 + 8 * b, (uint32_t)((k / kNbuf<NT>) & 1));
    if (g == 0 && a.utl && blockIdx.x == 0 && lane_id() == 0 && k < 4096) a.utl[4096 + k * 2] = clk64();
    __syncwarp();
    const uint32_t sst = *reinterpret_cast<volatile uint32_t*>(tc.slot + b);
    if (sst == 0) break;
    tc_fence_after();
    const uint64_t bd0 = smem_desc(sst + kW4UnitBytes, N * 16, 128);
    {
      const uint32_t d = tc.tbase + kAccColT<NT> + (uint32_t)(((k & (kNacc<NT> - 1)) * 2 + g) * N);
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        const int i = g * 8 + ks;
        const uint32_t at = tc.tbase + (uint32_t)(b * 128 + i * 8);
        const uint64_t bd = bd0 + (uint64_t)((i * 2 * N * 16) >> 4);
        asm volatile(
            "{\n\t.reg .pred p, e;\n\t"
            "elect.sync _|e, 0xffffffff;\n\t"
            "setp.ne.b32 p, %4, 0;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
            "r"(at), "l"(bd), "r"(idesc), "r"(ks))
            ;
      }
    }
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}"
        ::"r"(tc.mdone0 + 8 * (2 * b + g))
        : "memory");
    if (g == 0 && a.utl && blockIdx.x == 0 && lane_id() == 0 && k < 4096) a.utl[4096 + k * 2 + 1] = clk64();
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
// Tile-group tails are chains of dependent global accesses, so each first
// stages what it reads -- the tile-group's fp32 accumulator block, the
// per-token norm scales / positions -- into shared memory (the attention q
// area, idle during GEMM phases) with all loads in flight at once, then
// computes from shared memory.  New residual rows also stay there for the
// next GEMM's input.
SS_DEV float norm_scale(const float* ss, int t, int h, float eps) { return rsqrtf(__ldcg(ss + t) / (float)h + eps); }
// Deterministic mode (SS_DEBUG_DETERMINISTIC): the per-tile-group partial sums
// of squares are added as 2^-24 fixed point in 64-bit integers (exact, any
// order); the float entry holds only single-writer sums (the ingest kernel's).
constexpr double kSsFx = 16777216.0;
SS_DEV float norm_scale_a(const StepArgs& a, const float* ss, int t) {
  float v = __ldcg(ss + t);
  if (a.det) v += (float)((double)__ldcg(a.ssx + (ss - a.ss) + t) * (1.0 / kSsFx));
  return rsqrtf(v / (float)a.h + a.eps);
}

template <int NT>
struct TailSm {
  float* acc;  // [128][8 NT] accumulator block of the tile-group
  float* xn;   // [8 NT][128] new residual rows of the tile-group
  float* rs;   // [8 NT] per-token scale
  int* pos;    // [8 NT] positions
};
template <int NT>
SS_DEV TailSm<NT> tail_sm(uint8_t* base) {
  constexpr int TP = 8 * NT;
  TailSm<NT> t;
  t.acc = reinterpret_cast<float*>(base);
  t.xn = t.acc + 128 * TP;
  t.rs = t.xn + 128 * TP;
  t.pos = reinterpret_cast<int*>(t.rs + TP);
  return t;
}
// acc block (128 x 8 NT fp32) -> shared memory; caller synchronises
template <int NT>
SS_DEV void stage_acc(const float* acc, float* sm) {
  const float4* src = reinterpret_cast<const float4*>(acc);
  float4* dst = reinterpret_cast<float4*>(sm);
  float4 v[NT];
#pragma unroll
  for (int i = 0; i < NT; ++i) v[i] = __ldcg(src + threadIdx.x + i * 256);
#pragma unroll
  for (int i = 0; i < NT; ++i) dst[threadIdx.x + i * 256] = v[i];
}

SS_DEV uint32_t q_frag_index(int m, int j, int d, int rbmax, int kvh) {
  const int rb = m >> 4, r = m & 15, kk = j >> 4, c = j & 15;
  const int lane = ((r & 7) << 2) | ((c & 7) >> 1);
  const int reg = (r >> 3) + 2 * (c >> 3);
  return ((((uint32_t)kvh * rbmax + rb) * (d / 16) + kk) * 32 + lane) * 8 + reg * 2 + (c & 1);
}

// a4: deferred attn-norm scale, RoPE (R2), q hi/lo in fragment order,
// tree K/V rows: fp16 hi into the cache at L + t (R10), lo into the window.
template <int NT>
SS_DEV void epi_qkv(const StepArgs& a, int layer, int tg, const float* acc, const Sched& s, const TailSm<NT>& ts) {
  constexpr int TP = NT * 8, IT = 128 * TP / 256;
  const int T = s.T, L = s.L, d = a.d, half = d >> 1;
  const int R = L + s.T0;  // row of slot 0 (a non-square forward appends after the cached tree rows)
  const int nq = a.Hq_l * d, nk = a.Hkv_l * d;
  const float* ssa = a.ss + (size_t)layer * 2 * 64;
  const int wb = L & ~63;
  const int rbmax = 4 * a.G;
  const size_t qlo = (size_t)a.Hkv_l * rbmax * (d / 16) * 32 * 8;
  stage_acc<NT>(acc, ts.acc);
  if (threadIdx.x < T) {
    ts.rs[threadIdx.x] = norm_scale_a(a, ssa, threadIdx.x);
    ts.pos[threadIdx.x] = a.st->pos[s.T0 + threadIdx.x];
  }
  cbar();
  // each thread: a pair of adjacent rows (features j, j + 1 of one head) of one
  // token, so every q-fragment / cache store writes both halves at once
  constexpr int IT2 = IT / 2;
  float4 cs[IT2];
#pragma unroll
  for (int i = 0; i < IT2; ++i) {  // RoPE table entries first (independent loads)
    const int idx = threadIdx.x + i * 256, r = 2 * (idx / TP), t = idx % TP;
    const int row = tg * 128 + r, j = row % d;
    cs[i] = (t < T && row < nq + nk)
                ? __ldg(reinterpret_cast<const float4*>(&a.rope_cs[(size_t)ts.pos[t] * half + (j % half)]))
                : make_float4(1.f, 0.f, 1.f, 0.f);
  }
#pragma unroll
  for (int i = 0; i < IT2; ++i) {
    const int idx = threadIdx.x + i * 256, r = 2 * (idx / TP), t = idx % TP;
    if (t >= T) continue;
    const int row = tg * 128 + r, j = row % d;
    const float rs = ts.rs[t];
    float x0 = ts.acc[r * TP + t] * rs, x1 = ts.acc[(r + 1) * TP + t] * rs;
    if (row < nq + nk) {
      const int pr = (j < half) ? r + half : r - half;
      const float p0 = ts.acc[pr * TP + t] * rs, p1 = ts.acc[(pr + 1) * TP + t] * rs;
      if (j < half) {
        x0 = x0 * cs[i].x - p0 * cs[i].y;
        x1 = x1 * cs[i].z - p1 * cs[i].w;
      } else {
        x0 = x0 * cs[i].x + p0 * cs[i].y;
        x1 = x1 * cs[i].z + p1 * cs[i].w;
      }
    }
    uint32_t hi, lo2;
    split16(x0, x1, hi, lo2);
    if (row < nq) {
      const int hq = row / d, kvh = hq / a.G, jj = hq - kvh * a.G;
      const uint32_t fi = q_frag_index(t * a.G + jj, j, d, rbmax, kvh);  // j even: j + 1 at fi + 1
      *reinterpret_cast<uint32_t*>(a.qf + fi) = hi;
      *reinterpret_cast<uint32_t*>(a.qf + qlo + fi) = lo2;
    } else if (row < nq + 2 * nk) {
      const bool isk = row < nq + nk;
      const int kvh = (isk ? row - nq : row - nq - nk) / d;
      uint16_t* c = isk ? a.kc : a.vc;
      uint16_t* lo = isk ? a.klo : a.vlo;
      const size_t base = ((size_t)layer * a.Hkv_l + kvh) * a.max_ctx_pad * d;
      *reinterpret_cast<uint32_t*>(c + base + kv_elem_offset(R + t, j, d)) = hi;
      *reinterpret_cast<uint32_t*>(lo + (size_t)kvh * 128 * d + kv_elem_offset(R + t - wb, j, d)) = lo2;
    }
  }
  // zero the lo window rows outside this step's new rows of this tile-group's
  // K / V heads (a tree tile's prefix rows -- and the cached tree rows of a
  // non-square forward, fp16 like committed rows -- add q . 0).  The window is
  // per kv head, shared by the layers, and every layer of a step writes the
  // same rows [R, R + T): only the first layer has to clear the rest.
  const int row0 = tg * 128;
  if (layer == 0 && row0 + 127 >= nq && row0 < nq + 2 * nk) {
    for (int hd = 0; hd < 128 / d; ++hd) {
      const int row = row0 + hd * d;
      if (row < nq || row >= nq + 2 * nk) continue;
      const bool isk = row < nq + nk;
      const int kvh = (isk ? row - nq : row - nq - nk) / d;
      uint16_t* lo = (isk ? a.klo : a.vlo) + (size_t)kvh * 128 * d;
      for (int i = threadIdx.x; i < 128 * d / 8; i += 256) {
        const int w = i / (d / 8);
        const int pos = wb + w;
        if (pos >= R && pos < R + T) continue;
        *reinterpret_cast<uint4*>(lo + (size_t)w * d + (i % (d / 8)) * 8) = make_uint4(0, 0, 0, 0);
      }
    }
  }
}

// a8: deferred mlp-norm scale + SwiGLU (R4) -> down input (hi/lo, X)
template <int NT>
SS_DEV void epi_swiglu(const StepArgs& a, int layer, int tg, const float* acc, int T, const TailSm<NT>& ts) {
  const int TP = NT * 8;
  const float* ssm = a.ss + (size_t)layer * 2 * 64 + 64;
  const int warp = threadIdx.x >> 5, cp = threadIdx.x & 31;
  if constexpr (NT != 1) {  // several tokens per warp: stage the block once
    stage_acc<NT>(acc, ts.acc);
    if (threadIdx.x < T) ts.rs[threadIdx.x] = norm_scale_a(a, ssm, threadIdx.x);
    cbar();
  }
  for (int t = warp; t < T; t += 8) {
    float g0, g1, u0, u1;
    if constexpr (NT == 1) {
      // one token per warp: its sums straight from the split-K accumulator
      // with the token's norm scale, one round trip, no shared staging
      const float a0 = __ldcg(acc + (2 * cp) * TP + t), a1 = __ldcg(acc + (2 * cp + 1) * TP + t);
      const float a2 = __ldcg(acc + (64 + 2 * cp) * TP + t), a3 = __ldcg(acc + (64 + 2 * cp + 1) * TP + t);
      const float rs = norm_scale_a(a, ssm, t);
      g0 = a0 * rs; g1 = a1 * rs; u0 = a2 * rs; u1 = a3 * rs;
    } else {
      const float rs = ts.rs[t];
      g0 = ts.acc[(2 * cp) * TP + t] * rs;
      g1 = ts.acc[(2 * cp + 1) * TP + t] * rs;
      u0 = ts.acc[(64 + 2 * cp) * TP + t] * rs;
      u1 = ts.acc[(64 + 2 * cp + 1) * TP + t] * rs;
    }
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

// TP > 1: this rank's fp32 partial of tile-group tg (staged in shared memory)
// to every peer as LL lines (data1, flag1, data2, flag2, R15).
template <int NT>
SS_DEV void ar_send(const StepArgs& a, int tg, int T, int ar_seq, const TailSm<NT>& ts) {
  const int TP = NT * 8;
  const uint32_t flag = a.st->epoch + ar_seq;
  const int pairs = (T + 1) >> 1;
  const int ntg = a.h / 128;
  // two-shot: only the tile-group's home rank receives the partials.
  // Loopback emulation (one rank, rank 0, standing in for its peers): a home
  // tile-group receives P stand-in partials as in one-shot; a non-home one
  // stores its partial once (the remote store) and writes the home's
  // broadcast line itself (no wait for a real home).
  const int home = tg % a.P;
  const bool two = a.ar_mode == 1;
  const int p0 = two && !(a.loopback && home == a.rank) ? home : 0;
  const int p1 = two && !(a.loopback && home == a.rank) ? home + 1 : a.P;
  const size_t bl0 = a.bc_line0 + ((size_t)(ar_seq & 1) * ntg + tg) * 128 * (4 * NT);
  for (int idx = threadIdx.x; idx < 128 * pairs; idx += 256) {
    const int r = idx / pairs, tp = idx - r * pairs;
    const float2 v = *reinterpret_cast<const float2*>(ts.acc + r * TP + 2 * tp);
    if (two && a.loopback && home != a.rank)
      ll_store(reinterpret_cast<uint4*>(a.recv) + bl0 + (size_t)r * (4 * NT) + tp, __float_as_uint(v.x),
               __float_as_uint(v.y), flag);
    for (int p = p0; p < p1; ++p) {
      const int slot = (a.loopback && !(two && home != a.rank)) ? p : a.rank;
      const size_t line = (((size_t)(ar_seq & 1) * a.P + slot) * ntg + tg) * 128 * (4 * NT) + (size_t)r * (4 * NT) + tp;
      ll_store(reinterpret_cast<uint4*>(a.peer_recv[p]) + line, __float_as_uint(v.x), __float_as_uint(v.y), flag);
    }
  }
}

// Residual update of tile-group tg: x += acc (P == 1) or the rank-ordered sum
// of every rank's partial (TP all-reduce receive); the new rows also go to
// ts.xn for the next GEMM's input.
template <int NT>
SS_DEV void resid_update(const StepArgs& a, int tg, int T, int ar_seq, const TailSm<NT>& ts,
                         const float* accg = nullptr) {
  constexpr int TP = NT * 8;
  if (a.P == 1) {
    // the tile-group's sums straight from the split-K accumulator (no shared
    // staging): old residual and sums requested together, one round trip
    constexpr int IT = 128 * TP / 256;
    float xo[IT], ao[IT];
#pragma unroll
    for (int i = 0; i < IT; ++i) {
      const int idx = threadIdx.x + i * 256, t = idx >> 7, r = idx & 127;
      xo[i] = t < T ? __ldcg(a.x + (size_t)t * a.h + tg * 128 + r) : 0.f;
      ao[i] = t < T ? __ldcg(accg + r * TP + t) : 0.f;
    }
#pragma unroll
    for (int i = 0; i < IT; ++i) {
      const int idx = threadIdx.x + i * 256, t = idx >> 7, r = idx & 127;
      if (t < T) {
        const float v = xo[i] + ao[i];
        a.x[(size_t)t * a.h + tg * 128 + r] = v;
        ts.xn[t * 128 + r] = v;
      }
    }
    return;
  }
  constexpr int PP = 4 * NT;
  const uint32_t flag = a.st->epoch + ar_seq;
  const int pairs = (T + 1) >> 1;
  const int ntg = a.h / 128;
  const size_t pstride = (size_t)ntg * 128 * PP;
  const uint4* src0 = reinterpret_cast<const uint4*>(a.recv) + (((size_t)(ar_seq & 1) * a.P) * ntg + tg) * 128 * PP;
  for (int idx = threadIdx.x; idx < 128 * pairs; idx += 256) {
    const int tp = idx >> 7, r = idx & 127;
    const int t0 = 2 * tp;
    const uint4* src = src0 + (size_t)r * PP + tp;
    // the old residual values and every rank's line are requested together
    const float x0 = __ldcg(a.x + (size_t)t0 * a.h + tg * 128 + r);
    const float x1 = t0 + 1 < T ? __ldcg(a.x + (size_t)(t0 + 1) * a.h + tg * 128 + r) : 0.f;
    uint32_t d1[kMaxPeers], d2[kMaxPeers];
    unsigned ready = 0;
    const unsigned all = (1u << a.P) - 1u;
    unsigned spins = 0;
    unsigned long long tw = 0;
    while (ready != all) {
#pragma unroll
      for (int p = 0; p < kMaxPeers; ++p)
        if (p < a.P && !(ready & (1u << p)) && ll_try_load(src + p * pstride, flag, d1[p], d2[p])) ready |= 1u << p;
      if (ready != all && (++spins & 255u) == 0) {  // bounded: 2 s per line, or at once after another timeout
        if (!tw) tw = now_ns();
        if (now_ns() - tw > 2000000000ull || *reinterpret_cast<volatile int*>(&a.st->timeout)) {
          a.st->timeout = 1;
          break;
        }
      }
    }
    float s0 = 0.f, s1 = 0.f;
#pragma unroll
    for (int p = 0; p < kMaxPeers; ++p)
      if (p < a.P) {
        s0 += __uint_as_float(d1[p]);
        s1 += __uint_as_float(d2[p]);
      }
    if (a.ar_mode == 1) {
      // two-shot, home rank: broadcast the rank-ordered sum (every rank adds
      // it to the same residual: bit-identical rows on all ranks)
      const size_t bl = a.bc_line0 + ((size_t)(ar_seq & 1) * ntg + tg) * 128 * PP + (size_t)r * PP + tp;
      for (int p = 0; p < a.P; ++p)
        if (p != a.rank)  // loopback: peer_recv[p] is this rank's own buffer (stand-in stores)
          ll_store(reinterpret_cast<uint4*>(a.peer_recv[p]) + bl, __float_as_uint(s0), __float_as_uint(s1), flag);
    }
    float* xp = a.x + (size_t)t0 * a.h + tg * 128 + r;
    *xp = x0 + s0;
    ts.xn[t0 * 128 + r] = x0 + s0;
    if (t0 + 1 < T) {
      xp[a.h] = x1 + s1;
      ts.xn[(t0 + 1) * 128 + r] = x1 + s1;
    }
  }
}

// Two-shot all-reduce, a rank that is not tile-group tg's home: the home's
// broadcast of the rank-ordered sum, added to the residual.
template <int NT>
SS_DEV void resid_update_bcast(const StepArgs& a, int tg, int T, int ar_seq, const TailSm<NT>& ts) {
  constexpr int PP = 4 * NT;
  const uint32_t flag = a.st->epoch + ar_seq;
  const int pairs = (T + 1) >> 1;
  const int ntg = a.h / 128;
  const uint4* src0 = reinterpret_cast<const uint4*>(a.recv) + a.bc_line0 + ((size_t)(ar_seq & 1) * ntg + tg) * 128 * PP;
  for (int idx = threadIdx.x; idx < 128 * pairs; idx += 256) {
    const int tp = idx >> 7, r = idx & 127;
    const int t0 = 2 * tp;
    const float x0 = __ldcg(a.x + (size_t)t0 * a.h + tg * 128 + r);
    const float x1 = t0 + 1 < T ? __ldcg(a.x + (size_t)(t0 + 1) * a.h + tg * 128 + r) : 0.f;
    uint32_t d1 = 0, d2 = 0;
    unsigned spins = 0;
    unsigned long long tw = 0;
    while (!ll_try_load(src0 + (size_t)r * PP + tp, flag, d1, d2)) {
      if ((++spins & 255u) == 0) {
        if (!tw) tw = now_ns();
        if (now_ns() - tw > 2000000000ull || *reinterpret_cast<volatile int*>(&a.st->timeout)) {
          a.st->timeout = 1;
          break;
        }
      }
    }
    const float s0 = __uint_as_float(d1), s1 = __uint_as_float(d2);
    float* xp = a.x + (size_t)t0 * a.h + tg * 128 + r;
    *xp = x0 + s0;
    ts.xn[t0 * 128 + r] = x0 + s0;
    if (t0 + 1 < T) {
      xp[a.h] = x1 + s1;
      ts.xn[(t0 + 1) * 128 + r] = x1 + s1;
    }
  }
}

// After the residual of tile-group tg is final (its rows in ts.xn): the next
// GEMM's input for its 128 columns (x * g, fp16 hi/lo + X; or bf16 hi/lo for
// the LM head) and the token's sum of squares (the deferred RMSNorm scale, R5).
template <int NT>
SS_DEV void next_input(const StepArgs& a, int tg, int T, uint2 gw, float* ss, uint8_t* act, int lm,
                       const TailSm<NT>& ts) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int k = tg * 128 + lane * 4;
  for (int t = warp; t < T; t += 8) {
    const float4 v = *reinterpret_cast<const float4*>(ts.xn + t * 128 + lane * 4);
    const float q = warp_sum(v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w);
    if (lane == 0) {
      if (a.det) atomicAdd(a.ssx + (ss - a.ss) + t, __double2ull_rn((double)q * kSsFx));
      else atomicAdd(ss + t, q);
    }
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
SS_DEV void epi_argmax(const StepArgs& a, int tg, const float* acc, int T, const TailSm<NT>& ts) {
  const int TP = NT * 8;
  const float* ssf = a.ss + (size_t)a.n_layers * 2 * 64;
  (void)ts;
  const int r = threadIdx.x & 127;
  const int v = tg * 128 + r;
  const bool valid = v < a.V_l;
  constexpr int NI = NT * 4;  // tokens per thread (t = threadIdx.x / 128 + 2 i)
  float av[NI], rv[NI];
#pragma unroll
  for (int i = 0; i < NI; ++i) {  // sums and norm scales straight from global, all requested first
    const int t = (threadIdx.x >> 7) + 2 * i;
    if (t < T) {
      av[i] = __ldcg(acc + r * TP + t);
      rv[i] = norm_scale_a(a, ssf, t);
    }
  }
#pragma unroll
  for (int i = 0; i < NI; ++i) {
    const int t = (threadIdx.x >> 7) + 2 * i;
    if (t >= T) continue;
    const float val = valid ? av[i] * rv[i] : -INFINITY;
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
__device__ __noinline__ int2 gemm_phase(const StepArgs* __restrict__ ap, const Sched* __restrict__ sp, int layer,
                                        int u0, int u1, Ring ring, Tc tc, int tck, int* s_done, int* s_nd,
                                        uint8_t* s_tail) {
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
  const int tslot = PH == PH_LM ? a.n_layers * 5 : layer * 5 + PH;
  tmark(a, tslot, 0);
  where(a, WCODE(layer, PH, 1));
  if constexpr (PH == PH_LM) {
    float acc[NT][4];
#pragma unroll
    for (int n = 0; n < NT; ++n) acc[n][0] = acc[n][1] = acc[n][2] = acc[n][3] = 0.f;
    for (int u = u0; u < u1; ++u) {
      const uint32_t sst = ring_wait<NT>(ring);
      if (u == u0) tmark(a, tslot, 1);
      lm_unit<NT>(sst, warp, lane, acc);
      ring_release<NT>(ring);
      const int tg = u / S;
      if (u + 1 == u1 || (u + 1) / S != tg) {  // flush this tile-group's partial
        float* base = accb + ((size_t)tg * 128 + warp * 16 + gq) * TP;
#pragma unroll
        for (int n = 0; n < NT; ++n) {
          red_add_v2(base + n * 8 + 2 * tq, acc[n][0], acc[n][1]);
          red_add_v2(base + 8 * TP + n * 8 + 2 * tq, acc[n][2], acc[n][3]);
          acc[n][0] = acc[n][1] = acc[n][2] = acc[n][3] = 0.f;
        }
      }
    }
  } else if constexpr (NT <= 2) {
    // two warp sets on alternating units, in lockstep pairs (p, p + 1): set s
    // dequantises unit p + s, runs the epilogue of its previous unit, hands the
    // new one to the MMA warps; after a barrier every warp releases the
    // previous pair's ring slots (once each: empty count 8)
    float y[8 * NT];
#pragma unroll
    for (int t = 0; t < 8 * NT; ++t) y[t] = 0.f;
    const int k0 = ring.k;
    const int ws = warp >> 2, qd = warp & 3;
    unsigned long long* utl =
        (a.utl && PH == PH_GU && layer == a.n_layers / 2 && blockIdx.x == 0 && (threadIdx.x & 127) == 0) ? a.utl
                                                                                                        : nullptr;
    if (utl && threadIdx.x == 0) { utl[127 * 8 + 7] = (unsigned long long)tck; utl[127 * 8 + 6] = (unsigned long long)(u1 - u0); }
    uint32_t sst_prev = 0;
    int u_prev = -1;
    auto release_pair = [&](int q0) {
      __syncwarp();
      if (lane == 0)
        for (int v = q0; v < q0 + 2 && v < u1; ++v) mbar_arrive_a(ring.empty0 + 8 * ((k0 + v - u0) % StepCfg<NT>::STAGES));
    };
    auto flush_prev = [&](int v) {
      const int tg = v / S;
      if (v + 2 >= u1 || (v + 2) / S != tg) {  // this set's next unit starts another tile-group
        float* row = accb + ((size_t)tg * 128 + 32 * qd + lane) * TP;
#pragma unroll
        for (int t = 0; t < 8 * NT; t += 4) {
          red_add_v4(row + t, y[t], y[t + 1], y[t + 2], y[t + 3]);
          y[t] = y[t + 1] = y[t + 2] = y[t + 3] = 0.f;
        }
      }
    };
    for (int p = u0; p < u1; p += 2) {
      const int um = p + ws;
      const bool have = um < u1;
      uint32_t sst = 0;
      // the A buffer's previous user (unit k - kNbuf) must have finished its
      // MMAs before the dequant below overwrites it
      if (have) tc_wait_buf<NT>(tc, tck + (um - u0));
      if (have) {
        if (utl && um - u0 < 127) utl[(um - u0) * 8 + 0] = clk64();
        sst = ring_wait_at<NT>(ring, k0 + (um - u0));
        if (utl && um - u0 < 127) utl[(um - u0) * 8 + 1] = clk64();
        if (p == u0) tmark(a, tslot, 1);
        tc_dequant_q(tc, sst, (tck + (um - u0)) % kNbuf<NT>, qd, lane);
        if (utl && um - u0 < 127) utl[(um - u0) * 8 + 2] = clk64();
      }
      // hand the new unit to the MMA warps first: its MMAs then run during
      // the previous unit's epilogue and are done before this set's next dequant
      if (have) tc_signal_q(tc, sst, (tck + (um - u0)) % kNbuf<NT>, qd, lane);
      if (u_prev >= 0) {
        where(a, WCODE(layer, PH, 3));
        // have: tc_wait_buf above waited for exactly u_prev's MMAs (unit k - 2)
        tc_epilogue_q<NT>(tc, sst_prev, tck + (u_prev - u0), qd, lane, y, have);
        if (utl && u_prev - u0 < 127) utl[(u_prev - u0) * 8 + 3] = clk64();
        flush_prev(u_prev);
      }
      cbar();
      if (p > u0) release_pair(p - 2);
      u_prev = have ? um : -1;
      sst_prev = sst;
    }
    if (u_prev >= 0) {
      tc_epilogue_q<NT>(tc, sst_prev, tck + (u_prev - u0), qd, lane, y, false);
      if (utl && u_prev - u0 < 127) utl[(u_prev - u0) * 8 + 3] = clk64();
      flush_prev(u_prev);
    }
    if (u1 > u0) {
      cbar();
      release_pair(u0 + ((u1 - 1 - u0) & ~1));
    }
    ring.k = k0 + (u1 - u0);
    tck += u1 - u0;
  } else {
    // software pipeline: dequant unit u into TMEM buffer (tck + u - u0) & 1
    // while the MMAs of unit u - 1 run, then its epilogue; flush per tile-group
    float y[8 * NT];
#pragma unroll
    for (int t = 0; t < 8 * NT; ++t) y[t] = 0.f;
    const int k0 = ring.k;
    uint32_t prev = 0;
    unsigned long long* utl =
        (a.utl && PH == PH_GU && layer == a.n_layers / 2 && blockIdx.x == 0 && threadIdx.x == 0) ? a.utl : nullptr;
    if (utl) { utl[127 * 8 + 7] = (unsigned long long)tck; utl[127 * 8 + 6] = (unsigned long long)(u1 - u0); }
    // per iteration: the TMEM stores of unit u are issued, then the epilogue of
    // unit u - 1 runs while they drain, then unit u is handed to the MMA warp
    for (int u = u0; u <= u1; ++u) {
      uint32_t sst = 0;
      if (u < u1) {
        if (utl && u - u0 < 127) utl[(u - u0) * 8 + 0] = clk64();
        sst = ring_wait_at<NT>(ring, k0 + (u - u0));
        if (utl && u - u0 < 127) utl[(u - u0) * 8 + 1] = clk64();
        if (u == u0) tmark(a, tslot, 1);
        tc_wait_buf<NT>(tc, tck + (u - u0));  // satisfied: the epilogue of unit u - 2 waited on the same MMAs
        tc_dequant<NT>(tc, sst, (tck + (u - u0)) % kNbuf<NT>, warp, lane);
        if (utl && u - u0 < 127) utl[(u - u0) * 8 + 2] = clk64();
      }
      if (u > u0) {
        const int v = u - 1;
        where(a, WCODE(layer, PH, 3));
        tc_epilogue<NT>(tc, prev, tck + (v - u0), warp, lane, y);
        if (utl && v - u0 < 127) utl[(v - u0) * 8 + 3] = clk64();
      }
      if (u < u1) tc_signal(tc, sst, (tck + (u - u0)) % kNbuf<NT>, warp, lane);
      if (u > u0) {
        const int v = u - 1;
        ring_release_at<NT>(ring, k0 + (v - u0));
        const int tg = v / S;
        if (v + 1 == u1 || (v + 1) / S != tg) {  // flush: row 32 qd + lane, group half of the warp
          float* row = accb + ((size_t)tg * 128 + 32 * (warp & 3) + lane) * TP;
#pragma unroll
          for (int t = 0; t < 8 * NT; t += 4) {
            red_add_v4(row + t, y[t], y[t + 1], y[t + 2], y[t + 3]);
            y[t] = y[t + 1] = y[t + 2] = y[t + 3] = 0.f;
          }
        }
      }
      prev = sst;
    }
    ring.k = k0 + (u1 - u0);
    tck += u1 - u0;
  }
  where(a, WCODE(layer, PH, 4));
  // arrivals: the barrier orders every warp's reductions before thread 0's
  // GPU-scope fence (cumulative) and arrival counts
  const unsigned long long tl0 = clk64();
  cbar();
  if (threadIdx.x == 0) {
    int nd = 0;
    if (u1 > u0) {
      for (int tg = u0 / S; tg <= (u1 - 1) / S; ++tg) {
        const int nst = min(u1, (tg + 1) * S) - max(u0, tg * S);
        // release: this CTA's partials; acquire (last arriver): the others'
        if (atom_add_acqrel_gpu(&arr[tg], nst) + nst == S) s_done[nd++] = tg;
      }
    }
    *s_nd = nd;
  }
  __syncwarp();
  cbar();
  const int nd = *s_nd;
  // tail timeline (trace mode): the finaliser of tile-group 0, middle layer
  unsigned long long* ttl = (a.utl && PH != PH_LM && layer == a.n_layers / 2 && nd > 0 && s_done[0] == 0 &&
                             threadIdx.x == 0) ? a.utl + 30000 + PH * 16 : nullptr;
  if (ttl) { ttl[0] = tl0; ttl[1] = clk64(); ttl[8] = (unsigned long long)nd; }
  if (nd == 0) {
    tmark(a, tslot, 2);
    return make_int2(ring.k, tck);
  }
  int* ctr = a.ctr + (size_t)layer * kCtrPerLayer;
  const TailSm<NT> ts = tail_sm<NT>(s_tail);
  if constexpr (PH == PH_QKV || PH == PH_GU || PH == PH_LM) {
    for (int i = 0; i < nd; ++i) {
      const int tg = s_done[i];
      const float* accp = accb + (size_t)tg * 128 * TP;
      if constexpr (PH == PH_QKV) epi_qkv<NT>(a, layer, tg, accp, s, ts);
      else if constexpr (PH == PH_GU) epi_swiglu<NT>(a, layer, tg, accp, T, ts);
      else epi_argmax<NT>(a, tg, accp, T, ts);
      cbar();  // shared staging reused by the next tile-group
    }
  } else {
    // residual phases: sends of every completed tile-group first, then the
    // receives (no rank waits on a tile-group it has not sent yet)
    const int ar_seq = 2 * layer + (PH == PH_DN ? 1 : 0);
    where(a, WCODE(layer, PH, 6));
    if (a.P > 1)
      for (int i = 0; i < nd; ++i) {
        stage_acc<NT>(accb + (size_t)s_done[i] * 128 * TP, ts.acc);
        cbar();
        ar_send<NT>(a, s_done[i], T, ar_seq, ts);
        cbar();
      }
    if (ttl) ttl[2] = clk64();
    where(a, WCODE(layer, PH, 7));
    const bool last = PH == PH_DN && layer + 1 == a.n_layers;
    const uint16_t* gain = PH == PH_O ? a.layers[layer].mlp_norm
                                      : (last ? a.final_norm : a.layers[layer + 1].attn_norm);
    float* ssn = a.ss + (size_t)(PH == PH_O ? layer * 2 + 1 : (layer + 1) * 2) * 64;
    uint8_t* act = last ? a.act_lm : a.act_h;
    // two-shot: the tile-groups this rank is home of first (their sums are
    // what the other ranks wait for; homes wait only on the sends above)
    const bool two = a.ar_mode == 1 && a.P > 1;
    for (int pass = 0; pass < (two ? 2 : 1); ++pass)
      for (int i = 0; i < nd; ++i) {
        const bool home = !two || s_done[i] % a.P == a.rank;
        if (two && home != (pass == 0)) continue;
        // the next norm's gains for this tile-group's 128 columns, requested
        // before the residual's round trips
        const uint2 gw = __ldg(reinterpret_cast<const uint2*>(gain + s_done[i] * 128 + (threadIdx.x & 31) * 4));
        if (home) resid_update<NT>(a, s_done[i], T, ar_seq, ts, accb + (size_t)s_done[i] * 128 * TP);
        else resid_update_bcast<NT>(a, s_done[i], T, ar_seq, ts);
        cbar();
        if (ttl && i == 0) ttl[3] = clk64();
        next_input<NT>(a, s_done[i], T, gw, ssn, act, last ? 1 : 0, ts);
        cbar();
      }
    where(a, WCODE(layer, PH, 8));
    if constexpr (PH == PH_O) {
      // zero the down input's X slots (the SwiGLU epilogues of this layer add into them)
      const int ngrp = a.I_l / 128;
      for (int i = 0; i < nd; ++i)
        for (int g = s_done[i]; g < ngrp; g += a.o_tg)
          for (int t = threadIdx.x; t < 8 * NT; t += 256)
            *reinterpret_cast<float*>(a.act_d + a2_xsum(t, g, NT)) = 0.f;
    }
  }
  if (ttl) ttl[4] = clk64();
  cbar();
  // self-clean the accumulators and arrival counters for the next layer
  for (int i = 0; i < nd; ++i) {
    float* accw = accb + (size_t)s_done[i] * 128 * TP;
    for (int j = threadIdx.x; j < 128 * TP; j += 256) accw[j] = 0.f;
    if (threadIdx.x == 0) arr[s_done[i]] = 0;
  }
  cbar();
  if (threadIdx.x == 0) {
    // the completion counts carry release semantics (cumulative over the
    // epilogue outputs and the cleaning, ordered by the barrier above)
    if constexpr (PH == PH_LM) {
      int* lmc = a.ctr + (size_t)a.n_layers * kCtrPerLayer;
      if (atom_add_acqrel_gpu(lmc, nd) + nd == a.lm_tg) {
        where(a, WCODE(layer, PH, 0x10));
        if (a.P > 1) {
          const ArgmaxXArgs x{a.P, a.rank, a.loopback, 2 * a.n_layers, a.h / 128, a.recv, a.peer_recv};
          argmax_exchange(x, a.st);
        }
        accept_walk_dev(a.st);
      }
    } else {
      const int ci = PH == PH_QKV ? C_QKV : PH == PH_O ? C_O : PH == PH_GU ? C_GU : C_DN;
      if (ttl) ttl[5] = clk64();
      red_release_gpu_add(ctr + ci, nd);
      if (ttl) ttl[6] = clk64();
    }
  }
  __syncwarp();
  tmark(a, tslot, 2);
  where(a, WCODE(layer, PH, 9));
  return make_int2(ring.k, tck);
}

// Tree-masked attention (a5, R11) of one work item: (kv head,
// 64-row chunk z, key split).  Two tile streams: warps 0-3 take the item's
// even tiles, warps 4-7 the odd ones; warp (stream, rb) owns query rows
// rb*16 .. rb*16+15 of the chunk over ALL keys of its tiles, so the scores
// stay in registers: S = q K^T (q hi + lo fragments from global / L1 -- the
// QKV epilogue wrote them -- times the K tile from the ring; tree tiles add
// q_hi K_lo), online softmax on the S fragments, P (fp16) reused in place as
// the A fragments of O += P V (+ P V_lo on tree tiles).  No shared-memory P
// exchange, no barriers inside the tile loop.  Each stream's unnormalised
// partial (m, l, O) goes to the workspace (2 partials per item); after the
// group's items meet, the 2S partials are merged by log-sum-exp, several
// warps per output row.
template <int NT, int D>
__device__ __forceinline__ int attn_item(const StepArgs* __restrict__ ap, const Sched* __restrict__ sp, int layer,
                                      Ring ring, float* s_merge, uint8_t* s_q) {
  const StepArgs& a = *ap;
  const Sched& s = *sp;
  constexpr int KT = 4096 / D, NB = KT / 8, DB = D / 8;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rb = warp & 3, ws = warp >> 2;
  const int gq = lane >> 2, tq = lane & 3;
  const int b = s.att_item;
  const int grp = b / s.att_S, split = b % s.att_S;
  const int kvh = grp / s.att_Z, z = grp % s.att_Z;
  const int G = a.G, T = s.T, L = s.L;
  const int Mrows = G * T;
  const int rbmax = 4 * G;
  const size_t qlo = (size_t)a.Hkv_l * rbmax * (D / 16) * 32 * 8;
  int* ctr = a.ctr + (size_t)layer * kCtrPerLayer;
  tmark(a, layer * 5 + PH_ATT, 0);
  where(a, WCODE(layer, PH_ATT, 1));
  unsigned long long* atl =
      (a.utl && layer == a.n_layers / 2 && blockIdx.x == 0 && threadIdx.x == 0) ? a.utl + 28672 : nullptr;
  if (atl) atl[0] = clk64();
  wait_counter(ctr + C_QKV, a.qkv_tg);  // q, tree rows and their lo parts are written
  if (atl) atl[1] = clk64();
  where(a, WCODE(layer, PH_ATT, 2));
  const DevState* st = a.st;
  const int rbg = z * 4 + rb;
  const int ra = rb * 16 + gq, rbr = ra + 8;  // rows within the chunk
  const int rowA = z * 64 + ra, rowB = z * 64 + rbr;
  const int tokA = min(s.T0 + rowA / G, SS_MAX_TREE - 1), tokB = min(s.T0 + rowB / G, SS_MAX_TREE - 1);
  const unsigned long long ancA = st->anc[tokA], ancB = st->anc[tokB];
  const bool okA = rowA < Mrows, okB = rowB < Mrows;
  const float sl2 = rsqrtf((float)D) * 1.4426950408889634f;
  // the chunk's q fragments (4 row blocks x d/16 k-steps x 32 lanes x 16 B,
  // hi then lo) -> shared memory once; the tile loop reads them with LDS
  // (from global they were L2 round trips every tile: the ring leaves ~30 KB of L1)
  {
    constexpr int NQ = 4 * (D / 16) * 32;  // uint4 per part
    const uint4* gh = reinterpret_cast<const uint4*>(a.qf) + ((size_t)kvh * rbmax + z * 4) * (D / 16) * 32;
    const uint4* gl = reinterpret_cast<const uint4*>(a.qf + qlo) + ((size_t)kvh * rbmax + z * 4) * (D / 16) * 32;
    uint4* sq = reinterpret_cast<uint4*>(s_q);
    for (int i = threadIdx.x; i < NQ; i += 256) {
      sq[i] = __ldcg(gh + i);
      sq[NQ + i] = __ldcg(gl + i);
    }
    cbar();
  }
  const uint32_t qh = smem_u32(s_q) + (uint32_t)((rb * (D / 16)) * 32 + lane) * 16;
  const uint32_t ql = qh + (uint32_t)(4 * (D / 16) * 32) * 16;
  // ring position of tile it: one unit per tile, two for a tree tile (hi, lo)
  const int t0 = s.att_t0, t1 = s.att_t1, ft = L / KT, k0 = ring.k;
  auto ring_of = [&](int it) { return k0 + (it - t0) + max(0, it - max(t0, ft)); };
  float mA = -INFINITY, mB = -INFINITY, lA = 0.f, lB = 0.f;
  float o[DB][4];
#pragma unroll
  for (int n = 0; n < DB; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
  // Tiles go in groups of two (one per stream) -- one when the pair would
  // need more ring units than there are stages: both streams wait for their
  // tile's units, compute, meet at a barrier, then every warp releases every
  // unit of the group once (empty count 8).  Consumption stays in ring order.
  constexpr int STG = StepCfg<NT>::STAGES;
  auto units_of = [&](int x) { return x >= ft ? 2 : 1; };
  for (int g0 = t0; g0 < t1;) {
    const int g1 = (g0 + 1 < t1 && units_of(g0) + units_of(g0 + 1) <= STG) ? g0 + 2 : g0 + 1;
    const int it = g0 + ws;
    if (it < g1) {
    const bool tree = it >= ft;
    const int ri = ring_of(it);
    const uint32_t shi = ring_wait_at<NT>(ring, ri);
    const uint32_t slo = tree ? ring_wait_at<NT>(ring, ri + 1) : shi;
    if (atl && it - t0 < 64) atl[16 + (it - t0) * 2] = clk64();
    // S = q K^T: the k16 chains alternate between two accumulator sets
    float sc[1][NB][4];
#pragma unroll
    for (int n = 0; n < NB; ++n) sc[0][n][0] = sc[0][n][1] = sc[0][n][2] = sc[0][n][3] = 0.f;
#pragma unroll 2
    for (int kk = 0; kk < D / 16; ++kk) {
      const uint4 fh = lds128(qh + kk * 512), fl = lds128(ql + kk * 512);
      const uint32_t ah[4] = {fh.x, fh.y, fh.z, fh.w}, al[4] = {fl.x, fl.y, fl.z, fl.w};
      float(&sk)[NB][4] = sc[0];
#pragma unroll
      for (int np = 0; np < NB / 2; ++np) {
        const int key = np * 16 + (lane & 7) + ((lane >> 4) << 3);
        const int ch = kk * 2 + ((lane >> 3) & 1);
        const uint32_t koff = (uint32_t)(key * D + ((ch ^ (key & 7)) << 3)) * 2;
        uint32_t kb[4];
        asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                     : "=r"(kb[0]), "=r"(kb[1]), "=r"(kb[2]), "=r"(kb[3]) : "r"(shi + koff));
        mma_f16_16816(sk[2 * np], ah, kb[0], kb[1]);
        mma_f16_16816(sk[2 * np + 1], ah, kb[2], kb[3]);
        mma_f16_16816(sk[2 * np], al, kb[0], kb[1]);
        mma_f16_16816(sk[2 * np + 1], al, kb[2], kb[3]);
        if (tree) {
          asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                       : "=r"(kb[0]), "=r"(kb[1]), "=r"(kb[2]), "=r"(kb[3]) : "r"(slo + koff));
          mma_f16_16816(sk[2 * np], ah, kb[0], kb[1]);
          mma_f16_16816(sk[2 * np + 1], ah, kb[2], kb[3]);
        }
      }
    }
    if (atl && it - t0 < 8) atl[200 + (it - t0) * 4] = clk64();
    // mask (prefix always visible; tree keys -- cached and new -- by ancestor
    // bit, the non-square mask of P:321; beyond L + T0 + T never), scale, tile
    // row maxima over the quad
    const int kbase = it * KT;
    float mxA = -INFINITY, mxB = -INFINITY;
#pragma unroll
    for (int n = 0; n < NB; ++n)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int key = kbase + n * 8 + 2 * tq + (e & 1);
        const unsigned long long anc = (e < 2) ? ancA : ancB;
        const bool ok = (e < 2) ? okA : okB;
        const bool vis = ok && (key < L || (key < L + s.T0 + T && ((anc >> (key - L)) & 1ull)));
        const float v = vis ? sc[0][n][e] * sl2 : -INFINITY;
        sc[0][n][e] = v;
        if (e < 2) mxA = fmaxf(mxA, v); else mxB = fmaxf(mxB, v);
      }
    mxA = fmaxf(mxA, __shfl_xor_sync(0xffffffffu, mxA, 1));
    mxA = fmaxf(mxA, __shfl_xor_sync(0xffffffffu, mxA, 2));
    mxB = fmaxf(mxB, __shfl_xor_sync(0xffffffffu, mxB, 1));
    mxB = fmaxf(mxB, __shfl_xor_sync(0xffffffffu, mxB, 2));
    const float mnA = fmaxf(mA, mxA), mnB = fmaxf(mB, mxB);
    const float uA = (mnA == -INFINITY) ? 0.f : mnA, uB = (mnB == -INFINITY) ? 0.f : mnB;
    const float alA = exp2f(mA - uA), alB = exp2f(mB - uB);
    mA = mnA;
    mB = mnB;
    // P = exp2(s - m) as fp16 A fragments (the C fragments of n-blocks 2j, 2j+1
    // are the A fragment of keys 16j .. 16j+15)
    uint32_t pf[NB / 2][4];
    float sumA = 0.f, sumB = 0.f;
#pragma unroll
    for (int j = 0; j < NB / 2; ++j) {
      const float p00 = exp2f(sc[0][2 * j][0] - uA), p01 = exp2f(sc[0][2 * j][1] - uA);
      const float p02 = exp2f(sc[0][2 * j][2] - uB), p03 = exp2f(sc[0][2 * j][3] - uB);
      const float p10 = exp2f(sc[0][2 * j + 1][0] - uA), p11 = exp2f(sc[0][2 * j + 1][1] - uA);
      const float p12 = exp2f(sc[0][2 * j + 1][2] - uB), p13 = exp2f(sc[0][2 * j + 1][3] - uB);
      sumA += (p00 + p01) + (p10 + p11);
      sumB += (p02 + p03) + (p12 + p13);
      pf[j][0] = pack_half2(p00, p01);
      pf[j][1] = pack_half2(p02, p03);
      pf[j][2] = pack_half2(p10, p11);
      pf[j][3] = pack_half2(p12, p13);
    }
    lA = lA * alA + sumA;  // this thread's keys; the quad is summed at the end
    lB = lB * alB + sumB;
    if (__any_sync(0xffffffffu, alA != 1.f || alB != 1.f)) {
#pragma unroll
      for (int n = 0; n < DB; ++n) {
        o[n][0] *= alA; o[n][1] *= alA; o[n][2] *= alB; o[n][3] *= alB;
      }
    }
    if (atl && it - t0 < 8) atl[200 + (it - t0) * 4 + 1] = clk64();
    // O += P V (V hi; tree tiles also V lo)
    const uint32_t vh = shi + KT * D * 2, vl = slo + KT * D * 2;
#pragma unroll
    for (int j = 0; j < NB / 2; ++j) {
#pragma unroll
      for (int dp = 0; dp < D / 16; ++dp) {
        const int key = j * 16 + (lane & 7) + (((lane >> 3) & 1) << 3);
        const int ch = dp * 2 + (lane >> 4);
        const uint32_t voff = (uint32_t)(key * D + ((ch ^ (key & 7)) << 3)) * 2;
        uint32_t vb[4];
        asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                     : "=r"(vb[0]), "=r"(vb[1]), "=r"(vb[2]), "=r"(vb[3]) : "r"(vh + voff));
        mma_f16_16816(o[2 * dp], pf[j], vb[0], vb[1]);
        mma_f16_16816(o[2 * dp + 1], pf[j], vb[2], vb[3]);
        if (tree) {
          asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                       : "=r"(vb[0]), "=r"(vb[1]), "=r"(vb[2]), "=r"(vb[3]) : "r"(vl + voff));
          mma_f16_16816(o[2 * dp], pf[j], vb[0], vb[1]);
          mma_f16_16816(o[2 * dp + 1], pf[j], vb[2], vb[3]);
        }
      }
    }
    if (atl && it - t0 < 8) atl[200 + (it - t0) * 4 + 2] = clk64();
    if (atl && it - t0 < 64) atl[16 + (it - t0) * 2 + 1] = clk64();
    }
    cbar();
    if (lane == 0)
      for (int x = g0; x < g1; ++x) {
        const int rx = ring_of(x);
        mbar_arrive_a(ring.empty0 + 8 * (rx % STG));
        if (x >= ft) mbar_arrive_a(ring.empty0 + 8 * ((rx + 1) % STG));
      }
    g0 = g1;
  }
  // this stream's partial -> workspace: O (16 rows x D per warp) and (m, l)
  {
    lA += __shfl_xor_sync(0xffffffffu, lA, 1);
    lA += __shfl_xor_sync(0xffffffffu, lA, 2);
    lB += __shfl_xor_sync(0xffffffffu, lB, 1);
    lB += __shfl_xor_sync(0xffffffffu, lB, 2);
    const size_t pidx = (size_t)b * 2 + ws;
    float* wsp = a.att_ws + pidx * 64 * D;
#pragma unroll
    for (int n = 0; n < DB; ++n) {
      const int c = n * 8 + 2 * tq;
      *reinterpret_cast<float2*>(wsp + (size_t)ra * D + c) = make_float2(o[n][0], o[n][1]);
      *reinterpret_cast<float2*>(wsp + (size_t)rbr * D + c) = make_float2(o[n][2], o[n][3]);
    }
    if (tq == 0) {
      a.att_ml[pidx * 64 + ra] = make_float2(mA, lA);
      a.att_ml[pidx * 64 + rbr] = make_float2(mB, lB);
    }
  }
  // meet the other splits of this (kv head, row chunk)
  where(a, WCODE(layer, PH_ATT, 4));
  if (atl) atl[2] = clk64();
  cbar();
  if (threadIdx.x == 0) {
    atom_add_release_gpu(ctr + C_MEET + grp, 1);
    spin_until_geq(ctr + C_MEET + grp, s.att_S);
  }
  cbar();
  if (atl) atl[3] = clk64();
  // merge this item's slice of the row groups (one 128-wide group of the O
  // input: one head at d = 128, two at d = 64) over the group's 2S partials:
  // W warps per row group, each summing every W-th partial, then combined
  // through shared memory (R11 log-sum-exp)
  constexpr int RPG = 128 / D;             // rows per group
  constexpr int NRG = 64 / RPG;
  const int rg0 = split * NRG / s.att_S, rg1 = (split + 1) * NRG / s.att_S;
  const int nrg = rg1 - rg0;
  const int P2 = 2 * s.att_S;
  const size_t pb0 = (size_t)grp * P2;
  const int W = nrg > 0 ? max(1, 8 / nrg) : 1;
  for (int base = 0; base < nrg; base += 8 / W) {
    const int rgl = base + warp / W, sub = warp % W;
    const bool act = rgl < nrg && warp / W < 8 / W;
    const int rg = rg0 + rgl;
    const int rr = rg * RPG + (RPG == 2 ? (lane >> 4) : 0);  // row within the chunk
    const int c4 = (RPG == 2 ? (lane & 15) : lane) * 4;       // 4 columns
    float mx = -INFINITY, l = 0.f;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (act) {
      // one pass: online log-sum-exp (the running max rescales what was summed),
      // so every partial's (m, l) and O are requested together
      for (int p0 = sub; p0 < P2; p0 += 4 * W) {
        float2 v8[4];
        float4 o8[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          v8[j] = make_float2(-INFINITY, 0.f);
          if (p0 + j * W < P2) {
            const size_t pp = pb0 + p0 + j * W;
            v8[j] = __ldcg(&a.att_ml[pp * 64 + rr]);
            o8[j] = __ldcg(reinterpret_cast<const float4*>(a.att_ws + (pp * 64 + rr) * D + c4));
          }
        }
        float mn = mx;
#pragma unroll
        for (int j = 0; j < 4; ++j) mn = fmaxf(mn, v8[j].x);
        if (mn != -INFINITY) {
          const float sc = (mx == -INFINITY) ? 0.f : exp2f(mx - mn);
          l *= sc;
          acc.x *= sc; acc.y *= sc; acc.z *= sc; acc.w *= sc;
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (p0 + j * W < P2 && v8[j].x != -INFINITY) {
              const float w = exp2f(v8[j].x - mn);
              l += w * v8[j].y;
              acc.x += w * o8[j].x;
              acc.y += w * o8[j].y;
              acc.z += w * o8[j].z;
              acc.w += w * o8[j].w;
            }
          mx = mn;
        }
      }
      if (W > 1) {
        float* sm = s_merge + warp * 132;
        *reinterpret_cast<float4*>(sm + lane * 4) = acc;
        if ((lane & 15) == 0) {
          sm[128 + (lane >> 4) * 2] = mx;
          sm[129 + (lane >> 4) * 2] = l;
        }
      }
    }
    if (W > 1) cbar();
    if (act && sub == 0) {
      if (W > 1) {  // combine the W warps of this row group
        float M = -INFINITY;
        const int half = RPG == 2 ? (lane >> 4) : 0;
        for (int v = 0; v < W; ++v) M = fmaxf(M, s_merge[(warp + v) * 132 + 128 + half * 2]);
        float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
        float lt = 0.f;
        for (int v = 0; v < W; ++v) {
          const float* sm = s_merge + (warp + v) * 132;
          const float mv = sm[128 + half * 2];
          const float w = (mv == -INFINITY) ? 0.f : exp2f(mv - M);
          lt += w * sm[129 + half * 2];
          const float4 q4 = *reinterpret_cast<const float4*>(sm + lane * 4);
          t.x += w * q4.x; t.y += w * q4.y; t.z += w * q4.z; t.w += w * q4.w;
        }
        acc = t;
        l = lt;
      }
      const int m = z * 64 + rr;
      const bool valid = m < Mrows;
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
      // the warp's columns are exactly one 128-group of one token (at d = 64
      // the two rows are consecutive heads of the same token: G is even)
      xs = warp_sum(valid ? xs : 0.f);
      if (lane == 0 && valid) *reinterpret_cast<float*>(a.act_o + a2_xsum(t, k >> 7, NT)) = xs;
    }
    if (W > 1) cbar();
  }
  cbar();
  if (threadIdx.x == 0) red_release_gpu_add(ctr + C_ATT, 1);
  if (atl) { atl[4] = clk64(); atl[5] = (unsigned long long)(t1 - t0); atl[6] = (unsigned long long)s.att_S; }
  tmark(a, layer * 5 + PH_ATT, 2);
  where(a, WCODE(layer, PH_ATT, 9));
  return ring_of(t1);
}

template <int NT, int D>
__global__ void __launch_bounds__(StepCfg<NT>::THREADS, StepCfg<NT>::CTAS_PER_SM)
    step_kernel(const StepArgs* __restrict__ ap_g) {
  using C = StepCfg<NT>;
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[C::STAGES], empty[C::STAGES], ardy[2], mdone[4];
  __shared__ int s_done[128];
  __shared__ int s_nd;
  __shared__ float s_rmax[2 * 64];
  __shared__ Sched s_sched;
  __shared__ __align__(16) float s_merge[8 * 132];
  __shared__ uint32_t s_tmem, s_slot[2];
  // the arguments and the per-layer pointer table live in shared memory: the
  // producer's per-unit address arithmetic must not chase global pointers
  __shared__ __align__(16) StepArgs s_args;
  __shared__ __align__(16) LayerPtrs s_lp[kStepMaxLayers];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  {
    const uint64_t* src = reinterpret_cast<const uint64_t*>(ap_g);
    uint64_t* dst = reinterpret_cast<uint64_t*>(&s_args);
    for (int i = threadIdx.x; i < (int)(sizeof(StepArgs) / 8); i += blockDim.x) dst[i] = src[i];
    const uint64_t* lsrc = reinterpret_cast<const uint64_t*>(ap_g->layers);
    uint64_t* ldst = reinterpret_cast<uint64_t*>(s_lp);
    const int nl = ap_g->n_layers;
    for (int i = threadIdx.x; i < nl * (int)(sizeof(LayerPtrs) / 8); i += blockDim.x) ldst[i] = lsrc[i];
  }
#ifdef SS_WATCHDOG_RECORD
  if (threadIdx.x == 0 && blockIdx.x == 0 && !g_panic_map && g_panic) {  // barrier map (first launch)
    g_panic_map = 1;
    g_panic[8] = smem_u32(full);
    g_panic[9] = smem_u32(empty);
    g_panic[10] = smem_u32(ardy);
    g_panic[11] = smem_u32(mdone);
    g_panic[12] = C::STAGES;
  }
#endif
  if (threadIdx.x == 0) {
    for (int i = 0; i < C::STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 8);
    }
    for (int i = 0; i < kNbuf<NT>; ++i) mbar_init(&ardy[i], 8);
    for (int i = 0; i < 2 * kNbuf<NT>; ++i) mbar_init(&mdone[i], 1);
    fence_mbar_init();
  }
  if (warp == 0) {  // the whole TMEM of the SM (one CTA per SM)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) s_args.layers = s_lp;
  __syncthreads();
  const StepArgs* __restrict__ ap = &s_args;
  const uint32_t sm0 = smem_u32(smem), full0 = smem_u32(full), empty0 = smem_u32(empty);
  const Tc tc{s_tmem, smem_u32(ardy), smem_u32(mdone), s_slot};
  // everything below reads the ingest kernel's outputs (T, L, tree, counters)
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x == 0) make_sched(*ap, blockIdx.x, ap->st->L, ap->st->T, ap->st->T0, NT, s_sched);
  __syncthreads();
  if (warp >= 8) {  // warpgroup 2: producer, MMA issuer, two idle warps
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(C::REG_AUX));
    if (warp == 8) {
      if (lane == 0) producer<NT>(ap, &s_sched, sm0, full0, empty0);
      where(*ap, WCODE(0xFFFF, 0x40, 0xFF));
    } else if (warp == 9 || warp == 10) {
      mma_warp<NT>(ap, tc, warp - 9);
      where(*ap, WCODE(0xFFFF, 0x20, 0xFF));
    }
    return;
  }
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(C::REG_CONSUMER));
  Ring ring{sm0, full0, empty0, 0};
  uint8_t* s_tail = smem + C::STAGES * C::SLOT;
  int tck = 0;  // W4 units consumed (TMEM buffer / barrier phase)
  const int n_layers = ap->n_layers;
  const bool att = s_sched.att_item >= 0;
  int2 r;
  for (int l = 0; l < n_layers; ++l) {
    r = gemm_phase<NT, PH_QKV>(ap, &s_sched, l, s_sched.qkv0, s_sched.qkv1, ring, tc, tck, s_done, &s_nd, s_tail);
    ring.k = r.x; tck = r.y;
    if (att) ring.k = attn_item<NT, D>(ap, &s_sched, l, ring, s_merge, smem + C::STAGES * C::SLOT);
    r = gemm_phase<NT, PH_O>(ap, &s_sched, l, s_sched.o0, s_sched.o1, ring, tc, tck, s_done, &s_nd, s_tail);
    ring.k = r.x; tck = r.y;
    r = gemm_phase<NT, PH_GU>(ap, &s_sched, l, s_sched.gu0, s_sched.gu1, ring, tc, tck, s_done, &s_nd, s_tail);
    ring.k = r.x; tck = r.y;
    r = gemm_phase<NT, PH_DN>(ap, &s_sched, l, s_sched.dn0, s_sched.dn1, ring, tc, tck, s_done, &s_nd, s_tail);
    ring.k = r.x; tck = r.y;
  }
  // stop the MMA warp: an empty A buffer announcement (thread 0 writes the slot
  // before its own arrival; every consumer warp's lane 0 arrives)
  if (threadIdx.x == 0) s_slot[tck % kNbuf<NT>] = 0;
  if (lane == 0) mbar_arrive_a(tc.ardy0 + 8 * (tck % kNbuf<NT>));
  where(*ap, WCODE(0xFFFE, 0, 0));
  gemm_phase<NT, PH_LM>(ap, &s_sched, 0, s_sched.lm0, s_sched.lm1, ring, tc, tck, s_done, &s_nd, s_tail);
  tc_fence_before();
  cbar();
  __syncwarp();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(s_tmem), "r"(kTmemCols));
  where(*ap, WCODE(0xFFFF, 0xFF, 0xFF));
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

// Watchdog panic record (debugging aid, always armed: one mapped host page).
static unsigned long long* g_panic_host = nullptr;
void arm_watchdog_record() {
  if (g_panic_host) return;
  unsigned long long* dev = nullptr;
  if (cudaHostAlloc((void**)&g_panic_host, 64 * 1024 * 8, cudaHostAllocMapped) != cudaSuccess) {
    g_panic_host = nullptr;
    cudaGetLastError();
    return;
  }
  memset(g_panic_host, 0, 64 * 1024 * 8);
  cudaHostGetDevicePointer((void**)&dev, g_panic_host, 0);
  cudaMemcpyToSymbol(g_panic, &dev, sizeof(dev));
}
const unsigned long long* watchdog_record() { return g_panic_host; }

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
