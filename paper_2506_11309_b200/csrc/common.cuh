// common.cuh -- sm_100a device helpers shared by the swiftspec kernels:
// mbarrier + cp.async.bulk (TMA bulk engine) pipeline primitives, mma.sync
// wrappers, int4 -> bf16 dequant, LL-style flagged 16-byte lines, packed
// layouts.  No model arithmetic lives here.
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>

#define SS_DEV __device__ __forceinline__

namespace ss {

// ---------------------------------------------------------------- layouts
// W4 unit (tile-group of 128 output rows x one K-stage of 256):
//   [warp 0..7][kblock 0..3][lane 0..31][4 x u32 nibble words] = 16384 B
//   [warp][group 0..1][gq 0..7] bf16x2 (s[gq], s[gq+8])         =   512 B
//   [warp][group 0..1][gq 0..7] byte   z[gq] | z[gq+8] << 4      =   128 B
// (gq = lane / 4: one 32-bit and one 8-bit shared load give a lane the
// scales and zeros of both of its rows)
// BF16 unit (LM head; 128 rows x K-stage of 64):
//   [warp][k16 step 0..3][lane][4 x u32 bf16x2]                 = 16384 B
constexpr int kTG = 128;             // rows per tile-group (8 warps x 16)
constexpr int kW4KS = 256;           // K per W4 unit
constexpr int kBFKS = 64;            // K per BF16 unit
constexpr int kW4Bytes = 16384;
constexpr int kW4MetaBytes = 640;
constexpr int kW4UnitBytes = kW4Bytes + kW4MetaBytes;   // 17024
constexpr int kBFUnitBytes = 16384;
constexpr int kKvTile = 64;          // keys per attention tile

// Activation "fragment order" (B operand of mma.m16n8k16, col layout).  W4
// GEMM inputs are fp16; the LM-head input is split bf16 hi/lo in 2*NT n-tiles.
// Inside one 32-deep k block, element (token tt, k) sits at
//   ((k/32 * NT + tt/8) * 32 + lane) * 16 + ((k/16)%2) * 8 + word * 4 + half * 2  bytes,
//   lane = (tt%8)*4 + ((k%16)%8)/2, word = (k%16)/8, half = k%2,
// so one LDS.128 per lane yields the B fragments of two consecutive k16 steps.
SS_DEV uint32_t frag_offset(int tt, int k, int NT) {
  int kk = k & 15;
  int lane = ((tt & 7) << 2) | ((kk & 7) >> 1);
  int word = kk >> 3;
  return ((uint32_t)(((k >> 5) * NT + (tt >> 3)) * 32 + lane) << 4) + (((k >> 4) & 1) << 3) + (word << 2) +
         ((k & 1) << 1);
}
// W4 GEMM input: one chunk per 256-deep K stage = the fp16 fragments (NT*4 KB)
// followed by X[2 groups][8*NT] fp32, the per-(128-group, token) sums of the
// fp16 values (the zero-point correction of gemm.cu).
SS_DEV constexpr uint32_t w4_act_stage_bytes(int NT) { return (uint32_t)NT * 4096u + (uint32_t)NT * 64u; }
SS_DEV uint32_t act_frag_offset(int tt, int k, int NT) {
  return (uint32_t)(k >> 8) * w4_act_stage_bytes(NT) + frag_offset(tt, k & 255, NT);
}
SS_DEV uint32_t act_xsum_offset(int tt, int g, int NT) {
  return (uint32_t)(g >> 1) * w4_act_stage_bytes(NT) + (uint32_t)NT * 4096u + (uint32_t)(((g & 1) * 8 * NT + tt) * 4);
}

// Swizzled KV cache row layout: 64-row blocks, 16-byte chunk index XORed
// with (row % 8) so ldmatrix reads of 8 rows are bank-conflict free.
SS_DEV uint32_t kv_elem_offset(int pos, int j, int d) {
  int r = pos & 63;
  int c = (j >> 3) ^ (r & 7);
  return (uint32_t)(pos - r) * d + r * d + c * 8 + (j & 7);
}

// ---------------------------------------------------------------- PTX
SS_DEV uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

SS_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
SS_DEV void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
SS_DEV void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
SS_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
SS_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared.b64 P, [%0], %1;\n\t"
      "@!P bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// Opaque copy: the compiler keeps the value in a register instead of
// rematerialising it (e.g. a shared-window base) inside a hot loop.
SS_DEV uint32_t opaque(uint32_t v) {
  uint32_t r;
  asm volatile("mov.b32 %0, %1;" : "=r"(r) : "r"(v));
  return r;
}
// Same on precomputed shared-window addresses (keeps the address arithmetic
// out of hot loops: no generic->shared conversion per access).
SS_DEV void mbar_wait_a(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared.b64 P, [%0], %1;\n\t"
      "@!P bra WAIT_%=;\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
SS_DEV void mbar_arrive_a(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(bar) : "memory");
}
SS_DEV uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
SS_DEV float2 lds64f(uint32_t a) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0,%1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a));
  return v;
}
SS_DEV uint32_t lds32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
SS_DEV uint32_t lds8(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
// 1-D bulk async copy global -> shared (TMA bulk engine, SASS UBLKCP),
// completion counted on an mbarrier; L2 evict-first policy for streamed data.
SS_DEV void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
SS_DEV void bulk_g2s_nohint(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// Bulk prefetch of global memory into L2 (no shared memory, no completion).
SS_DEV void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
SS_DEV uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
SS_DEV uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// Programmatic dependent launch (PDL): the next kernel in the stream may start
// its prologue while this one drains; it must wait before reading our outputs.
#ifndef SS_SPIN_NS
#define SS_SPIN_NS 100  // back-off of the grid-level spin waits (experiment knob)
#endif
SS_DEV void spin_pause() { if (SS_SPIN_NS > 0) __nanosleep(SS_SPIN_NS); }
SS_DEV void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
SS_DEV void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Order this thread's (and, after a barrier, the CTA's) generic-proxy shared
// memory accesses before subsequent async-proxy (TMA / bulk copy) accesses.
SS_DEV void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Release/acquire fence at GPU scope (lighter than __threadfence's fence.sc,
// which also invalidates L1).
SS_DEV void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

// Named barrier over nthreads threads.  The non-.aligned form: threads of a
// warp may arrive from divergent paths (the producer warp's lanes run
// different loops; synccheck flags bar.sync there).
SS_DEV void named_bar_sync(int id, int nthreads) {
  asm volatile("barrier.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
// Non-blocking mbarrier phase test (the step kernel's producer polls several
// conditions without blocking on any one of them).
SS_DEV bool mbar_test_a(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 P, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
// expect_tx without an arrival (the first part of a unit whose second part is
// issued later by the same producer thread, with mbar_arrive_expect_tx_a).
SS_DEV void mbar_expect_tx_noarrive_a(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
SS_DEV void mbar_arrive_expect_tx_a(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
// 1-D bulk copies with precomputed shared addresses.
SS_DEV void bulk_g2s_a(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          dst),
      "l"(src), "r"(bytes), "r"(bar), "l"(policy)
      : "memory");
}
SS_DEV void bulk_g2s_nohint_a(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
// Order this thread's earlier generic-proxy observations of global memory
// (data other CTAs wrote, acquired through a flag) before its later
// async-proxy (TMA) reads of that memory.
SS_DEV void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
SS_DEV int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
SS_DEV void red_release_gpu_add(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// D = A(16x16 bf16, row) * B(16x8 bf16, col) + D, fp32 accumulate.
SS_DEV void mma_bf16_16816(float* d, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

SS_DEV void ldmatrix_x4(uint32_t* r, const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_u32(p)));
}
SS_DEV void ldmatrix_x4_trans(uint32_t* r, const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_u32(p)));
}

// Vector fp32 reduction into global memory (sm_90+).
SS_DEV void red_add_v2(float* p, float a, float b) {
  asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(a), "f"(b) : "memory");
}

// int4 nibble word -> the 4 f16x2 A-fragment registers of one m16n8k16 step.
// Nibble e_p sits at bits [4p, 4p+4); (e0,e4) -> r0, (e1,e5) -> r1, (e2,e6)
// -> r2, (e3,e7) -> r3.  lop3 with the fp16 exponent 0x6400 (1024, ulp 1)
// turns a nibble at bits 0-3 of a half into 1024 + e and one at bits 4-7
// into 1024 + 16 e; the second pair needs w >> 8, done as mul.hi on the FMA
// pipe so the ALU pipe only runs the four lop3.  r1/r3 carry the factor 16,
// which the zero-point fma removes exactly (see gemm.cu).
SS_DEV void dequant8(uint32_t w, uint32_t* r) {
  const uint32_t lo = 0x000F000Fu, hi = 0x00F000F0u, magic = 0x64006400u;
  uint32_t w8;
  asm("mul.hi.u32 %0, %1, %2;" : "=r"(w8) : "r"(w), "r"(0x01000000u));
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r[0]) : "r"(w), "r"(lo), "r"(magic));
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r[1]) : "r"(w), "r"(hi), "r"(magic));
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r[2]) : "r"(w8), "r"(lo), "r"(magic));
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r[3]) : "r"(w8), "r"(hi), "r"(magic));
}
SS_DEV uint32_t f16x2_fma(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t r;
  asm("fma.rn.f16x2 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
  return r;
}
SS_DEV uint32_t f16x2_sub(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("sub.rn.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
// D = A(16x16 f16, row) * B(16x8 f16, col) + D, fp32 accumulate.
SS_DEV void mma_f16_16816(float* d, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
SS_DEV uint32_t pack_half2(float lo, float hi) {
  __half2 v = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

SS_DEV uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
SS_DEV float bf16_lo(uint32_t v) { return __uint_as_float(v << 16); }
SS_DEV float bf16_hi(uint32_t v) { return __uint_as_float(v & 0xFFFF0000u); }
SS_DEV float bf16_bits_to_f32(uint16_t b) { return __uint_as_float(((uint32_t)b) << 16); }
SS_DEV uint16_t f32_to_bf16_bits(float f) {
  __nv_bfloat16 h = __float2bfloat16_rn(f);
  return *reinterpret_cast<uint16_t*>(&h);
}

SS_DEV uint16_t f32_to_f16_bits(float f) {
  __half h = __float2half_rn(f);
  return *reinterpret_cast<uint16_t*>(&h);
}

SS_DEV float half2_sum(uint32_t p) {
  const __half2 h = *reinterpret_cast<const __half2*>(&p);
  return __low2float(h) + __high2float(h);
}

SS_DEV float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
SS_DEV float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Order-preserving float key for packed (value, index) argmax with
// lowest-index tie break: key = (ordered(v) << 32) | (0xFFFFFFFF - idx).
SS_DEV uint64_t argmax_key(float v, uint32_t idx) {
  uint32_t b = __float_as_uint(v);
  uint32_t o = (b & 0x80000000u) ? ~b : (b | 0x80000000u);
  return ((uint64_t)o << 32) | (uint64_t)(0xFFFFFFFFu - idx);
}
SS_DEV uint32_t argmax_key_index(uint64_t k) { return 0xFFFFFFFFu - (uint32_t)(k & 0xFFFFFFFFu); }

// LL line (Alg. 2, reading R15: NCCL order data1, flag1, data2, flag2):
// each 8-byte (data, flag) half is written/read atomically by one v4 access.
SS_DEV void ll_store(uint4* dst, uint32_t d1, uint32_t d2, uint32_t flag) {
  asm volatile("st.volatile.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "r"(d1), "r"(flag), "r"(d2),
               "r"(flag)
               : "memory");
}
SS_DEV bool ll_try_load(const uint4* src, uint32_t flag, uint32_t& d1, uint32_t& d2) {
  uint32_t a, f1, b, f2;
#ifdef SS_EXP_LLRELAXED
  asm volatile("ld.relaxed.sys.global.v4.u32 {%0, %1, %2, %3}, [%4];"
#else
  asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
#endif
               : "=r"(a), "=r"(f1), "=r"(b), "=r"(f2)
               : "l"(src)
               : "memory");
  d1 = a;
  d2 = b;
  return f1 == flag && f2 == flag;
}

}  // namespace ss
