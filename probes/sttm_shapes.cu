// Probe: tcgen05.st throughput by shape (8 warps, 8 KB per warp per iteration,
// i.e. one W4 unit's fp16 A operand per iteration), alone and with a thread
// issuing 128x16x16 TS MMAs on another TMEM region.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("err %s line %d\n", cudaGetErrorString(e), __LINE__); exit(1);}}while(0)
__device__ __forceinline__ uint32_t smem_u32(const void* p){ return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t bdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}
#define R16(v) "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
// shape: 0 = 16x256b.x4 (4 per iter), 1 = 32x32b.x16 (4 per iter), 2 = 16x256b.x16 (1 per iter, 64 regs), 3 = 32x32b.x64
__global__ void k(int shape, int mma, int wait_each, int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 16384; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) { asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(&bar))); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  if (warp == 0) { asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(512)); asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;"); }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tb = tbase;
  long long t0 = clock64();
  if (warp < 8) {
    const int q = warp & 3, h = warp >> 2;
    uint32_t v[64];
    for (int i = 0; i < 64; ++i) v[i] = lane * 7 + i;
    for (int it = 0; it < iters; ++it) {
      const uint32_t base = tb + (it & 1) * 128;
      if (shape == 0) {
        const uint32_t ta = base + ((uint32_t)(32 * q + 16 * h) << 16);
        for (int c = 0; c < 4; ++c)
          asm volatile("tcgen05.st.sync.aligned.16x256b.x4.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(ta + c * 32), R16(v) : "memory");
      } else if (shape == 1) {
        const uint32_t ta = base + ((uint32_t)(32 * q) << 16) + h * 64;
        for (int c = 0; c < 4; ++c)
          asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(ta + c * 16), R16(v) : "memory");
      } else if (shape == 2) {
        const uint32_t ta = base + ((uint32_t)(32 * q + 16 * h) << 16);
        asm volatile("tcgen05.st.sync.aligned.16x256b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63,%64};" ::"r"(ta),
                     R16(v), R16((v + 16)), R16((v + 32)), R16((v + 48)) : "memory");
      } else {
        const uint32_t ta = base + ((uint32_t)(32 * q) << 16) + h * 64;
        asm volatile("tcgen05.st.sync.aligned.32x32b.x64.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63,%64};" ::"r"(ta),
                     R16(v), R16((v + 16)), R16((v + 32)), R16((v + 48)) : "memory");
      }
      if (wait_each) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      v[0] += 1;
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    long long t1 = clock64();
    if (lane == 0) out[warp] = t1 - t0;
  }
  if (warp == 8 && mma && lane == 0) {
    const uint64_t bd0 = bdesc(smem_u32(smem), 16 * 16, 128);
    for (int it = 0; it < iters * 16; ++it) {
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tb + 256 + (it & 7) * 16),
                   "r"(tb + ((it >> 4) & 1) * 128 + (it & 15) * 8), "l"(bd0 + (uint64_t)(((it & 15) * 512) >> 4)), "r"((1u << 4) | (2u << 17) | (8u << 24)), "r"(1u));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    asm volatile("{\n\t.reg .pred P;\n\tW: mbarrier.try_wait.parity.shared.b64 P, [%0], 0;\n\t@!P bra W;\n\t}" ::"r"(smem_u32(&bar)));
    out[31] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(512));
}
int main() {
  long long* d; CK(cudaMalloc(&d, 32 * 8));
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
  const char* names[4] = {"16x256b.x4 x4", "32x32b.x16 x4", "16x256b.x16", "32x32b.x64"};
  for (int mma = 0; mma < 2; ++mma)
    for (int we = 0; we < 2; ++we)
      for (int shape = 0; shape < 4; ++shape) {
        const int iters = 512;
        CK(cudaMemset(d, 0, 32 * 8));
        k<<<1, 288, 65536>>>(shape, mma, we, iters, d);
        CK(cudaDeviceSynchronize());
        long long h[32]; CK(cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost));
        double st = 0; for (int w = 0; w < 8; ++w) st = h[w] > st ? h[w] : st;
        printf("%-14s mma=%d wait_each=%d: %.0f cyc per 64 KB (all 8 warps) = %.0f B/cyc; mma %.1f cyc/MMA\n", names[shape], mma, we,
               st / iters, 65536.0 * iters / st, mma ? (double)h[31] / (iters * 16) : 0.0);
      }
  return 0;
}
