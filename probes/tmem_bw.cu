// Probe: tcgen05.st / tcgen05.ld throughput (registers <-> TMEM) with 4 or 8
// warps, alone and while one thread issues 128xNx16 TS MMAs.
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

// mode bit0: do STTM in warps 0..NW-1; bit1: MMAs from warp NW (lane 0); bit2: use .x32 stores; bit3: LDTM instead of STTM
template <int NW>
__global__ void k(int mode, int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 16384; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tb = tbase;
  long long t0 = clock64();
  if (warp < NW && (mode & 1)) {
    const uint32_t ta = tb + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 128;
    uint32_t v[32];
    for (int i = 0; i < 32; ++i) v[i] = lane * 7 + i;
    for (int it = 0; it < iters; ++it) {
      if (mode & 8) {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                       "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                     : "r"(ta + (it & 3) * 16));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      } else {
        for (int c = 0; c < 4; ++c)
          asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                       ::"r"(ta + c * 16), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
                       "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]) : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      }
      v[0] += 1;
    }
    long long t1 = clock64();
    if (lane == 0) out[warp] = t1 - t0;
  }
  if (warp == NW && (mode & 2) && lane == 0) {
    const uint64_t bd0 = bdesc(smem_u32(smem), 16 * 16, 128);
    for (int it = 0; it < iters; ++it)
      for (int kk = 0; kk < 8; ++kk) {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tb + 256 + (kk & 1) * 16),
                     "r"(tb + 384 + kk * 8), "l"(bd0 + (uint64_t)((kk * 512) >> 4)), "r"((1u << 4) | (2u << 17) | (8u << 24)), "r"(1u));
      }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    asm volatile("{\n\t.reg .pred P;\n\tW: mbarrier.try_wait.parity.shared.b64 P, [%0], 0;\n\t@!P bra W;\n\t}" ::"r"(smem_u32(&bar)));
    out[31] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(512));
}

template <int NW>
void run(int mode, int iters) {
  long long* d; CK(cudaMalloc(&d, 32 * 8)); CK(cudaMemset(d, 0, 32 * 8));
  CK(cudaFuncSetAttribute(k<NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
  k<NW><<<1, (NW + 1) * 32, 65536>>>(mode, iters, d);
  CK(cudaDeviceSynchronize());
  long long h[32]; CK(cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost));
  double st = 0; for (int w = 0; w < NW; ++w) st = h[w] > st ? h[w] : st;
  const char* what = (mode & 8) ? "LDTM.x16" : "STTM.x16 x4";
  printf("NW=%d mode=%d: %s per iter (per warp) %.1f cyc; MMA: %.1f cyc/MMA\n", NW, mode, what,
         (mode & 1) ? st / iters : 0.0, (mode & 2) ? (double)h[31] / (iters * 8) : 0.0);
  cudaFree(d);
}

int main() {
  run<4>(1, 256);
  run<8>(1, 256);
  run<4>(2, 256);
  run<4>(3, 256);
  run<8>(3, 256);
  run<4>(9, 256);
  run<8>(9, 256);
  run<8>(11, 256);
  return 0;
}
