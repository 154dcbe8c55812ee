// Probe: tcgen05.mma kind::f16 with A from TMEM (written by tcgen05.st from
// registers), B from shared memory (K-major, no swizzle), D fp32 in TMEM.
// Verifies the layout assumptions the W4 GEMM relies on:
//   A: lane = row m, column = k/2, low half = even k
//   B: [kstep][c 2][n N][8 fp16], LBO = N*16 B (c step), SBO = 128 B (8 rows)
//   D: lane = row m, column = n
// and times back-to-back 128xNx16 MMAs.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("err %s line %d\n", cudaGetErrorString(e), __LINE__); exit(1);}}while(0)

__device__ __forceinline__ uint32_t smem_u32(const void* p){ return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t bdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version = 1 (sm100)
  return d;                // base_offset 0, lbo_mode 0, layout SWIZZLE_NONE (0)
}
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) {
  return (1u << 4)                      // D f32
       | (0u << 7) | (0u << 10)         // A, B f16
       | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

template <int N, bool SS = false, int NACC = 1, int MM = 128, int NISS = 1>
__global__ void k_ts(const uint16_t* A, const uint16_t* B, float* D, int K, long long* cyc, int reps) {
  // A: [128][K] fp16 row-major; B: [N][K] fp16; D: [128][N]
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // B into smem in the canonical layout
  for (int i = threadIdx.x; i < N * K; i += blockDim.x) {
    int n = i / K, k = i % K;
    int ks = k / 16, c = (k / 8) % 2, e = k % 8;
    reinterpret_cast<uint16_t*>(smem)[((ks * 2 + c) * N + n) * 8 + e] = B[(size_t)n * K + k];
  }
  for (int i = threadIdx.x; i < 128 * K; i += blockDim.x) {
    int m = i / K, k = i % K;
    int ks = k / 16, c = (k / 8) % 2, e = k % 8;
    reinterpret_cast<uint16_t*>(smem + N * K * 2)[((ks * 2 + c) * 128 + m) * 8 + e] = A[(size_t)m * K + k];
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(NISS));
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
  // A: warp w (w < 4) writes rows 32w..32w+31; columns [0, K/2) ; D at columns 128..
  if (warp < 4) {
    const int r = warp * 32 + lane;
    for (int c0 = 0; c0 < K / 2; c0 += 8) {
      uint32_t v[8];
      for (int j = 0; j < 8; ++j) {
        uint32_t lo = A[(size_t)r * K + 2 * (c0 + j)], hi = A[(size_t)r * K + 2 * (c0 + j) + 1];
        v[j] = lo | (hi << 16);
      }
      uint32_t ta = tb + ((uint32_t)(warp * 32) << 16) + c0;
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(ta), "r"(v[0]),
                   "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t dcol = 128;
  if ((threadIdx.x & 31) == 0 && threadIdx.x / 32 < NISS) {
    const uint32_t dcol2 = dcol + (threadIdx.x / 32) * 128;
    long long t0 = clock64();
    const uint64_t bd0 = bdesc(smem_u32(smem), N * 16, 128);
    const uint64_t ad0 = bdesc(smem_u32(smem) + N * K * 2, 128 * 16, 128);
    for (int rep = 0; rep < reps; ++rep) {
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        const uint64_t bd = bd0 + (uint64_t)((ks * 2 * N * 16) >> 4);
        const uint32_t acc = (ks >= NACC || rep > 0) ? 1u : 0u;
        if constexpr (SS) {
          const uint64_t ad = ad0 + (uint64_t)((ks * 2 * 128 * 16) >> 4);
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tb + dcol),
                       "l"(ad), "l"(bd), "r"(idesc_f16(128, N)), "r"(acc));
        } else {
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tb + dcol2 + (ks % NACC) * N),
                       "r"(tb + ks * 8), "l"(bd), "r"(idesc_f16(MM, N)), "r"(acc));
        }
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    asm volatile("{\n\t.reg .pred P;\n\tW: mbarrier.try_wait.parity.shared.b64 P, [%0], 0;\n\t@!P bra W;\n\t}" ::"r"(
        smem_u32(&bar)));
    if (threadIdx.x == 0) cyc[0] = clock64() - t0;
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp < 4) {
    const int r = warp * 32 + lane;
    for (int c0 = 0; c0 < N; c0 += 8) {
      uint32_t v[8];
      uint32_t ta = tb + ((uint32_t)(warp * 32) << 16) + dcol + c0;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                   : "r"(ta));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      for (int j = 0; j < 8; ++j) D[(size_t)r * N + c0 + j] = __uint_as_float(v[j]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(512));
}

static uint16_t f2h(float f) { __half h = __float2half(f); return *reinterpret_cast<uint16_t*>(&h); }

template <int N, bool SS = false, int NACC = 1, int MM = 128, int NISS = 1>
int run(int K, int reps) {
  std::vector<uint16_t> A(128 * K), B(N * K);
  std::vector<float> Af(128 * K), Bf(N * K), Dref(128 * N, 0.f), D(128 * N);
  srand(1);
  for (int i = 0; i < 128 * K; ++i) { Af[i] = (float)(rand() % 31 - 15); A[i] = f2h(Af[i]); }
  for (int i = 0; i < N * K; ++i) { Bf[i] = (float)(rand() % 9 - 4) * 0.25f; B[i] = f2h(Bf[i]); }
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < N; ++n) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += (double)Af[m * K + k] * Bf[n * K + k];
      Dref[m * N + n] = (float)(s * reps);
    }
  uint16_t *dA, *dB; float* dD; long long* dc;
  CK(cudaMalloc(&dA, A.size() * 2)); CK(cudaMalloc(&dB, B.size() * 2)); CK(cudaMalloc(&dD, D.size() * 4));
  CK(cudaMalloc(&dc, 8));
  CK(cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice));
  int smem = N * K * 2 + 128 * K * 2 + 1024;
  CK(cudaFuncSetAttribute(k_ts<N, SS, NACC, MM, NISS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  k_ts<N, SS, NACC, MM, NISS><<<1, 256, smem>>>(dA, dB, dD, K, dc, reps);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
  long long cyc; CK(cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost));
  int bad = 0; double maxe = 0;
  for (int i = 0; i < 128 * N; ++i) {
    double e = fabs(D[i] - Dref[i]);
    maxe = e > maxe ? e : maxe;
    if (NACC == 1 && MM == 128 && NISS == 1 && e > 1e-3 * (1 + fabs(Dref[i]))) { if (bad < 5) printf("  mismatch m=%d n=%d got %f want %f\n", i / N, i % N, D[i], Dref[i]); ++bad; }
  }
  printf("M=%d NISS=%d NACC=%d %s N=%d K=%d reps=%d: %s (max err %.3g), %lld cycles for %d MMAs = %.1f cyc/MMA\n", MM, NISS, NACC, SS ? "SS" : "TS", N, K, reps,
         bad ? "FAIL" : "OK", maxe, cyc, reps * K / 16, (double)cyc / (NISS * reps * K / 16));
  cudaFree(dA); cudaFree(dB); cudaFree(dD); cudaFree(dc);
  return bad;
}

int main() {
  int bad = 0;
  bad += run<16>(128, 64);
  bad += run<16, false, 1, 64>(128, 64);
  bad += run<32, false, 1, 64>(128, 64);
  bad += run<16, false, 1, 128, 2>(128, 64);
  bad += run<16, false, 1, 128, 4>(128, 64);
  bad += run<16, false, 1, 64, 2>(128, 64);
  printf(bad ? "PROBE FAIL\n" : "PROBE OK\n");
  return bad ? 1 : 0;
}
