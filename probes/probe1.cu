// Round-1 B200 probes: HBM streaming (LDG.128 vs cp.async.bulk ring), mma.sync bf16 rate.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("err %s line %d\n", cudaGetErrorString(e), __LINE__); return 1;}}while(0)

__global__ void ldg_stream(const int4* __restrict__ p, size_t n, int4* out) {
  int4 acc = make_int4(0,0,0,0);
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  #pragma unroll 8
  for (; i < n; i += stride) {
    int4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x),"=r"(v.y),"=r"(v.z),"=r"(v.w) : "l"(p+i));
    acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
  }
  if (acc.x == 0x12345 && acc.y == 7) out[0] = acc;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p){ return (uint32_t)__cvta_generic_to_shared(p); }

template<int STAGES, int CHUNK>
__global__ void bulk_stream(const char* __restrict__ p, size_t nchunks, int* out) {
  extern __shared__ __align__(128) char sm[];
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
  int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  int nconsumer = blockDim.x/32 - 1;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      asm volatile("mbarrier.init.shared.b64 [%0], %1;" :: "r"(smem_u32(&full[s])), "r"(1));
      asm volatile("mbarrier.init.shared.b64 [%0], %1;" :: "r"(smem_u32(&empty[s])), "r"(nconsumer));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  size_t first = blockIdx.x, step = gridDim.x;
  if (warp == nconsumer) {
    if (lane == 0) {
      int s = 0; uint32_t ph = 0;
      for (size_t c = first; c < nchunks; c += step) {
        // wait empty
        asm volatile("{ .reg .pred P; W: mbarrier.try_wait.parity.shared.b64 P, [%0], %1; @!P bra W; }" :: "r"(smem_u32(&empty[s])), "r"(ph ^ 1));
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" :: "r"(smem_u32(&full[s])), "r"(CHUNK));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
          :: "r"(smem_u32(sm + s*CHUNK)), "l"(p + c*CHUNK), "r"(CHUNK), "r"(smem_u32(&full[s])) : "memory");
        if (++s == STAGES) { s = 0; ph ^= 1; }
      }
    }
  } else {
    int s = 0; uint32_t ph = 0; int acc = 0;
    for (size_t c = first; c < nchunks; c += step) {
      asm volatile("{ .reg .pred P; W: mbarrier.try_wait.parity.shared.b64 P, [%0], %1; @!P bra W; }" :: "r"(smem_u32(&full[s])), "r"(ph));
      const int4* q = (const int4*)(sm + s*CHUNK);
      for (int i = warp*32 + lane; i < CHUNK/16; i += nconsumer*32) { int4 v = q[i]; acc ^= v.x ^ v.w; }
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared.b64 _, [%0];" :: "r"(smem_u32(&empty[s])));
      if (++s == STAGES) { s = 0; ph ^= 1; }
    }
    if (acc == 0x7777777) out[0] = acc;
  }
}

__global__ void mma_rate(int iters, float* out) {
  uint32_t a0 = threadIdx.x, a1 = a0*3, a2 = a0*5, a3 = a0*7, b0 = a0*11, b1 = a0*13;
  float c[4][4] = {};
  for (int i = 0; i < iters; ++i) {
    #pragma unroll
    for (int j = 0; j < 4; ++j)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3]) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0; for (int j = 0; j < 4; ++j) for (int k = 0; k < 4; ++k) s += c[j][k];
  if (s == 1.2345f) out[0] = s;
}

__global__ void dequant_rate(int iters, const uint32_t* in, uint32_t* out) {
  uint32_t w = in[threadIdx.x & 31] + threadIdx.x;
  uint32_t acc = 0;
  for (int i = 0; i < iters; ++i) {
    #pragma unroll
    for (int j = 0; j < 8; ++j) {
      uint32_t r0, r1, r2, r3;
      uint32_t w1 = w >> 4, w2 = w >> 8, w3 = w >> 12;
      asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r0) : "r"(w), "r"(0x000F000Fu), "r"(0x43004300u));
      asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r1) : "r"(w1), "r"(0x000F000Fu), "r"(0x43004300u));
      asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r2) : "r"(w2), "r"(0x000F000Fu), "r"(0x43004300u));
      asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r3) : "r"(w3), "r"(0x000F000Fu), "r"(0x43004300u));
      acc += r0 ^ r1 ^ r2 ^ r3;  // stand-in consumer
      w = w * 1664525u + 1013904223u;
    }
  }
  if (acc == 0x1234567) out[0] = acc;
}

int main() {
  int dev = 0; cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, dev));
  printf("device %s SMs %d L2 %d MB smemOptin %zu KB clock %d MHz\n", prop.name, prop.multiProcessorCount, prop.l2CacheSize>>20, prop.sharedMemPerBlockOptin>>10, prop.clockRate/1000);
  size_t bytes = 4ull << 30;
  char* buf; CK(cudaMalloc(&buf, bytes)); CK(cudaMemset(buf, 1, bytes));
  int* dout; CK(cudaMalloc(&dout, 1024));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int nsm = prop.multiProcessorCount;
  for (int bpsm : {1, 2, 4, 8}) for (int threads : {256, 512}) {
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); ldg_stream<<<nsm*bpsm, threads>>>((const int4*)buf, bytes/16, (int4*)dout); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    printf("LDG.128 stream grid=%d*%d thr=%d: %.1f GB/s\n", nsm, bpsm, threads, bytes / best / 1e6);
  }
  CK(cudaGetLastError());
#define RUNBULK(ST, CH, BPSM, THR) { \
    auto k = bulk_stream<ST, CH>; size_t sm = (size_t)ST*CH; CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)); \
    float best = 1e9; for (int r = 0; r < 5; ++r) { cudaEventRecord(e0); k<<<nsm*BPSM, THR, sm>>>(buf, bytes/CH, dout); cudaEventRecord(e1); cudaEventSynchronize(e1); \
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms; } CK(cudaGetLastError()); \
    printf("bulk stream stages=%d chunk=%d bpsm=%d thr=%d: %.1f GB/s\n", ST, CH, BPSM, THR, bytes/best/1e6); }
  RUNBULK(4, 16384, 1, 288); RUNBULK(6, 16384, 1, 288); RUNBULK(8, 16384, 1, 288); RUNBULK(4, 16384, 2, 288);
  RUNBULK(12, 8192, 1, 288); RUNBULK(6, 8192, 2, 288); RUNBULK(4, 32768, 1, 288); RUNBULK(3, 32768, 2, 288);
  float* fo; CK(cudaMalloc(&fo, 64));
  for (int wpsm : {4, 8, 16, 32}) {
    int iters = 4096; float best = 1e9;
    for (int r = 0; r < 3; ++r) { cudaEventRecord(e0); mma_rate<<<nsm, wpsm*32>>>(iters, fo); cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms; }
    double flops = 2.0 * 16 * 8 * 16 * 4.0 * iters * wpsm * nsm;
    printf("mma.sync m16n8k16 bf16 warps/SM=%d: %.1f TFLOP/s\n", wpsm, flops / best / 1e9);
  }
  for (int wpsm : {8, 16, 32}) {
    int iters = 4096; float best = 1e9;
    for (int r = 0; r < 3; ++r) { cudaEventRecord(e0); dequant_rate<<<nsm, wpsm*32>>>(iters, (uint32_t*)dout, (uint32_t*)dout); cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms; }
    double w = 8.0 * 8 * iters * wpsm * 32 * nsm;
    printf("dequant lop3 (8 int4/iter) warps/SM=%d: %.2f Tweights/s\n", wpsm, w / best / 1e9 / 1e3);
  }
  CK(cudaGetLastError());
  return 0;
}
