// attention.cu -- tree-masked GQA attention.
//
// Every tree node attends to the committed prefix [0, L) plus its
// ancestors-or-self among the tree rows [L, L+T) (square mask P:321, one
// ancestor bitmask per node).  One CTA = (kv head, key split, row chunk).
// The rows are the G query heads x T nodes that share the kv head (GQA), so
// each K/V tile is read from HBM once per kv head.  Warps are laid out as
// (16-row block) x (key slice of every 64-key tile), so a CTA keeps 8 warps
// busy even for the 64 rows of a T=8 tree.  K/V tiles (pre-swizzled in the
// cache layout) arrive through the TMA bulk engine into a double-buffered
// ring; prefix tiles are requested before the PDL wait because they do not
// depend on the QKV kernel.  QK^T and PV run on mma.sync (fp16, fp32
// accumulate); online softmax in fp32 (R11).
//
// The split partials are merged inside the same kernel ("the
// threadblocks aggregate the sum ... without explicit synchronization across
// thread blocks or extra kernel launches"): the CTAs of one kv head meet at a
// flag counter and each then merges a slice of the rows by log-sum-exp,
// writing fp16 straight into the O-projection's fragment-ordered input.
#include <cooperative_groups.h>

#include "common.cuh"
#include "internal.h"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace ss {

template <int D, int RB, bool CL = false>
struct AttnCfg {
  static constexpr int KS = (8 / RB) < 1 ? 1 : ((8 / RB) > 4 ? 4 : (8 / RB));  // key slices
  static constexpr int WARPS = RB * KS;
  static constexpr int ROWS = RB * 16;
  static constexpr int KEYS = kKvTile / KS;   // keys per warp per tile (64, 32 or 16)
  static constexpr int NTK = KEYS / 8;        // score n-tiles per warp
  static constexpr int TILE_ELEMS = kKvTile * D;
  // K/V tiles in flight: a CTA's whole range at L=4K; the cluster variant
  // keeps 2 so that two CTAs fit an SM (16-CTA clusters must be co-resident)
#ifdef SS_EXP_ANBUF
  static constexpr int NBUF = CL ? 2 : SS_EXP_ANBUF;
#else
  static constexpr int NBUF = CL ? 2 : 4;
#endif
  static constexpr size_t SMEM = (size_t)ROWS * D * 2 + 2 * NBUF * (size_t)TILE_ELEMS * 2;
  // the in-CTA key-slice merge (and the cluster variant's published partial
  // plus its merge weights) reuse the K/V ring
  static_assert((size_t)(KS - 1) * ROWS * (D + 2) * 4 <= 2 * NBUF * (size_t)TILE_ELEMS * 2, "merge buffer");
  static_assert(!CL || (size_t)ROWS * D * 4 + 2 * 16 * 16 * 4 <= 2 * NBUF * (size_t)TILE_ELEMS * 2, "cluster buffer");
};

#ifdef SS_ATTN_TRACE
__device__ unsigned long long g_at[256 * 8];
__device__ unsigned long long g_att[256 * 16];  // per CTA: [tile][waited, computed]
SS_DEV unsigned long long gtime_at() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define ATR(ev) do { if (threadIdx.x == 0 && a.layer == 0) { const int cta = (blockIdx.y * gridDim.x + blockIdx.x) * gridDim.z + blockIdx.z; if (cta < 256) g_at[cta * 8 + (ev)] = gtime_at(); } } while (0)
#else
#define ATR(ev) do {} while (0)
#endif
// CL = true: the S splits of a (kv head, row chunk) form one thread-block
// cluster and merge their partials through distributed shared memory (no
// global workspace, no grid-level meet); CL = false: global workspace merge.
template <int D, int RB, bool CL>
__global__ void __launch_bounds__(AttnCfg<D, RB, CL>::WARPS * 32, 1) attn_kernel(AttnArgs a) {
  using C = AttnCfg<D, RB, CL>;
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int NBUF = C::NBUF;
  __shared__ __align__(8) uint64_t full[NBUF];
  __shared__ __align__(8) uint64_t qbar;
  constexpr int ROWS = C::ROWS, TILE_ELEMS = C::TILE_ELEMS, NTHR = C::WARPS * 32;
  uint16_t* Qs = reinterpret_cast<uint16_t*>(smem);  // [ROWS][D] fp16, swizzled
  uint16_t* Ks = Qs + ROWS * D;                      // [NBUF][64][D]
  uint16_t* Vs = Ks + NBUF * TILE_ELEMS;

  const int split = blockIdx.x, kvh = blockIdx.y, z = blockIdx.z;
  const int S = gridDim.x, Z = gridDim.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rb = warp % RB, ks = warp / RB;
  const int gq = lane >> 2, tq = lane & 3;
  DevState* st = a.st;
  // L (committed by an earlier step) and T (written by this step's ingest
  // kernel, which completed before the QKV kernel could trigger our launch)
  // are stable here; only the tree rows [L, L+T) and q come from the QKV
  // kernel this launch depends on.
  const int L = st->L, T = st->T;
  const int G = a.G;
  const int Mrows = G * T;
  const int m0 = z * ROWS;
  const int ntiles = (L + T + kKvTile - 1) / kKvTile;
  // Split count from the RUNTIME length (a captured graph replays at any L):
  // the fewest splits with the same longest split; surplus CTAs leave at once
  // (the cluster variant keeps all S CTAs: they meet in cl.sync).
  const int per = (ntiles + S - 1) / S;
  const int SE = CL ? S : (ntiles + per - 1) / per;
  if (!CL && split >= SE) return;
  const int t0 = CL ? (int)((long)split * ntiles / S) : split * per;
  const int t1 = CL ? (int)((long)(split + 1) * ntiles / S) : min(ntiles, t0 + per);
  const size_t head_base = ((size_t)a.layer * a.Hkv_l + kvh) * a.max_ctx_pad * D;
  ATR(0);

  if (threadIdx.x == 0) {
    for (int i = 0; i < NBUF; ++i) mbar_init(&full[i], 1);
    mbar_init(&qbar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  int issued = 0;
  if (threadIdx.x == 0) {  // prefix tiles: independent of the QKV kernel
    for (int i = 0; i < NBUF && t0 + i < t1; ++i) {
      const int tile = t0 + i;
      if ((tile + 1) * kKvTile > L) break;
      mbar_expect_tx(&full[i], 2 * TILE_ELEMS * 2);
      bulk_g2s_nohint(Ks + i * TILE_ELEMS, a.kc + head_base + (size_t)tile * TILE_ELEMS, TILE_ELEMS * 2, &full[i]);
      bulk_g2s_nohint(Vs + i * TILE_ELEMS, a.vc + head_base + (size_t)tile * TILE_ELEMS, TILE_ELEMS * 2, &full[i]);
      ++issued;
    }
  }
  pdl_wait();
  pdl_trigger();
  ATR(1);
  if (threadIdx.x == 0) {
    for (int i = issued; i < NBUF && t0 + i < t1; ++i) {
      const int tile = t0 + i;
      mbar_expect_tx(&full[i], 2 * TILE_ELEMS * 2);
      bulk_g2s_nohint(Ks + i * TILE_ELEMS, a.kc + head_base + (size_t)tile * TILE_ELEMS, TILE_ELEMS * 2, &full[i]);
      bulk_g2s_nohint(Vs + i * TILE_ELEMS, a.vc + head_base + (size_t)tile * TILE_ELEMS, TILE_ELEMS * 2, &full[i]);
    }
    // q rows [m0, m0 + ROWS) of this kv head (fp16, swizzled by the QKV
    // epilogue).  Rows >= G*T are stale but finite and masked below.
    mbar_expect_tx(&qbar, ROWS * D * 2);
    bulk_g2s_nohint(Qs, a.qbuf + ((size_t)kvh * (G * SS_MAX_TREE) + m0) * D, ROWS * D * 2, &qbar);
  }
  mbar_wait(&qbar, 0);
  ATR(2);
  const int qr = rb * 16 + (lane & 15);
  const uint16_t* qrow = Qs + qr * D;
  // the warp's Q fragments stay in registers for all tiles (shared-memory
  // bandwidth, not math, bounds this loop: K/V are re-read by every row block)
  uint32_t qf[D / 16][4];
#pragma unroll
  for (int kk = 0; kk < D / 16; ++kk) ldmatrix_x4(qf[kk], qrow + (((kk * 2 + (lane >> 4)) ^ (qr & 7)) << 3));

  const int rowA = m0 + rb * 16 + gq, rowB = rowA + 8;
  const int tokA = min(rowA / G, SS_MAX_TREE - 1), tokB = min(rowB / G, SS_MAX_TREE - 1);
  const unsigned long long ancA = st->anc[tokA], ancB = st->anc[tokB];
  const bool okA = rowA < Mrows, okB = rowB < Mrows;
  const float sl2 = rsqrtf((float)D) * 1.4426950408889634f;
  const int kofs = ks * C::KEYS;  // this warp's key slice inside each tile

  float mA = -INFINITY, mB = -INFINITY, lA = 0.f, lB = 0.f;
  float o[D / 8][4];
#pragma unroll
  for (int n = 0; n < D / 8; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;

  for (int it = t0; it < t1; ++it) {
    const int b = (it - t0) % NBUF;
    const uint32_t phase = ((it - t0) / NBUF) & 1;
    mbar_wait(&full[b], phase);
#ifdef SS_ATTN_TRACE
    if (threadIdx.x == 0 && a.layer == 0 && it - t0 < 8) {
      const int cta = (blockIdx.y * gridDim.x + blockIdx.x) * gridDim.z + blockIdx.z;
      if (cta < 256) g_att[cta * 16 + (it - t0) * 2] = gtime_at();
    }
#endif
    const uint16_t* Kt = Ks + b * TILE_ELEMS;
    const uint16_t* Vt = Vs + b * TILE_ELEMS;

    float sc[C::NTK][4];
#pragma unroll
    for (int n = 0; n < C::NTK; ++n) sc[n][0] = sc[n][1] = sc[n][2] = sc[n][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
#pragma unroll
      for (int np = 0; np < C::NTK / 2; ++np) {
        const int key = kofs + np * 16 + (lane & 7) + ((lane >> 4) << 3);
        const int ch = kk * 2 + ((lane >> 3) & 1);
        uint32_t kb[4];
        ldmatrix_x4(kb, Kt + key * D + ((ch ^ (key & 7)) << 3));
        mma_f16_16816(sc[2 * np], qf[kk], kb[0], kb[1]);
        mma_f16_16816(sc[2 * np + 1], qf[kk], kb[2], kb[3]);
      }
    }
    // mask: prefix always visible; tree rows by ancestor bit; beyond L+T never
    const int kbase = it * kKvTile + kofs;
    float mxA = -INFINITY, mxB = -INFINITY;
#pragma unroll
    for (int n = 0; n < C::NTK; ++n) {
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
    }
    mxA = fmaxf(mxA, __shfl_xor_sync(0xffffffffu, mxA, 1));
    mxA = fmaxf(mxA, __shfl_xor_sync(0xffffffffu, mxA, 2));
    mxB = fmaxf(mxB, __shfl_xor_sync(0xffffffffu, mxB, 1));
    mxB = fmaxf(mxB, __shfl_xor_sync(0xffffffffu, mxB, 2));
    const float mnA = fmaxf(mA, mxA), mnB = fmaxf(mB, mxB);
    const float uA = (mnA == -INFINITY) ? 0.f : mnA, uB = (mnB == -INFINITY) ? 0.f : mnB;
    const float alA = exp2f(mA - uA), alB = exp2f(mB - uB);
    float sumA = 0.f, sumB = 0.f;
    uint32_t pa[C::NTK / 2][4];
#pragma unroll
    for (int n = 0; n < C::NTK; ++n) {
      const float p0 = exp2f(sc[n][0] - uA), p1 = exp2f(sc[n][1] - uA);
      const float p2 = exp2f(sc[n][2] - uB), p3 = exp2f(sc[n][3] - uB);
      sumA += p0 + p1;
      sumB += p2 + p3;
      pa[n >> 1][(n & 1) * 2 + 0] = pack_half2(p0, p1);
      pa[n >> 1][(n & 1) * 2 + 1] = pack_half2(p2, p3);
    }
    sumA += __shfl_xor_sync(0xffffffffu, sumA, 1);
    sumA += __shfl_xor_sync(0xffffffffu, sumA, 2);
    sumB += __shfl_xor_sync(0xffffffffu, sumB, 1);
    sumB += __shfl_xor_sync(0xffffffffu, sumB, 2);
    lA = lA * alA + sumA;
    lB = lB * alB + sumB;
    mA = mnA;
    mB = mnB;
    if (__any_sync(0xffffffffu, alA != 1.f || alB != 1.f)) {  // running max moved: rescale
#pragma unroll
      for (int n = 0; n < D / 8; ++n) {
        o[n][0] *= alA; o[n][1] *= alA; o[n][2] *= alB; o[n][3] *= alB;
      }
    }
#pragma unroll
    for (int kk = 0; kk < C::NTK / 2; ++kk) {
#pragma unroll
      for (int dp = 0; dp < D / 16; ++dp) {
        const int key = kofs + kk * 16 + (lane & 7) + (((lane >> 3) & 1) << 3);
        const int ch = dp * 2 + (lane >> 4);
        uint32_t vb[4];
        ldmatrix_x4_trans(vb, Vt + key * D + ((ch ^ (key & 7)) << 3));
        mma_f16_16816(o[2 * dp], pa[kk], vb[0], vb[1]);
        mma_f16_16816(o[2 * dp + 1], pa[kk], vb[2], vb[3]);
      }
    }
    if (it + NBUF < t1) {
      __syncthreads();  // every warp is done with buffer b: refill it with tile it + NBUF
      if (threadIdx.x == 0) {
        fence_proxy_async_smem();  // the ldmatrix reads above before the TMA overwrite
        mbar_expect_tx(&full[b], 2 * TILE_ELEMS * 2);
        bulk_g2s_nohint(Ks + b * TILE_ELEMS, a.kc + head_base + (size_t)(it + NBUF) * TILE_ELEMS, TILE_ELEMS * 2,
                        &full[b]);
        bulk_g2s_nohint(Vs + b * TILE_ELEMS, a.vc + head_base + (size_t)(it + NBUF) * TILE_ELEMS, TILE_ELEMS * 2,
                        &full[b]);
      }
    }
  }

  ATR(3);
  // ---- merge the KS key-slice partials of each row inside the CTA (shared
  // memory, reusing the K/V ring), so only one partial per split goes out
  const int grp = kvh * Z + z;
  const int P = SE;  // partials per (kv head, row chunk)
  const int ra = rb * 16 + gq, rbb = ra + 8;
  if constexpr (C::KS > 1) {
    __syncthreads();  // every warp is done with the K/V ring
    float* so = reinterpret_cast<float*>(Ks);          // [KS-1][ROWS][D]
    float* sml = so + (C::KS - 1) * ROWS * D;          // [KS-1][ROWS][2]
    if (ks > 0) {
      float* dst = so + (size_t)(ks - 1) * ROWS * D;
#pragma unroll
      for (int n = 0; n < D / 8; ++n) {
        *reinterpret_cast<float2*>(dst + ra * D + n * 8 + 2 * tq) = make_float2(o[n][0], o[n][1]);
        *reinterpret_cast<float2*>(dst + rbb * D + n * 8 + 2 * tq) = make_float2(o[n][2], o[n][3]);
      }
      if (tq == 0) {
        *reinterpret_cast<float2*>(sml + ((ks - 1) * ROWS + ra) * 2) = make_float2(mA, lA);
        *reinterpret_cast<float2*>(sml + ((ks - 1) * ROWS + rbb) * 2) = make_float2(mB, lB);
      }
    }
    __syncthreads();
    if (ks == 0) {
#pragma unroll
      for (int k2 = 1; k2 < C::KS; ++k2) {
        const float* src = so + (size_t)(k2 - 1) * ROWS * D;
        const float2 mlA = *reinterpret_cast<const float2*>(sml + ((k2 - 1) * ROWS + ra) * 2);
        const float2 mlB = *reinterpret_cast<const float2*>(sml + ((k2 - 1) * ROWS + rbb) * 2);
        const float nA = fmaxf(mA, mlA.x), nB = fmaxf(mB, mlB.x);
        const float a1A = (mA == -INFINITY) ? 0.f : exp2f(mA - nA), a2A = (mlA.x == -INFINITY) ? 0.f : exp2f(mlA.x - nA);
        const float a1B = (mB == -INFINITY) ? 0.f : exp2f(mB - nB), a2B = (mlB.x == -INFINITY) ? 0.f : exp2f(mlB.x - nB);
#pragma unroll
        for (int n = 0; n < D / 8; ++n) {
          const float2 pa = *reinterpret_cast<const float2*>(src + ra * D + n * 8 + 2 * tq);
          const float2 pb = *reinterpret_cast<const float2*>(src + rbb * D + n * 8 + 2 * tq);
          o[n][0] = o[n][0] * a1A + pa.x * a2A;
          o[n][1] = o[n][1] * a1A + pa.y * a2A;
          o[n][2] = o[n][2] * a1B + pb.x * a2B;
          o[n][3] = o[n][3] * a1B + pb.y * a2B;
        }
        lA = lA * a1A + mlA.y * a2A;
        lB = lB * a1B + mlB.y * a2B;
        mA = nA;
        mB = nB;
      }
    }
  }
  if constexpr (CL) {
    // ---- publish the split's partial in shared memory, merge a slice of the
    // rows from every split of the cluster (DSMEM), R11 log-sum-exp
    __shared__ float2 s_pml[256];                      // (m, l) per row
    float* pub = reinterpret_cast<float*>(Ks);         // [ROWS][D] fp32
    __syncthreads();                                   // the in-CTA merge is done reading the ring
    if (ks == 0) {
#pragma unroll
      for (int n = 0; n < D / 8; ++n) {
        *reinterpret_cast<float2*>(pub + ra * D + n * 8 + 2 * tq) = make_float2(o[n][0], o[n][1]);
        *reinterpret_cast<float2*>(pub + rbb * D + n * 8 + 2 * tq) = make_float2(o[n][2], o[n][3]);
      }
      if (tq == 0) {
        s_pml[ra] = make_float2(mA, lA);
        s_pml[rbb] = make_float2(mB, lB);
      }
    }
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();
    ATR(5);
    float* s_w = reinterpret_cast<float*>(Ks) + ROWS * D;  // [rows_here][S] weights (after pub)
    const int rows_per = (ROWS + S - 1) / S;
    const int r_first = split * rows_per, r_end = min(ROWS, r_first + rows_per);
    const int nr = r_end > r_first ? r_end - r_first : 0;
    for (int i = threadIdx.x; i < nr * S; i += NTHR) {
      const int rr = i / S, p2 = i - rr * S;
      const float2* pml = cl.map_shared_rank(s_pml, p2);
      const float2 v = pml[r_first + rr];
      s_w[i] = v.x;
      s_w[nr * S + i] = v.y;
    }
    __syncthreads();
    for (int rr = warp; rr < nr; rr += C::WARPS) {  // one warp per row: m*, l*, weights
      float mx = -INFINITY;
      for (int p2 = lane; p2 < S; p2 += 32) mx = fmaxf(mx, s_w[rr * S + p2]);
      mx = warp_max(mx);
      float l = 0.f;
      for (int p2 = lane; p2 < S; p2 += 32) {
        const float ms = s_w[rr * S + p2];
        const float w = (ms == -INFINITY) ? 0.f : exp2f(ms - mx);
        l += w * s_w[nr * S + rr * S + p2];
        s_w[rr * S + p2] = w;
      }
      l = warp_sum(l);
      __syncwarp();
      const float inv = l > 0.f ? 1.f / l : 0.f;
      for (int p2 = lane; p2 < S; p2 += 32) s_w[rr * S + p2] *= inv;
    }
    __syncthreads();
    for (int itm = threadIdx.x; itm < nr * (D / 4); itm += NTHR) {
      const int r = r_first + itm / (D / 4), c4 = itm % (D / 4);
      const int m = m0 + r;
      if (m >= Mrows) continue;
      const float* wr = s_w + (r - r_first) * S;
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
      for (int p2 = 0; p2 < S; ++p2) {
        const float w = wr[p2];
        const float4 ov = *reinterpret_cast<const float4*>(cl.map_shared_rank(pub, p2) + r * D + 4 * c4);
        acc.x += w * ov.x;
        acc.y += w * ov.y;
        acc.z += w * ov.z;
        acc.w += w * ov.w;
      }
      const int t = m / G, hq = kvh * G + (m % G);
      const int k = hq * D + 4 * c4;
      const uint32_t p01 = pack_half2(acc.x, acc.y), p23 = pack_half2(acc.z, acc.w);
      *reinterpret_cast<uint32_t*>(a.act_out + act_frag_offset(t, k, a.NT)) = p01;
      *reinterpret_cast<uint32_t*>(a.act_out + act_frag_offset(t, k + 2, a.NT)) = p23;
      // group sum X of the O-projection input (slots zeroed by the QKV kernel)
      atomicAdd(reinterpret_cast<float*>(a.act_out + act_xsum_offset(t, k >> 7, a.NT)),
                half2_sum(p01) + half2_sum(p23));
    }
    ATR(6);
    cl.sync();  // peers may still be reading this CTA's partial
    return;
  }
  // ---- the split's partial -> workspace
  if (ks == 0) {
    float* ws = a.ws + (((size_t)grp * P + split) * 256) * D;
    float* ml = a.ml + (((size_t)grp * P + split) * 256) * 2;
#pragma unroll
    for (int n = 0; n < D / 8; ++n) {
      *reinterpret_cast<float2*>(ws + (size_t)ra * D + n * 8 + 2 * tq) = make_float2(o[n][0], o[n][1]);
      *reinterpret_cast<float2*>(ws + (size_t)rbb * D + n * 8 + 2 * tq) = make_float2(o[n][2], o[n][3]);
    }
    if (tq == 0) {
      *reinterpret_cast<float2*>(ml + ra * 2) = make_float2(mA, lA);
      *reinterpret_cast<float2*>(ml + rbb * 2) = make_float2(mB, lB);
    }
  }
  // ---- meet the other splits of this (kv head, row chunk): the barrier
  // orders every thread's partial stores before thread 0's GPU-scope fence
  // (cumulative), which precedes its arrival; thread 0 spins, fences again
  // (acquire side) and releases the CTA.
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    ATR(4);
    atomicAdd(&a.bar[grp * 2], 1);
    while (*reinterpret_cast<volatile int*>(&a.bar[grp * 2]) < SE) spin_pause();
    __threadfence();
    ATR(5);
  }
  __syncthreads();
  // ---- merge a slice of the rows across the P partials (log-sum-exp, R11).
  // Items = (row, 4-float chunk); the CTA's items are a contiguous slice.  The
  // per-(row, partial) weights exp2(m_p - m*) / l* go through shared memory and
  // every thread issues its P loads back to back (no serial L2 chain).
  {
    float* s_w = reinterpret_cast<float*>(Ks);  // reuse the K/V ring: [rows_here][P] x 2
    const int n_items = ROWS * (D / 4);
    const int i_lo = (int)((long)split * n_items / SE), i_hi = (int)((long)(split + 1) * n_items / SE);
    const int r_first = i_lo / (D / 4), r_last = (i_hi - 1) / (D / 4);
    const int nr = (i_hi > i_lo) ? r_last - r_first + 1 : 0;
    const float* wsg = a.ws + ((size_t)grp * P * 256) * D;
    const float* mlg = a.ml + ((size_t)grp * P * 256) * 2;
    for (int i = threadIdx.x; i < nr * P; i += NTHR) {
      const int rr = i / P, p2 = i % P;
      const float2 v = __ldcg(reinterpret_cast<const float2*>(mlg + ((size_t)p2 * 256 + r_first + rr) * 2));
      s_w[i] = v.x;
      s_w[nr * P + i] = v.y;
    }
    __syncthreads();
    for (int rr = warp; rr < nr; rr += C::WARPS) {  // one warp per row: m*, l*, weights
      float mx = -INFINITY;
      for (int p2 = lane; p2 < P; p2 += 32) mx = fmaxf(mx, s_w[rr * P + p2]);
      mx = warp_max(mx);
      float l = 0.f;
      for (int p2 = lane; p2 < P; p2 += 32) {
        const float ms = s_w[rr * P + p2];
        const float w = (ms == -INFINITY) ? 0.f : exp2f(ms - mx);
        l += w * s_w[nr * P + rr * P + p2];
        s_w[rr * P + p2] = w;
      }
      l = warp_sum(l);
      __syncwarp();
      const float inv = l > 0.f ? 1.f / l : 0.f;
      for (int p2 = lane; p2 < P; p2 += 32) s_w[rr * P + p2] *= inv;
    }
    __syncthreads();
    for (int itm = i_lo + threadIdx.x; itm < i_hi; itm += NTHR) {
      const int r = itm / (D / 4), c4 = itm % (D / 4);
      const int m = m0 + r;
      if (m >= Mrows) continue;
      const float* wr = s_w + (r - r_first) * P;
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 8
      for (int p2 = 0; p2 < P; ++p2) {
        const float w = wr[p2];
        const float4 ov = __ldcg(reinterpret_cast<const float4*>(wsg + ((size_t)p2 * 256 + r) * D + 4 * c4));
        acc.x += w * ov.x;
        acc.y += w * ov.y;
        acc.z += w * ov.z;
        acc.w += w * ov.w;
      }
      const int t = m / G, hq = kvh * G + (m % G);
      const int k = hq * D + 4 * c4;
      const uint32_t p01 = pack_half2(acc.x, acc.y), p23 = pack_half2(acc.z, acc.w);
      *reinterpret_cast<uint32_t*>(a.act_out + act_frag_offset(t, k, a.NT)) = p01;
      *reinterpret_cast<uint32_t*>(a.act_out + act_frag_offset(t, k + 2, a.NT)) = p23;
      // group sum X of the O-projection input (slots zeroed by the QKV kernel)
      atomicAdd(reinterpret_cast<float*>(a.act_out + act_xsum_offset(t, k >> 7, a.NT)), half2_sum(p01) + half2_sum(p23));
    }
  }
  __syncthreads();
  ATR(6);
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&a.bar[grp * 2 + 1], 1) == SE - 1) {
      a.bar[grp * 2] = 0;
      a.bar[grp * 2 + 1] = 0;
    }
  }
}

template <int D, int RB, bool CL>
static int occ_of() {
  static int occ_dev[kMaxDevices] = {0};  // per device (the smem opt-in is per device)
  using C = AttnCfg<D, RB, CL>;
  const int dev = current_device();
  if (!occ_dev[dev]) {
    int occ = 1;
    cudaFuncSetAttribute(attn_kernel<D, RB, CL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, attn_kernel<D, RB, CL>, C::WARPS * 32, C::SMEM);
    occ_dev[dev] = occ < 1 ? 1 : occ;
  }
  return occ_dev[dev];
}

static int rb_for(int G, int NT) {
  int rb = (G * NT * 8 + 15) / 16;
  int r = 1;
  while (r < rb && r < 16) r <<= 1;
  return r;
}

constexpr int kAttnCluster = 16;  // splits per (kv head, row chunk) in the cluster variant (non-portable size)

// Whether 16-CTA clusters of the cluster variant can be scheduled (queried once).
template <int D, int RB>
static bool cluster_ok() {
  static int ok_dev[kMaxDevices] = {0};  // 0 unknown, 1 yes, 2 no (per device)
  const int dev = current_device();
  int& ok = ok_dev[dev];
  if (ok == 0) {
    using C = AttnCfg<D, RB, true>;
    auto k = attn_kernel<D, RB, true>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(kAttnCluster, 1, 1);
    cfg.blockDim = dim3(C::WARPS * 32, 1, 1);
    cfg.dynamicSmemBytes = C::SMEM;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = kAttnCluster;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    ok = (cudaOccupancyMaxActiveClusters(&n, k, &cfg) == cudaSuccess && n >= 1) ? 1 : 2;
    cudaGetLastError();
  }
  return ok == 1;
}

template <int D, int RB>
static int launch_rb(AttnArgs a, int max_ctas, cudaStream_t st) {
  const int rows = a.G * a.NT * 8;
  int n_sm = 148;
  cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, current_device());
  // SS_ATTN_CLUSTER = 0 / 1 forces the variant (experiment builds)
  static const int force = exp_env_int("SS_ATTN_CLUSTER", -1);
  if constexpr (RB <= 4) {
    using C = AttnCfg<D, RB, true>;
    // The cluster variant has 16 CTAs per (kv head, row chunk): it wins when
    // there are few of those (TP 4-8 shards, <= 2 kv heads per GPU: measured
    // 7.33 -> 7.04 ms per TP8-rank step); with 8 kv heads (TP 1) the global
    // merge over 18 splits per head is faster (more CTAs, deeper K/V ring).
    // Uncapped launches only (fake-peer TP caps the CTAs per rank).
    const int groups = a.Hkv_l * ((rows + C::ROWS - 1) / C::ROWS);
    const bool want = force >= 0 ? force == 1 : groups <= 2;
    if (want && max_ctas <= 0 && cluster_ok<D, RB>()) {
      // optional dynamic shared-memory padding (KB) that keeps one cluster
      // CTA per SM (two would share an SM's tensor pipe)
      static const int pad_kb = exp_env_int("SS_ATTN_CL_SMEM_KB", 0);
      const int smem = std::max((int)C::SMEM, pad_kb * 1024);
      static int attr_smem[kMaxDevices] = {0};
      if (smem > attr_smem[current_device()]) {
        cudaFuncSetAttribute(attn_kernel<D, RB, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        attr_smem[current_device()] = smem;
      }
      a.splits = kAttnCluster;
      a.zchunks = (rows + C::ROWS - 1) / C::ROWS;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(kAttnCluster, a.Hkv_l, a.zchunks);
      cfg.blockDim = dim3(C::WARPS * 32, 1, 1);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = st;
      cudaLaunchAttribute at[2];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = kAttnCluster;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[1].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      cfg.numAttrs = (exp_env("SS_NO_PDL") || ss_pdl_off) ? 1 : 2;
      cudaLaunchKernelEx(&cfg, attn_kernel<D, RB, true>, a);
      return 1;
    }
  }
  using C = AttnCfg<D, RB, false>;
  const int Z = (rows + C::ROWS - 1) / C::ROWS;
#ifdef SS_EXP_AOCC1
  int cap = n_sm;  // experiment: one split per SM even if two CTAs would fit
#else
  int cap = n_sm * occ_of<D, RB, false>();
#endif
  if (max_ctas > 0 && cap > max_ctas) cap = max_ctas;
  int S = cap / (a.Hkv_l * Z);
  const int max_tiles = (a.max_ctx_pad + kKvTile - 1) / kKvTile;
  if (S > max_tiles) S = max_tiles;
  if (S > 64) S = 64;  // workspace holds 64 partials (one per split) per row chunk
  if (S < 1) S = 1;
  a.splits = S;
  a.zchunks = Z;
  launch_pdl(attn_kernel<D, RB, false>, dim3(S, a.Hkv_l, Z), dim3(C::WARPS * 32), C::SMEM, st, a);
  return 1;
}

template <int D>
static int launch_d(const AttnArgs& a, int max_ctas, cudaStream_t st) {
  int rb = rb_for(a.G, a.NT);
  // With <= 2 kv heads per GPU (TP 4 / 8) the few CTAs per head are bound by
  // each CTA's tile loop, so split the rows over two chunks of 2 row blocks
  // (twice the CTAs, each half the rows): TP4-rank step 6.64 -> 6.48 ms, TP8
  // 6.08 -> 5.97 ms.  With 8 kv heads (TP 1) it costs 1.5 us per layer.
  // SS_ATTN_RB overrides the cap (tuning aid).  The workspace and meet
  // counters hold two row chunks per kv head, so Z = rows / (16 rb) <= 2.
  static const int rb_env = exp_env_int("SS_ATTN_RB", 0);
  const int rb_cap = rb_env > 0 ? rb_env : (a.Hkv_l <= 2 ? 2 : 0);
  const int rows = a.G * a.NT * 8;
  while (rb_cap > 0 && rb > rb_cap && rows <= (rb / 2) * 16 * 2) rb /= 2;
  switch (rb) {
    case 1: return launch_rb<D, 1>(a, max_ctas, st);
    case 2: return launch_rb<D, 2>(a, max_ctas, st);
    case 4: return launch_rb<D, 4>(a, max_ctas, st);
    case 8: return launch_rb<D, 8>(a, max_ctas, st);
    default: return launch_rb<D, 16>(a, max_ctas, st);
  }
}

template <int D>
static void warm_d() {
  cudaFuncAttributes at;
  cudaFuncGetAttributes(&at, attn_kernel<D, 1, false>);
  cudaFuncGetAttributes(&at, attn_kernel<D, 2, false>);
  cudaFuncGetAttributes(&at, attn_kernel<D, 4, false>);
  cudaFuncGetAttributes(&at, attn_kernel<D, 8, false>);
  cudaFuncGetAttributes(&at, attn_kernel<D, 16, false>);
  cudaFuncGetAttributes(&at, attn_kernel<D, 1, true>);
  cudaFuncGetAttributes(&at, attn_kernel<D, 2, true>);
  cudaFuncGetAttributes(&at, attn_kernel<D, 4, true>);
}
// see warm_misc_kernels (misc.cu)
void warm_attention_kernels() {
  warm_d<64>();
  warm_d<128>();
}

int launch_attention(const AttnArgs& a, int max_ctas, cudaStream_t st) {
  return a.d == 64 ? launch_d<64>(a, max_ctas, st) : launch_d<128>(a, max_ctas, st);
}

}  // namespace ss

#ifdef SS_ATTN_TRACE
extern "C" int ss_debug_attn_trace(unsigned long long* out) {
  cudaDeviceSynchronize();
  return cudaMemcpyFromSymbol(out, ss::g_at, sizeof(ss::g_at)) == cudaSuccess ? 0 : -1;
}
extern "C" int ss_debug_attn_tiles(unsigned long long* out) {
  cudaDeviceSynchronize();
  return cudaMemcpyFromSymbol(out, ss::g_att, sizeof(ss::g_att)) == cudaSuccess ? 0 : -1;
}
#endif
