// attention.cu -- tree-masked GQA attention.
//
// Every tree node attends to the committed prefix [0, L) plus its
// ancestors-or-self among the tree rows [L, L+T) (square mask P:321, bitmask
// per node).  One CTA = (kv head, key split, row chunk); the rows are the
// G query heads x T nodes that share the kv head (GQA), so K/V tiles are
// read from HBM once per kv head.  K/V tiles (64 keys, pre-swizzled in the
// cache layout) arrive via the TMA bulk engine into a double-buffered ring;
// QK^T and PV run on mma.sync with ldmatrix; online softmax in fp32 (R11).
// The split partials are combined inside the same kernel: CTAs of one kv head
// meet at a flag counter (the paper's intra-GPU LL aggregation, "without
// explicit synchronization across thread blocks or extra kernel launches")
// and each CTA then merges a slice of the rows, writing the bf16 result
// straight into the O-projection's fragment-ordered input.
#include "common.cuh"
#include "internal.h"
#include "kernels.h"

namespace ss {

template <int D, int NW>
__global__ void __launch_bounds__(NW * 32, 1) attn_kernel(AttnArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[2];
  constexpr int ROWS = NW * 16;
  constexpr int QS = D + 8;  // padded Q row stride (elements)
  constexpr int TILE_ELEMS = kKvTile * D;
  uint16_t* Qs = reinterpret_cast<uint16_t*>(smem);
  uint16_t* Ks = Qs + 2 * ROWS * QS;  // [2][64*D] after the Q hi / lo planes
  uint16_t* Vs = Ks + 2 * TILE_ELEMS;

  const int split = blockIdx.x, kvh = blockIdx.y, z = blockIdx.z;
  const int S = gridDim.x, Z = gridDim.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gq = lane >> 2, tq = lane & 3;
  DevState* st = a.st;
  pdl_wait();
  pdl_trigger();
  const int L = st->L, T = st->T;
  const int G = a.G;
  const int Mrows = G * T;
  const int m0 = z * ROWS;
  const int ntiles = (L + T + kKvTile - 1) / kKvTile;
  const int t0 = (int)((long)split * ntiles / S), t1 = (int)((long)(split + 1) * ntiles / S);
  const size_t head_base = ((size_t)a.layer * a.Hkv_l + kvh) * a.max_ctx_pad * D;

  if (threadIdx.x == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0 && t0 < t1) {
    mbar_expect_tx(&full[0], 2 * TILE_ELEMS * 2);
    bulk_g2s_nohint(Ks, a.kc + head_base + (size_t)t0 * TILE_ELEMS, TILE_ELEMS * 2, &full[0]);
    bulk_g2s_nohint(Vs, a.vc + head_base + (size_t)t0 * TILE_ELEMS, TILE_ELEMS * 2, &full[0]);
  }
  // Q rows [m0, m0 + ROWS) of this kv head (post-RoPE, from the QKV epilogue),
  // as bf16 hi and lo planes: q = hi + lo carries ~16 mantissa bits, so the
  // QK^T product is not limited by a bf16 rounding of q.
  const uint16_t* qsrc = a.qbuf + ((size_t)kvh * (G * SS_MAX_TREE) + m0) * D;
  const size_t qplane = (size_t)a.Hkv_l * G * SS_MAX_TREE * D;
  for (int i = threadIdx.x; i < ROWS * (D / 8); i += NW * 32) {
    int r = i / (D / 8), c = i % (D / 8);
    uint4 v = make_uint4(0, 0, 0, 0), w = make_uint4(0, 0, 0, 0);
    if (m0 + r < Mrows) {
      v = *reinterpret_cast<const uint4*>(qsrc + (size_t)r * D + c * 8);
      w = *reinterpret_cast<const uint4*>(qsrc + qplane + (size_t)r * D + c * 8);
    }
    *reinterpret_cast<uint4*>(Qs + r * QS + c * 8) = v;
    *reinterpret_cast<uint4*>(Qs + (ROWS + r) * QS + c * 8) = w;
  }
  __syncthreads();
  const uint16_t* qrow = Qs + (warp * 16 + (lane & 15)) * QS + (lane >> 4) * 8;

  const int rowA = m0 + warp * 16 + gq, rowB = rowA + 8;
  const int tokA = min(rowA / G, SS_MAX_TREE - 1), tokB = min(rowB / G, SS_MAX_TREE - 1);
  const unsigned long long ancA = st->anc[tokA], ancB = st->anc[tokB];
  const bool okA = rowA < Mrows, okB = rowB < Mrows;
  const float sl2 = rsqrtf((float)D) * 1.4426950408889634f;

  float mA = -INFINITY, mB = -INFINITY, lA = 0.f, lB = 0.f;
  float o[D / 8][4];
#pragma unroll
  for (int n = 0; n < D / 8; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;

  for (int it = t0; it < t1; ++it) {
    const int b = (it - t0) & 1;
    const uint32_t phase = ((it - t0) >> 1) & 1;
    if (threadIdx.x == 0 && it + 1 < t1) {
      fence_proxy_async_smem();  // ldmatrix reads of this buffer (previous tile) before the TMA overwrite
      mbar_expect_tx(&full[b ^ 1], 2 * TILE_ELEMS * 2);
      bulk_g2s_nohint(Ks + (b ^ 1) * TILE_ELEMS, a.kc + head_base + (size_t)(it + 1) * TILE_ELEMS, TILE_ELEMS * 2,
                      &full[b ^ 1]);
      bulk_g2s_nohint(Vs + (b ^ 1) * TILE_ELEMS, a.vc + head_base + (size_t)(it + 1) * TILE_ELEMS, TILE_ELEMS * 2,
                      &full[b ^ 1]);
    }
    mbar_wait(&full[b], phase);
    const uint16_t* Kt = Ks + b * TILE_ELEMS;
    const uint16_t* Vt = Vs + b * TILE_ELEMS;

    float sc[8][4];
#pragma unroll
    for (int n = 0; n < 8; ++n) sc[n][0] = sc[n][1] = sc[n][2] = sc[n][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
      uint32_t qh[4], ql[4];
      ldmatrix_x4(qh, qrow + kk * 16);
      ldmatrix_x4(ql, qrow + ROWS * QS + kk * 16);
#pragma unroll
      for (int np = 0; np < 4; ++np) {
        const int key = np * 16 + (lane & 7) + ((lane >> 4) << 3);
        const int ch = kk * 2 + ((lane >> 3) & 1);
        uint32_t kb[4];
        ldmatrix_x4(kb, Kt + key * D + ((ch ^ (key & 7)) << 3));
        mma_bf16_16816(sc[2 * np], qh, kb[0], kb[1]);
        mma_bf16_16816(sc[2 * np + 1], qh, kb[2], kb[3]);
        mma_bf16_16816(sc[2 * np], ql, kb[0], kb[1]);
        mma_bf16_16816(sc[2 * np + 1], ql, kb[2], kb[3]);
      }
    }
    // mask (prefix always visible; tree rows by ancestor bit; beyond L+T never)
    const int kbase = it * kKvTile;
    float mxA = -INFINITY, mxB = -INFINITY;
#pragma unroll
    for (int n = 0; n < 8; ++n) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int key = kbase + n * 8 + 2 * tq + (e & 1);
        const unsigned long long anc = (e < 2) ? ancA : ancB;
        const bool ok = (e < 2) ? okA : okB;
        bool vis = ok && (key < L || (key < L + T && ((anc >> (key - L)) & 1ull)));
        float v = vis ? sc[n][e] * sl2 : -INFINITY;
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
    // probabilities as bf16 hi + lo (V is bf16 in the cache)
    uint32_t pa[4][4], pl[4][4];
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      float p0 = exp2f(sc[n][0] - uA), p1 = exp2f(sc[n][1] - uA);
      float p2 = exp2f(sc[n][2] - uB), p3 = exp2f(sc[n][3] - uB);
      sumA += p0 + p1;
      sumB += p2 + p3;
      uint32_t h01 = pack_bf16x2(p0, p1), h23 = pack_bf16x2(p2, p3);
      pa[n >> 1][(n & 1) * 2 + 0] = h01;
      pa[n >> 1][(n & 1) * 2 + 1] = h23;
      pl[n >> 1][(n & 1) * 2 + 0] = pack_bf16x2(p0 - bf16_lo(h01), p1 - bf16_hi(h01));
      pl[n >> 1][(n & 1) * 2 + 1] = pack_bf16x2(p2 - bf16_lo(h23), p3 - bf16_hi(h23));
    }
    sumA += __shfl_xor_sync(0xffffffffu, sumA, 1);
    sumA += __shfl_xor_sync(0xffffffffu, sumA, 2);
    sumB += __shfl_xor_sync(0xffffffffu, sumB, 1);
    sumB += __shfl_xor_sync(0xffffffffu, sumB, 2);
    lA = lA * alA + sumA;
    lB = lB * alB + sumB;
    mA = mnA;
    mB = mnB;
#pragma unroll
    for (int n = 0; n < D / 8; ++n) {
      o[n][0] *= alA; o[n][1] *= alA; o[n][2] *= alB; o[n][3] *= alB;
    }
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
#pragma unroll
      for (int dp = 0; dp < D / 16; ++dp) {
        const int key = kk * 16 + (lane & 7) + (((lane >> 3) & 1) << 3);
        const int ch = dp * 2 + (lane >> 4);
        uint32_t vb[4];
        ldmatrix_x4_trans(vb, Vt + key * D + ((ch ^ (key & 7)) << 3));
        mma_bf16_16816(o[2 * dp], pa[kk], vb[0], vb[1]);
        mma_bf16_16816(o[2 * dp + 1], pa[kk], vb[2], vb[3]);
        mma_bf16_16816(o[2 * dp], pl[kk], vb[0], vb[1]);
        mma_bf16_16816(o[2 * dp + 1], pl[kk], vb[2], vb[3]);
      }
    }
    __syncthreads();  // buffer b is refilled two iterations later
  }

  // ---- partials to the workspace
  const int grp = kvh * Z + z;
  float* ws = a.ws + (((size_t)grp * S + split) * 256) * D;
  float* ml = a.ml + (((size_t)grp * S + split) * 256) * 2;
  {
    const int ra = warp * 16 + gq, rb = ra + 8;
#pragma unroll
    for (int n = 0; n < D / 8; ++n) {
      *reinterpret_cast<float2*>(ws + (size_t)ra * D + n * 8 + 2 * tq) = make_float2(o[n][0], o[n][1]);
      *reinterpret_cast<float2*>(ws + (size_t)rb * D + n * 8 + 2 * tq) = make_float2(o[n][2], o[n][3]);
    }
    if (tq == 0) {
      *reinterpret_cast<float2*>(ml + ra * 2) = make_float2(mA, lA);
      *reinterpret_cast<float2*>(ml + rb * 2) = make_float2(mB, lB);
    }
  }
  // ---- meet the other splits of this (kv head, row chunk): every thread
  // fences its partial stores, one thread arrives and spins on the flag.
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicAdd(&a.bar[grp * 2], 1);
    while (*reinterpret_cast<volatile int*>(&a.bar[grp * 2]) < S) {
    }
    __threadfence();
  }
  __syncthreads();
  __threadfence();
  // ---- merge a slice of the rows across the S splits (log-sum-exp, R11).
  // Items = (row, 4-float chunk); the CTA's items are a contiguous slice.  The
  // per-(row, split) weights exp2(m_s - m*) / l* go through shared memory, and
  // every thread issues its S partial loads back to back (no serial L2 chain).
  {
    float* s_w = reinterpret_cast<float*>(Ks);  // reuse the K/V ring: [rows_here][S]
    const int n_items = ROWS * (D / 4);
    const int i_lo = (int)((long)split * n_items / S), i_hi = (int)((long)(split + 1) * n_items / S);
    const int r_first = i_lo / (D / 4), r_last = (i_hi - 1) / (D / 4);
    const int nr = (i_hi > i_lo) ? r_last - r_first + 1 : 0;
    const float* wsg = a.ws + ((size_t)grp * S * 256) * D;
    const float* mlg = a.ml + ((size_t)grp * S * 256) * 2;
    for (int i = threadIdx.x; i < nr * S; i += NW * 32) {
      int rr = i / S, s2 = i % S;
      float2 v = __ldcg(reinterpret_cast<const float2*>(mlg + ((size_t)s2 * 256 + r_first + rr) * 2));
      s_w[i] = v.x;
      s_w[nr * S + i] = v.y;
    }
    __syncthreads();
    for (int rr = warp; rr < nr; rr += NW) {  // one warp per row: m*, l*, weights
      float mx = -INFINITY;
      for (int s2 = lane; s2 < S; s2 += 32) mx = fmaxf(mx, s_w[rr * S + s2]);
      mx = warp_max(mx);
      float l = 0.f;
      for (int s2 = lane; s2 < S; s2 += 32) {
        float ms = s_w[rr * S + s2];
        float w = (ms == -INFINITY) ? 0.f : exp2f(ms - mx);
        l += w * s_w[nr * S + rr * S + s2];
        s_w[rr * S + s2] = w;
      }
      l = warp_sum(l);
      __syncwarp();
      const float inv = l > 0.f ? 1.f / l : 0.f;
      for (int s2 = lane; s2 < S; s2 += 32) s_w[rr * S + s2] *= inv;
    }
    __syncthreads();
    for (int it = i_lo + threadIdx.x; it < i_hi; it += NW * 32) {
      const int r = it / (D / 4), c4 = it % (D / 4);
      const int m = m0 + r;
      if (m >= Mrows) continue;
      const float* wr = s_w + (r - r_first) * S;
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 8
      for (int s2 = 0; s2 < S; ++s2) {
        const float w = wr[s2];
        const float4 ov = __ldcg(reinterpret_cast<const float4*>(wsg + ((size_t)s2 * 256 + r) * D + 4 * c4));
        acc.x += w * ov.x;
        acc.y += w * ov.y;
        acc.z += w * ov.z;
        acc.w += w * ov.w;
      }
      const int t = m / G, hq = kvh * G + (m % G);
      const int k = hq * D + 4 * c4;
      *reinterpret_cast<uint32_t*>(a.act_out + act_frag_offset(t, k, a.NT)) = pack_half2(acc.x, acc.y);
      *reinterpret_cast<uint32_t*>(a.act_out + act_frag_offset(t, k + 2, a.NT)) = pack_half2(acc.z, acc.w);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&a.bar[grp * 2 + 1], 1) == S - 1) {
      a.bar[grp * 2] = 0;
      a.bar[grp * 2 + 1] = 0;
    }
  }
}

template <int D, int NW>
static size_t attn_smem() {
  return 2 * (size_t)NW * 16 * (D + 8) * 2 + 4 * (size_t)kKvTile * D * 2;
}

template <int D, int NW>
static int occ_of() {
  static int occ = -1;
  if (occ < 0) {
    cudaFuncSetAttribute(attn_kernel<D, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)attn_smem<D, NW>());
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, attn_kernel<D, NW>, NW * 32, attn_smem<D, NW>());
    if (occ < 1) occ = 1;
  }
  return occ;
}

static int nw_for(int G, int NT) {
  int rb = (G * NT * 8 + 15) / 16;
  int nw = 1;
  while (nw < rb && nw < 16) nw <<= 1;
  return nw;
}

template <int D>
static int occ_dispatch(int nw) {
  switch (nw) {
    case 1: return occ_of<D, 1>();
    case 2: return occ_of<D, 2>();
    case 4: return occ_of<D, 4>();
    case 8: return occ_of<D, 8>();
    default: return occ_of<D, 16>();
  }
}

template <int D>
static int launch_d(const AttnArgs& a0, int max_ctas, cudaStream_t st) {
  AttnArgs a = a0;
  int nw = nw_for(a.G, a.NT);
  int rows = a.G * a.NT * 8;
  int Z = (rows + nw * 16 - 1) / (nw * 16);
  int n_sm = 148;
  cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, 0);
  int cap = n_sm * occ_dispatch<D>(nw);
  if (max_ctas > 0 && cap > max_ctas) cap = max_ctas;
  int S = cap / (a.Hkv_l * Z);
  int max_tiles = (a.max_ctx_pad + kKvTile - 1) / kKvTile;
  if (S > max_tiles) S = max_tiles;
  if (S > 64) S = 64;
  if (S < 1) S = 1;
  a.splits = S;
  a.zchunks = Z;
  dim3 grid(S, a.Hkv_l, Z);
  switch (nw) {
    case 1: launch_pdl(attn_kernel<D, 1>, grid, dim3(32), attn_smem<D, 1>(), st, a); break;
    case 2: launch_pdl(attn_kernel<D, 2>, grid, dim3(64), attn_smem<D, 2>(), st, a); break;
    case 4: launch_pdl(attn_kernel<D, 4>, grid, dim3(128), attn_smem<D, 4>(), st, a); break;
    case 8: launch_pdl(attn_kernel<D, 8>, grid, dim3(256), attn_smem<D, 8>(), st, a); break;
    default: launch_pdl(attn_kernel<D, 16>, grid, dim3(512), attn_smem<D, 16>(), st, a); break;
  }
  return 1;
}

int launch_attention(const AttnArgs& a, int max_ctas, cudaStream_t st) {
  return a.d == 64 ? launch_d<64>(a, max_ctas, st) : launch_d<128>(a, max_ctas, st);
}

}  // namespace ss
