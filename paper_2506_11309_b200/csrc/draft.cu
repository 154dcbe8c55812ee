// draft.cu -- device pieces of the draft worker:
//  * topk_kernel: per computed leaf, the top-K tokens of this rank's vocab
//    slice with their logits and the slice's log-sum-exp -- the maximum-
//    likelihood expansion's children and node values ("the logarithm
//    of the softmax probability as the value of each node");
//  * reroot_kernel: the draft KV reorganisation: the verified
//    chain's K/V move into the prefix cache and the kept subtree's K/V are
//    packed right after it ("reorganizes the remaining sub-tree ... into the
//    next positions available"), with the tree metadata re-indexed on the
//    device so the next non-square forward (ss_extend_tree) reads it.
#include "common.cuh"
#include "internal.h"
#include "kernels.h"

namespace ss {

// (value, lowest index) as one ordered 64-bit key: larger value first, then
// the lower index (ties -> lowest token id, R6).
SS_DEV unsigned long long topk_key(float v, int i) {
  const uint32_t u = __float_as_uint(v);
  const uint32_t o = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
  return ((unsigned long long)o << 32) | (0xFFFFFFFFu - (uint32_t)i);
}

constexpr int kTopkThreads = 1024;

template <typename T, typename Op>
SS_DEV T block_reduce_1024(T v, T* s, Op op) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = v;
  __syncthreads();
  T r = s[0];
#pragma unroll
  for (int i = 1; i < kTopkThreads / 32; ++i) r = op(r, s[i]);
  return r;
}

// One CTA per row (a computed node's logits over this rank's V_l tokens).
__global__ void __launch_bounds__(kTopkThreads) topk_kernel(const float* logits, int ld, int V_l, int V_off,
                                                            int K, int32_t* tok, float* val, float* lse) {
  __shared__ float s_f[32];
  __shared__ unsigned long long s_k[32];
  const float* x = logits + (size_t)blockIdx.x * ld;
  float m = -INFINITY;
  for (int i = threadIdx.x; i < V_l; i += kTopkThreads) m = fmaxf(m, x[i]);
  m = block_reduce_1024(m, s_f, [](float a, float b) { return fmaxf(a, b); });
  float s = 0.f;
  for (int i = threadIdx.x; i < V_l; i += kTopkThreads) s += __expf(x[i] - m);
  s = block_reduce_1024(s, s_f, [](float a, float b) { return a + b; });
  if (threadIdx.x == 0) lse[blockIdx.x] = m + logf(s);
  // K rounds: the largest key strictly below the previous round's
  unsigned long long prev = ~0ull;
  for (int r = 0; r < K; ++r) {
    unsigned long long best = 0ull;
    for (int i = threadIdx.x; i < V_l; i += kTopkThreads) {
      const unsigned long long k = topk_key(x[i], i);
      if (k < prev && k > best) best = k;
    }
    best = block_reduce_1024(best, s_k, [](unsigned long long a, unsigned long long b) { return a > b ? a : b; });
    if (threadIdx.x == 0) {
      const int i = (int)(0xFFFFFFFFu - (uint32_t)(best & 0xFFFFFFFFull));
      const bool ok = best != 0ull && i < V_l;
      tok[blockIdx.x * K + r] = ok ? V_off + i : -1;
      val[blockIdx.x * K + r] = ok ? x[i] : -INFINITY;
    }
    prev = best;
  }
}

void launch_topk(ss_shard* s, int w, int K, int32_t* d_tok, float* d_val, float* d_lse, cudaStream_t st) {
  topk_kernel<<<w, kTopkThreads, 0, st>>>(s->logits_dev, s->V_l_pad, s->V_l, s->V_off, K, d_tok, d_val, d_lse);
}

// Two-phase copy per (kv head, layer): rows L + commit_chain[k] -> L + k, then
// rows L + keep[j] -> L + n + j (all loads before any store: the ranges
// overlap).  The last CTA advances L by n and re-indexes the kept nodes'
// metadata (token, parent, position -- unchanged: pos = L + depth and both
// move by n --, ancestor mask, argmax) as nodes 0 .. m-1 of the pending tree.
__global__ void __launch_bounds__(256) reroot_kernel(DevState* st, uint16_t* kc, uint16_t* vc, int Hkv_l, int d,
                                                     int max_ctx_pad) {
  const int kvh = blockIdx.x, layer = blockIdx.y;
  const int n = st->commit_n, m = st->keep_n;
  const int L = st->L;
  const int cpr = d / 8;
  const size_t base = ((size_t)layer * Hkv_l + kvh) * max_ctx_pad * d;
  uint4 buf[2][8];
  const int total = (n + m) * cpr;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int idx = threadIdx.x + i * 256;
    if (idx < total) {
      const int k = idx / cpr, c = idx % cpr;
      const int src = L + (k < n ? st->commit_chain[k] : st->keep[k - n]);
      const size_t off = base + (size_t)src * d + ((c ^ (src & 7)) << 3);
      buf[0][i] = *reinterpret_cast<const uint4*>(kc + off);
      buf[1][i] = *reinterpret_cast<const uint4*>(vc + off);
    }
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int idx = threadIdx.x + i * 256;
    if (idx < total) {
      const int k = idx / cpr, c = idx % cpr;
      const int dst = L + k;
      const size_t off = base + (size_t)dst * d + ((c ^ (dst & 7)) << 3);
      *reinterpret_cast<uint4*>(kc + off) = buf[0][i];
      *reinterpret_cast<uint4*>(vc + off) = buf[1][i];
    }
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const int old = atomicAdd(&st->commit_done, 1);
    if (old == (int)(gridDim.x * gridDim.y) - 1) {
      __threadfence();
      st->commit_done = 0;
      // keep[j] >= j (ascending, distinct): node keep[j] is read before index j is written
      for (int j = 0; j < m; ++j) {
        const int o = st->keep[j];
        const int po = st->parents[o];
        int pn = -1;
        for (int i = 0; i < j; ++i)
          if (st->keep[i] == po) pn = i;
        st->tokens[j] = st->tokens[o];
        st->parents[j] = pn;
        st->pos[j] = st->pos[o];
        st->anc[j] = (pn >= 0 ? st->anc[pn] : 0ull) | (1ull << j);
        st->result.argmax[j] = st->result.argmax[o];
      }
      for (int j = m; j < SS_MAX_TREE; ++j) {
        st->anc[j] = 0ull;
        st->tokens[j] = -1;
        st->parents[j] = -2;
      }
      st->L = L + n;
      st->max_written = max(st->max_written, L + n + m);
      st->T0 = 0;
      st->T = m;
      st->have_verify = m > 0 ? 1 : 0;
    }
  }
}

void launch_reroot(ss_shard* s, cudaStream_t st) {
  dim3 grid(s->Hkv_l, s->cfg.n_layers);
  reroot_kernel<<<grid, 256, 0, st>>>(s->dstate, s->kcache, s->vcache, s->Hkv_l, s->cfg.head_dim,
                                      s->max_ctx_pad);
}

void warm_draft_kernels() {
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, topk_kernel);
  cudaFuncGetAttributes(&a, reroot_kernel);
}

}  // namespace ss
