// accept.cuh -- the greedy accept walk (a11) and the TP argmax all-gather,
// run by the CTA that finalises the last LM-head tile-group (gemm.cu per-phase
// path and step.cu persistent kernel).
#pragma once
#include "common.cuh"
#include "internal.h"
#include "kernels.h"

namespace ss {

// tp > 1: all-gather the per-rank (logit, id) keys of every node through LL
// lines (one 8-byte key per 16-byte line) and keep the max (ties -> lowest id);
// every rank then walks the same accepted path.
struct ArgmaxXArgs {
  int P, rank, loopback, ar_seq, n_tg_total;
  float* recv;
  float* const* peer_recv;
};
__device__ inline void argmax_exchange(const ArgmaxXArgs& e, DevState* st) {
  const uint32_t flag = st->epoch + e.ar_seq;
  const size_t base = (size_t)2 * e.P * e.n_tg_total * 128 * 32;
  const int T = st->T;
  for (int t = 0; t < T; ++t) {
    unsigned long long k = __ldcg(&st->argmax_key[t]);
    for (int p = 0; p < e.P; ++p)
      ll_store(reinterpret_cast<uint4*>(e.peer_recv[p]) + base + (size_t)(e.loopback ? p : e.rank) * 64 + t,
               (uint32_t)k, (uint32_t)(k >> 32), flag);
  }
  for (int t = 0; t < T; ++t) {
    unsigned long long best = 0;
    for (int p = 0; p < e.P; ++p) {
      const uint4* src = reinterpret_cast<const uint4*>(e.recv) + base + (size_t)p * 64 + t;
      uint32_t d1, d2;
      long spins = 0;
      while (!ll_try_load(src, flag, d1, d2)) {
        if (++spins > (1L << 26)) { st->timeout = 1; break; }
      }
      unsigned long long k = ((unsigned long long)d2 << 32) | d1;
      best = k > best ? k : best;
    }
    st->argmax_key[t] = best;
  }
}

// Greedy accept walk (a11; R6, R7) on the device.
// A non-square forward (T0 > 0, ss_extend_tree) computed slots t = nodes
// T0 + t; the cached nodes keep the argmax of the call that computed them, and
// the walk runs over the whole grown tree of T0 + T nodes.
__device__ inline void accept_walk_dev(DevState* st) {
  const int T0 = st->T0;
  const int T = T0 + st->T;
  ss_verify_result& res = st->result;
  for (int i = T0; i < SS_MAX_TREE; ++i) {
    const int t = i - T0;  // slot of node i
    res.argmax[i] = i < T ? (int)argmax_key_index(__ldcg(&st->argmax_key[t])) : 0;
  }
  for (int t = 0; t < SS_MAX_TREE; ++t) st->argmax_key[t] = 0ull;
  int cur = 0, n = 1;
  res.accepted[0] = 0;
  while (true) {
    int tok = res.argmax[cur];
    int nxt = -1;
    for (int c = cur + 1; c < T; ++c)
      if (st->parents[c] == cur && st->tokens[c] == tok) { nxt = c; break; }
    if (nxt < 0) { res.bonus_token = tok; break; }
    res.accepted[n++] = nxt;
    cur = nxt;
  }
  for (int i = n; i < SS_MAX_TREE; ++i) res.accepted[i] = -1;
  res.n_accepted = n;
  // a peer poll that ran out of budget makes the step's result invalid
  res.status = st->timeout ? SS_ETIMEOUT : st->status;
  st->timeout = 0;
  st->have_verify = 1;
  // a13: post the verified path to the draft group's outbox (Alg. 1
  // "Send the verified tokens"; P:293 STOP at the end of generation): lines
  // 1..n = (node index, token), then line 0 = (n | -status << 16 | stop << 31,
  // bonus).  A failed step posts n = 0 and its status; an inbox message that
  // timed out gets no post and is polled again by the next step (the sequence
  // number does not advance).
  if (st->mbox_mode) {
    const uint32_t seq = st->mbox_cur;
    const bool ok = res.status == SS_OK;
    if (st->mbox_post && st->mbox_out && !st->mbox_tmo) {
      const int np = ok ? n : 0;
      for (int k = 0; k < np; ++k)
        ll_store(st->mbox_out + 1 + k, (uint32_t)res.accepted[k], (uint32_t)st->tokens[res.accepted[k]], seq);
      const uint32_t stop = (ok && st->eos >= 0 && res.bonus_token == st->eos) ? 1u : 0u;
      ll_store(st->mbox_out, (uint32_t)np | ((uint32_t)(-res.status) & 0xFFu) << 16 | (stop << 31),
               ok ? (uint32_t)res.bonus_token : 0u, seq);
    }
    if (!st->mbox_tmo) st->mbox_seq = seq;
  }
}


}  // namespace ss
