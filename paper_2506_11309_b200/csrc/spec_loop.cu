// spec_loop.cu -- Alg. 1: the draft worker and the target worker
// of SwiftSpec's parallel tree generation, linked only by the a13 mailboxes
// ("the two groups communicate using NVLink"; here LL lines in
// device memory).  Host code: the draft loop runs on the calling thread
// (draft_tree.h decides, the draft shard computes: ss_extend_tree_topk,
// ss_reroot); the target loop runs on its own thread and only enqueues
// mailbox-driven verify steps (ss_verify_tree_mailbox: the step polls its
// inbox on the device, verifies, commits, posts the path).  In async mode the
// draft keeps expanding while the target verifies (the paper's design); in
// serial mode it waits for each verify (SwiftSpec-base-like baseline).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "draft_tree.h"
#include "internal.h"

namespace {

ss_status fail(ss_shard* s, ss_status code, const std::string& m) {
  if (s) s->err = m;
  return code;
}

constexpr int kSpareSms = 8;

struct Outbox {
  void* dev = nullptr;     // (1 + SS_MAX_TREE) LL lines the target posts into
  int32_t* res = nullptr;  // device copy of a received result: [4 + 2 * SS_MAX_TREE]
  int32_t* host = nullptr; // pinned
};

}  // namespace

extern "C" ss_status ss_speculative_decode(ss_shard* target, ss_shard* draft, int32_t root_token,
                                           const ss_spec_cfg* cfg, int32_t* out_tokens, ss_spec_stats* stats,
                                           void* target_stream, void* draft_stream) {
  if (!target || !draft || !cfg || !out_tokens) return fail(target, SS_EINVAL, "null argument");
  if (target->P != 1 || draft->P != 1)
    return fail(target, SS_EINVAL, "the loop drives single-rank target / draft shards");
  if (target->device != draft->device) return fail(target, SS_EINVAL, "target and draft on different devices");
  const int bs = cfg->bs, w = cfg->w, d = cfg->d, K = cfg->K > 0 ? cfg->K : cfg->w;
  if (bs < 1 || bs > target->cfg.max_tree || w < 1 || w > 32 || d < 0 || K < 1 || K > 32 || cfg->n_tokens < 1)
    return fail(target, SS_EINVAL, "bs / w / d / K / n_tokens out of range");
  if (root_token < 0 || root_token >= target->cfg.vocab || target->cfg.vocab != draft->cfg.vocab)
    return fail(target, SS_EINVAL, "root token / vocabularies");
  if (target->hs.have_verify || draft->hs.have_verify) return fail(target, SS_ESTATE, "a verify is pending");
  cudaSetDevice(target->device);
  cudaStream_t ts = (cudaStream_t)target_stream, ds = (cudaStream_t)draft_stream;
  if (cfg->mode == 0) {
    // async: both groups' kernels must be resident at once -- the target's
    // step (launched early under PDL) waits on the inbox the draft fills
    if (ts == ds) return fail(target, SS_EINVAL, "async mode needs two different streams");
    // the two persistent grids plus room for the small kernels (ingest, commit,
    // top-K, re-root, mailbox): a persistent grid that waits for an SM held by
    // a small kernel of the other group would deadlock on the group hand-off
    if (target->launch_cap <= 0 || draft->launch_cap <= 0 ||
        target->launch_cap + draft->launch_cap > target->n_sm - kSpareSms)
      return fail(target, SS_EINVAL, "async mode: cap both grids (ss_set_launch_cap) to a split of the SMs "
                                     "that leaves 8 SMs free");
  }

  Outbox ob;
  if (cudaMalloc(&ob.dev, (1 + SS_MAX_TREE) * 16) != cudaSuccess ||
      cudaMalloc((void**)&ob.res, (4 + 2 * SS_MAX_TREE) * 4) != cudaSuccess ||
      cudaMallocHost((void**)&ob.host, (4 + 2 * SS_MAX_TREE) * 4) != cudaSuccess)
    return fail(target, SS_ECUDA, "outbox allocation");
  auto cleanup = [&]() {
    cudaFree(ob.dev);
    cudaFree(ob.res);
    cudaFreeHost(ob.host);
  };
  cudaMemset(ob.dev, 0, (1 + SS_MAX_TREE) * 16);
  ss_status r = ss_attach_mailbox(target, ob.dev, cfg->eos);
  void* inbox = nullptr;
  if (r == SS_OK) r = ss_mailbox_inbox(target, &inbox);
  uint32_t seq = 0;
  if (r == SS_OK && cudaMemcpy(&seq, &target->dstate->mbox_seq, 4, cudaMemcpyDeviceToHost) != cudaSuccess)
    r = SS_ECUDA;
  if (r != SS_OK) {
    cleanup();
    return r;
  }

  ss::draft::Tree tree;
  tree.max_slots = draft->cfg.max_tree;
  tree.reset(root_token);
  ss_spec_stats st{};
  std::vector<int32_t> toks, pars, sel, ctoks, cpars, cmap;
  std::vector<int32_t> top_tok((size_t)w * K);
  std::vector<float> top_val((size_t)w * K), lse(w);
  std::vector<double> lp(K);
  ss_verify_result vres;
  ss_status err = SS_OK;

  // one expansion of the w most probable leaves (Alg. 1)
  auto expand = [&]() -> int {
    sel = tree.select(w);
    if (sel.empty()) return 0;
    tree.forward_inputs(sel, toks, pars);
    ss_status e = ss_extend_tree_topk(draft, toks.data(), pars.data(), tree.n_slots, (int32_t)sel.size(), K,
                                      top_tok.data(), top_val.data(), lse.data(), &vres, ds);
    if (e != SS_OK) {
      err = e;
      return -1;
    }
    tree.computed(sel);
    for (size_t i = 0; i < sel.size(); ++i) {
      int k = 0;
      for (; k < K && top_tok[i * K + k] >= 0; ++k) lp[k] = (double)top_val[i * K + k] - (double)lse[i];
      tree.add_children(sel[i], &top_tok[i * K], lp.data(), k);
    }
    ++st.expansions;
    return (int)sel.size();
  };
  auto grow_to_bs = [&]() {
    while (err == SS_OK && tree.size_from_troot() < bs)
      if (expand() <= 0) break;
  };
  // Single-GPU emulation of the two GPU groups: the target launches its next
  // step only once the draft has enqueued that step's tree.  The hand-off
  // itself stays on the device (LL lines), but a step whose inbox poll
  // started early would hold SM resources the draft's own persistent kernel
  // needs to produce the tree.
  std::atomic<uint32_t> posted{seq};
  auto post = [&]() {
    tree.subgraph(bs, ctoks, cpars, cmap);
    ++seq;
    ss_status e = ss_mailbox_post_tree(inbox, ctoks.data(), cpars.data(), (int32_t)ctoks.size(), seq, ds);
    if (e != SS_OK) err = e;
    posted.store(seq);
  };

  // target worker (Alg. 1 target branch): get the tree, verify, post the path
  std::atomic<bool> stop{false};
  std::atomic<int> target_err{SS_OK};
  std::atomic<int> target_steps{0};
  const bool async = cfg->mode == 0;
  uint32_t tseq = seq;  // last message the target took (target thread only)
  auto target_step = [&]() -> bool {
    while (posted.load() <= tseq) {
      if (stop.load()) return false;
      std::this_thread::yield();
    }
    ++tseq;
    ss_status e = ss_verify_tree_mailbox_n(target, bs, 1, ts);
    if (e == SS_OK && cudaStreamSynchronize(ts) != cudaSuccess) e = SS_ECUDA;
    // the committed length after the step's device commit, read on the target
    // stream (the generic refresh synchronises the whole device, which would
    // wait on the draft's mailbox poll -- and that waits on this thread)
    int32_t Lw[2] = {0, 0};
    if (e == SS_OK && (cudaMemcpyAsync(&Lw[0], &target->dstate->L, 4, cudaMemcpyDeviceToHost, ts) != cudaSuccess ||
                       cudaMemcpyAsync(&Lw[1], &target->dstate->max_written, 4, cudaMemcpyDeviceToHost, ts) !=
                           cudaSuccess ||
                       cudaStreamSynchronize(ts) != cudaSuccess))
      e = SS_ECUDA;
    if (e == SS_OK) {
      target->hs.L = Lw[0];
      target->hs.L_known = true;
      target->hs.max_written = std::max(target->hs.max_written, std::max(Lw[0], Lw[1]));
    }
    if (e != SS_OK) {
      target_err = e;
      return false;
    }
    ++target_steps;
    return true;
  };
  std::thread tthread;
  if (async)
    tthread = std::thread([&]() {
      cudaSetDevice(target->device);
      while (!stop.load() && target_step()) {
      }
    });

  auto expand_d = [&]() {
    for (int i = 0; i < d && err == SS_OK; ++i)
      if (expand() <= 0) break;
  };
  const auto t0 = std::chrono::steady_clock::now();
  if (!async) expand_d();
  grow_to_bs();
  if (err == SS_OK) post();
  int emitted = 0;
  while (err == SS_OK && target_err.load() == SS_OK) {
    // async: the draft expands d times while the target verifies the posted
    // tree; serial: the target verifies while the draft waits
    if (async) expand_d();
    else if (!target_step()) break;
    // "Get verified tokens from the target worker"
    if (ss_mailbox_recv_result(ob.dev, seq, ob.res, ds) != SS_OK ||
        cudaMemcpyAsync(ob.host, ob.res, (4 + 2 * SS_MAX_TREE) * 4, cudaMemcpyDeviceToHost, ds) != cudaSuccess ||
        cudaStreamSynchronize(ds) != cudaSuccess) {
      err = SS_ECUDA;
      break;
    }
    const int n = ob.host[0], bonus = ob.host[1], stopbit = ob.host[2];
    if (n < 1 || ob.host[3] != SS_OK) {
      err = n < 0 ? SS_ETIMEOUT : (ss_status)(ob.host[3] != SS_OK ? ob.host[3] : SS_ECONSISTENCY);
      break;
    }
    ++st.steps;
    std::vector<int32_t> path(n);
    for (int k = 0; k < n; ++k) path[k] = cmap[ob.host[4 + 2 * k]];
    for (int k = 1; k < n && emitted < cfg->n_tokens; ++k) out_tokens[emitted++] = ob.host[5 + 2 * k];
    if (emitted < cfg->n_tokens) out_tokens[emitted++] = bonus;
    st.accepted += n - 1;
    if (emitted >= cfg->n_tokens || stopbit) break;
    // "Update KV Cache and draft tree based on verified tokens"
    std::vector<int32_t> commit, keep;
    tree.reroot(path, bonus, commit, keep);
    if (!commit.empty() || !keep.empty()) {
      ss_status e = ss_reroot(draft, commit.data(), (int32_t)commit.size(), keep.data(), (int32_t)keep.size(), ds);
      if (e != SS_OK) {
        err = e;
        break;
      }
    }
    // "While Tree size < bs: expand"; send the most probable subgraph
    if (!async) expand_d();
    grow_to_bs();
    if (err != SS_OK) break;
    post();
  }
  const auto t1 = std::chrono::steady_clock::now();
  if (async) {
    stop = true;  // the target thread takes no further tree (none was posted)
    tthread.join();
  }
  cudaStreamSynchronize(ds);
  cudaStreamSynchronize(ts);
  st.n_emitted = emitted;
  st.target_steps = target_steps.load();
  st.wall_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
  if (stats) *stats = st;
  cleanup();
  if (err == SS_OK && target_err.load() != SS_OK) err = (ss_status)target_err.load();
  if (err != SS_OK) return fail(target, err, "speculative decode loop failed (" + std::to_string((int)err) + ")");
  // the draft's pending tree rows are discarded; both shards end without a pending verify
  if (draft->hs.have_verify) ss_set_committed_len(draft, ss_committed_len(draft));
  return SS_OK;
}
