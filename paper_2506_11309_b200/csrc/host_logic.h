// host_logic.h -- the C-ABI's host-side argument checks and call-order state
// machine (include/swiftspec.h "Errors").  Pure C++ (no CUDA):
// shard.cu runs these checks before any launch, and tests/host_logic_harness.cpp
// compiles this same header with g++ so the CPU test suite covers every
// host-detected error code without a GPU.
//
// Order of checks for a verify call: SS_EINVAL (tree shape), then
// SS_ESTATE (weights / peers missing, or a verify still pending: "two
// verifies without a commit"), then SS_ECAPACITY (L + T >
// max_ctx: no eviction).
#pragma once
#include <stdint.h>
#include <string>

#include "../../include/swiftspec.h"

namespace ss {
namespace host {

struct CallState {
  int32_t max_ctx = 0, max_tree = 0, vocab = 0;
  int32_t L = 0;                 // committed length (an upper bound when !L_known)
  bool L_known = true;
  bool weights_ready = false;
  bool peers_ready = true;       // false while tp_size > 1 and peers are not imported
  bool have_verify = false;      // a verify whose tree rows are not committed / discarded yet
  int32_t last_T = 0;
  int32_t last_parents[SS_MAX_TREE] = {0};
  int32_t max_written = 0;       // KV rows ever written (prefix + tree rows)
};

// Root first, topological parents, tokens in the vocabulary.
inline ss_status check_tree(const CallState& c, const int32_t* tokens, const int32_t* parents, int32_t T,
                            std::string& err) {
  if (!tokens || !parents) { err = "null tree"; return SS_EINVAL; }
  if (T < 1 || T > c.max_tree) { err = "T out of [1, max_tree]"; return SS_EINVAL; }
  if (parents[0] != -1) { err = "parents[0] must be -1 (root first)"; return SS_EINVAL; }
  for (int i = 1; i < T; ++i)
    if (parents[i] < 0 || parents[i] >= i) { err = "parents[i] must be in [0, i)"; return SS_EINVAL; }
  for (int i = 0; i < T; ++i)
    if (tokens[i] < 0 || tokens[i] >= c.vocab) { err = "token out of vocab"; return SS_EINVAL; }
  return SS_OK;
}

// State and capacity for a verify of T nodes (auto_commit: the step commits
// its own accepted path, so no verify stays pending).
inline ss_status check_verify(const CallState& c, int32_t T, std::string& err) {
  if (!c.weights_ready) { err = "weights not fully loaded"; return SS_ESTATE; }
  if (!c.peers_ready) { err = "peers not imported (tp_size > 1)"; return SS_ESTATE; }
  if (c.have_verify) {
    err = "a verify is pending: commit it (ss_commit_kv / ss_commit_accepted) or discard it "
          "(ss_set_committed_len) first";
    return SS_ESTATE;
  }
  if ((int64_t)c.L + T > c.max_ctx) { err = "L + T exceeds max_ctx"; return SS_ECAPACITY; }
  return SS_OK;
}

// A non-square forward (ss_extend_tree): w new nodes on the first T0 nodes of
// the pending tree.  Parents index the whole tree.
inline ss_status check_extend(const CallState& c, const int32_t* tokens, const int32_t* parents, int32_t T0,
                              int32_t w, std::string& err) {
  if (!tokens || !parents) { err = "null tree"; return SS_EINVAL; }
  if (w < 1 || w > 32) { err = "w out of [1, 32]"; return SS_EINVAL; }
  if (T0 < 0 || T0 + w > c.max_tree) { err = "T0 + w out of [1, max_tree]"; return SS_EINVAL; }
  for (int i = 0; i < w; ++i) {
    const int node = T0 + i;
    if (node == 0 ? parents[i] != -1 : (parents[i] < 0 || parents[i] >= node)) {
      err = "parents[i] must be in [0, T0 + i) (-1 only for node 0)";
      return SS_EINVAL;
    }
    if (tokens[i] < 0 || tokens[i] >= c.vocab) { err = "token out of vocab"; return SS_EINVAL; }
  }
  if (!c.weights_ready) { err = "weights not fully loaded"; return SS_ESTATE; }
  if (!c.peers_ready) { err = "peers not imported (tp_size > 1)"; return SS_ESTATE; }
  if (T0 > 0 && (!c.have_verify || T0 > c.last_T)) {
    err = "T0 > 0 needs a pending tree of at least T0 nodes";
    return SS_ESTATE;
  }
  if (T0 == 0 && c.have_verify) {
    err = "a verify is pending: commit or discard it, or extend it (T0 > 0)";
    return SS_ESTATE;
  }
  if ((int64_t)c.L + T0 + w > c.max_ctx) { err = "L + T0 + w exceeds max_ctx"; return SS_ECAPACITY; }
  return SS_OK;
}

// A commit of a root-anchored chain of the last verified tree.
inline ss_status check_commit(const CallState& c, const int32_t* accepted, int32_t n, std::string& err) {
  if (!accepted) { err = "null argument"; return SS_EINVAL; }
  if (!c.have_verify) { err = "commit without a preceding verify"; return SS_ESTATE; }
  if (n < 1 || n > c.last_T) { err = "n out of [1, T]"; return SS_EINVAL; }
  if (accepted[0] != 0) { err = "chain must start at the root (node 0)"; return SS_EINVAL; }
  for (int k = 1; k < n; ++k)
    if (accepted[k] <= 0 || accepted[k] >= c.last_T || c.last_parents[accepted[k]] != accepted[k - 1]) {
      err = "accepted is not a root-anchored chain of the last tree";
      return SS_EINVAL;
    }
  return SS_OK;
}

// ss_reroot (draft KV reorganisation): commit a root-anchored
// chain path[0..n) of the pending tree and keep the subtree keep[0..m)
// (ascending node indices; keep[0] a child of path[n-1], or the root when
// n == 0; every other kept node's parent kept before it) as the new pending
// tree, packed right after the new prefix.
inline ss_status check_reroot(const CallState& c, const int32_t* path, int32_t n, const int32_t* keep, int32_t m,
                              std::string& err) {
  if ((n > 0 && !path) || (m > 0 && !keep)) { err = "null argument"; return SS_EINVAL; }
  if (!c.have_verify) { err = "re-root without a pending tree"; return SS_ESTATE; }
  if (n < 0 || m < 0 || n + m < 1 || n + m > c.last_T) { err = "n, m out of range"; return SS_EINVAL; }
  if (n > 0) {
    ss_status r = check_commit(c, path, n, err);
    if (r != SS_OK) return r;
  }
  for (int j = 0; j < m; ++j) {
    if (keep[j] < 0 || keep[j] >= c.last_T || (j > 0 && keep[j] <= keep[j - 1])) {
      err = "keep must be ascending node indices of the pending tree";
      return SS_EINVAL;
    }
    const int32_t p = c.last_parents[keep[j]];
    bool ok;
    if (j == 0) {
      ok = n > 0 ? p == path[n - 1] : keep[0] == 0;
    } else {
      ok = false;
      for (int i = 0; i < j; ++i) ok = ok || keep[i] == p;
    }
    if (!ok) {
      err = "keep is not a subtree rooted at a child of the chain's last node";
      return SS_EINVAL;
    }
  }
  return SS_OK;
}

// ss_set_committed_len: truncate, or grow only over rows that hold data.
inline ss_status check_set_len(const CallState& c, int32_t L, std::string& err) {
  if (L < 0 || (int64_t)L + c.max_tree > c.max_ctx) { err = "length out of range"; return SS_ECAPACITY; }
  if (L > c.max_written) { err = "length beyond the KV rows ever written"; return SS_EINVAL; }
  return SS_OK;
}

// State transitions.
inline void on_verify(CallState& c, int32_t T, const int32_t* parents, bool auto_commit) {
  c.last_T = T;
  for (int i = 0; i < T && i < SS_MAX_TREE; ++i) c.last_parents[i] = parents ? parents[i] : 0;
  if (c.L_known && c.L + T > c.max_written) c.max_written = c.L + T;
  if (auto_commit) {
    c.L_known = false;  // the device decides n <= T
    c.L += T;           // upper bound until read back
    c.have_verify = false;
  } else {
    c.have_verify = true;
  }
}
inline void on_extend(CallState& c, int32_t T0, int32_t w, const int32_t* parents) {
  for (int i = 0; i < w && T0 + i < SS_MAX_TREE; ++i) c.last_parents[T0 + i] = parents[i];
  c.last_T = T0 + w;
  if (c.L_known && c.L + T0 + w > c.max_written) c.max_written = c.L + T0 + w;
  c.have_verify = true;
}
inline void on_commit(CallState& c, int32_t n) {
  c.L += n;
  if (c.L > c.max_written) c.max_written = c.L;
  c.have_verify = false;
}
inline void on_reroot(CallState& c, const int32_t* path, int32_t n, const int32_t* keep, int32_t m) {
  int32_t par[SS_MAX_TREE];
  for (int j = 0; j < m; ++j) {
    const int32_t p = c.last_parents[keep[j]];
    par[j] = -1;
    for (int i = 0; i < j; ++i)
      if (keep[i] == p) par[j] = i;
  }
  for (int j = 0; j < m; ++j) c.last_parents[j] = par[j];
  (void)path;
  c.L += n;
  if (c.L + m > c.max_written) c.max_written = c.L + m;
  c.last_T = m;
  c.have_verify = m > 0;
}
inline void on_set_len(CallState& c, int32_t L) {
  c.L = L;
  c.L_known = true;
  c.have_verify = false;
}

}  // namespace host
}  // namespace ss
