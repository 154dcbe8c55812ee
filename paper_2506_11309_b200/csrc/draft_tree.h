// draft_tree.h -- the draft worker's token tree: the host
// side of Alg. 1's draft branch, maximum-likelihood expansion
// (P:259), the most probable subgraph of size bs, and the re-root with
// the draft KV reorganisation.  Pure C++ (no CUDA): the draft loop
// (draft.cu) drives it, and tests/native/draft_tree_harness.cpp compiles this
// same header with g++ so the CPU suite compares it with oracle/draft_tree.py.
//
// Nodes.  Node ids are topological (a parent's id is below its children's);
// node 0 is the draft root.  A node is *computed* once a draft forward ran on
// it: its K/V sit in the draft's tree cache at row L + slot ("the KV states of
// the tree are stored right after the prefix") and its top-K children
// (the K most probable next tokens under the draft) were added as uncomputed
// leaves.  The weight of a node is the sum of log-softmax values from the root
// ("We use the logarithm of the softmax probability as the value of each node,
// and use the sum of values from the root to each node as the weight");
// ties are broken by the lower node id everywhere.
//
// troot is the node of the last verified token -- the target's next root (R9:
// the root is the last bonus, not yet in any KV cache).  The draft root may sit
// above it: verified tokens whose draft K/V was never computed stay in the tree
// as a weight-0 chain from the draft root to troot, are expanded first (they
// are the most probable nodes) and committed at the next re-root.
#pragma once
#include <stdint.h>

#include <algorithm>
#include <vector>

namespace ss {
namespace draft {

struct Node {
  int32_t token;
  int32_t parent;  // node id, -1 for the root
  double weight;   // sum of log-probabilities from the draft root (<= 0)
  int32_t slot;    // tree-cache row offset (computed nodes), -1 if not computed
};

struct Tree {
  std::vector<Node> nodes;
  int32_t n_slots = 0;    // computed nodes = tree-cache rows in use
  int32_t troot = 0;      // node of the target's next root
  int32_t max_slots = 64; // tree-cache capacity (the draft shard's max_tree)

  void reset(int32_t root_token) {
    nodes.assign(1, Node{root_token, -1, 0.0, -1});
    n_slots = 0;
    troot = 0;
  }

  // (weight desc, id asc): the order of "most probable"
  bool before(int32_t a, int32_t b) const {
    if (nodes[a].weight != nodes[b].weight) return nodes[a].weight > nodes[b].weight;
    return a < b;
  }

  bool in_subtree(int32_t n, int32_t r) const {
    for (int32_t j = n; j != -1; j = nodes[j].parent)
      if (j == r) return true;
    return false;
  }

  // Nodes of troot's subtree: what a subgraph can be drawn from ("Tree size").
  int32_t size_from_troot() const {
    int32_t c = 0;
    for (int32_t i = 0; i < (int32_t)nodes.size(); ++i) c += in_subtree(i, troot) ? 1 : 0;
    return c;
  }

  // "Expand the w most probable leaves" (Alg. 1): the w most probable
  // uncomputed nodes, at most the free tree-cache rows, returned in id order
  // (a selected node's uncomputed parent is more probable, so it is selected
  // too and comes first).
  std::vector<int32_t> select(int32_t w) const {
    std::vector<int32_t> c;
    for (int32_t i = 0; i < (int32_t)nodes.size(); ++i)
      if (nodes[i].slot < 0) c.push_back(i);
    std::sort(c.begin(), c.end(), [&](int32_t a, int32_t b) { return before(a, b); });
    const int32_t n = std::min<int32_t>({w, (int32_t)c.size(), max_slots - n_slots});
    c.resize(std::max<int32_t>(n, 0));
    std::sort(c.begin(), c.end());
    return c;
  }

  // Forward inputs of a selection: tokens and parents as tree-cache slots
  // (the slots the selection is about to get: n_slots + its index).
  void forward_inputs(const std::vector<int32_t>& sel, std::vector<int32_t>& toks,
                      std::vector<int32_t>& pars) const {
    toks.clear();
    pars.clear();
    for (size_t i = 0; i < sel.size(); ++i) {
      const Node& nd = nodes[sel[i]];
      toks.push_back(nd.token);
      int32_t ps = -1;
      if (nd.parent >= 0) {
        ps = nodes[nd.parent].slot;
        if (ps < 0)
          for (size_t j = 0; j < i; ++j)
            if (sel[j] == nd.parent) ps = n_slots + (int32_t)j;
      }
      pars.push_back(ps);
    }
  }

  // The selection was computed: slots n_slots.. in selection order.
  void computed(const std::vector<int32_t>& sel) {
    for (int32_t n : sel) nodes[n].slot = n_slots++;
  }

  // Top-K children of a computed node (tokens, log-probabilities).
  void add_children(int32_t node, const int32_t* tok, const double* logp, int32_t k) {
    for (int32_t i = 0; i < k; ++i) nodes.push_back(Node{tok[i], node, nodes[node].weight + logp[i], -1});
  }

  // "Get the most probable subgraph of size bs from the draft tree" (Alg. 1,
  // P:285): the bs most probable nodes of troot's subtree (troot has the
  // largest weight there and every chosen node's parent is more probable, so
  // the choice is a tree rooted at troot), renumbered in id order: toks[i],
  // pars[i] (local, root -1) and map[i] = node id.
  void subgraph(int32_t bs, std::vector<int32_t>& toks, std::vector<int32_t>& pars,
                std::vector<int32_t>& map) const {
    std::vector<int32_t> c;
    for (int32_t i = 0; i < (int32_t)nodes.size(); ++i)
      if (in_subtree(i, troot)) c.push_back(i);
    std::sort(c.begin(), c.end(), [&](int32_t a, int32_t b) { return before(a, b); });
    if ((int32_t)c.size() > bs) c.resize(bs);
    std::sort(c.begin(), c.end());
    map = c;
    toks.clear();
    pars.clear();
    for (size_t i = 0; i < c.size(); ++i) {
      toks.push_back(nodes[c[i]].token);
      int32_t p = -1;
      if (i > 0)
        for (size_t j = 0; j < i; ++j)
          if (c[j] == nodes[c[i]].parent) p = (int32_t)j;
      pars.push_back(p);
    }
  }

  // Re-root after the target verified path (node ids [troot, d1 .. dk]) and
  // sampled `bonus`.  The verified nodes from the draft root down
  // to dk are S; the computed prefix of S is committed to the draft's prefix
  // cache (commit_slots: a root-anchored chain of tree-cache slots); the new
  // target root is dk's child carrying `bonus` (created if the tree lacks
  // it).  If all of S was computed the new draft root is that child and the
  // computed nodes of its subtree stay in the tree cache, re-packed right
  // after the new prefix (keep_slots, ascending); otherwise the new draft root
  // is the first uncomputed verified node, and the rest of S plus the bonus
  // node stay as a weight-0 chain (nothing is kept).  Every other node is
  // discarded; ids are renumbered in order.  Returns the number committed.
  int32_t reroot(const std::vector<int32_t>& path, int32_t bonus, std::vector<int32_t>& commit_slots,
                 std::vector<int32_t>& keep_slots) {
    std::vector<int32_t> S;
    for (int32_t j = path[0]; j != -1; j = nodes[j].parent) S.push_back(j);
    std::reverse(S.begin(), S.end());  // draft root .. troot
    for (size_t i = 1; i < path.size(); ++i) S.push_back(path[i]);
    int32_t p = 0;
    while (p < (int32_t)S.size() && nodes[S[p]].slot >= 0) ++p;
    commit_slots.clear();
    keep_slots.clear();
    for (int32_t i = 0; i < p; ++i) commit_slots.push_back(nodes[S[i]].slot);
    const int32_t last = S.back();
    int32_t e = -1;
    for (int32_t i = last + 1; i < (int32_t)nodes.size() && e < 0; ++i)
      if (nodes[i].parent == last && nodes[i].token == bonus) e = i;
    if (e < 0) {
      nodes.push_back(Node{bonus, last, nodes[last].weight, -1});
      e = (int32_t)nodes.size() - 1;
    }
    const int32_t new_root = p < (int32_t)S.size() ? S[p] : e;
    // retained nodes: new_root's subtree
    std::vector<int32_t> keep_nodes;
    for (int32_t i = 0; i < (int32_t)nodes.size(); ++i)
      if (in_subtree(i, new_root)) keep_nodes.push_back(i);
    // weights: the verified chain is certain (0); the bonus node's subtree is
    // re-based on the bonus node
    const double we = nodes[e].weight;
    std::vector<double> nw(nodes.size(), 0.0);
    for (int32_t i : keep_nodes) nw[i] = in_subtree(i, e) ? nodes[i].weight - we : 0.0;
    // tree-cache rows that stay: computed retained nodes in slot order
    std::vector<int32_t> comp;
    for (int32_t i : keep_nodes)
      if (nodes[i].slot >= 0) comp.push_back(i);
    std::sort(comp.begin(), comp.end(), [&](int32_t a, int32_t b) { return nodes[a].slot < nodes[b].slot; });
    std::vector<int32_t> new_slot(nodes.size(), -1);
    for (size_t j = 0; j < comp.size(); ++j) {
      keep_slots.push_back(nodes[comp[j]].slot);
      new_slot[comp[j]] = (int32_t)j;
    }
    // renumber
    std::vector<int32_t> new_id(nodes.size(), -1);
    std::vector<Node> nn;
    for (int32_t i : keep_nodes) {
      new_id[i] = (int32_t)nn.size();
      nn.push_back(Node{nodes[i].token, i == new_root ? -1 : new_id[nodes[i].parent], nw[i], new_slot[i]});
    }
    troot = new_id[e];
    nodes.swap(nn);
    n_slots = (int32_t)comp.size();
    return p;
  }
};

}  // namespace draft
}  // namespace ss
