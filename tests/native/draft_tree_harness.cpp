// CPU test harness: the draft worker's tree (paper_2506_11309_b200/csrc/
// draft_tree.h, the header the draft loop uses) behind extern "C" functions so
// tests/test_draft_tree.py can compare it with oracle/draft_tree.py.  Test
// infrastructure only.
#include <vector>

#include "../../paper_2506_11309_b200/csrc/draft_tree.h"

using ss::draft::Tree;

extern "C" {
void* dt_new(int root_token, int max_slots) {
  Tree* t = new Tree();
  t->max_slots = max_slots;
  t->reset(root_token);
  return t;
}
void dt_free(void* p) { delete static_cast<Tree*>(p); }
int dt_n_nodes(void* p) { return (int)static_cast<Tree*>(p)->nodes.size(); }
int dt_n_slots(void* p) { return static_cast<Tree*>(p)->n_slots; }
int dt_troot(void* p) { return static_cast<Tree*>(p)->troot; }
int dt_size(void* p) { return static_cast<Tree*>(p)->size_from_troot(); }
// node i -> (token, parent, slot), weight
void dt_node(void* p, int i, int* out3, double* w) {
  const auto& n = static_cast<Tree*>(p)->nodes[i];
  out3[0] = n.token;
  out3[1] = n.parent;
  out3[2] = n.slot;
  *w = n.weight;
}
// select + forward inputs: returns the count; sel / toks / pars sized >= w
int dt_select(void* p, int w, int* sel, int* toks, int* pars) {
  Tree* t = static_cast<Tree*>(p);
  std::vector<int32_t> s = t->select(w), tk, pr;
  t->forward_inputs(s, tk, pr);
  for (size_t i = 0; i < s.size(); ++i) {
    sel[i] = s[i];
    toks[i] = tk[i];
    pars[i] = pr[i];
  }
  return (int)s.size();
}
void dt_computed(void* p, const int* sel, int n) {
  static_cast<Tree*>(p)->computed(std::vector<int32_t>(sel, sel + n));
}
void dt_add_children(void* p, int node, const int* tok, const double* logp, int k) {
  static_cast<Tree*>(p)->add_children(node, tok, logp, k);
}
int dt_subgraph(void* p, int bs, int* toks, int* pars, int* map) {
  std::vector<int32_t> tk, pr, mp;
  static_cast<Tree*>(p)->subgraph(bs, tk, pr, mp);
  for (size_t i = 0; i < tk.size(); ++i) {
    toks[i] = tk[i];
    pars[i] = pr[i];
    map[i] = mp[i];
  }
  return (int)tk.size();
}
// returns n committed; *nc / *nk = list lengths
int dt_reroot(void* p, const int* path, int n, int bonus, int* commit, int* nc, int* keep, int* nk) {
  std::vector<int32_t> c, k;
  int r = static_cast<Tree*>(p)->reroot(std::vector<int32_t>(path, path + n), bonus, c, k);
  for (size_t i = 0; i < c.size(); ++i) commit[i] = c[i];
  for (size_t i = 0; i < k.size(); ++i) keep[i] = k[i];
  *nc = (int)c.size();
  *nk = (int)k.size();
  return r;
}
}
