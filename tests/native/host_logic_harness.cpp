// CPU test harness: exposes the C-ABI's host-side checks and call-order state
// machine (paper_2506_11309_b200/csrc/host_logic.h, the same header shard.cu
// uses) through extern "C" functions so tests/test_host_logic.py can drive
// every host-detected error code without a GPU.  Test infrastructure only.
#include <string>

#include "../../paper_2506_11309_b200/csrc/host_logic.h"

using ss::host::CallState;
static thread_local std::string g_msg;

extern "C" {
void* hl_new(int max_ctx, int max_tree, int vocab) {
  CallState* c = new CallState();
  c->max_ctx = max_ctx;
  c->max_tree = max_tree;
  c->vocab = vocab;
  return c;
}
void hl_free(void* p) { delete static_cast<CallState*>(p); }
void hl_set(void* p, int weights_ready, int peers_ready, int L, int max_written) {
  CallState* c = static_cast<CallState*>(p);
  c->weights_ready = weights_ready != 0;
  c->peers_ready = peers_ready != 0;
  c->L = L;
  c->max_written = max_written;
}
int hl_check_tree(void* p, const int32_t* t, const int32_t* par, int T) {
  return ss::host::check_tree(*static_cast<CallState*>(p), t, par, T, g_msg);
}
int hl_check_verify(void* p, int T) { return ss::host::check_verify(*static_cast<CallState*>(p), T, g_msg); }
int hl_check_commit(void* p, const int32_t* a, int n) {
  return ss::host::check_commit(*static_cast<CallState*>(p), a, n, g_msg);
}
int hl_check_extend(void* p, const int32_t* t, const int32_t* par, int T0, int w) {
  return ss::host::check_extend(*static_cast<CallState*>(p), t, par, T0, w, g_msg);
}
void hl_on_extend(void* p, int T0, int w, const int32_t* par) {
  ss::host::on_extend(*static_cast<CallState*>(p), T0, w, par);
}
int hl_check_reroot(void* p, const int32_t* path, int n, const int32_t* keep, int m) {
  return ss::host::check_reroot(*static_cast<CallState*>(p), path, n, keep, m, g_msg);
}
void hl_on_reroot(void* p, const int32_t* path, int n, const int32_t* keep, int m) {
  ss::host::on_reroot(*static_cast<CallState*>(p), path, n, keep, m);
}
int hl_last_T(void* p) { return static_cast<CallState*>(p)->last_T; }
int hl_check_set_len(void* p, int L) { return ss::host::check_set_len(*static_cast<CallState*>(p), L, g_msg); }
void hl_on_verify(void* p, int T, const int32_t* par, int auto_commit) {
  ss::host::on_verify(*static_cast<CallState*>(p), T, par, auto_commit != 0);
}
void hl_on_commit(void* p, int n) { ss::host::on_commit(*static_cast<CallState*>(p), n); }
void hl_on_set_len(void* p, int L) { ss::host::on_set_len(*static_cast<CallState*>(p), L); }
int hl_L(void* p) { return static_cast<CallState*>(p)->L; }
int hl_have_verify(void* p) { return static_cast<CallState*>(p)->have_verify ? 1 : 0; }
int hl_max_written(void* p) { return static_cast<CallState*>(p)->max_written; }
const char* hl_msg() { return g_msg.c_str(); }
}
