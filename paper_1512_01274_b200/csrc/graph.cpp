// Native graph builder: reverse-mode gradient structure and the bind-time
// launch order, over the flat index form of a symbol graph.
//
// The host layer (symbol.py / executor.py) flattens a graph into arrays
// indexed by topological position and turns the records produced here back
// into nodes.  Node names come from the host's counters in record order, so
// the records must be emitted in exactly the order the reference creates its
// nodes (symbol.py:227-298):
//   * the reverse topological walk visits an operator only if something
//     feeds it a gradient (a seeded output, a consumer's Backward) or it is a
//     loss head;
//   * its incoming contributions are folded left to right into a chain of
//     ElementwiseAdd records (`add` counter) just before its Backward records;
//   * one Backward record per input slot, in slot order (`bwd` counter),
//     whose inputs are the values its kernel reads (roles);
//   * after the walk, each requested argument gets its folded sum, or a
//     ZerosLike record (`zeros` counter) if no gradient reaches it.
// The launch order (executor.py:143-185) is a min-heap over (phase, index)
// on the graph's edges plus the planner's extra ordering edges.

#include <cstdint>
#include <queue>
#include <utility>
#include <vector>

#include "mgx.h"

namespace mgx {
void set_error(const char* fmt, ...);
}

namespace {

// Endpoint codes: [0, n) original nodes, [n, n+nseed) head-gradient
// variables, [n+nseed, ...) records emitted here.  kNone = "no value".
constexpr int64_t kNone = -1;

struct GradWriter {
  int32_t cap;
  int32_t count = 0;
  int32_t in_count = 0;
  int32_t in_cap;
  int32_t* kind;
  int64_t* a;
  int64_t* b;
  int32_t* in_ptr;
  int64_t* in_idx;
  int64_t base;  // endpoint code of record 0

  bool room(int32_t extra_inputs) const {
    return count < cap && in_count + extra_inputs <= in_cap;
  }
  int64_t emit(int32_t k, int64_t x, int64_t y) {
    kind[count] = k;
    a[count] = x;
    b[count] = y;
    in_ptr[count + 1] = in_count;
    return base + count++;
  }
};

}  // namespace

extern "C" int mgx_grad_build(int32_t n, const uint8_t* is_var, const uint8_t* is_loss,
                              const uint8_t* differentiable, const int32_t* in_ptr,
                              const int32_t* in_idx, int32_t nseed, const int32_t* seed_node,
                              const int32_t* role_ptr, const int32_t* role_code, int32_t nwrt,
                              const int32_t* wrt_node, int32_t cap, int32_t in_cap,
                              int32_t* rec_kind, int64_t* rec_a, int64_t* rec_b,
                              int32_t* rec_in_ptr, int64_t* rec_in_idx, int64_t* wrt_out,
                              int32_t* n_rec, int32_t* bad_node) {
  if (n < 0 || nseed < 0 || nwrt < 0 || cap < 0 || !n_rec || !bad_node) {
    mgx::set_error("mgx_grad_build: bad sizes");
    return MGX_BAD_ARGUMENT;
  }
  *bad_node = -1;
  GradWriter w{cap, 0, 0, in_cap, rec_kind, rec_a, rec_b, rec_in_ptr, rec_in_idx,
               static_cast<int64_t>(n) + nseed};
  rec_in_ptr[0] = 0;

  // gradient contributions reaching each original node, in arrival order
  std::vector<std::vector<int64_t>> arrivals(n);
  for (int32_t s = 0; s < nseed; ++s) arrivals[seed_node[s]].push_back(n + s);

  // fold a contribution list left to right: ((c0 + c1) + c2) + ...
  auto fold = [&](const std::vector<int64_t>& parts, int64_t* out) -> bool {
    int64_t acc = parts[0];
    for (size_t p = 1; p < parts.size(); ++p) {
      if (!w.room(0)) return false;
      acc = w.emit(MGX_GREC_ADD, acc, parts[p]);
    }
    *out = acc;
    return true;
  };
  auto overflow = [&]() {
    mgx::set_error("mgx_grad_build: record capacity %d exceeded", cap);
    return MGX_INTERNAL;
  };

  for (int32_t i = n - 1; i >= 0; --i) {
    if (is_var[i]) continue;
    const std::vector<int64_t>& mine = arrivals[i];
    if (mine.empty() && !is_loss[i]) continue;
    if (!differentiable[i]) {
      *bad_node = i;
      mgx::set_error("mgx_grad_build: node %d has no backward", i);
      return MGX_BAD_ARGUMENT;
    }
    int64_t og = kNone;
    if (!is_loss[i] && !fold(mine, &og)) return overflow();
    const int32_t nin = in_ptr[i + 1] - in_ptr[i];
    for (int32_t k = 0; k < nin; ++k) {
      const int32_t pair = in_ptr[i] + k;  // (node, slot) pairs share in_ptr
      const int32_t r0 = role_ptr[pair], r1 = role_ptr[pair + 1];
      if (!w.room(r1 - r0)) return overflow();
      for (int32_t r = r0; r < r1; ++r) {
        const int32_t code = role_code[r];
        int64_t ep;
        if (code == MGX_ROLE_OG) ep = og;
        else if (code == MGX_ROLE_OUT) ep = i;
        else ep = in_idx[in_ptr[i] + code];
        w.in_idx[w.in_count++] = ep;
      }
      const int64_t rec = w.emit(MGX_GREC_BACKWARD, i, k);
      arrivals[in_idx[pair]].push_back(rec);
    }
  }
  for (int32_t j = 0; j < nwrt; ++j) {
    const std::vector<int64_t>& mine = arrivals[wrt_node[j]];
    if (mine.empty()) {
      if (!w.room(0)) return overflow();
      wrt_out[j] = w.emit(MGX_GREC_ZEROS, wrt_node[j], 0);
    } else if (!fold(mine, &wrt_out[j])) {
      return overflow();
    }
  }
  *n_rec = w.count;
  return MGX_OK;
}

extern "C" int mgx_push_order(int32_t n, const uint8_t* is_var, const int32_t* phase,
                              const int32_t* in_ptr, const int32_t* in_idx, int32_t nextra,
                              const int32_t* extra, int32_t* order, int32_t* n_order) {
  if (n < 0 || nextra < 0 || !n_order) {
    mgx::set_error("mgx_push_order: bad sizes");
    return MGX_BAD_ARGUMENT;
  }
  // successor lists over operator nodes: graph edges first, then the extra
  // ordering edges, each in input order (a node may appear twice, matching
  // a multigraph's in-degree)
  std::vector<std::vector<int32_t>> next(n);
  std::vector<int32_t> pending(n, 0);
  int32_t ops = 0;
  for (int32_t i = 0; i < n; ++i) {
    if (is_var[i]) continue;
    ++ops;
    for (int32_t p = in_ptr[i]; p < in_ptr[i + 1]; ++p) {
      const int32_t u = in_idx[p];
      if (is_var[u]) continue;
      next[u].push_back(i);
      ++pending[i];
    }
  }
  for (int32_t e = 0; e < nextra; ++e) {
    const int32_t u = extra[2 * e], v = extra[2 * e + 1];
    if (u < 0 || v < 0 || u >= n || v >= n || is_var[u] || is_var[v]) continue;
    next[u].push_back(v);
    ++pending[v];
  }
  using Key = std::pair<int32_t, int32_t>;  // (phase, topo index)
  std::priority_queue<Key, std::vector<Key>, std::greater<Key>> ready;
  for (int32_t i = 0; i < n; ++i)
    if (!is_var[i] && pending[i] == 0) ready.push({phase[i], i});
  std::vector<uint8_t> emitted(n, 0);
  int32_t count = 0;
  while (!ready.empty()) {
    const int32_t i = ready.top().second;
    ready.pop();
    if (emitted[i]) continue;
    emitted[i] = 1;
    order[count++] = i;
    for (int32_t c : next[i])
      if (--pending[c] == 0) ready.push({phase[c], c});
  }
  *n_order = count;
  if (count != ops) {
    mgx::set_error("mgx_push_order: graph plus extra edges is not acyclic");
    return MGX_BAD_ARGUMENT;
  }
  return MGX_OK;
}
