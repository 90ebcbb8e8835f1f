// Static memory planner (native core).
//
// Restates planner.py:221-348 (_plan_view, _longest_path_order) over the flat
// index view built by the host layer (planner.py:164-200).  The plan must be
// bit-exact with the reference, so every iteration order the reference
// depends on is reproduced here:
//   * op visit order: sorted (phase, i) for none/inplace; for coshare/both a
//     heap over (phase, depth-to-sink, i)            (planner.py:232-236, 317-348)
//   * free-pool pops are LIFO per exact byte size     (planner.py:282-284)
//   * freed inputs are appended to the pools in the iteration order of a
//     CPython set built from the node's input list   (planner.py:298-304);
//     that order is emulated exactly by PySmallIntSet below
//   * extra edges are a set, returned sorted          (planner.py:307)

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <map>
#include <queue>
#include <set>
#include <tuple>
#include <utility>
#include <vector>

#include "mgx.h"

namespace mgx {
void set_error(const char* fmt, ...);
}

namespace {

// Iteration order of CPython's set(list_of_small_non_negative_ints).
// CPython 3.x setobject.c: hash(i) == i, open addressing with LINEAR_PROBES=9
// then perturbed probing, table starts at 8 slots and is resized to
// used*4 (next power of two) when fill*5 >= mask*3; iteration walks the table.
class PySmallIntSet {
 public:
  explicit PySmallIntSet(const std::vector<int64_t>& keys) {
    table_.assign(8, kEmpty);
    mask_ = 7;
    for (int64_t k : keys) add(k);
  }
  std::vector<int64_t> order() const {
    std::vector<int64_t> out;
    for (int64_t v : table_)
      if (v != kEmpty) out.push_back(v);
    return out;
  }

 private:
  static constexpr int64_t kEmpty = -1;
  static constexpr size_t kLinearProbes = 9;
  static constexpr int kPerturbShift = 5;

  void add(int64_t key) {
    size_t hash = static_cast<size_t>(key);
    size_t perturb = hash;
    size_t i = hash & mask_;
    while (true) {
      size_t probes = (i + kLinearProbes <= mask_) ? kLinearProbes : 0;
      size_t j = i;
      while (true) {
        if (table_[j] == kEmpty) {
          table_[j] = key;
          ++fill_;
          ++used_;
          if (fill_ * 5 >= mask_ * 3) resize(used_ > 50000 ? used_ * 2 : used_ * 4);
          return;
        }
        if (table_[j] == key) return;
        if (probes == 0) break;
        --probes;
        ++j;
      }
      perturb >>= kPerturbShift;
      i = (i * 5 + 1 + perturb) & mask_;
    }
  }

  void resize(size_t minused) {
    size_t newsize = 8;
    while (newsize <= minused) newsize <<= 1;
    std::vector<int64_t> old = table_;
    table_.assign(newsize, kEmpty);
    mask_ = newsize - 1;
    fill_ = used_;
    for (int64_t key : old) {
      if (key == kEmpty) continue;
      insert_clean(key);
    }
  }

  void insert_clean(int64_t key) {
    size_t hash = static_cast<size_t>(key);
    size_t perturb = hash;
    size_t i = hash & mask_;
    while (true) {
      if (table_[i] == kEmpty) {
        table_[i] = key;
        return;
      }
      if (i + kLinearProbes <= mask_) {
        for (size_t j = 1; j <= kLinearProbes; ++j) {
          if (table_[i + j] == kEmpty) {
            table_[i + j] = key;
            return;
          }
        }
      }
      perturb >>= kPerturbShift;
      i = (i * 5 + 1 + perturb) & mask_;
    }
  }

  std::vector<int64_t> table_;
  size_t mask_ = 7;
  size_t fill_ = 0;
  size_t used_ = 0;
};

}  // namespace

extern "C" int mgx_py_set_order(const int64_t* keys, int32_t n, int64_t* out, int32_t* n_out) {
  if (n < 0 || (n > 0 && (!keys || !out)) || !n_out) {
    mgx::set_error("mgx_py_set_order: bad arguments");
    return MGX_BAD_ARGUMENT;
  }
  for (int32_t i = 0; i < n; ++i) {
    if (keys[i] < 0) {
      mgx::set_error("mgx_py_set_order: keys must be non-negative");
      return MGX_BAD_ARGUMENT;
    }
  }
  std::vector<int64_t> v(keys, keys + n);
  auto order = PySmallIntSet(v).order();
  for (size_t i = 0; i < order.size(); ++i) out[i] = order[i];
  *n_out = static_cast<int32_t>(order.size());
  return MGX_OK;
}

extern "C" int mgx_plan_memory(int32_t n, const uint8_t* is_var, const int64_t* nbytes,
                               const uint8_t* dedicated, const int32_t* in_ptr,
                               const int32_t* in_idx, const int32_t* ip_ptr,
                               const int32_t* ip_pos, const int32_t* phase_in,
                               int32_t strategy, int32_t* slot_of, int64_t* slot_bytes,
                               uint8_t* slot_dedicated, int32_t* n_slots, int32_t* edges,
                               int32_t edge_cap, int32_t* n_edges,
                               int64_t* total_internal_bytes, int64_t* visits_out) {
  if (n < 0 || strategy < 0 || strategy > 3 || !is_var || !nbytes || !dedicated ||
      !in_ptr || !ip_ptr || !slot_of || !slot_bytes || !slot_dedicated || !n_slots ||
      !n_edges || !total_internal_bytes || !visits_out || (edge_cap > 0 && !edges)) {
    mgx::set_error("mgx_plan_memory: bad arguments");
    return MGX_BAD_ARGUMENT;
  }
  const bool use_pool = strategy != 0;
  const bool use_claims = strategy == 1 || strategy == 3;
  const bool coshare = strategy == 2 || strategy == 3;
  int64_t visits = 0;

  std::vector<std::vector<int32_t>> inputs(n), consumers(n);
  for (int32_t i = 0; i < n; ++i) {
    for (int32_t e = in_ptr[i]; e < in_ptr[i + 1]; ++e) {
      int32_t u = in_idx[e];
      if (u < 0 || u >= n) {
        mgx::set_error("mgx_plan_memory: input index %d out of range", u);
        return MGX_BAD_ARGUMENT;
      }
      inputs[i].push_back(u);
    }
  }
  for (int32_t i = 0; i < n; ++i)
    for (int32_t u : inputs[i]) consumers[u].push_back(i);
  std::vector<int32_t> phase(n, 0);
  if (phase_in)
    for (int32_t i = 0; i < n; ++i) phase[i] = phase_in[i];

  std::vector<int32_t> op_nodes;
  for (int32_t i = 0; i < n; ++i)
    if (!is_var[i]) op_nodes.push_back(i);

  // ---- allocation order (planner.py:232-236)
  std::vector<int32_t> order;
  if (coshare) {
    // _longest_path_order (planner.py:317-348)
    std::vector<uint8_t> isop(n, 0);
    for (int32_t i : op_nodes) isop[i] = 1;
    std::vector<int64_t> depth(n, 1);
    for (auto it = op_nodes.rbegin(); it != op_nodes.rend(); ++it) {
      int32_t i = *it;
      ++visits;
      for (int32_t c : consumers[i])
        if (isop[c] && phase[c] == phase[i]) depth[i] = std::max(depth[i], 1 + depth[c]);
    }
    std::vector<int64_t> indeg(n, 0);
    for (int32_t i : op_nodes)
      for (int32_t u : inputs[i])
        if (isop[u]) ++indeg[i];
    using Key = std::tuple<int64_t, int64_t, int64_t>;
    std::priority_queue<Key, std::vector<Key>, std::greater<Key>> ready;
    for (int32_t i : op_nodes)
      if (indeg[i] == 0) ready.emplace(phase[i], depth[i], i);
    while (!ready.empty()) {
      int32_t cur = static_cast<int32_t>(std::get<2>(ready.top()));
      ready.pop();
      ++visits;
      order.push_back(cur);
      for (int32_t c : consumers[cur]) {
        ++visits;
        if (!isop[c]) continue;
        if (--indeg[c] == 0) ready.emplace(phase[c], depth[c], c);
      }
    }
    if (order.size() < op_nodes.size()) {
      mgx::set_error("allocation scheduler stalled (cycle?)");
      return MGX_INTERNAL;
    }
  } else {
    order = op_nodes;
    std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) {
      return std::make_pair(phase[a], a) < std::make_pair(phase[b], b);
    });
  }

  // ---- slot assignment (planner.py:238-304)
  int32_t next_slot = 0;
  std::vector<int64_t> sbytes;
  std::vector<uint8_t> sded;
  for (int32_t i = 0; i < n; ++i) slot_of[i] = -1;
  auto fresh = [&](int32_t i, bool ded) {
    int32_t s = next_slot++;
    slot_of[i] = s;
    sbytes.push_back(nbytes[i]);
    sded.push_back(ded ? 1 : 0);
  };
  for (int32_t i = 0; i < n; ++i)
    if (is_var[i]) fresh(i, true);

  std::vector<int64_t> refcount(n);
  for (int32_t i = 0; i < n; ++i) refcount[i] = static_cast<int64_t>(consumers[i].size());
  std::map<int64_t, std::vector<std::pair<int32_t, int32_t>>> pool;
  std::vector<uint8_t> transferred(n, 0);
  std::set<std::pair<int32_t, int32_t>> extra;

  auto in_inputs = [&](int32_t v, int32_t c) {
    return std::find(inputs[v].begin(), inputs[v].end(), c) != inputs[v].end();
  };

  for (int32_t v : order) {
    ++visits;
    bool placed = false;
    if (dedicated[v]) {
      fresh(v, true);
      placed = true;
    }
    if (!placed && use_claims) {
      const auto& ins = inputs[v];
      for (int32_t e = ip_ptr[v]; e < ip_ptr[v + 1]; ++e) {
        int32_t pos = ip_pos[e];
        if (pos < 0 || pos >= static_cast<int32_t>(ins.size())) continue;
        int32_t u = ins[pos];
        int64_t cnt = std::count(ins.begin(), ins.end(), u);
        if (!dedicated[u] && !is_var[u] && refcount[u] == 1 && cnt == 1 &&
            nbytes[u] == nbytes[v]) {
          slot_of[v] = slot_of[u];
          transferred[u] = 1;
          for (int32_t c : consumers[u]) {
            ++visits;
            if (c != v && !in_inputs(v, c)) extra.emplace(c, v);
          }
          placed = true;
          break;
        }
      }
    }
    if (!placed && use_pool) {
      auto it = pool.find(nbytes[v]);
      if (it != pool.end() && !it->second.empty()) {
        auto [slot, owner] = it->second.back();
        it->second.pop_back();
        slot_of[v] = slot;
        const auto& cons = consumers[owner];
        if (!cons.empty()) {
          std::set<int32_t> uniq(cons.begin(), cons.end());
          for (int32_t c : uniq) {
            ++visits;
            if (c != v && !in_inputs(v, c)) extra.emplace(c, v);
          }
        } else if (!in_inputs(v, owner)) {
          extra.emplace(owner, v);
        }
        placed = true;
      }
    }
    if (!placed) fresh(v, false);
    std::vector<int64_t> ins64(inputs[v].begin(), inputs[v].end());
    for (int64_t u64 : PySmallIntSet(ins64).order()) {
      int32_t u = static_cast<int32_t>(u64);
      ++visits;
      if (dedicated[u]) continue;
      refcount[u] -= std::count(inputs[v].begin(), inputs[v].end(), u);
      if (refcount[u] == 0 && !transferred[u]) pool[nbytes[u]].emplace_back(slot_of[u], u);
    }
  }

  // ---- acyclicity invariant (planner.py:351-373)
  {
    std::vector<std::vector<int32_t>> adj(n);
    std::vector<int64_t> indeg(n, 0);
    for (int32_t i = 0; i < n; ++i)
      for (int32_t u : inputs[i]) {
        adj[u].push_back(i);
        ++indeg[i];
      }
    for (auto& e : extra) {
      adj[e.first].push_back(e.second);
      ++indeg[e.second];
    }
    std::vector<int32_t> stack;
    for (int32_t i = 0; i < n; ++i)
      if (indeg[i] == 0) stack.push_back(i);
    int32_t seen = 0;
    while (!stack.empty()) {
      int32_t x = stack.back();
      stack.pop_back();
      ++seen;
      for (int32_t y : adj[x])
        if (--indeg[y] == 0) stack.push_back(y);
    }
    if (seen != n) {
      mgx::set_error("extra dependency edges introduced a cycle");
      return MGX_INTERNAL;
    }
  }

  int64_t total = 0;
  for (size_t s = 0; s < sbytes.size(); ++s) {
    slot_bytes[s] = sbytes[s];
    slot_dedicated[s] = sded[s];
    if (!sded[s]) total += sbytes[s];
  }
  *n_slots = next_slot;
  int32_t ne = 0;
  for (auto& e : extra) {
    if (ne < edge_cap) {
      edges[2 * ne] = e.first;
      edges[2 * ne + 1] = e.second;
    }
    ++ne;
  }
  *n_edges = ne;
  *total_internal_bytes = total;
  *visits_out = visits;
  if (ne > edge_cap) {
    mgx::set_error("mgx_plan_memory: %d edges exceed capacity %d", ne, edge_cap);
    return MGX_BAD_ARGUMENT;
  }
  return MGX_OK;
}
