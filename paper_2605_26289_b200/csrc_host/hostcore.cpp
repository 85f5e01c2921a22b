// Native host core: the unified cell allocator / page tables and the radix
// prefix trie of the coordination thread, behind the same
// Python API as kvcache.UnifiedKvCache and radix.RadixTrie.
//
// Same observable semantics as the reference (and as the Python restatement,
// which stays selectable with DS_HOST_CORE=python):
//  * first-fit allocation from the lowest free address, possibly several runs
//    (reference kvcache.py:116-131), coalescing frees (:133-148), int32
//    refcounts, one span per append / alias (:191-255), span-slicing trim
//    (:257-279) - cell ids are part of the parity contract;
//  * radix walk touching every visited node (radix.py:81-100), delta-only
//    save with split on divergence and path-protected eviction (:104-163),
//    leaf-oldest eviction keyed by (last_touch, first token) (:167-196);
//  * every page-table mutation recorded as a device op (int32 x5: kind, seq,
//    pos, first cell, length) for ds_kv_apply.
// The hot spots this replaces are the reference's Python _common_len, radix
// save / lookup and allocator / decref (radix.py:43-163, kvcache.py:116-183).
#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include <algorithm>
#include <cstdint>
#include <queue>
#include <stdexcept>
#include <string>
#include <tuple>
#include <unordered_map>
#include <vector>

namespace py = pybind11;

namespace {

using Run = std::pair<int64_t, int64_t>;  // (first cell, length)
enum { KV_MAP = 0, KV_UNMAP = 1, KV_TRIE_INC = 2, KV_TRIE_DEC = 3 };

py::object g_capacity_exc, g_donor_exc, g_budget_exc;

[[noreturn]] void raise_py(const py::object& cls, const std::string& msg) {
  PyErr_SetString(cls.ptr(), msg.c_str());
  throw py::error_already_set();
}
[[noreturn]] void raise_value(const std::string& msg) { throw py::value_error(msg); }

std::vector<Run> slice_runs(const std::vector<Run>& runs, int64_t offset, int64_t length) {
  std::vector<Run> out;
  if (length <= 0) return out;
  const int64_t stop = offset + length;
  int64_t base = 0;
  for (const auto& r : runs) {
    const int64_t lo = std::max(offset, base), hi = std::min(stop, base + r.second);
    if (hi > lo) out.emplace_back(r.first + lo - base, hi - lo);
    base += r.second;
    if (base >= stop) break;
  }
  return out;
}

int64_t run_cells(const std::vector<Run>& runs) {
  int64_t n = 0;
  for (const auto& r : runs) n += r.second;
  return n;
}

std::vector<Run> to_runs(const py::iterable& it) {
  std::vector<Run> out;
  for (auto h : it) {
    auto t = h.cast<py::sequence>();
    out.emplace_back(t[0].cast<int64_t>(), t[1].cast<int64_t>());
  }
  return out;
}

py::list runs_list(const std::vector<Run>& runs) {
  py::list l;
  for (const auto& r : runs) l.append(py::make_tuple(r.first, r.second));
  return l;
}

struct Span {
  int64_t start, length;
  std::vector<Run> runs;
  bool owned;
  int64_t end() const { return start + length; }
};

class KvCore {
 public:
  explicit KvCore(int64_t capacity) : cap_(capacity), rc_(capacity, 0) {
    if (capacity <= 0) raise_value("capacity_cells must be positive");
    fstart_.push_back(0);
    flen_.push_back(capacity);
    free_ = capacity;
  }

  bool record_ops = false;
  int64_t capacity() const { return cap_; }
  int64_t free_cells() const { return free_; }
  int64_t occupancy() const { return cap_ - free_; }

  int64_t seq_len(int64_t seq) const {
    auto it = tables_.find(seq);
    return (it == tables_.end() || it->second.empty()) ? 0 : it->second.back().end();
  }
  int64_t span_count(int64_t seq) const {
    auto it = tables_.find(seq);
    return it == tables_.end() ? 0 : static_cast<int64_t>(it->second.size());
  }
  std::vector<int64_t> sequences() const {
    std::vector<int64_t> out;
    for (int64_t s : order_) {
      auto it = tables_.find(s);
      if (it != tables_.end() && !it->second.empty()) out.push_back(s);
    }
    return out;
  }
  int32_t refcount(int64_t cell) const {
    if (cell < 0 || cell >= cap_) throw py::index_error("cell out of range");
    return rc_[cell];
  }
  py::array_t<int32_t> refcounts() const {
    py::array_t<int32_t> a(cap_);
    std::copy(rc_.begin(), rc_.end(), a.mutable_data());
    return a;
  }

  py::array_t<int32_t> take_ops() {
    const py::ssize_t n = static_cast<py::ssize_t>(ops_.size() / 5);
    py::array_t<int32_t> a({n, static_cast<py::ssize_t>(5)});
    if (n) std::copy(ops_.begin(), ops_.end(), a.mutable_data());
    ops_.clear();
    return a;
  }

  // -- refcounting --
  void incref_runs(const std::vector<Run>& runs) {
    std::vector<Run> done;
    try {
      for (const auto& r : runs) {  // per-run check-then-increment (kvcache.py:154-158)
        check_live(r, "incref of a dead cell");
        for (int64_t c = r.first; c < r.first + r.second; ++c) ++rc_[c];
        done.push_back(r);
      }
    } catch (...) {
      emit(KV_TRIE_INC, -1, 0, done);
      throw;
    }
    emit(KV_TRIE_INC, -1, 0, done);
  }
  // the device log gets exactly the runs whose drop happened (a run failing
  // its liveness check raises before it changes anything)
  int64_t decref_runs(const std::vector<Run>& runs) {
    std::vector<Run> done;
    int64_t freed = 0;
    try {
      for (const auto& r : runs) {
        freed += drop(std::vector<Run>{r});
        done.push_back(r);
      }
    } catch (...) {
      emit(KV_TRIE_DEC, -1, 0, done);
      throw;
    }
    emit(KV_TRIE_DEC, -1, 0, done);
    return freed;
  }

  // -- sequence operations --
  std::pair<int64_t, int64_t> append_cells(int64_t seq, int64_t n) {
    if (n <= 0) raise_value("n must be positive");
    auto runs = allocate(n);
    for (const auto& r : runs)
      std::fill(rc_.begin() + r.first, rc_.begin() + r.first + r.second, 1);
    const int64_t p = append_span(seq, n, runs, true);
    emit(KV_MAP, seq, p, runs);
    return {p, p + n};
  }

  std::vector<Run> resolve_runs(int64_t seq, int64_t start, int64_t end) const {
    std::vector<Run> out;
    if (start >= end) return out;
    const int64_t len = seq_len(seq);
    if (len < end)
      raise_py(g_donor_exc, "seq " + std::to_string(seq) + " covers " + std::to_string(len) +
                                " < " + std::to_string(end));
    const auto& table = tables_.at(seq);
    // spans tile [0, len) in order: start at the one holding `start`
    auto it = std::upper_bound(table.begin(), table.end(), start,
                               [](int64_t v, const Span& s) { return v < s.start; });
    size_t i = it == table.begin() ? 0 : static_cast<size_t>(it - table.begin()) - 1;
    for (; i < table.size(); ++i) {
      const Span& sp = table[i];
      if (sp.start >= end) break;
      const int64_t lo = std::max(start, sp.start), hi = std::min(end, sp.end());
      if (hi > lo) {
        auto part = slice_runs(sp.runs, lo - sp.start, hi - lo);
        out.insert(out.end(), part.begin(), part.end());
      }
    }
    return out;
  }

  void seq_alias(int64_t donor, int64_t dest, int64_t start, int64_t end) {
    if (start >= end) raise_value("empty alias range");
    const int64_t dl = seq_len(donor);
    if (dl < end)
      raise_py(g_donor_exc, "donor " + std::to_string(donor) + " covers " + std::to_string(dl) +
                                " < " + std::to_string(end));
    if (seq_len(dest) != start)
      raise_value("dest " + std::to_string(dest) + " must hold exactly [0, " +
                  std::to_string(start) + ") before aliasing");
    auto runs = resolve_runs(donor, start, end);
    for (const auto& r : runs)
      for (int64_t c = r.first; c < r.first + r.second; ++c) ++rc_[c];
    table(dest).push_back(Span{start, end - start, runs, false});
    emit(KV_MAP, dest, start, runs);
  }

  void alias_runs(int64_t dest, const std::vector<Run>& runs) {
    const int64_t n = run_cells(runs);
    if (n == 0) return;
    std::vector<Run> done;
    for (const auto& r : runs) {  // per-run check-then-increment (kvcache.py:248-252)
      try {
        check_live(r, "alias of a dead cell");
      } catch (...) {
        // the runs already incremented stay held (reference semantics): the
        // device mirrors them as holds without a mapping (exact refcount)
        emit(KV_TRIE_INC, -1, 0, done);
        throw;
      }
      for (int64_t c = r.first; c < r.first + r.second; ++c) ++rc_[c];
      done.push_back(r);
    }
    const int64_t p = append_span(dest, n, runs, false);
    emit(KV_MAP, dest, p, runs);
  }

  int64_t trim(int64_t seq, int64_t from_pos) {
    const int64_t length = seq_len(seq);
    if (from_pos > length)
      raise_value("trim beyond length (" + std::to_string(from_pos) + " > " +
                  std::to_string(length) + ")");
    auto it = tables_.find(seq);
    if (it == tables_.end()) return 0;
    auto& t = it->second;
    int64_t freed = 0;
    while (!t.empty() && t.back().end() > from_pos) {
      Span& sp = t.back();
      const int64_t keep = std::max<int64_t>(0, from_pos - sp.start);
      auto dropped = slice_runs(sp.runs, keep, sp.length - keep);
      freed += drop(dropped);
      emit(KV_UNMAP, seq, sp.start + keep, dropped);
      if (keep) {
        sp.runs = slice_runs(sp.runs, 0, keep);
        sp.length = keep;
        break;
      }
      t.pop_back();
    }
    return freed;
  }

  int64_t release_sequence(int64_t seq) {
    int64_t freed = 0;
    if (tables_.count(seq)) {
      freed = trim(seq, 0);
      tables_.erase(seq);
      order_.erase(std::remove(order_.begin(), order_.end(), seq), order_.end());
    }
    return freed;
  }

  std::vector<int64_t> cell_ids(int64_t seq, int64_t start, int64_t end) const {
    std::vector<int64_t> out;
    for (const auto& r : resolve_runs(seq, start, end))
      for (int64_t c = r.first; c < r.first + r.second; ++c) out.push_back(c);
    return out;
  }

 private:
  void check_live(const Run& r, const char* msg) const {
    for (int64_t c = r.first; c < r.first + r.second; ++c)
      if (rc_[c] < 1) raise_value(msg);
  }

  void emit(int kind, int64_t seq, int64_t pos, const std::vector<Run>& runs) {
    if (!record_ops) return;
    for (const auto& r : runs) {
      ops_.push_back(kind);
      ops_.push_back(static_cast<int32_t>(seq));
      ops_.push_back(static_cast<int32_t>(pos));
      ops_.push_back(static_cast<int32_t>(r.first));
      ops_.push_back(static_cast<int32_t>(r.second));
      pos += r.second;
    }
  }

  std::vector<Span>& table(int64_t seq) {
    auto it = tables_.find(seq);
    if (it == tables_.end()) {
      order_.push_back(seq);
      it = tables_.emplace(seq, std::vector<Span>{}).first;
    }
    return it->second;
  }

  int64_t append_span(int64_t seq, int64_t length, const std::vector<Run>& runs, bool owned) {
    auto& t = table(seq);
    const int64_t p = t.empty() ? 0 : t.back().end();
    t.push_back(Span{p, length, runs, owned});
    return p;
  }

  std::vector<Run> allocate(int64_t n) {
    if (n > free_)
      raise_py(g_capacity_exc,
               "need " + std::to_string(n) + " cells, " + std::to_string(free_) + " free");
    std::vector<Run> out;
    size_t used = 0;  // whole runs consumed from the front
    while (n) {
      const int64_t start = fstart_[used], ln = flen_[used];
      const int64_t take = ln <= n ? ln : n;
      out.emplace_back(start, take);
      if (take == ln) {
        ++used;
      } else {
        fstart_[used] = start + take;
        flen_[used] = ln - take;
      }
      n -= take;
      free_ -= take;
    }
    if (used) {
      fstart_.erase(fstart_.begin(), fstart_.begin() + used);
      flen_.erase(flen_.begin(), flen_.begin() + used);
    }
    return out;
  }

  void release_run(int64_t start, int64_t length) {
    const size_t i = std::lower_bound(fstart_.begin(), fstart_.end(), start) - fstart_.begin();
    const bool mp = i > 0 && fstart_[i - 1] + flen_[i - 1] == start;
    const bool mn = i < fstart_.size() && start + length == fstart_[i];
    if (mp && mn) {
      flen_[i - 1] += length + flen_[i];
      fstart_.erase(fstart_.begin() + i);
      flen_.erase(flen_.begin() + i);
    } else if (mp) {
      flen_[i - 1] += length;
    } else if (mn) {
      fstart_[i] = start;
      flen_[i] += length;
    } else {
      fstart_.insert(fstart_.begin() + i, start);
      flen_.insert(flen_.begin() + i, length);
    }
    free_ += length;
  }

  // decrement every cell of runs; consecutive cells reaching zero return to
  // the free pool as one run each, in ascending order (kvcache.py:172-182)
  int64_t drop(const std::vector<Run>& runs) {
    int64_t freed = 0;
    for (const auto& r : runs) {
      check_live(r, "refcount underflow");
      int64_t a = -1;
      for (int64_t j = 0; j < r.second; ++j) {
        const bool dead = --rc_[r.first + j] == 0;
        if (dead && a < 0) {
          a = j;
        } else if (!dead && a >= 0) {
          release_run(r.first + a, j - a);
          freed += j - a;
          a = -1;
        }
      }
      if (a >= 0) {
        release_run(r.first + a, r.second - a);
        freed += r.second - a;
      }
    }
    return freed;
  }

  int64_t cap_;
  std::vector<int32_t> rc_;
  std::vector<int64_t> fstart_, flen_;
  int64_t free_ = 0;
  std::unordered_map<int64_t, std::vector<Span>> tables_;
  std::vector<int64_t> order_;  // table creation order (sequences())
  std::vector<int32_t> ops_;
};

// ---------------------------------------------------------------------------

int64_t common_len(const int32_t* a, int64_t na, const int32_t* b, int64_t nb) {
  const int64_t n = std::min(na, nb);
  int64_t i = 0;
  while (i < n && a[i] == b[i]) ++i;
  return i;
}

struct Node {
  std::vector<int32_t> seg;
  std::vector<Run> runs;
  int64_t donor = -1;  // -1: None
  int parent = -1;
  int64_t last_touch = 0;
  std::vector<std::pair<int32_t, int>> kids;  // insertion-ordered (first token, node)
};

class RadixCore {
 public:
  RadixCore(KvCore& kv, int64_t cell_budget) : kv_(kv), budget_(cell_budget) {
    nodes_.emplace_back();  // root
  }

  int64_t cell_budget() const { return budget_; }
  int64_t total_cells() const { return cells_; }
  int64_t evicted_cells_total = 0;

  int64_t node_count() const {
    int64_t n = 0;
    std::vector<int> stack{0};
    while (!stack.empty()) {
      const int x = stack.back();
      stack.pop_back();
      n += static_cast<int64_t>(nodes_[x].kids.size());
      for (const auto& k : nodes_[x].kids) stack.push_back(k.second);
    }
    return n;
  }

  // (length, runs, donor or None) - touches every node on the path
  py::tuple longest_prefix(const std::vector<int32_t>& tokens) {
    const int64_t tick = ++clock_;
    int64_t length = 0, donor = -1;
    std::vector<Run> runs;
    walk(tokens, tick, [&](int child, int64_t k, int64_t pos) {
      auto part = slice_runs(nodes_[child].runs, 0, k);
      runs.insert(runs.end(), part.begin(), part.end());
      donor = nodes_[child].donor;
      length = pos;
      return true;
    });
    return py::make_tuple(length, runs_list(runs),
                          donor < 0 ? py::object(py::none()) : py::object(py::int_(donor)));
  }

  int64_t save(const std::vector<int32_t>& tokens, int64_t seq) {
    const int64_t tick = ++clock_;
    int node = 0;
    int64_t i = 0;
    std::vector<char> prot(nodes_.size() + 1, 0);
    prot[0] = 1;
    const int64_t n = static_cast<int64_t>(tokens.size());
    walk(tokens, tick, [&](int child, int64_t k, int64_t pos) {
      mark(prot, child);
      i = pos;
      if (k < static_cast<int64_t>(nodes_[child].seg.size())) {
        if (i < n) {
          node = split(child, static_cast<int>(k));
          mark(prot, node);
        } else {
          node = child;
        }
        return false;
      }
      node = child;
      return true;
    });
    if (i >= n) return 0;
    const int64_t delta = n - i;
    if (cells_ + delta > budget_) {
      evict_impl(cells_ + delta - budget_, &prot);
      if (cells_ + delta > budget_)
        raise_py(g_budget_exc, "delta of " + std::to_string(delta) + " cells does not fit");
    }
    auto runs = kv_.resolve_runs(seq, i, n);
    kv_.incref_runs(runs);
    const int leaf = new_node();
    Node& nd = nodes_[leaf];
    nd.seg.assign(tokens.begin() + i, tokens.end());
    nd.runs = runs;
    nd.donor = seq;
    nd.parent = node;
    nd.last_touch = tick;
    nodes_[node].kids.emplace_back(tokens[i], leaf);
    cells_ += delta;
    return delta;
  }

  int64_t evict(int64_t needed) { return evict_impl(needed, nullptr); }
  int64_t clear() { return cells_ ? evict_impl(cells_, nullptr) : 0; }

  // (prefix_len, cells, last_touch, donor) per node, pre-order then stably
  // sorted by (prefix_len, last_touch)
  py::list dump() const {
    struct Row {
      int64_t plen, cells, touch, donor;
    };
    std::vector<Row> rows;
    std::vector<std::pair<int, int64_t>> stack;
    const auto& rk = nodes_[0].kids;
    for (auto it = rk.rbegin(); it != rk.rend(); ++it) stack.emplace_back(it->second, 0);
    while (!stack.empty()) {
      auto [x, depth] = stack.back();
      stack.pop_back();
      const Node& nd = nodes_[x];
      const int64_t end = depth + static_cast<int64_t>(nd.seg.size());
      rows.push_back(Row{end, run_cells(nd.runs), nd.last_touch, nd.donor});
      for (auto it = nd.kids.rbegin(); it != nd.kids.rend(); ++it) stack.emplace_back(it->second, end);
    }
    std::stable_sort(rows.begin(), rows.end(), [](const Row& a, const Row& b) {
      return a.plen != b.plen ? a.plen < b.plen : a.touch < b.touch;
    });
    py::list out;
    for (const auto& r : rows) {
      py::dict d;
      d["prefix_len"] = r.plen;
      d["cells"] = r.cells;
      d["last_touch"] = r.touch;
      d["donor"] = r.donor < 0 ? py::object(py::none()) : py::object(py::int_(r.donor));
      out.append(d);
    }
    return out;
  }

 private:
  static void mark(std::vector<char>& prot, int x) {
    if (static_cast<size_t>(x) >= prot.size()) prot.resize(x + 1, 0);
    prot[x] = 1;
  }
  static bool is_prot(const std::vector<char>* prot, int x) {
    return prot && static_cast<size_t>(x) < prot->size() && (*prot)[x];
  }

  int find_kid(int x, int32_t tok) const {
    for (const auto& k : nodes_[x].kids)
      if (k.first == tok) return k.second;
    return -1;
  }

  template <typename F>
  void walk(const std::vector<int32_t>& tokens, int64_t tick, F&& visit) {
    int node = 0;
    int64_t i = 0;
    const int64_t n = static_cast<int64_t>(tokens.size());
    while (i < n) {
      const int child = find_kid(node, tokens[i]);
      if (child < 0) return;
      Node& c = nodes_[child];
      const int64_t sl = static_cast<int64_t>(c.seg.size());
      const int64_t k = common_len(c.seg.data(), sl, tokens.data() + i, std::min(sl, n - i));
      c.last_touch = tick;
      i += k;
      if (!visit(child, k, i)) return;
      if (k < sl) return;
      node = child;
    }
  }

  int new_node() {
    if (!free_nodes_.empty()) {
      const int x = free_nodes_.back();
      free_nodes_.pop_back();
      nodes_[x] = Node{};
      return x;
    }
    nodes_.emplace_back();
    return static_cast<int>(nodes_.size()) - 1;
  }

  int split(int x, int at) {
    const int up = new_node();
    {
      Node& nd = nodes_[x];
      Node& u = nodes_[up];
      u.seg.assign(nd.seg.begin(), nd.seg.begin() + at);
      u.runs = slice_runs(nd.runs, 0, at);
      u.donor = nd.donor;
      u.parent = nd.parent;
      u.last_touch = nd.last_touch;
    }
    Node& nd = nodes_[x];
    std::vector<int32_t> rest(nd.seg.begin() + at, nd.seg.end());
    nd.runs = slice_runs(nd.runs, at, static_cast<int64_t>(rest.size()));
    nd.seg = std::move(rest);
    nodes_[up].kids.clear();
    nodes_[up].kids.emplace_back(nd.seg[0], x);
    for (auto& k : nodes_[nd.parent].kids)  // same key, same position in the parent
      if (k.first == nodes_[up].seg[0]) k.second = up;
    nd.parent = up;
    return up;
  }

  int64_t evict_impl(int64_t needed, const std::vector<char>* prot) {
    int64_t released = 0;
    using Key = std::tuple<int64_t, int32_t, int64_t, int>;  // (touch, first token, rank, node)
    std::priority_queue<Key, std::vector<Key>, std::greater<Key>> heap;
    if (needed > 0) {
      // evictable leaves in the Python restatement's scan order
      std::vector<int> stack;
      for (const auto& k : nodes_[0].kids) stack.push_back(k.second);
      int64_t rank = 0;
      while (!stack.empty()) {
        const int x = stack.back();
        stack.pop_back();
        const Node& nd = nodes_[x];
        if (!nd.kids.empty()) {
          for (const auto& k : nd.kids) stack.push_back(k.second);
        } else if (!is_prot(prot, x)) {
          heap.emplace(nd.last_touch, nd.seg[0], rank++, x);
        }
      }
    }
    while (released < needed && !heap.empty()) {
      const auto [touch, tok, rank, v] = heap.top();
      heap.pop();
      (void)touch;
      (void)tok;
      Node& vn = nodes_[v];
      kv_.decref_runs(vn.runs);
      const int64_t len = static_cast<int64_t>(vn.seg.size());
      released += len;
      cells_ -= len;
      const int p = vn.parent;
      auto& pk = nodes_[p].kids;
      const int32_t key = vn.seg[0];
      pk.erase(std::find_if(pk.begin(), pk.end(), [&](const auto& k) { return k.first == key; }));
      vn = Node{};
      free_nodes_.push_back(v);
      if (p != 0 && nodes_[p].kids.empty() && !is_prot(prot, p))
        heap.emplace(nodes_[p].last_touch, nodes_[p].seg[0], rank, p);
    }
    evicted_cells_total += released;
    return released;
  }

  KvCore& kv_;
  int64_t budget_;
  std::vector<Node> nodes_;
  std::vector<int> free_nodes_;
  int64_t clock_ = 0;
  int64_t cells_ = 0;
};

}  // namespace

// FNV-1a 64 over UTF-8 bytes (reference _native.pyx fnv1a64_bytes)
uint64_t fnv1a64(const char* p, size_t n) {
  uint64_t h = 0xCBF29CE484222325ull;
  for (size_t i = 0; i < n; ++i) {
    h ^= static_cast<uint8_t>(p[i]);
    h *= 0x100000001B3ull;
  }
  return h;
}

// FNV-1a over the 4-byte little-endian serialisation of tokens[start:end]
// (reference _native.pyx:36-59: uint32 reinterpretation), straight from a
// Python list (no int32 array conversion) or any int32-convertible buffer
template <typename H, H kPrime>
H fnv_tokens(py::handle seq, py::ssize_t start, py::ssize_t end, H h) {
  auto step = [&](uint32_t u) {
    for (int b = 0; b < 4; ++b) {
      h ^= static_cast<uint8_t>(u >> (8 * b));
      h *= kPrime;
    }
  };
  if (PyList_Check(seq.ptr())) {
    const py::ssize_t n = PyList_GET_SIZE(seq.ptr());
    if (end > n) end = n;
    for (py::ssize_t i = start; i < end; ++i) {
      const long v = PyLong_AsLong(PyList_GET_ITEM(seq.ptr(), i));
      if (v == -1 && PyErr_Occurred()) throw py::error_already_set();
      step(static_cast<uint32_t>(static_cast<int32_t>(v)));
    }
    return h;
  }
  auto a = py::array_t<int32_t, py::array::c_style | py::array::forcecast>::ensure(seq);
  if (!a) throw py::type_error("tokens must be a list or an int32-convertible array");
  const int32_t* d = a.data();
  if (end > a.size()) end = a.size();
  for (py::ssize_t i = start; i < end; ++i) step(static_cast<uint32_t>(d[i]));
  return h;
}

PYBIND11_MODULE(_hostcore, m) {
  m.def("fnv1a64_tokens", [](py::handle seq, py::ssize_t start, py::ssize_t end, uint64_t state) {
    return fnv_tokens<uint64_t, 0x100000001B3ull>(seq, start, end, state);
  });
  m.def("fnv1a32_tokens", [](py::handle seq, py::ssize_t start, py::ssize_t end, uint32_t state) {
    return fnv_tokens<uint32_t, 0x01000193u>(seq, start, end, state);
  });
  m.def("fnv1a64_bytes", [](const py::bytes& b) {
    const std::string s = b;
    return fnv1a64(s.data(), s.size());
  });
  // tokenizer piece ids: fnv1a64(utf-8 piece) mod modulus (engine.py:228-230)
  m.def("piece_ids", [](const py::list& pieces, uint64_t modulus) {
    std::vector<int64_t> out;
    out.reserve(pieces.size());
    for (auto h : pieces) {
      Py_ssize_t n = 0;
      const char* p = PyUnicode_AsUTF8AndSize(h.ptr(), &n);
      if (!p) throw py::error_already_set();
      out.push_back(static_cast<int64_t>(fnv1a64(p, static_cast<size_t>(n)) % modulus));
    }
    return out;
  });
  m.doc() = "deltaserve B200 native host core: cell allocator / page tables and radix trie";
  m.def("set_exceptions", [](py::object cap, py::object donor, py::object budget) {
    g_capacity_exc = cap;
    g_donor_exc = donor;
    g_budget_exc = budget;
  });
  m.def("common_prefix_len", [](const std::vector<int32_t>& a, const std::vector<int32_t>& b) {
    return common_len(a.data(), static_cast<int64_t>(a.size()), b.data(),
                      static_cast<int64_t>(b.size()));
  });
  py::class_<KvCore>(m, "KvCore")
      .def(py::init<int64_t>())
      .def_readwrite("record_ops", &KvCore::record_ops)
      .def_property_readonly("capacity_cells", &KvCore::capacity)
      .def_property_readonly("free_cells", &KvCore::free_cells)
      .def_property_readonly("occupancy", &KvCore::occupancy)
      .def("seq_len", &KvCore::seq_len)
      .def("span_count", &KvCore::span_count)
      .def("sequences", &KvCore::sequences)
      .def("refcount", &KvCore::refcount)
      .def("refcounts", &KvCore::refcounts)
      .def("take_ops", &KvCore::take_ops)
      .def("incref_runs", [](KvCore& k, const py::iterable& r) { k.incref_runs(to_runs(r)); })
      .def("decref_runs", [](KvCore& k, const py::iterable& r) { return k.decref_runs(to_runs(r)); })
      .def("append_cells", &KvCore::append_cells)
      .def("resolve_runs",
           [](const KvCore& k, int64_t s, int64_t a, int64_t b) { return runs_list(k.resolve_runs(s, a, b)); })
      .def("seq_alias", &KvCore::seq_alias)
      .def("alias_runs", [](KvCore& k, int64_t d, const py::iterable& r) { k.alias_runs(d, to_runs(r)); })
      .def("trim", &KvCore::trim)
      .def("release_sequence", &KvCore::release_sequence)
      .def("cell_ids", &KvCore::cell_ids);
  py::class_<RadixCore>(m, "RadixCore")
      .def(py::init<KvCore&, int64_t>(), py::keep_alive<1, 2>())
      .def_property_readonly("cell_budget", &RadixCore::cell_budget)
      .def_property_readonly("total_cells", &RadixCore::total_cells)
      .def_readwrite("evicted_cells_total", &RadixCore::evicted_cells_total)
      .def("node_count", &RadixCore::node_count)
      .def("longest_prefix", &RadixCore::longest_prefix)
      .def("save", &RadixCore::save)
      .def("evict", &RadixCore::evict)
      .def("clear", &RadixCore::clear)
      .def("dump", &RadixCore::dump);
}
