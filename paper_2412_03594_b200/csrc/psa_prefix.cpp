// psa_prefix.cpp — native host preprocessing: compact prefix (radix) tree over
// all prompts, first-level reuse enlargement, and prefix-sharing group
// extraction. A restatement of the reference's prefix_tree.py:
//   build_tree        (prefix_tree.py:107-159)  insertion + canonical child order
//   maximize_reuse    (prefix_tree.py:187-245)  bottom-up fork of grandchildren
//   extract_groups    (prefix_tree.py:271-301)  first-level children -> groups
// producing exactly the reference's groups (same order, same members, same
// member order) — tests/test_prefix.py compares them on the reference's own
// workloads. Edge spans are (request, offset, length) views into the prompts,
// never copies: a span always sits at its path depth in the prompt it names.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/psa.h"

namespace {

struct Node {
  int32_t src = -1;  // request whose prompt holds the span
  int64_t beg = 0;   // span = prompt(src)[beg, beg + len): beg is the path depth
  int64_t len = 0;
  std::vector<int32_t> children;
  std::vector<int32_t> leaf;  // requests whose prompt ends here
};

struct Tree {
  const int64_t* cu;
  const int32_t* tok;
  std::vector<Node> nodes;

  const int32_t* span(const Node& n) const { return tok + cu[n.src] + n.beg; }

  // Python tuple order of the two spans (lexicographic, a proper prefix first).
  bool less(int32_t a, int32_t b) const {
    const Node& x = nodes[a];
    const Node& y = nodes[b];
    const int32_t* p = span(x);
    const int32_t* q = span(y);
    const int64_t m = std::min(x.len, y.len);
    for (int64_t i = 0; i < m; ++i)
      if (p[i] != q[i]) return p[i] < q[i];
    return x.len < y.len;
  }
  void sort_children(int32_t n) {
    auto& c = nodes[n].children;
    std::stable_sort(c.begin(), c.end(), [&](int32_t a, int32_t b) { return less(a, b); });
  }
};

// prefix_tree.py:107-151: strict radix tree, children looked up by first token.
void build(Tree& t, int32_t R) {
  t.nodes.emplace_back();  // root
  std::vector<std::unordered_map<int32_t, int32_t>> index(1);
  for (int32_t r = 0; r < R; ++r) {
    const int32_t* s = t.tok + t.cu[r];
    const int64_t n = t.cu[r + 1] - t.cu[r];
    int32_t node = 0;
    int64_t pos = 0;
    for (;;) {
      if (pos == n) {
        t.nodes[node].leaf.push_back(r);
        break;
      }
      auto it = index[node].find(s[pos]);
      if (it == index[node].end()) {
        Node leaf;
        leaf.src = r;
        leaf.beg = pos;
        leaf.len = n - pos;
        leaf.leaf.push_back(r);
        const int32_t id = int32_t(t.nodes.size());
        t.nodes.push_back(std::move(leaf));
        t.nodes[node].children.push_back(id);
        index[node][s[pos]] = id;
        index.emplace_back();
        break;
      }
      const int32_t child = it->second;
      const int32_t* sp = t.span(t.nodes[child]);
      const int64_t m = std::min(t.nodes[child].len, n - pos);
      int64_t k = 0;
      while (k < m && sp[k] == s[pos + k]) ++k;
      if (k < t.nodes[child].len) {  // split: child keeps span[:k], `rest` the remainder
        Node rest;
        rest.src = t.nodes[child].src;
        rest.beg = t.nodes[child].beg + k;
        rest.len = t.nodes[child].len - k;
        rest.children = std::move(t.nodes[child].children);
        rest.leaf = std::move(t.nodes[child].leaf);
        const int32_t rid = int32_t(t.nodes.size());
        const int32_t first = t.span(rest)[0];
        t.nodes.push_back(std::move(rest));
        index.emplace_back(std::move(index[child]));
        Node& c = t.nodes[child];
        c.len = k;
        c.children.assign(1, rid);
        c.leaf.clear();
        index[child].clear();
        index[child][first] = rid;
      }
      node = child;
      pos += k;
    }
  }
  for (int32_t n = 0; n < int32_t(t.nodes.size()); ++n) t.sort_children(n);
}

// prefix_tree.py:219-245 for one node whose children are solved.
void enlarge(Tree& t, int32_t node, std::vector<int64_t>& counts) {
  const std::vector<int32_t> kids = t.nodes[node].children;
  for (int32_t child : kids) {
    if (t.nodes[child].children.empty()) continue;
    const int64_t penalty = t.nodes[child].len;
    const std::vector<int32_t> gkids = t.nodes[child].children;
    for (int32_t g : gkids) {
      const int64_t gleaves = counts[g];
      const int64_t gain = (gleaves - 1) * t.nodes[g].len;
      if (gain > penalty) {
        Node forked;
        forked.src = t.nodes[g].src;
        forked.beg = t.nodes[g].beg - t.nodes[child].len;
        forked.len = t.nodes[child].len + t.nodes[g].len;
        forked.children = t.nodes[g].children;
        forked.leaf = t.nodes[g].leaf;
        const int32_t id = int32_t(t.nodes.size());
        t.nodes.push_back(std::move(forked));
        counts.push_back(gleaves);
        auto& cc = t.nodes[child].children;
        cc.erase(std::find(cc.begin(), cc.end(), g));
        counts[child] -= gleaves;
        t.nodes[node].children.push_back(id);
      }
    }
    Node& c = t.nodes[child];
    if (c.leaf.empty() && c.children.empty()) {
      auto& nc = t.nodes[node].children;
      nc.erase(std::find(nc.begin(), nc.end(), child));
    } else if (c.leaf.empty() && c.children.size() == 1) {
      const int32_t only = c.children[0];
      const Node o = t.nodes[only];
      Node& c2 = t.nodes[child];
      c2.src = o.src;
      c2.beg = o.beg - c2.len;
      c2.len = c2.len + o.len;
      c2.children = o.children;
      c2.leaf = o.leaf;
    }
  }
  t.sort_children(node);
  int64_t total = int64_t(t.nodes[node].leaf.size());
  for (int32_t c : t.nodes[node].children) total += counts[c];
  counts[node] = total;
}

std::vector<int64_t> subtree_counts(const Tree& t) {
  std::vector<int64_t> counts(t.nodes.size(), 0);
  // children always have larger ids than... not after forks: use an explicit post-order
  std::vector<std::pair<int32_t, bool>> st{{0, false}};
  while (!st.empty()) {
    auto [n, ready] = st.back();
    st.pop_back();
    if (!ready) {
      st.push_back({n, true});
      for (int32_t c : t.nodes[n].children) st.push_back({c, false});
      continue;
    }
    int64_t total = int64_t(t.nodes[n].leaf.size());
    for (int32_t c : t.nodes[n].children) total += counts[c];
    counts[n] = total;
  }
  return counts;
}

thread_local std::string g_prefix_error;

}  // namespace

extern "C" {

psa_status psa_prefix_groups(int32_t num_requests, const int64_t* cu_tokens, const int32_t* tokens,
                             const int32_t* id_rank, int32_t maximize, int32_t* num_groups,
                             int64_t* group_prefix_len, int32_t* cu_members, int32_t* members,
                             int64_t* saved_tokens) {
  if (num_requests < 0 || !cu_tokens || (!tokens && num_requests > 0 && cu_tokens[num_requests]) ||
      !id_rank || !num_groups || !group_prefix_len || !cu_members || !members)
    return PSA_INVALID_ARGUMENT;
  for (int32_t r = 0; r < num_requests; ++r)
    if (cu_tokens[r + 1] <= cu_tokens[r]) return PSA_INVALID_ARGUMENT;  // empty prompt
  Tree t{cu_tokens, tokens, {}};
  t.nodes.reserve(size_t(num_requests) * 3 + 1);
  build(t, num_requests);
  std::vector<int64_t> counts;
  if (maximize) {
    counts.assign(t.nodes.size(), 0);
    std::vector<std::pair<int32_t, bool>> st{{0, false}};
    while (!st.empty()) {  // post-order over the tree as it is before any fork
      auto [n, ready] = st.back();
      st.pop_back();
      if (!ready) {
        st.push_back({n, true});
        for (int32_t c : t.nodes[n].children) st.push_back({c, false});
        continue;
      }
      enlarge(t, n, counts);
    }
  } else {
    counts = subtree_counts(t);
  }
  // prefix_tree.py:271-301: first-level children in order; members by a
  // pre-order walk, identical prompts ordered by request id (id_rank).
  int32_t G = 0, nm = 0;
  int64_t saved = 0;
  cu_members[0] = 0;
  std::vector<int32_t> st;
  for (int32_t child : t.nodes[0].children) {
    const int64_t leaves = counts[child];
    group_prefix_len[G] = leaves >= 2 ? t.nodes[child].len : 0;
    if (leaves >= 2) saved += (leaves - 1) * t.nodes[child].len;
    st.assign(1, child);
    while (!st.empty()) {
      const int32_t n = st.back();
      st.pop_back();
      std::vector<int32_t> ids = t.nodes[n].leaf;
      std::sort(ids.begin(), ids.end(), [&](int32_t a, int32_t b) { return id_rank[a] < id_rank[b]; });
      for (int32_t r : ids) members[nm++] = r;
      const auto& ch = t.nodes[n].children;
      for (auto it = ch.rbegin(); it != ch.rend(); ++it) st.push_back(*it);
    }
    cu_members[++G] = nm;
  }
  *num_groups = G;
  if (saved_tokens) *saved_tokens = saved;
  return nm == num_requests ? PSA_OK : PSA_INVALID_ARGUMENT;
}

}  // extern "C"
