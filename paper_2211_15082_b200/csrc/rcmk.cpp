// Host-side reverse Cuthill-McKee (reference: reorder.py:55-123 rcmk and
// reorder.py:55-69 _symmetrized_adjacency).  Pure C++ over host arrays; the
// Python per-node BFS costs ~65 us/node, this is
// O(E log d).  Tie rules reproduced exactly:
//   * undirected neighbour lists = union of in- and out-edges, self loops
//     dropped, duplicates merged, ascending id;
//   * components discovered by seed id order; each component starts at its
//     minimum (degree, id) node; components are processed in ascending order
//     of their start node;
//   * BFS appends each frontier node's unvisited neighbours sorted by
//     (degree, id);
//   * the whole sequence is reversed.
#include <stdint.h>

#include <algorithm>
#include <vector>

#include "../../include/glint_b200.h"

extern "C" int glint_rcmk_host(int64_t n, const int64_t* indptr, const int64_t* indices,
                               int64_t* perm_out) {
  if (n < 0 || (n > 0 && (!indptr || !perm_out))) return GLINT_EINVAL;
  if (n == 0) return GLINT_OK;
  const int64_t m = indptr[n];
  // 1. symmetrised adjacency (CSR), sorted + deduplicated per row
  std::vector<int64_t> cnt(n + 1, 0);
  for (int64_t v = 0; v < n; ++v) {
    for (int64_t e = indptr[v]; e < indptr[v + 1]; ++e) {
      const int64_t u = indices[e];
      if (u < 0 || u >= n) return GLINT_EINVAL;
      if (u == v) continue;
      ++cnt[u + 1];
      ++cnt[v + 1];
    }
  }
  for (int64_t v = 0; v < n; ++v) cnt[v + 1] += cnt[v];
  std::vector<int64_t> adj(cnt[n]);
  {
    std::vector<int64_t> fill(cnt.begin(), cnt.end() - 1);
    for (int64_t v = 0; v < n; ++v) {
      for (int64_t e = indptr[v]; e < indptr[v + 1]; ++e) {
        const int64_t u = indices[e];
        if (u == v) continue;
        adj[fill[u]++] = v;
        adj[fill[v]++] = u;
      }
    }
  }
  std::vector<int64_t> ptr(n + 1, 0);
  {
    int64_t w = 0;
    for (int64_t v = 0; v < n; ++v) {
      auto b = adj.begin() + cnt[v];
      auto e = adj.begin() + cnt[v + 1];
      std::sort(b, e);
      auto last = std::unique(b, e);
      ptr[v] = w;
      for (auto it = b; it != last; ++it) adj[w++] = *it;
    }
    ptr[n] = w;
    adj.resize(w);
  }
  (void)m;
  std::vector<int64_t> deg(n);
  for (int64_t v = 0; v < n; ++v) deg[v] = ptr[v + 1] - ptr[v];

  // 2. components in seed order; start = min (deg, id) member
  std::vector<int64_t> comp(n, -1);
  std::vector<int64_t> starts;
  std::vector<int64_t> stack;
  for (int64_t seed = 0; seed < n; ++seed) {
    if (comp[seed] >= 0) continue;
    const int64_t c = static_cast<int64_t>(starts.size());
    int64_t best = seed;
    comp[seed] = c;
    stack.push_back(seed);
    while (!stack.empty()) {
      const int64_t u = stack.back();
      stack.pop_back();
      if (deg[u] < deg[best] || (deg[u] == deg[best] && u < best)) best = u;
      for (int64_t e = ptr[u]; e < ptr[u + 1]; ++e) {
        const int64_t v = adj[e];
        if (comp[v] < 0) {
          comp[v] = c;
          stack.push_back(v);
        }
      }
    }
    starts.push_back(best);
  }
  std::sort(starts.begin(), starts.end());

  // 3. BFS per start, candidates ordered by (degree, id)
  std::vector<char> visited(n, 0);
  std::vector<int64_t> seq(n);
  std::vector<int64_t> cand;
  int64_t pos = 0;
  for (int64_t s : starts) {
    seq[pos] = s;
    visited[s] = 1;
    int64_t head = pos++;
    while (head < pos) {
      const int64_t u = seq[head++];
      cand.clear();
      for (int64_t e = ptr[u]; e < ptr[u + 1]; ++e)
        if (!visited[adj[e]]) cand.push_back(adj[e]);
      std::sort(cand.begin(), cand.end(), [&](int64_t a, int64_t b) {
        return deg[a] != deg[b] ? deg[a] < deg[b] : a < b;
      });
      for (int64_t v : cand) {
        visited[v] = 1;
        seq[pos++] = v;
      }
    }
  }
  if (pos != n) return GLINT_ECUDA;  // internal invariant
  for (int64_t i = 0; i < n; ++i) perm_out[i] = seq[n - 1 - i];
  return GLINT_OK;
}

// Same ordering from a pre-sorted symmetrised adjacency: row v of (ptr, adj)
// holds v's distinct neighbours (self loops dropped) already ordered by
// (degree, id), degree = ptr[v+1] - ptr[v].  The device builds it (two sorts,
// reorder.py _sorted_adjacency_device), so the host pass is two linear sweeps:
// components in seed order (start = min (degree, id) member, components in
// ascending start order), then the BFS, whose per-node candidate list is the
// row filtered by `visited` -- the (degree, id) order is preserved by the
// filter, so no per-node sort remains.
extern "C" int glint_rcmk_sorted_host(int64_t n, const int64_t* ptr, const int32_t* adj,
                                      int64_t* perm_out) {
  if (n < 0 || (n > 0 && (!ptr || !perm_out))) return GLINT_EINVAL;
  if (n == 0) return GLINT_OK;
  auto deg = [&](int64_t v) { return ptr[v + 1] - ptr[v]; };
  std::vector<int32_t> comp(n, -1);
  std::vector<int64_t> starts;
  std::vector<int64_t> stack;
  for (int64_t seed = 0; seed < n; ++seed) {
    if (comp[seed] >= 0) continue;
    const int32_t c = static_cast<int32_t>(starts.size());
    int64_t best = seed;
    comp[seed] = c;
    stack.push_back(seed);
    while (!stack.empty()) {
      const int64_t u = stack.back();
      stack.pop_back();
      if (deg(u) < deg(best) || (deg(u) == deg(best) && u < best)) best = u;
      for (int64_t e = ptr[u]; e < ptr[u + 1]; ++e) {
        const int64_t v = adj[e];
        if (v < 0 || v >= n) return GLINT_EINVAL;
        if (comp[v] < 0) {
          comp[v] = c;
          stack.push_back(v);
        }
      }
    }
    starts.push_back(best);
  }
  std::sort(starts.begin(), starts.end());
  std::vector<char> visited(n, 0);
  std::vector<int64_t> seq(n);
  int64_t pos = 0;
  for (int64_t s : starts) {
    seq[pos] = s;
    visited[s] = 1;
    int64_t head = pos++;
    while (head < pos) {
      const int64_t u = seq[head++];
      for (int64_t e = ptr[u]; e < ptr[u + 1]; ++e) {
        const int64_t v = adj[e];
        if (!visited[v]) {
          visited[v] = 1;
          seq[pos++] = v;
        }
      }
    }
  }
  if (pos != n) return GLINT_ECUDA;  // internal invariant
  for (int64_t i = 0; i < n; ++i) perm_out[i] = seq[n - 1 - i];
  return GLINT_OK;
}

// Host int64 -> int32 id narrowing on `threads` threads (the e2e upload path
// narrows CSR chunks on the CPU while the features cross PCIe, so the CSR
// crosses as int32 -- half the bytes).  Ids must already be validated
// (CscGraph checks [0, N) on construction); returns the count of ids that do
// not fit int32 as a guard.
#include <thread>

extern "C" int64_t glint_narrow_ids_host(const int64_t* src, int32_t* dst, int64_t n,
                                         int32_t threads) {
  if (n <= 0) return 0;
  if (!src || !dst) return -1;
  int t = threads < 1 ? 1 : (threads > 64 ? 64 : threads);
  if (n < (1 << 16)) t = 1;
  std::vector<int64_t> bad(t, 0);
  auto work = [&](int k) {
    const int64_t lo = n * k / t, hi = n * (k + 1) / t;
    int64_t b = 0;
    for (int64_t i = lo; i < hi; ++i) {
      const int64_t v = src[i];
      b += (v < INT32_MIN || v > INT32_MAX);
      dst[i] = static_cast<int32_t>(v);
    }
    bad[k] = b;
  };
  std::vector<std::thread> pool;
  for (int k = 1; k < t; ++k) pool.emplace_back(work, k);
  work(0);
  for (auto& th : pool) th.join();
  int64_t total = 0;
  for (int64_t b : bad) total += b;
  return total;
}
