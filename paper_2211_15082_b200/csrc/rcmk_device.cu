// Device building blocks of reverse Cuthill-McKee (reference: reorder.py:72-123
// rcmk), used by reorder.rcmk for a DeviceGraph.  The host orchestrates a
// level-synchronous, multi-source BFS that reproduces the sequential order
// exactly:
//   * components: union-find over the symmetrised adjacency (hooking the
//     larger root under the smaller, so a root is its component's minimum id);
//   * each component's start = its minimum (degree, id) member
//     (glint_rcmk_starts: one 64-bit atomicMin per member);
//   * components are visited in ascending order of their start;
//   * BFS level L+1 of a component = its unvisited neighbours of level L; a
//     node's parent is its FIRST level-L neighbour in sequence order
//     (glint_rcmk_expand: atomicMin of the parent's index in the level list),
//     and the level is ordered by (parent index, (degree, id) rank) -- the
//     order in which the sequential BFS appends them.
#include "common.cuh"

namespace glint {
namespace {

__device__ __forceinline__ int32_t cc_find(int32_t* parent, int32_t v) {
  int32_t p = parent[v];
  while (p != v) {   // path halving
    const int32_t gp = parent[p];
    if (gp != p) parent[v] = gp;
    v = p;
    p = gp;
  }
  return v;
}

__global__ void cc_init_kernel(int64_t n, int32_t* parent) {
  for (int64_t v = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; v < n;
       v += static_cast<int64_t>(gridDim.x) * blockDim.x)
    parent[v] = static_cast<int32_t>(v);
}

// one thread per row v: every neighbour u < v (each undirected edge once)
__global__ void cc_hook_kernel(int64_t n, const int64_t* __restrict__ ptr,
                               const int32_t* __restrict__ adj, int32_t* parent) {
  for (int64_t v = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; v < n;
       v += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    for (int64_t e = ptr[v]; e < ptr[v + 1]; ++e) {
      const int32_t u = adj[e];
      if (u >= v) continue;
      int32_t a = cc_find(parent, static_cast<int32_t>(v));
      int32_t b = cc_find(parent, u);
      while (a != b) {
        if (a < b) { const int32_t t = a; a = b; b = t; }   // hook the larger root a under b
        const int32_t old = atomicCAS(parent + a, a, b);
        if (old == a) break;
        a = cc_find(parent, old);
        b = cc_find(parent, b);
      }
    }
  }
}

// Final labels: every thread writes only its own slot, and only a root, so no
// path-splitting write can land after it (which cc_find's would: another
// thread's splitting step may store a stale grandparent into parent[v] after
// v's thread wrote the root).
__global__ void cc_compress_kernel(int64_t n, int32_t* parent) {
  for (int64_t v = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; v < n;
       v += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int32_t r = parent[v];
    while (true) {
      const int32_t up = parent[r];
      if (up == r) break;
      r = up;
    }
    parent[v] = r;
  }
}

// start_key[root] = min over members of (degree << 32 | id)
__global__ void starts_kernel(int64_t n, const int64_t* __restrict__ ptr,
                              const int32_t* __restrict__ comp, unsigned long long* start_key) {
  for (int64_t v = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; v < n;
       v += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const unsigned long long key = (static_cast<unsigned long long>(ptr[v + 1] - ptr[v]) << 32) |
                                   static_cast<unsigned long long>(v);
    atomicMin(start_key + comp[v], key);
  }
}

// frontier[i] (level list in sequence order): each unvisited neighbour u gets
// best[u] = min(best[u], i) -- the index of its first parent
__global__ void expand_kernel(int64_t n_front, const int32_t* __restrict__ frontier,
                              const int64_t* __restrict__ ptr, const int32_t* __restrict__ adj,
                              const int32_t* __restrict__ level, long long* best) {
  // one warp per frontier node, lanes over its neighbours
  const int64_t warp = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t i = warp; i < n_front; i += nwarps) {
    const int32_t v = frontier[i];
    for (int64_t e = ptr[v] + lane; e < ptr[v + 1]; e += 32) {
      const int32_t u = adj[e];
      if (level[u] < 0) atomicMin(best + u, static_cast<long long>(i));
    }
  }
}

int grid_for(int64_t n, int per = 256) {
  return static_cast<int>(std::min<int64_t>(std::max<int64_t>(ceil_div(n, per), 1),
                                            static_cast<int64_t>(sm_count()) * 16));
}

}  // namespace
}  // namespace glint

using namespace glint;

extern "C" int glint_rcmk_components(int64_t n, const int64_t* ptr, const int32_t* adj,
                                     int32_t* comp_out, glint_stream_t stream) {
  GLINT_REQUIRE(n >= 0 && n < (1LL << 31), "rcmk_components: n out of range");
  if (n == 0) return GLINT_OK;
  GLINT_REQUIRE(ptr && comp_out, "rcmk_components: null argument");   // adj may be empty
  cudaStream_t s = as_stream(stream);
  const int g = grid_for(n);
  cc_init_kernel<<<g, 256, 0, s>>>(n, comp_out);
  cc_hook_kernel<<<g, 256, 0, s>>>(n, ptr, adj, comp_out);
  cc_compress_kernel<<<g, 256, 0, s>>>(n, comp_out);
  return launch_status("rcmk_components");
}

extern "C" int glint_rcmk_starts(int64_t n, const int64_t* ptr, const int32_t* comp,
                                 uint64_t* start_key, glint_stream_t stream) {
  GLINT_REQUIRE(n >= 0 && n < (1LL << 31), "rcmk_starts: n out of range");
  if (n == 0) return GLINT_OK;
  GLINT_REQUIRE(ptr && comp && start_key, "rcmk_starts: null argument");
  cudaStream_t s = as_stream(stream);
  GLINT_CUDA(cudaMemsetAsync(start_key, 0xff, static_cast<size_t>(n) * sizeof(uint64_t), s));
  starts_kernel<<<grid_for(n), 256, 0, s>>>(n, ptr, comp,
                                            reinterpret_cast<unsigned long long*>(start_key));
  return launch_status("rcmk_starts");
}

extern "C" int glint_rcmk_expand(int64_t n_front, const int32_t* frontier, const int64_t* ptr,
                                 const int32_t* adj, const int32_t* level, int64_t* best,
                                 glint_stream_t stream) {
  GLINT_REQUIRE(n_front >= 0, "rcmk_expand: n_front must be >= 0");
  if (n_front == 0) return GLINT_OK;
  GLINT_REQUIRE(frontier && ptr && level && best, "rcmk_expand: null argument");   // adj may be empty
  expand_kernel<<<grid_for(n_front * 32), 256, 0, as_stream(stream)>>>(
      n_front, frontier, ptr, adj, level, reinterpret_cast<long long*>(best));
  return launch_status("rcmk_expand");
}
