// lbvh.cu -- on-device LBVH build (helios_build_accel).
//
// Replaces the paper's CPU kd-tree (Sec. 5.1: recursive search,
// x/y/z split cycling by depth) with a linear BVH built entirely on the GPU:
//   K1 centroid bounds (block reduce + ordered-int atomics)
//   K1 Morton codes of the centroids: 3 x kMortonBits bits over an isotropic
//      grid (kMortonBits = 21 -> 63-bit codes; DESIGN.md s.8 says why not 30)
//   K2 stable LSD radix sort of (code, index), 8 bits per pass (sort_scan.cu)
//   K3 Karras hierarchy: N-1 internal nodes, delta = clz(code_i ^ code_j),
//      index tie-break (64 + clz(i ^ j)) for duplicate codes
//   K4 bottom-up AABB refit (second-arriving child computes the parent)
//   K5 layout: 64-B child-pair nodes, subtrees of <= kLeafMax triangles
//      collapsed into leaves, triangles permuted to leaf order (48 B).
// fp32 min/max of fp32 vertices is exact, so every box contains its
// triangles exactly; traversal adds the conservative slack (trace.cu).
#include <vector>

#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "internal.cuh"

namespace helios {
namespace {

__device__ __forceinline__ unsigned f2ord(float f) {
  unsigned u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float ord2f(unsigned u) {
  return __uint_as_float((u & 0x80000000u) ? (u & 0x7FFFFFFFu) : ~u);
}

__global__ void k_centroid_bounds(const float* __restrict__ xyz, uint32_t n,
                                  unsigned* __restrict__ bounds /* [6] ordered */) {
  float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const float* t = xyz + 9ull * i;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      float c = (t[a] + t[3 + a] + t[6 + a]) * (1.0f / 3.0f);
      lo[a] = fminf(lo[a], c);
      hi[a] = fmaxf(hi[a], c);
    }
  }
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    for (int o = 16; o > 0; o >>= 1) {
      lo[a] = fminf(lo[a], __shfl_xor_sync(0xffffffffu, lo[a], o));
      hi[a] = fmaxf(hi[a], __shfl_xor_sync(0xffffffffu, hi[a], o));
    }
  }
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      atomicMin(bounds + a, f2ord(lo[a]));
      atomicMax(bounds + 3 + a, f2ord(hi[a]));
    }
  }
}

// spread the low 21 bits of v to every third bit of a 63-bit word
__device__ __forceinline__ uint64_t expand21(uint64_t v) {
  v &= 0x1FFFFFull;
  v = (v | (v << 32)) & 0x1F00000000FFFFull;
  v = (v | (v << 16)) & 0x1F0000FF0000FFull;
  v = (v | (v << 8)) & 0x100F00F00F00F00Full;
  v = (v | (v << 4)) & 0x10C30C30C30C30C3ull;
  v = (v | (v << 2)) & 0x1249249249249249ull;
  return v;
}

// Morton code of the centroid over an ISOTROPIC grid: every axis uses the
// largest extent of the centroid AABB, so on flat scenes (2 km x 2 km x
// 0.2 km) the top levels split x/y first instead of slicing the whole scene
// into thin z slabs that every nadir ray crosses.  kMortonBits per axis.
__global__ void k_morton(const float* __restrict__ xyz, uint32_t n,
                         const unsigned* __restrict__ bounds, uint64_t* __restrict__ codes,
                         uint32_t* __restrict__ idx, int bits, int isotropic) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float* t = xyz + 9ull * i;
  float lo[3], ex[3], ext = 0.0f;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    lo[a] = ord2f(bounds[a]);
    ex[a] = ord2f(bounds[3 + a]) - lo[a];
    ext = fmaxf(ext, ex[a]);
  }
  const double cells = (double)(1u << bits);
  uint64_t q[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double c = ((double)t[a] + (double)t[3 + a] + (double)t[6 + a]) / 3.0;
    const float e = isotropic ? ext : ex[a];
    const double f = e > 0.0f ? (c - (double)lo[a]) / (double)e : 0.0;
    long long k = (long long)(f * cells);
    q[a] = (uint64_t)min(max(k, 0ll), (long long)(cells - 1));
  }
  codes[i] = (expand21(q[0]) << 2) | (expand21(q[1]) << 1) | expand21(q[2]);
  idx[i] = i;
}

__device__ __forceinline__ int delta(const uint64_t* __restrict__ codes, int n, int i, int j) {
  if (j < 0 || j >= n) return -1;
  const uint64_t a = codes[i], b = codes[j];
  if (a == b) return 64 + __clz((unsigned)(i ^ j));
  return __clzll((long long)(a ^ b));
}

// Karras 2012 hierarchy: internal node i covers [first, last]; split gamma.
// child encoding: >= 0 internal node, < 0 sorted leaf ~k.
__global__ void k_karras(const uint64_t* __restrict__ codes, int n, int* __restrict__ child,
                         int* __restrict__ parent_int, int* __restrict__ parent_leaf,
                         int* __restrict__ range) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n - 1) return;
  int d = (delta(codes, n, i, i + 1) - delta(codes, n, i, i - 1)) >= 0 ? 1 : -1;
  int dmin = delta(codes, n, i, i - d);
  int lmax = 2;
  while (delta(codes, n, i, i + lmax * d) > dmin) lmax <<= 1;
  int l = 0;
  for (int t = lmax >> 1; t >= 1; t >>= 1)
    if (delta(codes, n, i, i + (l + t) * d) > dmin) l += t;
  int j = i + l * d;
  int dnode = delta(codes, n, i, j);
  int s = 0;
  int t = l;
  do {
    t = (t + 1) >> 1;
    if (delta(codes, n, i, i + (s + t) * d) > dnode) s += t;
  } while (t > 1);
  int gamma = i + s * d + min(d, 0);
  int first = min(i, j), last = max(i, j);
  int left = (first == gamma) ? ~gamma : gamma;
  int right = (last == gamma + 1) ? ~(gamma + 1) : gamma + 1;
  child[2 * i] = left;
  child[2 * i + 1] = right;
  range[2 * i] = first;
  range[2 * i + 1] = last;
  if (left < 0) parent_leaf[~left] = i; else parent_int[left] = i;
  if (right < 0) parent_leaf[~right] = i; else parent_int[right] = i;
  if (i == 0) parent_int[0] = -1;
}

struct Box {
  float lo[3], hi[3];
};

__device__ __forceinline__ Box tri_box(const float* __restrict__ xyz, uint32_t src) {
  const float* t = xyz + 9ull * src;
  Box b;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    b.lo[a] = fminf(fminf(t[a], t[3 + a]), t[6 + a]);
    b.hi[a] = fmaxf(fmaxf(t[a], t[3 + a]), t[6 + a]);
  }
  return b;
}

__device__ __forceinline__ Box load_box_cg(const float* p) {
  Box b;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    b.lo[a] = __ldcg(p + a);
    b.hi[a] = __ldcg(p + 3 + a);
  }
  return b;
}
__device__ __forceinline__ void store_box(float* p, const Box& b) {
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    __stcg(p + a, b.lo[a]);
    __stcg(p + 3 + a, b.hi[a]);
  }
}

__global__ void k_refit(const float* __restrict__ xyz, const uint32_t* __restrict__ sorted_idx,
                        int n, const int* __restrict__ child, const int* __restrict__ parent_int,
                        const int* __restrict__ parent_leaf, float* __restrict__ leafbox,
                        float* __restrict__ nodebox, unsigned* __restrict__ flags) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  Box b = tri_box(xyz, sorted_idx[k]);
  store_box(leafbox + 6ull * k, b);
  __threadfence();
  int p = parent_leaf[k];
  while (p >= 0) {
    if (atomicAdd(flags + p, 1u) == 0u) return;  // first arrival: sibling finishes
    __threadfence();
    Box u;
    int c0 = child[2 * p], c1 = child[2 * p + 1];
    Box b0 = load_box_cg(c0 < 0 ? leafbox + 6ull * (~c0) : nodebox + 6ull * c0);
    Box b1 = load_box_cg(c1 < 0 ? leafbox + 6ull * (~c1) : nodebox + 6ull * c1);
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      u.lo[a] = fminf(b0.lo[a], b1.lo[a]);
      u.hi[a] = fmaxf(b0.hi[a], b1.hi[a]);
    }
    store_box(nodebox + 6ull * p, u);
    __threadfence();
    p = parent_int[p];
  }
}

__device__ __forceinline__ int32_t make_ref(int c, const int* __restrict__ range) {
  if (c < 0) return leaf_ref((uint32_t)(~c), 1u);
  int first = range[2 * c], last = range[2 * c + 1];
  int size = last - first + 1;
  if (size <= kLeafMax) return leaf_ref((uint32_t)first, (uint32_t)size);
  return c;
}

__global__ void k_layout(int n, const int* __restrict__ child, const int* __restrict__ range,
                         const float* __restrict__ leafbox, const float* __restrict__ nodebox,
                         Node* __restrict__ nodes) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n - 1) return;
  int c0 = child[2 * i], c1 = child[2 * i + 1];
  const float* q0 = c0 < 0 ? leafbox + 6ull * (~c0) : nodebox + 6ull * c0;
  const float* q1 = c1 < 0 ? leafbox + 6ull * (~c1) : nodebox + 6ull * c1;
  // boxes padded outward (directed rounding): a ray lying exactly on a face of
  // a flat or axis-aligned box (zero direction component) is never culled
  float b0[6], b1[6];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    b0[a] = __fsub_rd(q0[a], fmaf(fabsf(q0[a]), 1e-6f, 1e-30f));
    b0[3 + a] = __fadd_ru(q0[3 + a], fmaf(fabsf(q0[3 + a]), 1e-6f, 1e-30f));
    b1[a] = __fsub_rd(q1[a], fmaf(fabsf(q1[a]), 1e-6f, 1e-30f));
    b1[3 + a] = __fadd_ru(q1[3 + a], fmaf(fabsf(q1[3 + a]), 1e-6f, 1e-30f));
  }
  Node nd;
  nd.xy0 = make_float4(b0[0], b0[3], b0[1], b0[4]);
  nd.xy1 = make_float4(b1[0], b1[3], b1[1], b1[4]);
  nd.z01 = make_float4(b0[2], b0[5], b1[2], b1[5]);
  nd.ref = make_float4(__int_as_float(make_ref(c0, range)), __int_as_float(make_ref(c1, range)),
                       0.0f, 0.0f);
  nodes[i] = nd;
}

// depth (internal nodes on the path from the root) of every non-collapsed node
__global__ void k_depth(int n, const int* __restrict__ range, const int* __restrict__ parent_int,
                        unsigned* __restrict__ max_depth) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n - 1) return;
  if (range[2 * i + 1] - range[2 * i] + 1 <= kLeafMax) return;  // collapsed into a leaf
  unsigned d = 1;
  for (int p = parent_int[i]; p >= 0; p = parent_int[p]) ++d;
  atomicMax(max_depth, d);
}

__global__ void k_permute(const float* __restrict__ xyz, const float* __restrict__ refl,
                          const uint32_t* __restrict__ sorted_idx, uint32_t n,
                          TriRecord* __restrict__ out, TriRecord* __restrict__ filt) {
  uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  uint32_t src = sorted_idx[k];
  const float* t = xyz + 9ull * src;
  float r = refl ? refl[src] : 0.5f;
  TriRecord rec;
  rec.a = make_float4(t[0], t[1], t[2], __uint_as_float(src));
  rec.b = make_float4(t[3], t[4], t[5], r);
  rec.c = make_float4(t[6], t[7], t[8], 0.0f);
  out[k] = rec;
  // K6's filter record: the fp32 edges (correctly rounded differences, the
  // same values the filter computed per test) and their 1-norms, summed in
  // the filter's order
  const float e1x = t[3] - t[0], e1y = t[4] - t[1], e1z = t[5] - t[2];
  const float e2x = t[6] - t[0], e2y = t[7] - t[1], e2z = t[8] - t[2];
  const float A = __fadd_rn(__fadd_rn(fabsf(e1x), fabsf(e1y)), fabsf(e1z));
  const float B = __fadd_rn(__fadd_rn(fabsf(e2x), fabsf(e2y)), fabsf(e2z));
  TriRecord f;
  f.a = make_float4(t[0], t[1], t[2], __fmul_rn(A, B));
  f.b = make_float4(e1x, e1y, e1z, A);
  f.c = make_float4(e2x, e2y, e2z, B);
  filt[k] = f;
}

// ---- PLOC (parallel locally-ordered clustering, Meister & Bittner 2018) ----
// The default hierarchy (the Karras LBVH stays available as builder 1): clusters start as the sorted
// triangles; each iteration every cluster finds, among the 2R clusters around
// it in Morton order, the one whose merged box has the smallest surface area
// (ties -> lower index); mutual nearest neighbours merge (the lower index
// keeps the slot), the array is compacted (one 64-bit scan carries both the
// compaction and the node-allocation counts: deterministic ids), until one
// cluster is left.  Leaves are then ordered depth-first (offsets top-down,
// iteration by iteration) so collapsed subtrees are contiguous triangle runs.
constexpr int kPlocBlock = 256;

__device__ __forceinline__ float merged_area(const float* a, const float* b) {
  const float dx = fmaxf(a[3], b[3]) - fminf(a[0], b[0]);
  const float dy = fmaxf(a[4], b[4]) - fminf(a[1], b[1]);
  const float dz = fmaxf(a[5], b[5]) - fminf(a[2], b[2]);
  return dx * dy + dy * dz + dz * dx;
}

__global__ void k_ploc_init(const float* __restrict__ xyz, const uint32_t* __restrict__ sorted_idx,
                            uint32_t n, int* __restrict__ cid, float* __restrict__ cbox,
                            uint32_t* __restrict__ size, float* __restrict__ leafbox) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const Box b = tri_box(xyz, sorted_idx[k]);
  cid[k] = (int)k;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    cbox[6ull * k + a] = b.lo[a];
    cbox[6ull * k + 3 + a] = b.hi[a];
  }
  store_box(leafbox + 6ull * k, b);  // cluster k's triangle box (the collapse costs)
  size[k] = 1;
}

__global__ void k_ploc_nn(const float* __restrict__ cbox, uint32_t m, int r, int* __restrict__ nn) {
  extern __shared__ float sb[];
  const int b0 = blockIdx.x * kPlocBlock;
  const int lo = max(0, b0 - r), hi = min((int)m, b0 + kPlocBlock + r);
  for (int t = threadIdx.x; t < (hi - lo) * 6; t += blockDim.x) sb[t] = cbox[6ll * lo + t];
  __syncthreads();
  const int i = b0 + threadIdx.x;
  if (i >= (int)m) return;
  const float* bi = sb + 6 * (i - lo);
  float best = INFINITY;
  int bj = -1;
  const int j0 = max(0, i - r), j1 = min((int)m - 1, i + r);
  for (int j = j0; j <= j1; ++j) {
    if (j == i) continue;
    const float a = merged_area(bi, sb + 6 * (j - lo));
    if (a < best) {
      best = a;
      bj = j;
    }
  }
  nn[i] = bj;
}

// low 32 bits: cluster survives; high 32 bits: cluster creates a node
__global__ void k_ploc_flags(const int* __restrict__ nn, uint32_t m,
                             unsigned long long* __restrict__ flags) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const int j = nn[i];
  const bool mutual = j >= 0 && nn[j] == (int)i;
  const unsigned long long keep = (mutual && (int)i > j) ? 0ull : 1ull;
  const unsigned long long create = (mutual && (int)i < j) ? 1ull : 0ull;
  flags[i] = keep | (create << 32);
}

__global__ void k_ploc_merge(const int* __restrict__ nn, uint32_t m,
                             const unsigned long long* __restrict__ flags,
                             const unsigned long long* __restrict__ incl, uint32_t n,
                             uint32_t node_base, const int* __restrict__ cid,
                             const float* __restrict__ cbox, int* __restrict__ cid2,
                             float* __restrict__ cbox2, int* __restrict__ child,
                             float* __restrict__ nodebox, uint32_t* __restrict__ size,
                             int* __restrict__ parent) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const unsigned long long f = flags[i];
  if (!(f & 0xFFFFFFFFull)) return;
  const unsigned long long ex = incl[i] - f;  // exclusive prefix
  const uint32_t dst = (uint32_t)(ex & 0xFFFFFFFFull);
  const float* bi = cbox + 6ull * i;
  if (f >> 32) {
    const int j = nn[i];
    const uint32_t u = node_base + (uint32_t)(ex >> 32);  // internal node index
    const int v = (int)(n + u);
    const int a = cid[i], b = cid[j];
    const float* bj = cbox + 6ull * j;
    float ub[6];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      ub[q] = fminf(bi[q], bj[q]);
      ub[3 + q] = fmaxf(bi[3 + q], bj[3 + q]);
    }
    child[2 * u] = a;
    child[2 * u + 1] = b;
    size[v] = size[a] + size[b];
    parent[a] = v;
    parent[b] = v;
#pragma unroll
    for (int q = 0; q < 6; ++q) {
      nodebox[6ull * u + q] = ub[q];
      cbox2[6ull * dst + q] = ub[q];
    }
    cid2[dst] = v;
  } else {
#pragma unroll
    for (int q = 0; q < 6; ++q) cbox2[6ull * dst + q] = bi[q];
    cid2[dst] = cid[i];
  }
}

// top-down leaf offsets for the nodes created in one PLOC iteration (their
// parents were created later, so are already placed); depth of kept nodes
// node flags of the leaf collapse: the node is a leaf itself / lies inside one
constexpr uint8_t kCollapsed = 1, kInside = 2;

__global__ void k_ploc_offsets(uint32_t u0, uint32_t cnt, uint32_t n,
                               const int* __restrict__ child, const uint32_t* __restrict__ size,
                               uint32_t* __restrict__ off, uint32_t* __restrict__ depth,
                               uint8_t* __restrict__ nflag, unsigned* __restrict__ max_depth) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= cnt) return;
  const uint32_t u = u0 + t, v = n + u;
  const int a = child[2 * u], b = child[2 * u + 1];
  const uint32_t o = off[v], d = depth[v];
  off[a] = o;
  off[b] = o + size[a];
  const uint8_t f = nflag[u];
  const bool emitted = !(f & (kCollapsed | kInside));
  // depth = emitted internal nodes on the path (the traversal stack bound)
  depth[a] = d + (emitted ? 1u : 0u);
  depth[b] = d + (emitted ? 1u : 0u);
  if (f & (kCollapsed | kInside)) {
    if ((uint32_t)a >= n) nflag[a - n] |= kInside;
    if ((uint32_t)b >= n) nflag[b - n] |= kInside;
  }
  if (emitted) atomicMax(max_depth, d);
}

// Leaf collapse by the surface-area heuristic, bottom-up (one launch per PLOC
// iteration, in creation order, so the children's costs exist): with a
// triangle test costing 1 and a node step r = HELIOS_SAH_NODE_COST,
//   split(v) = r + (A0 cost(c0) + A1 cost(c1)) / A,   leaf(v) = size(v),
// a cluster of <= kLeafMax triangles becomes one leaf iff leaf <= split, and
// cost(v) = min of the two (a triangle costs 1).  For a pair this reads
// A0 + A1 >= (2 - r) A: terrain and facade pairs (sharing an edge) share a
// leaf, scattered crown leaves keep a node step each (profiles/r02_leaf_ab.txt).
#ifndef HELIOS_SAH_NODE_COST
#define HELIOS_SAH_NODE_COST 0.5f
#endif
__device__ __forceinline__ float half_area(const float* __restrict__ b) {
  const float dx = b[3] - b[0], dy = b[4] - b[1], dz = b[5] - b[2];
  return dx * dy + dy * dz + dz * dx;
}
__global__ void k_ploc_cost(uint32_t u0, uint32_t cnt, uint32_t n, const int* __restrict__ child,
                            const uint32_t* __restrict__ size, const float* __restrict__ leafbox,
                            const float* __restrict__ nodebox, float* __restrict__ cost,
                            uint8_t* __restrict__ nflag) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= cnt) return;
  const uint32_t u = u0 + t;
  const int c[2] = {child[2 * u], child[2 * u + 1]};
  float acc = 0.0f;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const bool tri = (uint32_t)c[i] < n;
    const float a = half_area(tri ? leafbox + 6ull * c[i] : nodebox + 6ull * (c[i] - n));
    acc += a * (tri ? 1.0f : cost[c[i] - n]);
  }
  const float A = half_area(nodebox + 6ull * u);
  const float split = A > 0.0f ? HELIOS_SAH_NODE_COST + acc / A : INFINITY;
  const uint32_t sz = size[n + u];
  const bool leaf = sz <= (uint32_t)kLeafMax && (float)sz <= split;
  cost[u] = leaf ? (float)sz : split;
  nflag[u] = leaf ? kCollapsed : 0;
}

__global__ void k_ploc_order(const uint32_t* __restrict__ sorted_idx, uint32_t n,
                             const uint32_t* __restrict__ off, uint32_t* __restrict__ order) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  order[off[k]] = sorted_idx[k];
}

__device__ __forceinline__ int32_t ploc_ref(int c, uint32_t n, const uint32_t* __restrict__ size,
                                            const uint32_t* __restrict__ off,
                                            const uint8_t* __restrict__ nflag) {
  if ((uint32_t)c < n) return leaf_ref(off[c], 1u);
  if (nflag[c - n] & kCollapsed) return leaf_ref(off[c], size[c]);
  return (int32_t)((uint32_t)c - n);
}

__global__ void k_ploc_layout(uint32_t n, const int* __restrict__ child,
                              const uint32_t* __restrict__ size, const uint32_t* __restrict__ off,
                              const float* __restrict__ leafbox, const float* __restrict__ nodebox,
                              const uint8_t* __restrict__ nflag, Node* __restrict__ nodes) {
  const uint32_t u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= n - 1) return;
  if (nflag[u] & (kCollapsed | kInside)) return;  // a leaf, or inside one
  const int c0 = child[2 * u], c1 = child[2 * u + 1];
  const float* q0 = c0 < (int)n ? leafbox + 6ull * c0 : nodebox + 6ull * (c0 - n);
  const float* q1 = c1 < (int)n ? leafbox + 6ull * c1 : nodebox + 6ull * (c1 - n);
  float b0[6], b1[6];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    b0[a] = __fsub_rd(q0[a], fmaf(fabsf(q0[a]), 1e-6f, 1e-30f));
    b0[3 + a] = __fadd_ru(q0[3 + a], fmaf(fabsf(q0[3 + a]), 1e-6f, 1e-30f));
    b1[a] = __fsub_rd(q1[a], fmaf(fabsf(q1[a]), 1e-6f, 1e-30f));
    b1[3 + a] = __fadd_ru(q1[3 + a], fmaf(fabsf(q1[3 + a]), 1e-6f, 1e-30f));
  }
  Node nd;
  nd.xy0 = make_float4(b0[0], b0[3], b0[1], b0[4]);
  nd.xy1 = make_float4(b1[0], b1[3], b1[1], b1[4]);
  nd.z01 = make_float4(b0[2], b0[5], b1[2], b1[5]);
  nd.ref = make_float4(__int_as_float(ploc_ref(c0, n, size, off, nflag)),
                       __int_as_float(ploc_ref(c1, n, size, off, nflag)), 0.0f, 0.0f);
  nodes[u] = nd;
}

template <class T>
cudaError_t dalloc(T** p, size_t count, cudaStream_t s) {
  return dev_alloc((void**)p, sizeof(T) * (count ? count : 1), s);
}

}  // namespace

cudaError_t build_lbvh(const float* xyz, const float* refl, uint32_t n, int builder,
                       cudaStream_t s, BuildResult* out, char* err, size_t err_len) {
  out->tris = nullptr;
  out->filt = nullptr;
  out->nodes = nullptr;
  out->n_nodes = 0;
  out->root = kEmptyRef;
  out->max_depth = 0;
  out->ms = 0.f;
  if (n == 0) return cudaSuccess;
  cudaError_t e = cudaSuccess;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  unsigned* bounds = nullptr;
  uint64_t *codes = nullptr, *codes_s = nullptr;
  uint32_t *idx = nullptr, *idx_s = nullptr;
  int *child = nullptr, *parent_int = nullptr, *parent_leaf = nullptr, *range = nullptr;
  float *leafbox = nullptr, *nodebox = nullptr;
  unsigned *flags = nullptr, *dmax = nullptr;
  void* temp = nullptr;
  size_t temp_bytes = 0;
  const int T = 256;
  const unsigned nb = (n + T - 1) / T;
  const unsigned ni = n > 1 ? (n - 1 + T - 1) / T : 1;
  unsigned init_bounds[6] = {0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0u, 0u, 0u};
  unsigned hdepth = 0;
  uint32_t* idx_s_final = nullptr;  // leaf order (PLOC), else the Morton order
  // isotropic 63-bit Morton codes (DESIGN.md s.7.1); hierarchy: PLOC with
  // radius 32 (default) or Karras (builder = 1)
  const int bits = kMortonBits, isotropic = 1;
  const bool use_ploc = builder != 1;
#ifndef HELIOS_PLOC_R
#define HELIOS_PLOC_R 32
#endif
  constexpr int ploc_r = HELIOS_PLOC_R;
  int *pcid = nullptr, *pcid2 = nullptr, *pnn = nullptr, *pparent = nullptr;
  float *pbox = nullptr, *pbox2 = nullptr;
  uint32_t *psize = nullptr, *poff = nullptr, *pdepth = nullptr, *porder = nullptr;
  float* pcost = nullptr;
  uint8_t* pnflag = nullptr;
  unsigned long long *pflags = nullptr, *pincl = nullptr;
  void* ptemp = nullptr;
  size_t ptemp_bytes = 0;

#define CK(x)                 \
  do {                        \
    e = (x);                  \
    if (e != cudaSuccess) {   \
      snprintf(err, err_len, "build_lbvh: %s at %s:%d", cudaGetErrorString(e), __FILE__, __LINE__); \
      goto done;              \
    }                         \
  } while (0)

  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, s));
  CK(dalloc(&bounds, 6, s));
  CK(cudaMemcpyAsync(bounds, init_bounds, sizeof(init_bounds), cudaMemcpyHostToDevice, s));
  CK(dalloc(&codes, n, s));
  CK(dalloc(&idx, n, s));
  CK(dalloc(&out->tris, n, s));
  CK(dalloc(&out->filt, n, s));
  nvtxMarkA("build K1: centroid bounds + Morton codes");
  k_centroid_bounds<<<min(nb, 148u * 8u), T, 0, s>>>(xyz, n, bounds);
  CK(cudaGetLastError());
  k_morton<<<nb, T, 0, s>>>(xyz, n, bounds, codes, idx, bits, isotropic);
  CK(cudaGetLastError());
  temp_bytes = sort_temp_bytes(n);
  CK(dev_alloc(&temp, temp_bytes, s));
  nvtxMarkA("build K2: radix sort");
  CK(sort_pairs_u64(codes, idx, n, 3 * bits, temp, temp_bytes, s));
  codes_s = codes;  // sorted in place
  idx_s = idx;
  codes = nullptr;
  idx = nullptr;
  if (n <= (uint32_t)kLeafMax) {
    out->root = leaf_ref(0, n);
    out->max_depth = 0;
  } else if (use_ploc) {
    CK(dalloc(&pcid, n, s));
    CK(dalloc(&pcid2, n, s));
    CK(dalloc(&pnn, n, s));
    CK(dalloc(&pbox, 6ull * n, s));
    CK(dalloc(&pbox2, 6ull * n, s));
    CK(dalloc(&pflags, n, s));
    CK(dalloc(&pincl, n, s));
    CK(dalloc(&psize, 2ull * n - 1, s));
    CK(dalloc(&pparent, 2ull * n - 1, s));
    CK(dalloc(&poff, 2ull * n - 1, s));
    CK(dalloc(&pdepth, 2ull * n - 1, s));
    CK(dalloc(&porder, n, s));
    CK(dalloc(&pcost, n - 1, s));
    CK(dalloc(&pnflag, n - 1, s));
    CK(dalloc(&child, 2ull * (n - 1), s));
    CK(dalloc(&leafbox, 6ull * n, s));
    CK(dalloc(&nodebox, 6ull * (n - 1), s));
    CK(dalloc(&dmax, 1, s));
    CK(dalloc(&out->nodes, n - 1, s));
    CK(cudaMemsetAsync(dmax, 0, sizeof(unsigned), s));
    ptemp_bytes = scan_temp_bytes(n, sizeof(unsigned long long));
    CK(dev_alloc(&ptemp, ptemp_bytes, s));
    nvtxMarkA("build K3: PLOC clustering");
    k_ploc_init<<<nb, T, 0, s>>>(xyz, idx_s, n, pcid, pbox, psize, leafbox);
    CK(cudaGetLastError());
    {
      uint32_t m = n, base = 0;
      std::vector<uint32_t> it_base, it_cnt;
      const size_t smem = sizeof(float) * 6 * (kPlocBlock + 2 * ploc_r);
      while (m > 1) {
        const unsigned gb = (m + kPlocBlock - 1) / kPlocBlock;
        k_ploc_nn<<<gb, kPlocBlock, smem, s>>>(pbox, m, ploc_r, pnn);
        CK(cudaGetLastError());
        k_ploc_flags<<<(m + T - 1) / T, T, 0, s>>>(pnn, m, pflags);
        CK(cudaGetLastError());
        size_t tb = ptemp_bytes;
        CK(scan_u64(reinterpret_cast<const uint64_t*>(pflags), reinterpret_cast<uint64_t*>(pincl),
                    m, true, ptemp, tb, s));
        k_ploc_merge<<<(m + T - 1) / T, T, 0, s>>>(pnn, m, pflags, pincl, n, base, pcid, pbox,
                                                  pcid2, pbox2, child, nodebox, psize, pparent);
        CK(cudaGetLastError());
        unsigned long long tot = 0;
        CK(cudaMemcpyAsync(&tot, pincl + (m - 1), sizeof(tot), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        const uint32_t made = (uint32_t)(tot >> 32), keep = (uint32_t)(tot & 0xFFFFFFFFull);
        if (made == 0) {
          snprintf(err, err_len, "build_ploc: no merge in an iteration (m = %u)", m);
          e = cudaErrorUnknown;
          goto done;
        }
        it_base.push_back(base);
        it_cnt.push_back(made);
        base += made;
        m = keep;
        std::swap(pcid, pcid2);
        std::swap(pbox, pbox2);
      }
      // leaf collapse costs, bottom-up: iterations in creation order
      for (size_t t = 0; t < it_base.size(); ++t) {
        k_ploc_cost<<<(it_cnt[t] + T - 1) / T, T, 0, s>>>(it_base[t], it_cnt[t], n, child,
                                                         psize, leafbox, nodebox, pcost, pnflag);
        CK(cudaGetLastError());
      }
      // depth-first leaf offsets, top-down: iterations in reverse creation order
      const uint32_t root_v = n + (n - 2);
      const uint32_t one = 1, zero = 0;
      CK(cudaMemcpyAsync(poff + root_v, &zero, sizeof(uint32_t), cudaMemcpyHostToDevice, s));
      CK(cudaMemcpyAsync(pdepth + root_v, &one, sizeof(uint32_t), cudaMemcpyHostToDevice, s));
      for (size_t t = it_base.size(); t-- > 0;) {
        k_ploc_offsets<<<(it_cnt[t] + T - 1) / T, T, 0, s>>>(it_base[t], it_cnt[t], n, child,
                                                            psize, poff, pdepth, pnflag, dmax);
        CK(cudaGetLastError());
      }
    }
    k_ploc_order<<<nb, T, 0, s>>>(idx_s, n, poff, porder);
    CK(cudaGetLastError());
    k_ploc_layout<<<ni, T, 0, s>>>(n, child, psize, poff, leafbox, nodebox, pnflag, out->nodes);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(&hdepth, dmax, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
    out->n_nodes = n - 1;
    out->root = (int32_t)(n - 2);
    idx_s_final = porder;
  } else {
    CK(dalloc(&child, 2ull * (n - 1), s));
    CK(dalloc(&range, 2ull * (n - 1), s));
    CK(dalloc(&parent_int, n - 1, s));
    CK(dalloc(&parent_leaf, n, s));
    CK(dalloc(&leafbox, 6ull * n, s));
    CK(dalloc(&nodebox, 6ull * (n - 1), s));
    CK(dalloc(&flags, n - 1, s));
    CK(dalloc(&dmax, 1, s));
    CK(cudaMemsetAsync(flags, 0, sizeof(unsigned) * (n - 1), s));
    CK(cudaMemsetAsync(dmax, 0, sizeof(unsigned), s));
    CK(dalloc(&out->nodes, n - 1, s));
    nvtxMarkA("build K3: Karras hierarchy + refit");
    k_karras<<<ni, T, 0, s>>>(codes_s, (int)n, child, parent_int, parent_leaf, range);
    CK(cudaGetLastError());
    k_refit<<<nb, T, 0, s>>>(xyz, idx_s, (int)n, child, parent_int, parent_leaf, leafbox, nodebox,
                             flags);
    CK(cudaGetLastError());
    k_layout<<<ni, T, 0, s>>>((int)n, child, range, leafbox, nodebox, out->nodes);
    CK(cudaGetLastError());
    k_depth<<<ni, T, 0, s>>>((int)n, range, parent_int, dmax);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(&hdepth, dmax, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
    out->n_nodes = n - 1;
    out->root = 0;
  }
  nvtxMarkA("build K5: triangle records");
  k_permute<<<nb, T, 0, s>>>(xyz, refl, idx_s_final ? idx_s_final : idx_s, n, out->tris,
                              out->filt);
  CK(cudaGetLastError());
  CK(cudaEventRecord(e1, s));
  CK(cudaStreamSynchronize(s));
  CK(cudaEventElapsedTime(&out->ms, e0, e1));
  if (n > (uint32_t)kLeafMax) out->max_depth = hdepth;
  if (out->max_depth > (uint32_t)kStackSize) {
    snprintf(err, err_len, "build_lbvh: tree depth %u exceeds the traversal stack (%d)",
             out->max_depth, kStackSize);
    e = cudaErrorInvalidValue;
  }
#undef CK
done:
  cudaFreeAsync(bounds, s);
  cudaFreeAsync(codes, s);
  cudaFreeAsync(idx, s);
  cudaFreeAsync(codes_s, s);
  cudaFreeAsync(idx_s, s);
  cudaFreeAsync(temp, s);
  cudaFreeAsync(child, s);
  cudaFreeAsync(range, s);
  cudaFreeAsync(parent_int, s);
  cudaFreeAsync(parent_leaf, s);
  cudaFreeAsync(leafbox, s);
  cudaFreeAsync(nodebox, s);
  cudaFreeAsync(flags, s);
  cudaFreeAsync(dmax, s);
  cudaFreeAsync(pcid, s);
  cudaFreeAsync(pcid2, s);
  cudaFreeAsync(pnn, s);
  cudaFreeAsync(pbox, s);
  cudaFreeAsync(pbox2, s);
  cudaFreeAsync(pflags, s);
  cudaFreeAsync(pincl, s);
  cudaFreeAsync(psize, s);
  cudaFreeAsync(pparent, s);
  cudaFreeAsync(poff, s);
  cudaFreeAsync(pdepth, s);
  cudaFreeAsync(porder, s);
  cudaFreeAsync(pcost, s);
  cudaFreeAsync(pnflag, s);
  cudaFreeAsync(ptemp, s);
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  if (e != cudaSuccess) {
    cudaFreeAsync(out->tris, s);
    cudaFreeAsync(out->filt, s);
    cudaFreeAsync(out->nodes, s);
    out->tris = nullptr;
    out->filt = nullptr;
    out->nodes = nullptr;
  }
  cudaStreamSynchronize(s);
  return e;
}

}  // namespace helios
