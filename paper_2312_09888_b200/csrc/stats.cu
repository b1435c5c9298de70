// Field statistics (min, max, mean) with numpy's exact arithmetic -- the
// GPU side of the stats sink (reference StatsSink,
// sinks.py:366-393: `vals.min()`, `vals.max()`, `vals.mean()` of the
// concatenated field values).
//
// numpy's mean is np.add.reduce(a) / n, and add.reduce of a contiguous
// float64 array is 0.0 + pairwise(a, n) with (numpy/_core/src/umath/
// loops_utils.h.src, DOUBLE_pairwise_sum):
//   n < 8     : r = -0.0; r += a[i] in order
//   n <= 128  : 8 accumulators r[j] = a[j], r[j] += a[i+j] for i = 8, 16, ...
//               below n - n%8, then ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)),
//               then the n%8 tail added in order
//   otherwise : n2 = n/2 - (n/2)%8; pairwise(a, n2) + pairwise(a+n2, n-n2)
// The tree depends only on n, so the host cuts it into chunks (subtrees of
// at most kChunk values, split further at rank boundaries); one CTA
// evaluates one chunk bottom-up from a per-length shape table (leaves, then
// internal nodes level by level); the host adds the chunk sums up the top
// of the tree in the same order.  Every addition is an IEEE __dadd_rn in
// numpy's order, so the result is bit-identical (tests/test_gpu_stats.py).
#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>
#include <map>
#include <vector>

#include "nkb_internal.h"

namespace nkb {

namespace {

constexpr int kStatThreads = 256;

// sequential walk over the AoS (component-fastest) values of the segments
struct Walker {
  const StatsParams* p;
  int s;            // segment
  long long j;      // tuple within the segment
  int c;            // component
  __device__ void seek(long long i) {
    s = 0;
    while (s + 1 < p->nseg && i >= p->seg[s + 1].start) ++s;
    const long long r = i - p->seg[s].start;
    const int nc = p->seg[s].ncomp;
    j = r / nc;
    c = (int)(r - j * nc);
  }
  __device__ double next() {
    const StatSeg& g = p->seg[s];
    const double v = g.base[(long long)c * g.comp_stride + j];
    if (++c == g.ncomp) {
      c = 0;
      if (++j == g.n_tuples && s + 1 < p->nseg) {
        ++s;
        j = 0;
      }
    }
    return v;
  }
};

struct MinMax {
  double mn = INFINITY, mx = -INFINITY;
  int nan = 0;
  __device__ void add(double v) {
    if (v != v) nan = 1;
    mn = fmin(mn, v);
    mx = fmax(mx, v);
  }
};

// AoS value i through the segment table (slow path: leaves across segments)
__device__ double value_at(const StatsParams& p, long long i) {
  int s = 0;
  while (s + 1 < p.nseg && i >= p.seg[s + 1].start) ++s;
  const long long r = i - p.seg[s].start;
  const int nc = p.seg[s].ncomp;
  const long long j = r / nc;
  return p.seg[s].base[(long long)(r - j * nc) * p.seg[s].comp_stride + j];
}

// One leaf (57..128 values, or < 8 for a tiny root) summed by an OCTET of
// lanes: lane q owns numpy's accumulator r[q] (values q, q+8, q+16, ... in
// order), the octet then folds ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) with
// shuffles and lane 0 adds the n%8 tail.  Adjacent octets hold adjacent
// leaves, so a warp reads 4 x 64 contiguous bytes per step.
__device__ double octet_leaf(const StatsParams& p, long long off, int n, int q, unsigned mask, MinMax& m) {
  // locate (segment, tuple, component) of value off + q once; advance by 8
  int s = 0;
  while (s + 1 < p.nseg && off >= p.seg[s + 1].start) ++s;
  const StatSeg& g = p.seg[s];
  const bool one_seg = off + n <= g.start + g.n_tuples * g.ncomp;
  const int nc = g.ncomp, dj = 8 / nc, dc = 8 % nc;
  const long long r0 = off + q - g.start;
  long long j = r0 / nc;
  int c = (int)(r0 - j * nc);
  auto get = [&](long long i) -> double {          // i = offset of this lane's value in the leaf
    if (one_seg) {
      const double v = g.base[(long long)c * g.comp_stride + j];
      j += dj;
      c += dc;
      if (c >= nc) {
        c -= nc;
        ++j;
      }
      return v;
    }
    return value_at(p, off + i);
  };
  double res;
  if (n < 8) {
    res = -0.0;
    if (q == 0)
      for (int i = 0; i < n; ++i) {
        const double v = value_at(p, off + i);
        m.add(v);
        res = __dadd_rn(res, v);
      }
    return res;
  }
  const int lim = n - (n % 8), steps = lim / 8;   // <= 16
  double v[16];
#pragma unroll
  for (int k = 0; k < 16; ++k)                     // all loads first: 16 in flight per lane
    if (k < steps) v[k] = get(8 * k + q);
  double r = v[0];
  m.add(r);
#pragma unroll
  for (int k = 1; k < 16; ++k)
    if (k < steps) {
      m.add(v[k]);
      r = __dadd_rn(r, v[k]);
    }
  // fold in numpy's order: pairs, then quads, then the halves
  double o = __shfl_down_sync(mask, r, 1, 8);
  r = __dadd_rn(r, o);                             // lanes 0,2,4,6: r[q] + r[q+1]
  o = __shfl_down_sync(mask, r, 2, 8);
  r = __dadd_rn(r, o);                             // lanes 0,4
  o = __shfl_down_sync(mask, r, 4, 8);
  res = __dadd_rn(r, o);                           // lane 0
  if (q == 0)
    for (int i = lim; i < n; ++i) {
      const double v = value_at(p, off + i);
      m.add(v);
      res = __dadd_rn(res, v);
    }
  return res;
}

__global__ void __launch_bounds__(kStatThreads) pairwise_chunk_kernel(const StatsParams p) {
  __shared__ double val[2 * kMaxChunkLeaves];
  __shared__ double s_mn[kStatThreads / 32], s_mx[kStatThreads / 32];
  __shared__ int s_nan;
  const int tid = threadIdx.x;
  for (int ch = blockIdx.x; ch < p.n_chunks; ch += gridDim.x) {
    const StatChunk C = p.chunks[ch];
    const StatShape S = p.shapes[C.shape];
    if (tid == 0) s_nan = 0;
    MinMax m;
    const int oct = tid >> 3, q = tid & 7;
    const unsigned mask = 0xffu << (tid & 24);        // my octet's lanes
    for (int l0 = 0; l0 < S.n_leaves; l0 += kStatThreads / 8) {
      const int l = l0 + oct;
      if (l < S.n_leaves) {                          // whole octets take the branch together
        const int2 lf = p.leaves[S.leaf0 + l];         // (offset in chunk, length)
        const double v = octet_leaf(p, C.off + lf.x, lf.y, q, mask, m);
        if (q == 0) val[l] = v;
      }
    }
    __syncthreads();
    for (int lv = 0; lv < S.n_levels; ++lv) {
      const int a = p.level_start[S.level0 + lv], b = p.level_start[S.level0 + lv + 1];
      for (int k = a + tid; k < b; k += kStatThreads) {
        const int2 lr = p.nodes[S.node0 + k];           // children, indices into val
        val[S.n_leaves + k] = __dadd_rn(val[lr.x], val[lr.y]);
      }
      __syncthreads();
    }
    // chunk min / max (NaN-propagating, like numpy)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      m.mn = fmin(m.mn, __shfl_xor_sync(0xffffffffu, m.mn, o));
      m.mx = fmax(m.mx, __shfl_xor_sync(0xffffffffu, m.mx, o));
    }
    if (m.nan) s_nan = 1;
    if ((tid & 31) == 0) {
      s_mn[tid >> 5] = m.mn;
      s_mx[tid >> 5] = m.mx;
    }
    __syncthreads();
    if (tid == 0) {
      double mn = s_mn[0], mx = s_mx[0];
      for (int q = 1; q < kStatThreads / 32; ++q) {
        mn = fmin(mn, s_mn[q]);
        mx = fmax(mx, s_mx[q]);
      }
      const int root = S.n_leaves + S.n_nodes - 1;     // root is the last node (or the only leaf)
      p.out_sum[ch] = S.n_nodes ? val[root] : val[0];
      p.out_mm[3 * ch + 0] = mn;
      p.out_mm[3 * ch + 1] = mx;
      p.out_mm[3 * ch + 2] = s_nan ? 1.0 : 0.0;
    }
    __syncthreads();
  }
}

// first / last kWin AoS values of the local concatenation (for chunks that
// straddle rank boundaries)
__global__ void window_kernel(const StatsParams p, double* out) {
  const int i = threadIdx.x;                       // 0 .. 2*kWin-1
  const long long n = p.n;
  long long g = -1;
  if (i < kWin) {
    if (i < n) g = i;
  } else {
    const long long k = n - 2 * kWin + i;           // last kWin
    if (k >= 0 && k < n) g = k;
  }
  double v = NAN;
  if (g >= 0) {
    Walker w{&p, 0, 0, 0};
    w.seek(g);
    v = w.next();
  }
  out[i] = v;
}

}  // namespace

// ---- host: the pairwise tree ------------------------------------------------

static long long pw_split(long long n) {
  long long n2 = n / 2;
  return n2 - n2 % 8;
}

// owner rank of global value index i (rank_lo has nranks+1 entries)
static int owner_of(const std::vector<long long>& lo, long long i) {
  return (int)(std::upper_bound(lo.begin(), lo.end(), i) - lo.begin()) - 1;
}

static void plan_rec(long long off, long long n, const std::vector<long long>& lo, std::vector<PlanChunk>& out) {
  const int r0 = owner_of(lo, off), r1 = owner_of(lo, off + n - 1);
  if (r0 == r1 && n <= kChunk) {
    out.push_back({off, n, r0});
    return;
  }
  if (n <= 128) {                                  // a leaf across a rank boundary
    out.push_back({off, n, -1});
    return;
  }
  const long long n2 = pw_split(n);
  plan_rec(off, n2, lo, out);
  plan_rec(off + n2, n - n2, lo, out);
}

void pairwise_plan(long long n, const std::vector<long long>& rank_lo, std::vector<PlanChunk>& out) {
  out.clear();
  if (n > 0) plan_rec(0, n, rank_lo, out);
}

static double combine_rec(long long off, long long n, const std::vector<long long>& lo, const double* v,
                          size_t& k) {
  const int r0 = owner_of(lo, off), r1 = owner_of(lo, off + n - 1);
  if ((r0 == r1 && n <= kChunk) || n <= 128) return v[k++];
  const long long n2 = pw_split(n);
  const double a = combine_rec(off, n2, lo, v, k);
  const double b = combine_rec(off + n2, n - n2, lo, v, k);
  return a + b;                                    // host add, -ffp-contract=off: IEEE
}

double pairwise_combine(long long n, const std::vector<long long>& rank_lo, const std::vector<double>& chunk_sums) {
  size_t k = 0;
  return combine_rec(0, n, rank_lo, chunk_sums.data(), k);
}

// shape of the subtree of a chunk of length n: leaves left to right, then
// internal nodes grouped by level (children always in an earlier group)
static int shape_rec(long long rel, long long n, std::vector<int2>& leaves, std::vector<int2>& nodes,
                     std::vector<int>& level, int* depth) {
  if (n <= 128) {
    leaves.push_back(make_int2((int)rel, (int)n));
    *depth = 0;
    return (int)leaves.size() - 1;                 // leaf id >= 0
  }
  const long long n2 = pw_split(n);
  int dl, dr;
  const int l = shape_rec(rel, n2, leaves, nodes, level, &dl);
  const int r = shape_rec(rel + n2, n - n2, leaves, nodes, level, &dr);
  nodes.push_back(make_int2(l, r));                // child ids: leaf >= 0, node = -(k+1)
  *depth = 1 + std::max(dl, dr);
  level.push_back(*depth);
  return -(int)nodes.size();
}

void pairwise_shape(long long n, StatShapeHost& sh) {
  std::vector<int2> leaves, nodes;
  std::vector<int> level;
  int depth = 0;
  shape_rec(0, n, leaves, nodes, level, &depth);
  const int nl = (int)leaves.size(), nn = (int)nodes.size();
  // order internal nodes by level (stable), remap child ids into val[] slots
  std::vector<int> order(nn);
  for (int i = 0; i < nn; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return level[a] < level[b]; });
  std::vector<int> slot(nn);
  for (int k = 0; k < nn; ++k) slot[order[k]] = nl + k;
  auto map_child = [&](int id) { return id >= 0 ? id : slot[-id - 1]; };
  sh.leaves = leaves;
  sh.nodes.resize(nn);
  for (int k = 0; k < nn; ++k) sh.nodes[k] = make_int2(map_child(nodes[order[k]].x), map_child(nodes[order[k]].y));
  // level l (1..depth) occupies node slots [level_start[l-1], level_start[l])
  const int D = nn ? *std::max_element(level.begin(), level.end()) : 0;
  std::vector<int> cnt(D + 1, 0);
  for (int i = 0; i < nn; ++i) ++cnt[level[i]];
  sh.level_start.assign(1, 0);
  for (int l = 1; l <= D; ++l) sh.level_start.push_back(sh.level_start.back() + cnt[l]);
  sh.n_levels = D;
}

int launch_pairwise_chunks(const StatsParams& p, cudaStream_t s) {
  if (p.n_chunks <= 0) return NKB_OK;
  const int grid = std::min(p.n_chunks, 148 * 8);
  pairwise_chunk_kernel<<<grid, kStatThreads, 0, s>>>(p);
  NKB_CUDA(cudaGetLastError());
  return NKB_OK;
}

int launch_stat_windows(const StatsParams& p, double* out, cudaStream_t s) {
  window_kernel<<<1, 2 * kWin, 0, s>>>(p, out);
  NKB_CUDA(cudaGetLastError());
  return NKB_OK;
}

}  // namespace nkb
