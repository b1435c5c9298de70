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
// of the tree in the same order (a cached postfix program).  Every addition
// is an IEEE __dadd_rn in numpy's order, so the result is bit-identical
// (tests/test_gpu_stats.py).
//
// The chunk kernel is issue-bound unless the per-value work is a handful of
// instructions, so: leaves are summed in rounds of 32 (one per lane octet)
// whose values thread 0 moves into shared memory with bulk copies (TMA, one
// per component array, double-buffered so round r+1 streams in while round
// r is summed); a lane's shared-memory offsets are immediates (for 3
// components they repeat every 3 steps); min/max are plain compare-selects
// and the NaN test runs only for a chunk whose sum is NaN (a NaN value
// always makes the sum NaN).  min / max / NaN of all chunks reduce on the
// device to three words.  C4 velocity (12.9 GB): 5.66 -> 2.64 ms per launch.
#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>
#include <map>
#include <vector>

#include "nkb_internal.h"
#include "sem_dev.cuh"

namespace nkb {

namespace {

using dev::enc_ordered;

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

// Plain compare-and-select (3 instructions each, fmin/fmax cost ~10): a NaN
// value never survives the pairwise additions, so a chunk whose sum is not
// NaN has none and these equal numpy's min/max; a NaN sum triggers the exact
// scan below and numpy's NaN result.
struct MinMax {
  double mn = INFINITY, mx = -INFINITY;
  __device__ __forceinline__ void add(double v) {
    mn = v < mn ? v : mn;
    mx = v > mx ? v : mx;
  }
};

// AoS value i through the segment table (rounds that cross a segment
// boundary or whose arrays are not 16-byte aligned)
__device__ double value_at(const StatsParams& p, long long i) {
  int s = 0;
  while (s + 1 < p.nseg && i >= p.seg[s + 1].start) ++s;
  const long long r = i - p.seg[s].start;
  const int nc = p.seg[s].ncomp;
  const long long j = r / nc;
  return p.seg[s].base[(long long)(r - j * nc) * p.seg[s].comp_stride + j];
}

// mbarrier + bulk copy (one elected thread moves a contiguous run into smem)
__device__ __forceinline__ void st_mbar_init(unsigned long long* bar) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(a) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void st_expect(unsigned long long* bar, unsigned bytes) {
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
}
__device__ __forceinline__ void st_bulk(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(d), "l"(src), "r"(bytes), "r"(b) : "memory");
}
__device__ __forceinline__ void st_wait(unsigned long long* bar, unsigned parity) {
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n"
      ".reg .pred P;\n"
      "W_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
      "@!P bra W_%=;\n"
      "}\n" ::"r"(b), "r"(parity) : "memory");
}

constexpr int kRoundLeaves = kStatThreads / 8;          // one leaf per octet per round
constexpr int kCompSpan = 1380;                           // doubles per component (3 components); = 4 mod 16
                                                          // so an octet's 8 consecutive AoS values hit 8 banks
constexpr int kBufVals = 3 * kCompSpan;                   // >= 32 * 128 + 2 values (one component)

// A round: 32 consecutive leaves of a chunk, AoS values [v0, v1).  Fast when
// they sit in one segment of 1 or 3 components whose arrays are 16-byte
// aligned: thread 0 moves the tuples [ja, jb) of every component into the
// round's buffer with bulk copies (no per-value load instructions); buffer
// value of AoS index t (relative to the segment) = buf[(t % nc) * span + t / nc - ja].
struct Round {
  long long v0, v1, ja, jb;
  long long rel0;     // AoS index (segment-relative) of buffer tuple 0, component 0: nc * ja
  int seg, nc, fast;
};

__device__ __forceinline__ Round round_of(const StatsParams& p, const StatChunk& C, const StatShape& S, int l0) {
  Round R;
  const int l1 = min(l0 + kRoundLeaves, S.n_leaves);
  const int2 first = p.leaves[S.leaf0 + l0], last = p.leaves[S.leaf0 + l1 - 1];
  R.v0 = C.off + first.x;
  R.v1 = C.off + last.x + last.y;
  int s = 0;
  while (s + 1 < p.nseg && R.v0 >= p.seg[s + 1].start) ++s;
  const StatSeg& g = p.seg[s];
  R.seg = s;
  R.nc = g.ncomp;
  const long long t0 = R.v0 - g.start, t1 = R.v1 - g.start;
  R.ja = (t0 / R.nc) & ~1LL;
  R.jb = ((t1 + R.nc - 1) / R.nc + 1) & ~1LL;
  R.rel0 = R.ja * R.nc;
  bool ok = (R.nc == 1 || R.nc == 3) && t1 <= g.n_tuples * g.ncomp;
  for (int c = 0; c < R.nc && ok; ++c)
    ok = ((unsigned long long)(g.base + (long long)c * g.comp_stride + R.ja) & 15ULL) == 0;
  R.fast = ok;
  return R;
}

__device__ __forceinline__ void round_issue(const StatsParams& p, const Round& R, double* buf,
                                            unsigned long long* bar) {
  if (!R.fast) return;
  const StatSeg& g = p.seg[R.seg];
  const unsigned bytes = (unsigned)((R.jb - R.ja) * 8);
  st_expect(bar, bytes * (unsigned)R.nc);
  for (int c = 0; c < R.nc; ++c)
    st_bulk(buf + c * (R.nc == 1 ? 0 : kCompSpan), g.base + (long long)c * g.comp_stride + R.ja, bytes, bar);
}

// One leaf (57..128 values, or < 8 for a tiny root) summed by an OCTET of
// lanes: lane q owns numpy's accumulator r[q] (values q, q+8, q+16, ... in
// order), the octet then folds ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) with
// shuffles and lane 0 adds the n%8 tail in order.  `at(t)` = value of AoS
// index t relative to the round's segment; `step(k)` = value k of lane q's
// accumulator (t = t0 + q + 8k), specialised so the fast paths are one shared
// load at an immediate offset.
template <class At, class Step>
__device__ __forceinline__ double octet_leaf(int t0, int n, int q, unsigned mask, MinMax& m, At at,
                                             Step step) {
  double res;
  if (n < 8) {
    res = -0.0;
    if (q == 0)
      for (int i = 0; i < n; ++i) {
        const double v = at(t0 + i);
        m.add(v);
        res = __dadd_rn(res, v);
      }
    return res;
  }
  const int lim = n - (n % 8), steps = lim / 8;   // <= 16
  double r = step(0);
  m.add(r);
#pragma unroll
  for (int k = 1; k < 16; ++k)
    if (k < steps) {
      const double v = step(k);
      m.add(v);
      r = __dadd_rn(r, v);
    }
  double o = __shfl_down_sync(mask, r, 1, 8);
  r = __dadd_rn(r, o);                             // lanes 0,2,4,6: r[q] + r[q+1]
  o = __shfl_down_sync(mask, r, 2, 8);
  r = __dadd_rn(r, o);                             // lanes 0,4
  o = __shfl_down_sync(mask, r, 4, 8);
  res = __dadd_rn(r, o);                           // lane 0
  if (q == 0)
    for (int i = lim; i < n; ++i) {
      const double v = at(t0 + i);
      m.add(v);
      res = __dadd_rn(res, v);
    }
  return res;
}

// one CTA per chunk: rounds of 32 leaves, double-buffered bulk staging (round
// r+1 streams in while round r is summed), then the internal nodes of the
// chunk's subtree level by level
__global__ void __launch_bounds__(kStatThreads) pairwise_chunk_kernel(const StatsParams p) {
  extern __shared__ __align__(16) double s_dyn[];     // 2 x kBufVals: the round buffers
  double* const bufs = s_dyn;
  __shared__ double val[2 * kMaxChunkLeaves];
  __shared__ double s_mn[kStatThreads / 32], s_mx[kStatThreads / 32];
  __shared__ __align__(8) unsigned long long bar[2];
  __shared__ Round s_round[2];
  __shared__ int s_nan;
  const int tid = threadIdx.x;
  if (tid == 0) {
    st_mbar_init(&bar[0]);
    st_mbar_init(&bar[1]);
  }
  __syncthreads();
  unsigned phase = 0u;                               // bit b: parity of bar[b]
  for (int ch = blockIdx.x; ch < p.n_chunks; ch += gridDim.x) {
    const StatChunk C = p.chunks[ch];
    const StatShape S = p.shapes[C.shape];
    if (tid == 0) s_nan = 0;
    MinMax m;
    const int oct = tid >> 3, q = tid & 7;
    const unsigned mask = 0xffu << (tid & 24);        // my octet's lanes
    const int n_rounds = (S.n_leaves + kRoundLeaves - 1) / kRoundLeaves;
    // round descriptors are computed once by thread 0 and shared (slot = round parity)
    if (tid == 0) {
      s_round[0] = round_of(p, C, S, 0);
      round_issue(p, s_round[0], bufs, &bar[0]);
    }
    __syncthreads();
    for (int rr = 0; rr < n_rounds; ++rr) {
      const int b = rr & 1;
      if (tid == 0 && rr + 1 < n_rounds) {             // buf[b^1] was read in round rr-1: released below
        s_round[b ^ 1] = round_of(p, C, S, (rr + 1) * kRoundLeaves);
        round_issue(p, s_round[b ^ 1], bufs + (b ^ 1) * kBufVals, &bar[b ^ 1]);
      }
      const Round& cur = s_round[b];
      const int fast = cur.fast, nc = cur.nc;
      if (fast) {
        st_wait(&bar[b], (phase >> b) & 1u);
        phase ^= 1u << b;
      }
      const int l = rr * kRoundLeaves + oct;
      if (l < S.n_leaves) {                          // whole octets take the branch together
        const int2 lf = p.leaves[S.leaf0 + l];         // (offset in chunk, length)
        const double* B = bufs + b * kBufVals;
        double v;
        if (fast) {
          // buffer-relative AoS index of the leaf's first value (< 4100: 32-bit)
          const int r0 = (int)(C.off + lf.x - p.seg[cur.seg].start - cur.rel0);
          if (nc == 1) {
            const double* a = B + r0 + q;
            v = octet_leaf(r0, lf.y, q, mask, m, [&](int t) { return B[t]; }, [&](int k) { return a[8 * k]; });
          } else {                                     // 3 components: the lane's offsets repeat every 3 steps
            int off[3];
#pragma unroll
            for (int r = 0; r < 3; ++r) {
              const int t = r0 + q + 8 * r;
              off[r] = (t % 3) * kCompSpan + t / 3;
            }
            v = octet_leaf(r0, lf.y, q, mask, m, [&](int t) { return B[(t % 3) * kCompSpan + t / 3]; },
                           [&](int k) { return B[off[k % 3] + 8 * (k / 3)]; });
          }
        } else {
          const long long i0 = C.off + lf.x;
          v = octet_leaf(0, lf.y, q, mask, m, [&](int t) { return value_at(p, i0 + t); },
                         [&](int k) { return value_at(p, i0 + q + 8 * k); });
        }
        if (q == 0) val[l] = v;
      }
      __syncthreads();                               // buf[b] and s_round[b] free for round rr+2
    }
    for (int lv = 0; lv < S.n_levels; ++lv) {
      const int a = p.level_start[S.level0 + lv], b = p.level_start[S.level0 + lv + 1];
      for (int k = a + tid; k < b; k += kStatThreads) {
        const int2 lr = p.nodes[S.node0 + k];           // children, indices into val
        val[S.n_leaves + k] = __dadd_rn(val[lr.x], val[lr.y]);
      }
      __syncthreads();
    }
    // chunk min / max; NaN never survives an addition, so a chunk whose sum is
    // not NaN holds no NaN and only a NaN sum needs the exact (rare) scan
    const int root = S.n_leaves + S.n_nodes - 1;     // root is the last node (or the only leaf)
    const double sum = S.n_nodes ? val[root] : val[0];
    if (sum != sum) {
      const long long len = (long long)p.leaves[S.leaf0 + S.n_leaves - 1].x + p.leaves[S.leaf0 + S.n_leaves - 1].y;
      int any = 0;
      for (long long i = tid; i < len; i += kStatThreads) {
        const double v = value_at(p, C.off + i);
        any |= v != v;
      }
      if (any) s_nan = 1;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      m.mn = fmin(m.mn, __shfl_xor_sync(0xffffffffu, m.mn, o));
      m.mx = fmax(m.mx, __shfl_xor_sync(0xffffffffu, m.mx, o));
    }
    if ((tid & 31) == 0) {
      s_mn[tid >> 5] = m.mn;
      s_mx[tid >> 5] = m.mx;
    }
    __syncthreads();
    if (tid == 0) {
      double mn = s_mn[0], mx = s_mx[0];
      for (int w = 1; w < kStatThreads / 32; ++w) {
        mn = fmin(mn, s_mn[w]);
        mx = fmax(mx, s_mx[w]);
      }
      p.out_sum[ch] = sum;
      // min / max / NaN of all chunks: three words, reset by the host per launch
      if (mn <= mx) {
        atomicMin(&p.out_mm[0], enc_ordered(mn));
        atomicMax(&p.out_mm[1], enc_ordered(mx));
      }
      if (s_nan) atomicOr(&p.out_mm[2], 1ULL);
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

// the top of the tree above the chunks as a postfix program: k >= 0 pushes
// chunk sum k (plan order), -1 pops b, a and pushes a + b
static void combine_rec(long long off, long long n, const std::vector<long long>& lo, int& k,
                        std::vector<int>& prog) {
  const int r0 = owner_of(lo, off), r1 = owner_of(lo, off + n - 1);
  if ((r0 == r1 && n <= kChunk) || n <= 128) {
    prog.push_back(k++);
    return;
  }
  const long long n2 = pw_split(n);
  combine_rec(off, n2, lo, k, prog);
  combine_rec(off + n2, n - n2, lo, k, prog);
  prog.push_back(-1);
}

void pairwise_combine_program(long long n, const std::vector<long long>& rank_lo, std::vector<int>& prog) {
  prog.clear();
  int k = 0;
  if (n > 0) combine_rec(0, n, rank_lo, k, prog);
}

double pairwise_combine(const std::vector<int>& prog, const std::vector<double>& chunk_sums) {
  std::vector<double> st;
  st.reserve(64);
  for (const int op : prog) {
    if (op >= 0) {
      st.push_back(chunk_sums[op]);
    } else {
      const double b = st.back();
      st.pop_back();
      st.back() = st.back() + b;                   // host add, -ffp-contract=off: IEEE
    }
  }
  return st.empty() ? 0.0 : st.back();
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
  const size_t shm = 2 * kBufVals * sizeof(double);    // the two round buffers (66 KB)
  static bool attr = false;
  if (!attr) {
    NKB_CUDA(cudaFuncSetAttribute(pairwise_chunk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
    attr = true;
  }
  pairwise_chunk_kernel<<<p.n_chunks, kStatThreads, shm, s>>>(p);   // one chunk per CTA
  NKB_CUDA(cudaGetLastError());
  return NKB_OK;
}

int launch_stat_windows(const StatsParams& p, double* out, cudaStream_t s) {
  window_kernel<<<1, 2 * kWin, 0, s>>>(p, out);
  NKB_CUDA(cudaGetLastError());
  return NKB_OK;
}

}  // namespace nkb
