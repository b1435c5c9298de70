// K2 raster (triangles -> packed depth|scalar keys, order-independent
// atomicMin) and K3 resolve (keys -> RGBA8 + depth through the reference
// colormap).
//
// Reference anchors: colormap `ColorMap.apply` / DEFAULT_COLORMAP
// (sinks.py:190-213: clip, np.interp per channel, floor(v+0.5)); global range
// and degenerate-range rule of `render` (sinks.py:264-269); row 0 = top of
// the image (sinks.py:256-257).  Rasterisation itself (R15) has no reference
// implementation; oracle/sem_oracle.c restates it operation for operation.
#include <cuda_runtime.h>
#include <math.h>

#include "checked.cuh"
#include "nkb_internal.h"
#include "raster_dev.cuh"

namespace nkb {

namespace {

__device__ __forceinline__ double clip01(double t) { return t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t); }

__global__ void zbuf_clear_kernel(unsigned long long* z, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    z[i] = ~0ULL;
}

// one thread per triangle; blockIdx.y = triangle region (the count lives on
// the device).  The region's warps take 32 consecutive triangles each
// (coalesced reads) and are dealt round-robin over the region's blocks, so a
// region with few triangles still spreads over several SMs.
// (four CTAs per SM: 64 registers with a few bytes of spills beat three at
// 68 -- the kernel is issue- and latency-bound, profiles/r2/raster_lb4_ab.txt)
// kL lanes per triangle (each takes every kL-th pixel row): more warps with
// work when a step has few, large triangles (C1)
template <int kL>
__global__ void __launch_bounds__(256, 4) raster_kernel(const RasterParams p) {
  const int r = blockIdx.y;
  long long ntri = (long long)p.region_count[r];
  if (ntri > p.region_cap) ntri = p.region_cap;
  const float4* tri = p.tri + 3 * (long long)r * p.region_cap;
  const int W = p.width, H = p.height;
  constexpr int kPerWarp = 32 / kL;
  const long long gw = (long long)(threadIdx.x >> 5) * gridDim.x + blockIdx.x;   // region-local warp
  const long long nw = (long long)gridDim.x * (blockDim.x >> 5);
  const int lane = threadIdx.x & 31;
  for (long long t = gw * kPerWarp + lane / kL; t < ntri; t += nw * kPerWarp) {
    NKB_DCHECK(t >= 0 && t < p.region_cap && r < p.n_regions);
    rdev::raster_triangle(p.view, W, H, tri + 3 * t, p.zbuf, lane % kL, kL);
  }
}

// counters [1]=enc(min) [2]=enc(max) -> composite words: enc(min), ~enc(max);
// counters[6] = 1 when the step's triangles overflowed the buffer (a CTA
// region in FAST mode, the whole buffer in ordered mode).  Multi-rank steps
// share this word (P2P flags / an NCCL max) so that every rank decides alike
// whether the step must grow and re-run.
__device__ void range_words_body(unsigned long long* counters, unsigned long long* words,
                                 const unsigned long long* region_count, int n_regions, long long region_cap,
                                 long long tri_cap, unsigned long long* snap) {
  __shared__ int s_over;
  if (threadIdx.x == 0) {
    words[0] = counters[1];
    words[1] = ~counters[2];
    s_over = 0;
  }
  __syncthreads();
  int over = 0;
  if (region_count) {
    for (int r = threadIdx.x; r < n_regions; r += blockDim.x)
      over |= region_count[r] > (unsigned long long)region_cap;
  } else if (threadIdx.x == 0) {
    over = counters[0] > (unsigned long long)tri_cap;
  }
  if (over) s_over = 1;
  __syncthreads();
  if (threadIdx.x == 0) {
    counters[6] = (unsigned long long)s_over;
    // the step's counters for the composite stream (the next step resets them meanwhile)
    if (snap)
      for (int i = 0; i < 8; ++i) snap[i] = i == 6 ? (unsigned long long)s_over : counters[i];
  }
}

__global__ void __launch_bounds__(256) range_words_kernel(unsigned long long* counters, unsigned long long* words,
                                                          const unsigned long long* region_count, int n_regions,
                                                          long long region_cap, long long tri_cap,
                                                          unsigned long long* snap) {
  range_words_body(counters, words, region_count, n_regions, region_cap, tri_cap, snap);
}

// the step's report words straight into mapped pinned host memory: one
// kernel instead of 3-5 small D2H copies at the tail of every step
__device__ void report_body(const ReportParams& p) {
  const int t = threadIdx.x;
  if (p.part & 1) {
    if (t < 4) p.h_counters[t] = p.counters[t];
    // overflow words are sticky across stream-ordered steps: the host clears them
    if (t == 6 || t == 7) p.h_counters[t] |= p.counters[t];
  }
  if (!(p.part & 2)) return;
  if (t == 4 || t == 5) p.h_counters[t] = (unsigned long long)__double_as_longlong(p.range[t - 4]);
  if (p.h_res) {
    if (t == 0) p.h_res[0] = (unsigned long long)(unsigned)*p.err;
    if (t < kMaxRanks) p.h_res[1 + t] = *(volatile const unsigned long long*)(p.peer_counts + t);
    if (t == 32) {      // any rank overflowed (its flag was written before its "keys ready" release)
      unsigned long long any = 0;
      for (int q = 0; q < p.nranks; ++q) any |= *(volatile const unsigned long long*)(p.peer_overflow + q);
      p.h_res[1 + kMaxRanks] |= any;                 // sticky, like h_counters[6..7]
    }
  }
}

__global__ void __launch_bounds__(256) report_kernel(const ReportParams p) { report_body(p); }

constexpr int kResolvePx = 4;

template <bool kTail>
__global__ void __launch_bounds__(256) resolve_kernel(const ResolveParams p, const ReportParams rep) {
  double lo = p.vmin, hi = p.vmax;
  if (kTail) {                                       // the range straight from the step's counters
    const unsigned long long w0 = p.counters[1], w1 = p.counters[2];
    if (!(lo == lo)) lo = (w0 == ~0ULL) ? 0.0 : rdev::dec_ordered(w0);
    if (!(hi == hi)) hi = (w1 == 0ULL) ? 0.0 : rdev::dec_ordered(w1);
  } else if (p.range_words) {
    const unsigned long long w0 = p.range_words[0], w1 = ~p.range_words[1];
    if (!(lo == lo)) lo = (w0 == ~0ULL) ? 0.0 : rdev::dec_ordered(w0);
    if (!(hi == hi)) hi = (w1 == 0ULL) ? 0.0 : rdev::dec_ordered(w1);
  }
  const long long n = (long long)p.width * p.height;
  if (blockIdx.x == 0 && threadIdx.x == 0 && p.range_out) {
    p.range_out[0] = lo;
    p.range_out[1] = hi;
  }
  const double span = __dsub_rn(hi, lo);
  // kResolvePx pixels per thread per pass, every key load issued before the
  // first is used (the loop is load-latency-bound)
  const long long stride = (long long)gridDim.x * blockDim.x * kResolvePx;
  for (long long i0 = blockIdx.x * (long long)blockDim.x * kResolvePx + threadIdx.x; i0 < n; i0 += stride) {
    unsigned long long keys[kResolvePx];
#pragma unroll
    for (int k = 0; k < kResolvePx; ++k) {
      const long long i = i0 + (long long)k * blockDim.x;
      keys[k] = i < n ? p.zbuf[i] : ~0ULL;
    }
#pragma unroll
    for (int k = 0; k < kResolvePx; ++k) {
    const long long i = i0 + (long long)k * blockDim.x;
    if (i >= n) break;
    NKB_DCHECK(i >= 0 && i < n);
    const unsigned long long key = keys[k];
    uchar4 o;
    float dep;
    if (key == ~0ULL) {
      o = make_uchar4(p.bg[0], p.bg[1], p.bg[2], p.bg[3]);
      dep = INFINITY;
    } else {
      const double s = (double)__uint_as_float((unsigned)(key & 0xffffffffULL));
      dep = __uint_as_float((unsigned)(key >> 32));
      const double t = clip01(hi > lo ? __ddiv_rn(__dsub_rn(s, lo), span) : 0.0);
      o = rdev::cmap_rgba(p.cmap, t);
    }
    reinterpret_cast<uchar4*>(p.rgba)[i] = o;
    if (p.depth) p.depth[i] = dep;
    if (kTail) p.clear_next[i] = ~0ULL;
    }
  }
  if (!kTail) return;
  if (blockIdx.x == 0 && threadIdx.x < 2) p.clear_next[n + threadIdx.x] = ~0ULL;
  // the last CTA to finish: range words, overflow word and the step report.
  // It reads only what earlier kernels wrote plus block 0's range_out, which
  // block 0's thread 0 wrote itself and fences before its ticket -- one fence
  // per CTA, not per thread
  __shared__ int s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(p.ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  range_words_body(p.counters, p.words, p.region_count, p.n_regions, p.region_cap, p.tri_cap, nullptr);
  __syncthreads();
  report_body(rep);
  if (threadIdx.x == 0) *p.ticket = 0u;
}

// ---- reference 2D renderer (sinks.render) ---------------------------------

__device__ __forceinline__ unsigned long long enc_ordered(double d) {
  unsigned long long b = (unsigned long long)__double_as_longlong(d);
  return (b & 0x8000000000000000ULL) ? ~b : (b | 0x8000000000000000ULL);
}

__device__ __forceinline__ double structured_value(const StructuredParams& p, long long row,
                                                   long long col) {
  int b = 0;
  while (b + 1 < p.n_blocks && col >= p.col0[b + 1]) ++b;
  const long long ni = p.col0[b + 1] - p.col0[b];
  const double* v = p.values[b] + (size_t)p.comps * ((col - p.col0[b]) + ni * row);
  if (p.mode == 0) return v[0];
  // scalar_field ':mag' = sqrt(sum(grid**2, axis=-1)), left-to-right (sinks.py:240-241)
  double acc = __dmul_rn(v[0], v[0]);
  for (int c = 1; c < p.comps; ++c) acc = __dadd_rn(acc, __dmul_rn(v[c], v[c]));
  return __dsqrt_rn(acc);
}

__global__ void __launch_bounds__(256) structured_minmax_kernel(const StructuredParams p) {
  const long long n = p.ni_total * p.rows;
  double mn = INFINITY, mx = -INFINITY;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double v = structured_value(p, i / p.ni_total, i % p.ni_total);
    mn = fmin(mn, v);
    mx = fmax(mx, v);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if ((threadIdx.x & 31) == 0 && mn <= mx) {
    atomicMin(&p.minmax[0], enc_ordered(mn));
    atomicMax(&p.minmax[1], enc_ordered(mx));
  }
}

__global__ void __launch_bounds__(256) structured_render_kernel(const StructuredParams p) {
  double lo = p.vmin, hi = p.vmax;
  if (!(lo == lo)) lo = rdev::dec_ordered(p.minmax[0]);
  if (!(hi == hi)) hi = rdev::dec_ordered(p.minmax[1]);
  if (blockIdx.x == 0 && threadIdx.x == 0 && p.range_out) {
    p.range_out[0] = lo;
    p.range_out[1] = hi;
  }
  const long long ni = p.ni_total, nj = p.rows;
  const int W = p.width, H = p.height;
  const long long npx = (long long)W * H;
  const bool deg = !(hi > lo);
  const double span = __dsub_rn(hi, lo);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < npx;
       i += (long long)gridDim.x * blockDim.x) {
    const long long py = i / W, px = i % W;
    // sinks.py:271-281 pixel -> index space
    const double xf = (W > 1) ? __ddiv_rn((double)(px * (ni - 1)), (double)(W - 1)) : 0.0;
    const double yf = (H > 1) ? __ddiv_rn((double)((H - 1 - py) * (nj - 1)), (double)(H - 1)) : 0.0;
    const long long x0 = (ni > 1) ? min((long long)xf, ni - 2) : 0;
    const long long y0 = (nj > 1) ? min((long long)yf, nj - 2) : 0;
    const double ax = __dsub_rn(xf, (double)x0), ay = __dsub_rn(yf, (double)y0);
    const long long x1 = min(x0 + 1, ni - 1), y1 = min(y0 + 1, nj - 1);
    auto T = [&](long long r, long long c) {
      return deg ? 0.0 : __ddiv_rn(__dsub_rn(structured_value(p, r, c), lo), span);
    };
    const double t00 = T(y0, x0), t01 = T(y0, x1), t10 = T(y1, x0), t11 = T(y1, x1);
    const double omay = __dsub_rn(1.0, ay), omax = __dsub_rn(1.0, ax);
    // sinks.py:288-293, numpy left-to-right evaluation
    double s = __dmul_rn(__dmul_rn(t00, omay), omax);
    s = __dadd_rn(s, __dmul_rn(__dmul_rn(t01, omay), ax));
    s = __dadd_rn(s, __dmul_rn(__dmul_rn(t10, ay), omax));
    s = __dadd_rn(s, __dmul_rn(__dmul_rn(t11, ay), ax));
    const double t = clip01(s);
    const uchar4 o = rdev::cmap_rgba(p.cmap, t);
    p.rgb[3 * i + 0] = o.x;
    p.rgb[3 * i + 1] = o.y;
    p.rgb[3 * i + 2] = o.z;
  }
}

// RGBA8 -> packed RGB8 (the PPM payload): 4 pixels per thread, 16 B in, 12 B out
__global__ void pack_rgb_kernel(const uchar4* __restrict__ rgba, unsigned char* __restrict__ rgb, long long npx) {
  const long long n4 = npx / 4;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n4; q += (long long)gridDim.x * blockDim.x) {
    const uint4 v = reinterpret_cast<const uint4*>(rgba)[q];        // pixels 4q .. 4q+3, bytes r g b a
    uint3 o;
    o.x = __byte_perm(v.x, v.y, 0x4210);      // r0 g0 b0 r1
    o.y = __byte_perm(v.y, v.z, 0x5421);      // g1 b1 r2 g2
    o.z = __byte_perm(v.z, v.w, 0x6542);      // b2 r3 g3 b3
    reinterpret_cast<uint3*>(rgb)[q] = o;
  }
  if (blockIdx.x == 0 && threadIdx.x < (npx & 3)) {
    const long long i = n4 * 4 + threadIdx.x;
    const uchar4 c = rgba[i];
    rgb[3 * i] = c.x;
    rgb[3 * i + 1] = c.y;
    rgb[3 * i + 2] = c.z;
  }
}

inline unsigned grid_for(long long n, int threads, int max_blocks) {
  long long b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > max_blocks) b = max_blocks;
  return (unsigned)b;
}

}  // namespace

// the step's counter words {0, enc(+max) = ~0, 0, ...}: one graph node
__global__ void init_counters_kernel(unsigned long long* c) { c[threadIdx.x] = threadIdx.x == 1 ? ~0ULL : 0ULL; }

int launch_init_counters(unsigned long long* counters, cudaStream_t s) {
  init_counters_kernel<<<1, 8, 0, s>>>(counters);
  NKB_CUDA(cudaGetLastError());
  return NKB_OK;
}

int launch_zbuf_clear(unsigned long long* zbuf, int64_t n, cudaStream_t s) {
  zbuf_clear_kernel<<<grid_for(n, 256, 148 * 16), 256, 0, s>>>(zbuf, n);
  NKB_CUDA(cudaGetLastError());
  return NKB_OK;
}

int launch_raster(const RasterParams& p, cudaStream_t s) {
  const int bx = p.n_regions >= 148 ? 8 : (148 * 8 + p.n_regions - 1) / p.n_regions;
  if (p.lanes_per_tri == 4) raster_kernel<4><<<dim3(bx, p.n_regions), 256, 0, s>>>(p);
  else if (p.lanes_per_tri == 2) raster_kernel<2><<<dim3(bx, p.n_regions), 256, 0, s>>>(p);
  else raster_kernel<1><<<dim3(bx, p.n_regions), 256, 0, s>>>(p);
  NKB_CUDA(cudaGetLastError());
  return NKB_OK;
}

int launch_range_words(unsigned long long* counters, unsigned long long* words,
                       const unsigned long long* region_count, int n_regions, int64_t region_cap, int64_t tri_cap,
                       cudaStream_t s, unsigned long long* snap) {
  range_words_kernel<<<1, 256, 0, s>>>(counters, words, region_count, n_regions, (long long)region_cap,
                                       (long long)tri_cap, snap);
  NKB_CUDA(cudaGetLastError());
  return NKB_OK;
}

int launch_pack_rgb(const unsigned char* rgba, unsigned char* rgb, int64_t npx, cudaStream_t s) {
  if (npx <= 0) return NKB_OK;
  pack_rgb_kernel<<<grid_for(npx / 4 + 1, 256, 148 * 8), 256, 0, s>>>(reinterpret_cast<const uchar4*>(rgba), rgb,
                                                                     (long long)npx);
  NKB_CUDA(cudaGetLastError());
  return NKB_OK;
}

int launch_report(const ReportParams& p, cudaStream_t s) {
  report_kernel<<<1, 256, 0, s>>>(p);
  NKB_CUDA(cudaGetLastError());
  return NKB_OK;
}

int launch_resolve(const ResolveParams& p, cudaStream_t s) {
  resolve_kernel<false><<<grid_for(((long long)p.width * p.height + kResolvePx - 1) / kResolvePx, 256, 148 * 8), 256,
                          0, s>>>(p, ReportParams{});
  NKB_CUDA(cudaGetLastError());
  return NKB_OK;
}

int launch_resolve_tail(const ResolveParams& p, const ReportParams& rep, cudaStream_t s) {
  resolve_kernel<true><<<grid_for(((long long)p.width * p.height + kResolvePx - 1) / kResolvePx, 256, 148 * 8), 256, 0,
                         s>>>(p, rep);
  NKB_CUDA(cudaGetLastError());
  return NKB_OK;
}

int launch_structured_minmax(const StructuredParams& p, cudaStream_t s) {
  structured_minmax_kernel<<<grid_for(p.ni_total * p.rows, 256, 148 * 8), 256, 0, s>>>(p);
  NKB_CUDA(cudaGetLastError());
  return NKB_OK;
}

int launch_structured_render(const StructuredParams& p, cudaStream_t s) {
  structured_render_kernel<<<grid_for((long long)p.width * p.height, 256, 148 * 16), 256, 0, s>>>(p);
  NKB_CUDA(cudaGetLastError());
  return NKB_OK;
}

#ifdef NKB_CHECKED
// a check that always fails (NKB_CHECKED_SELFTEST=1): proves a violation
// reaches nkb_execute's error
__global__ void checked_selftest_kernel() { NKB_DCHECK(threadIdx.x > 0); }
int checked_selftest(cudaStream_t s) {
  checked_selftest_kernel<<<1, 32, 0, s>>>();
  NKB_CUDA(cudaGetLastError());
  return NKB_OK;
}
#else
int checked_selftest(cudaStream_t) { return NKB_OK; }
#endif

NKB_CHECKED_ACCESSOR(checked_read_raster)

}  // namespace nkb
