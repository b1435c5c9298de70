// K1s: the in situ pass for pipelines that need no velocity gradient --
// isosurfaces of |u| or of loaded scalars, slices, colour by |u| or a scalar
// (the C4 pebble-bed pipeline, and the surface pass
// of the continuous (DSSUM) pipeline, whose Q / |w| arrive as scalars).
//
// Without derivative pencils an element needs no shared staging at all, so
// the CTA-wide barriers of K1 (fused.cu) go away: every WARP owns one element
// at a time, start to finish.
//
//   node phase : lane l takes nodes 64k+2l, 64k+2l+1 (k = 0..7): 16-byte
//                loads straight from the SoA fields (512 B per warp load,
//                coalesced, each field byte read once), |u|, plane
//                distances, case bits (one byte per node, node order, into
//                the warp's 512 B of shared memory) and the colour range
//   vote       : warp AND / OR of the case bits; an element that no surface
//                crosses is done here (the common case)
//   classify   : 11 chunks of 32 sub-hexes in cell order: case byte per
//                surface, triangle count, a warp scan of the counts and a
//                ballot compaction of the active cells
//   emit       : one lane per active cell, triangles in (surface, table)
//                order at the cell's scanned offset; the few corner values
//                an edge needs are re-read through L1/L2 (the element was
//                streamed microseconds earlier)
//
// 24 warps per SM keep ~75 KB of loads in flight (Little's law at 6.5 TB/s
// and ~1 us needs ~45 KB), and warps emitting triangles overlap warps that
// stream.  Elements are handed out by a per-CTA counter, so heavy elements
// (many triangles) balance across warps.  Triangle slots, the CTA-private
// output regions, COUNT / ORDERED modes, the meta words and the colour-range
// atomics follow K1 exactly; every value is computed by the same functions in
// the same order (sem_dev.cuh), so triangles, images and ranges are
// bit-identical to K1 and to the CPU oracle.
#include <cuda_runtime.h>
#include <math.h>
#include <stdlib.h>

#define NKB_MC_NO_HOST_TABLES
#include "mc_tables.h"
#include "checked.cuh"
#include "nkb_internal.h"
#include "sem_dev.cuh"

namespace nkb {

namespace {

using namespace dev;

__device__ const unsigned char gs_mc_ntri[256] = {NKB_MC_NTRI_DATA};
__device__ const signed char gs_mc_tri[256][3 * NKB_MC_MAX_TRI] = {NKB_MC_TRI_DATA};
__device__ const unsigned char gs_mc_edge_v[12][2] = {NKB_MC_EDGE_V_DATA};

constexpr int kSMaxThreads = 1024;                 // block sizes: 768 (default), 896, 1024
constexpr int kChunks = (kNC + 31) / 32;   // 11 chunks of 32 sub-hexes

struct WarpScratch {
  unsigned long long rows[kNN / 8];   // case bits, one byte per node, node order
  unsigned cases[kNC];                // active cell a: case byte of surface s at bits 8s
  unsigned short cell[kNC];           // active cell a: sub-hex index
  unsigned short off[kNC];            // active cell a: exclusive triangle offset (cell order)
};

struct StreamFlags {
  int xyz;      // coordinates needed per node: bit c = some slice normal has a nonzero component c
  int umag;     // |u| needed per node
  int nsc;      // scalar fields loaded per node
};

__device__ __forceinline__ double2 ld2(const double* p) { return __ldg(reinterpret_cast<const double2*>(p)); }

}  // namespace

// kSProg: node program (cf. fused.cu node_prog).  0 = generic runtime
// dispatch; 1 = the C4 shape -- |u| iso (surface 0) + one slice plane
// (surface 1), colour |u|, no scalars: only u,v,w and the plane's coordinates
// are loaded and live, so the node loop needs fewer registers.
template <int kSThreads, int kSProg>
__global__ void __launch_bounds__(kSThreads, 1) stream_kernel(const FusedParams p, const StreamFlags fl) {
  constexpr int kSWarps = kSThreads / 32;
  extern __shared__ __align__(16) unsigned char s_raw[];
  __shared__ unsigned char t_ntri[256];
  __shared__ signed char t_tri[256][3 * NKB_MC_MAX_TRI];
  __shared__ unsigned char t_edge[12][2];
  __shared__ unsigned long long s_fill;               // FAST: triangles in this CTA's region
  __shared__ unsigned s_next;                         // next element (iteration) of this CTA
  __shared__ double s_mn[kSWarps], s_mx[kSWarps];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  WarpScratch& ws = reinterpret_cast<WarpScratch*>(s_raw)[warp];
  for (int i = tid; i < 256; i += kSThreads) t_ntri[i] = gs_mc_ntri[i];
  for (int i = tid; i < 256 * 3 * NKB_MC_MAX_TRI; i += kSThreads) (&t_tri[0][0])[i] = (&gs_mc_tri[0][0])[i];
  if (tid < 24) (&t_edge[0][0])[tid] = (&gs_mc_edge_v[0][0])[tid];
  if (tid == 0) {
    s_fill = 0;
    s_next = 0;
  }
  __syncthreads();

  const long long E = p.n_elements;
  const long long G = gridDim.x;
  const long long n_it = (E > blockIdx.x) ? (E - blockIdx.x + G - 1) / G : 0;
  const unsigned full = 0xffffffffu;
  const unsigned lt_mask = (1u << lane) - 1u;
  double cmin = INFINITY, cmax = -INFINITY;
  unsigned char* bytes = reinterpret_cast<unsigned char*>(ws.rows);

  for (;;) {
    unsigned it = 0;
    if (lane == 0) it = atomicAdd(&s_next, 1u);
    it = __shfl_sync(full, it, 0);
    if ((long long)it >= n_it) break;
    const long long e = blockIdx.x + (long long)it * G;
    const long long g0 = e * (long long)kNN;
    NKB_DCHECK(e >= 0 && e < E);

    // ---- node phase: 2 nodes per lane per step, 16-byte loads ----
    unsigned band = 0xffu, bor = 0u;
    if (kSProg == 1) {
#pragma unroll 1
      for (int k = 0; k < 8; ++k) {
        const long long gi = g0 + 64 * k + 2 * lane;
        double2 X = make_double2(0.0, 0.0), Y = X, Z = X;
        if (fl.xyz & 1) X = ld2(p.x + gi);
        if (fl.xyz & 2) Y = ld2(p.y + gi);
        if (fl.xyz & 4) Z = ld2(p.z + gi);
        const double2 U = ld2(p.vel[0] + gi), V = ld2(p.vel[1] + gi), W = ld2(p.vel[2] + gi);
        unsigned b2 = 0;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const double vu = mag3(h ? U.y : U.x, h ? V.y : V.x, h ? W.y : W.x);
          const double pd = plane_dist(p.surf_n[1], h ? X.y : X.x, h ? Y.y : Y.x, h ? Z.y : Z.x);
          const unsigned bits = (vu >= p.surf_iso[0] ? 1u : 0u) | ((pd >= p.surf_iso[1] ? 1u : 0u) << 1);
          b2 |= bits << (8 * h);
          cmin = fmin(cmin, vu);
          cmax = fmax(cmax, vu);
        }
        reinterpret_cast<unsigned short*>(bytes)[32 * k + lane] = (unsigned short)b2;
        band &= b2 & (b2 >> 8);
        bor |= (b2 | (b2 >> 8)) & 0xffu;
      }
    } else
#pragma unroll 1
    for (int k = 0; k < 8; ++k) {
      const long long gi = g0 + 64 * k + 2 * lane;
      double2 X = make_double2(0.0, 0.0), Y = X, Z = X, U = X, V = X, W = X, S[kMaxScalars];
      // an unloaded coordinate enters the distance as 0: its term is 0*x, which
      // can only flip the sign of a zero distance, and +-0 compare the same
      // against the iso value (emission recomputes distances from x,y,z)
      if (fl.xyz & 1) X = ld2(p.x + gi);
      if (fl.xyz & 2) Y = ld2(p.y + gi);
      if (fl.xyz & 4) Z = ld2(p.z + gi);
      if (fl.umag) {
        U = ld2(p.vel[0] + gi);
        V = ld2(p.vel[1] + gi);
        W = ld2(p.vel[2] + gi);
      }
#pragma unroll
      for (int c = 0; c < kMaxScalars; ++c) S[c] = (c < fl.nsc) ? ld2(p.scalar[c] + gi) : make_double2(0.0, 0.0);
      unsigned b2 = 0;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const double x = h ? X.y : X.x, y = h ? Y.y : Y.x, z = h ? Z.y : Z.x;
        double sc[kMaxScalars];
#pragma unroll
        for (int c = 0; c < kMaxScalars; ++c) sc[c] = h ? S[c].y : S[c].x;
        const double vu = fl.umag ? mag3(h ? U.y : U.x, h ? V.y : V.x, h ? W.y : W.x) : 0.0;
        auto scalar_of = [&](int src) -> double {
          double v = sc[0];
#pragma unroll
          for (int c = 1; c < kMaxScalars; ++c) v = (src == SRC_SCALAR0 + c) ? sc[c] : v;
          return v;
        };
        unsigned bits = 0;
#pragma unroll
        for (int s = 0; s < NKB_MAX_SURFACES; ++s) {
          if (s >= p.n_surf) break;
          const int src = p.surf_src[s];
          const double val = (src >= SRC_PLANE) ? plane_dist(p.surf_n[s], x, y, z)
                             : (src == SRC_UMAG) ? vu
                                                 : scalar_of(src);
          bits |= (val >= p.surf_iso[s] ? 1u : 0u) << s;
        }
        b2 |= bits << (8 * h);
        if (p.color_src >= 0) {
          const double c = (p.color_src == SRC_UMAG) ? vu : scalar_of(p.color_src);
          cmin = fmin(cmin, c);
          cmax = fmax(cmax, c);
        }
      }
      reinterpret_cast<unsigned short*>(bytes)[32 * k + lane] = (unsigned short)b2;   // nodes 64k+2l, +1
      band &= b2 & (b2 >> 8);
      bor |= (b2 | (b2 >> 8)) & 0xffu;
    }
    if (p.n_surf == 0) continue;
    band = __reduce_and_sync(full, band);
    bor = __reduce_or_sync(full, bor);
    if ((bor & ~band) == 0u) {                         // no surface crosses this element
      if (p.mode == FUSED_COUNT && lane == 0) p.elem_count[e] = 0;
      continue;
    }
    __syncwarp();

    // ---- classify: chunks of 32 sub-hexes in cell order ----
    int n_act = 0, total = 0;
    for (int m = 0; m < kChunks; ++m) {
      const int c = 32 * m + lane;
      unsigned packed = 0;
      int nc = 0;
      if (c < kNC) {
        const int a = c % kN, b = (c / kN) % kN, kk = c / (kN * kN);
        const unsigned long long w = corner_bytes(ws.rows, a, b, kk);
#pragma unroll
        for (int s = 0; s < NKB_MAX_SURFACES; ++s) {
          if (s >= p.n_surf) break;
          const unsigned cs = case_of(w, s);
          packed |= cs << (8 * s);
          nc += t_ntri[cs];
        }
      }
      int incl = nc;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(full, incl, o);
        if (lane >= o) incl += v;
      }
      const unsigned act = __ballot_sync(full, nc > 0);
      if (nc > 0) {
        const int a = n_act + __popc(act & lt_mask);
        NKB_DCHECK(a >= 0 && a < kNC && c < kNC);
        ws.cell[a] = (unsigned short)c;
        ws.cases[a] = packed;
        ws.off[a] = (unsigned short)(total + incl - nc);
      }
      n_act += __popc(act);
      total += __shfl_sync(full, incl, 31);
    }

    // ---- slots: CTA region (FAST), count (COUNT) or scanned offset (ORDERED) ----
    unsigned long long base = 0;
    if (lane == 0) {
      if (p.mode == FUSED_FAST) {
        base = (unsigned long long)blockIdx.x * (unsigned long long)p.region_cap +
               atomicAdd(&s_fill, (unsigned long long)total);
      } else if (p.mode == FUSED_COUNT) {
        p.elem_count[e] = total;
      } else {
        base = (unsigned long long)p.elem_offset[e];
      }
    }
    base = __shfl_sync(full, base, 0);
    if (p.mode == FUSED_COUNT || total == 0) continue;
    __syncwarp();

    // ---- emit: one lane per active cell ----
    const double* ex = p.x + g0;
    const double* ey = p.y + g0;
    const double* ez = p.z + g0;
    const double* eu = p.vel[0] + g0;
    const double* ev = p.vel[1] + g0;
    const double* ew = p.vel[2] + g0;
    auto value_at = [&](int src, int s, int n) -> double {
      if (src >= SRC_PLANE) return plane_dist(p.surf_n[s], ex[n], ey[n], ez[n]);
      if (src == SRC_UMAG) return mag3(eu[n], ev[n], ew[n]);
      return p.scalar[src - SRC_SCALAR0][g0 + n];
    };
    for (int a = lane; a < n_act; a += 32) {
      const int c = ws.cell[a];
      const unsigned packed = ws.cases[a];
      long long out = (long long)base + ws.off[a];
      const int ca = c % kN, cb = (c / kN) % kN, ck = c / (kN * kN);
      for (int s = 0; s < p.n_surf; ++s) {
        const unsigned cs = (packed >> (8 * s)) & 0xffu;
        const int nt = t_ntri[cs];
        const int src = p.surf_src[s];
        const double iso = p.surf_iso[s];
        for (int k = 0; k < nt; ++k, ++out) {
          const bool over = p.mode == FUSED_FAST ? (out - (long long)blockIdx.x * p.region_cap >= p.region_cap)
                                                 : (out >= p.tri_cap);
          if (over) continue;                          // counted, not written; the host grows and re-runs
          float4 v[3];
#pragma unroll
          for (int r = 0; r < 3; ++r) {
            const int ed = t_tri[cs][3 * k + r];
            const int va = t_edge[ed][0], vb = t_edge[ed][1];
            const int na = (ca + voff_i(va)) + kNP * (cb + voff_j(va)) + kNP * kNP * (ck + voff_k(va));
            const int nb = (ca + voff_i(vb)) + kNP * (cb + voff_j(vb)) + kNP * kNP * (ck + voff_k(vb));
            NKB_DCHECK(na >= 0 && na < kNN && nb >= 0 && nb < kNN && out >= 0 && out < p.tri_cap);
            const double sa = value_at(src, s, na), sb = value_at(src, s, nb);
            const double tv = __ddiv_rn(__dsub_rn(iso, sa), __dsub_rn(sb, sa));
            const double cla = (p.color_src == src) ? sa : (p.color_src >= 0 ? value_at(p.color_src, 0, na) : 0.0);
            const double clb = (p.color_src == src) ? sb : (p.color_src >= 0 ? value_at(p.color_src, 0, nb) : 0.0);
            const double xa = ex[na], ya = ey[na], za = ez[na];
            const double xb = ex[nb], yb = ey[nb], zb = ez[nb];
            v[r].x = __double2float_rn(__fma_rn(tv, __dsub_rn(xb, xa), xa));
            v[r].y = __double2float_rn(__fma_rn(tv, __dsub_rn(yb, ya), ya));
            v[r].z = __double2float_rn(__fma_rn(tv, __dsub_rn(zb, za), za));
            v[r].w = __double2float_rn(__fma_rn(tv, __dsub_rn(clb, cla), cla));
          }
          float4* dst = p.tri + 3 * out;
          dst[0] = v[0];
          dst[1] = v[1];
          dst[2] = v[2];
          if (p.meta)
            p.meta[out] = ((unsigned long long)e << 32) | ((unsigned long long)c << 16) |
                          ((unsigned long long)s << 12) | ((unsigned long long)k << 8) | cs;
        }
      }
    }
    __syncwarp();                                      // ws reused by the next element
  }

  // colour range of every node this CTA streamed: one ordered atomic pair
  if (p.color_src >= 0 && p.mode != FUSED_ORDERED) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      cmin = fmin(cmin, __shfl_xor_sync(full, cmin, o));
      cmax = fmax(cmax, __shfl_xor_sync(full, cmax, o));
    }
    if (lane == 0) {
      s_mn[warp] = cmin;
      s_mx[warp] = cmax;
    }
  }
  __syncthreads();
  if (tid == 0) {
    if (p.color_src >= 0 && p.mode != FUSED_ORDERED) {
      double mn = s_mn[0], mx = s_mx[0];
      for (int w = 1; w < kSWarps; ++w) {
        mn = fmin(mn, s_mn[w]);
        mx = fmax(mx, s_mx[w]);
      }
      if (mn <= mx) {
        atomicMin(&p.counters[1], enc_ordered(mn));
        atomicMax(&p.counters[2], enc_ordered(mx));
      }
    }
    if (p.mode == FUSED_FAST && p.region_count != nullptr) {
      p.region_count[blockIdx.x] = s_fill;
      if (s_fill) atomicAdd(&p.counters[0], s_fill);
    }
  }
}

// block size: the generic program 896 threads (28 warps, <= 72 registers:
// C4 3.90 -> 3.54 ms against 768; 1024 spills), node program 1 1024 threads
// (32 warps, no spills: C4 2.90 -> 2.85 ms against 896);
// NKB_STREAM_THREADS=768 / 896 / 1024 overrides (A/B runs)
static int stream_threads(int prog) {
  const char* v = getenv("NKB_STREAM_THREADS");
  const int n = v ? atoi(v) : (prog == 1 ? 1024 : 896);
  return (n == 768 || n == 1024) ? n : 896;
}

int launch_stream_prepare() {
#define NKB_SP(T, P)                                                                              \
  NKB_CUDA(cudaFuncSetAttribute(stream_kernel<T, P>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                (int)(sizeof(WarpScratch) * (T / 32))))
  NKB_SP(768, 0);
  NKB_SP(896, 0);
  NKB_SP(1024, 0);
  NKB_SP(768, 1);
  NKB_SP(896, 1);
  NKB_SP(1024, 1);
#undef NKB_SP
  return NKB_OK;
}

static bool aligned16(const void* q) { return ((uintptr_t)q & 15u) == 0; }

static StreamFlags stream_flags(const FusedParams& p) {
  StreamFlags fl{0, p.need_umag ? 1 : 0, p.n_scalars};
  for (int i = 0; i < p.n_surf; ++i)
    if (p.surf_src[i] >= SRC_PLANE)
      for (int c = 0; c < 3; ++c) fl.xyz |= (p.surf_n[i][c] != 0.0 ? 1 : 0) << c;
  return fl;
}

// the K1s node program of pipeline `p` (0 = generic)
int stream_prog_of(const FusedParams& p) {
  const char* v = getenv("NKB_NODE_PROGS");             // A/B: NKB_NODE_PROGS=0 forces the generic program
  if (v && v[0] == '0') return 0;
  const StreamFlags fl = stream_flags(p);
  return (p.n_surf == 2 && p.surf_src[0] == SRC_UMAG && p.surf_src[1] >= SRC_PLANE && p.color_src == SRC_UMAG &&
          fl.nsc == 0 && fl.umag) ? 1 : 0;
}


bool stream_eligible(const FusedParams& p) {
  if (p.need_grad || p.q_out || p.wmag_out || p.vort_out) return false;
  const StreamFlags fl = stream_flags(p);
  bool ok = true;
  if (fl.xyz) ok = ok && aligned16(p.x) && aligned16(p.y) && aligned16(p.z);
  if (fl.umag) ok = ok && aligned16(p.vel[0]) && aligned16(p.vel[1]) && aligned16(p.vel[2]);
  for (int c = 0; c < fl.nsc; ++c) ok = ok && aligned16(p.scalar[c]);
  return ok;                                           // else K1 (8-byte staging) handles the fields
}

int launch_stream(const FusedParams& p, int grid, cudaStream_t s) {
  const StreamFlags fl = stream_flags(p);
  const int prog = stream_prog_of(p);
  const int t = stream_threads(prog);
  const size_t sh = sizeof(WarpScratch) * (t / 32);
#define NKB_SL(T, P) stream_kernel<T, P><<<(unsigned)grid, T, sh, s>>>(p, fl)
  if (prog == 1) {
    if (t == 1024) NKB_SL(1024, 1);
    else if (t == 896) NKB_SL(896, 1);
    else NKB_SL(768, 1);
  } else {
    if (t == 1024) NKB_SL(1024, 0);
    else if (t == 896) NKB_SL(896, 0);
    else NKB_SL(768, 0);
  }
#undef NKB_SL
  NKB_CUDA(cudaGetLastError());
  return NKB_OK;
}

NKB_CHECKED_ACCESSOR(checked_read_stream)

}  // namespace nkb
