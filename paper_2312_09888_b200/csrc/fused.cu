// K1: the fused in situ pass -- SEM->VTK adaptor gather, tensor-product
// derivatives, Jacobian inverse, velocity gradient, vorticity, Q-criterion,
// marching-cubes classification of every linear sub-hex and triangle
// emission, in ONE read of the element's GLL fields.
//
// Persistent, warp-specialised: one CTA (512 threads, 16 warps) per SM walks
// the elements e_it = blockIdx.x + it*gridDim.x.  Iteration `it`:
//
//   warps 0-11  (pencils)  : 8-point derivatives of x,y,z | u,v,w along r,s,t
//                            for element it (384 threads x 3 fields)
//   warps 12-15 (MC + DMA) : cp.async prefetch of element it+1 (3-stage ring)
//                            and allocate / emit the triangles of element it-1
//                            (one triangle per thread)
//   ---- barrier ----
//   all 16 warps (nodes)   : one GLL node per thread: Jacobian inverse, grad u,
//                            Q, |w|, |u|, plane distances, case bits, colour range
//   ---- barrier ----
//   all warps (classify)   : one sub-hex per thread: case byte per surface and
//                            triangle count, kept for the MC warps of it+1
//
// The latency-bound MC work runs in the shadow of the FP64-bound pencils;
// the fields of every element are read from HBM exactly once.
//
// Output slots: FAST mode appends each element's triangles to a region of the
// triangle buffer private to the CTA (a shared counter, no global atomics);
// the raster walks the regions, an export compacts them.  Triangle order in
// the buffer therefore depends on the CTA schedule -- the image does not (the
// raster is an order-independent min); inside an element the order is
// (cell, surface, table) always.  Deterministic global order (emit_meta)
// runs COUNT mode, an exclusive scan of the per-element counts, then ORDERED.
//
// Shared memory is XOR-swizzled so node-parallel and r/s/t-pencil accesses
// are bank-conflict free (2 wavefronts per 64-bit warp access).
//
// Reference anchors: the adaptor copy `solver.snapshot_of` (solver.py:282-305)
// and the AoS layout (data_model.py:8-14) for R11; `scalar_field(':mag')`
// (sinks.py:227-242) for the ':mag' formula; the global colour range of
// `render` (sinks.py:264-265).  Rows R12-R14 have no reference
// implementation; the CPU oracle oracle/sem_oracle.c restates
// every floating-point operation below in the same order, so results are
// bit-identical (the library is compiled with -fmad=false; every FMA below is
// an explicit fma()).
#include <cuda_runtime.h>
#include <math.h>
#include <stdlib.h>

#define NKB_MC_NO_HOST_TABLES
#include "mc_tables.h"
#include "checked.cuh"
#include "nkb_internal.h"
#include "sem_dev.cuh"

namespace nkb {

__constant__ double c_D[kNP * kNP];
__constant__ double c_Ae[4][4];   // even half: 0.5*(D[i][m] + D[i][7-m])
__constant__ double c_Ao[4][4];   // odd half:  0.5*(D[i][m] - D[i][7-m])

// MC tables in global memory (read-only path; divergent indices)
__device__ const unsigned char g_mc_ntri[256] = {NKB_MC_NTRI_DATA};
__device__ const signed char g_mc_tri[256][3 * NKB_MC_MAX_TRI] = {NKB_MC_TRI_DATA};
__device__ const unsigned char g_mc_edge_v[12][2] = {NKB_MC_EDGE_V_DATA};

int set_dmat_constant(const double* dmat) {
  NKB_CUDA(cudaMemcpyToSymbol(c_D, dmat, sizeof(double) * kNP * kNP));
  double ae[4][4], ao[4][4];
  for (int i = 0; i < 4; ++i)
    for (int m = 0; m < 4; ++m) {   // host code, -ffp-contract=off (same as the oracle)
      ae[i][m] = 0.5 * (dmat[i * kNP + m] + dmat[i * kNP + (kNP - 1 - m)]);
      ao[i][m] = 0.5 * (dmat[i * kNP + m] - dmat[i * kNP + (kNP - 1 - m)]);
    }
  NKB_CUDA(cudaMemcpyToSymbol(c_Ae, ae, sizeof(ae)));
  NKB_CUDA(cudaMemcpyToSymbol(c_Ao, ao, sizeof(ao)));
  return NKB_OK;
}

namespace {

using namespace dev;

constexpr int kThreads = 512;
constexpr int kPencilThreads = 384;   // 2 groups x 3 dirs x 64 pencils
constexpr int kMcThreads = kThreads - kPencilThreads;   // 128
constexpr int kArr = kNN;             // 512 doubles per staged array
constexpr int kNumD = 18;             // derivative arrays: d(f)/d(r,s,t) for x,y,z,u,v,w
constexpr int kMaxIn = 8;
constexpr int kRing = 3;              // input ring: compute it, emit it-1, prefetch it+1

// node (i,j,k) -> shared-memory slot.  Within each 64 B line the 8 doubles
// are XOR-permuted by (j>>1 | (k&1)<<2); lines are XOR-permuted by (k&1).
// For every 16-lane half-warp pattern used below (node-parallel, r-, s- and
// t-pencils) the 16 accessed doubles fall in 16 distinct 8-byte bank pairs.
__device__ __forceinline__ int sw(int i, int j, int k) {
  return (i ^ ((j >> 1) | ((k & 1) << 2))) + 8 * (j ^ (k & 1)) + 64 * k;
}
__device__ __forceinline__ int sw_node(int n) { return sw(n & 7, (n >> 3) & 7, n >> 6); }


__device__ __forceinline__ void cp_async8(double* smem_dst, const double* gsrc) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async16(double* smem_dst, const double* gsrc) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// mbarrier + bulk (TMA) copy helpers: one elected thread moves a contiguous block
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void bulk_load(void* smem_dst, const void* gsrc, unsigned bytes, unsigned long long* bar) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(d), "l"(gsrc), "r"(bytes), "r"(b) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n"
      ".reg .pred P;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
      "@!P bra WAIT_%=;\n"
      "}\n" ::"r"(b), "r"(parity) : "memory");
}
// barrier among the 4 MC warps only (id 1; id 0 is __syncthreads)
__device__ __forceinline__ void mc_bar() { asm volatile("bar.sync 1, %0;" ::"n"(kMcThreads) : "memory"); }


constexpr int kMaxTriPerElem = kNC * NKB_MC_MAX_TRI * NKB_MAX_SURFACES;   // 6860

// even-odd 8-point derivatives of three staged fields along one pencil
// (oracle deriv8): e_m = v_m + v_{7-m}, o_m = v_m - v_{7-m},
// out[i] = E_i + O_i, out[7-i] = O_i - E_i; each coefficient feeds 3 DFMAs.
// kGeo (coordinate pencils, oracle deriv8_geo): a pencil whose 8 values all
// compare equal (every o_m == 0 and e_0 == e_1 == e_2 == e_3) has derivative
// exactly +0 -- the derivative of a constant -- instead of the rounding
// residue of D applied to it.  Extruded elements then have exact zeros in
// their Jacobian, which jinv's block branch and the compact cache rely on.
template <bool kGeo = false>
__device__ __forceinline__ void pencil3(const double* s0, const double* s1, const double* s2, double* d0,
                                        double* d1, double* d2, const int* off) {
  double e0[4], e1[4], e2[4], o0[4], o1[4], o2[4];
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    const double a0 = s0[off[m]], b0 = s0[off[kNP - 1 - m]];
    const double a1 = s1[off[m]], b1 = s1[off[kNP - 1 - m]];
    const double a2 = s2[off[m]], b2 = s2[off[kNP - 1 - m]];
    e0[m] = __dadd_rn(a0, b0);
    o0[m] = __dsub_rn(a0, b0);
    e1[m] = __dadd_rn(a1, b1);
    o1[m] = __dsub_rn(a1, b1);
    e2[m] = __dadd_rn(a2, b2);
    o2[m] = __dsub_rn(a2, b2);
  }
  bool c0 = false, c1 = false, c2 = false;
  if (kGeo) {
    c0 = o0[0] == 0.0 && o0[1] == 0.0 && o0[2] == 0.0 && o0[3] == 0.0 && e0[0] == e0[1] && e0[0] == e0[2] &&
         e0[0] == e0[3];
    c1 = o1[0] == 0.0 && o1[1] == 0.0 && o1[2] == 0.0 && o1[3] == 0.0 && e1[0] == e1[1] && e1[0] == e1[2] &&
         e1[0] == e1[3];
    c2 = o2[0] == 0.0 && o2[1] == 0.0 && o2[2] == 0.0 && o2[3] == 0.0 && e2[0] == e2[1] && e2[0] == e2[2] &&
         e2[0] == e2[3];
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const double ce = c_Ae[i][0], co = c_Ao[i][0];
    double E0 = __dmul_rn(ce, e0[0]), E1 = __dmul_rn(ce, e1[0]), E2 = __dmul_rn(ce, e2[0]);
    double O0 = __dmul_rn(co, o0[0]), O1 = __dmul_rn(co, o1[0]), O2 = __dmul_rn(co, o2[0]);
#pragma unroll
    for (int m = 1; m < 4; ++m) {
      const double ae = c_Ae[i][m], ao = c_Ao[i][m];
      E0 = __fma_rn(ae, e0[m], E0);
      E1 = __fma_rn(ae, e1[m], E1);
      E2 = __fma_rn(ae, e2[m], E2);
      O0 = __fma_rn(ao, o0[m], O0);
      O1 = __fma_rn(ao, o1[m], O1);
      O2 = __fma_rn(ao, o2[m], O2);
    }
    d0[off[i]] = c0 ? 0.0 : __dadd_rn(E0, O0);
    d1[off[i]] = c1 ? 0.0 : __dadd_rn(E1, O1);
    d2[off[i]] = c2 ? 0.0 : __dadd_rn(E2, O2);
    d0[off[kNP - 1 - i]] = c0 ? 0.0 : __dsub_rn(O0, E0);
    d1[off[kNP - 1 - i]] = c1 ? 0.0 : __dsub_rn(O1, E1);
    d2[off[kNP - 1 - i]] = c2 ? 0.0 : __dsub_rn(O2, E2);
  }
}

__device__ __forceinline__ void pencil_offsets(int dir, int pa, int pb, int* off) {
  if (dir == 0) {
#pragma unroll
    for (int m = 0; m < kNP; ++m) off[m] = sw(m, pa, pb);
  } else if (dir == 1) {
#pragma unroll
    for (int m = 0; m < kNP; ++m) off[m] = sw(pa, m, pb);
  } else {
#pragma unroll
    for (int m = 0; m < kNP; ++m) off[m] = sw(pa, pb, m);
  }
}

// Jacobian inverse d(r,s,t)/d(x,y,z) from the 9 reference derivatives
// G = (xr,xs,xt, yr,ys,yt, zr,zs,zt): cofactors, det, 1/det (oracle order).
// J[3d + b] = d r_d / d x_b.  When xt = yt = zr = zs = 0 exactly (an element
// extruded along t: x, y independent of t and z of r, s -- the coordinate
// pencils of kGeo give exact zeros there), the Jacobian is block diagonal and
// its inverse is taken blockwise (oracle jinv, same branch): the 2x2 block
// [[ys, -xs], [-yr, xr]] / (xr ys - xs yr) and 1/zt, +0 elsewhere.  Its
// entries then depend on (i, j) and on k only, which the compact cache uses.
__device__ __forceinline__ void jinv(const double* G, double* J) {
  const double xr = G[0], xs = G[1], xt = G[2];
  const double yr = G[3], ys = G[4], yt = G[5];
  const double zr = G[6], zs = G[7], zt = G[8];
  if (xt == 0.0 && yt == 0.0 && zr == 0.0 && zs == 0.0) {
    const double r2 = __drcp_rn(__fma_rn(xr, ys, -__dmul_rn(xs, yr)));
    J[0] = __dmul_rn(ys, r2);
    J[1] = __dmul_rn(-xs, r2);
    J[2] = 0.0;
    J[3] = __dmul_rn(-yr, r2);
    J[4] = __dmul_rn(xr, r2);
    J[5] = 0.0;
    J[6] = 0.0;
    J[7] = 0.0;
    J[8] = __drcp_rn(zt);
    return;
  }
  J[0] = __fma_rn(ys, zt, -__dmul_rn(yt, zs));
  J[1] = __fma_rn(xt, zs, -__dmul_rn(xs, zt));
  J[2] = __fma_rn(xs, yt, -__dmul_rn(xt, ys));
  J[3] = __fma_rn(yt, zr, -__dmul_rn(yr, zt));
  J[4] = __fma_rn(xr, zt, -__dmul_rn(xt, zr));
  J[5] = __fma_rn(xt, yr, -__dmul_rn(xr, yt));
  J[6] = __fma_rn(yr, zs, -__dmul_rn(ys, zr));
  J[7] = __fma_rn(xs, zr, -__dmul_rn(xr, zs));
  J[8] = __fma_rn(xr, ys, -__dmul_rn(xs, yr));
  const double det = __fma_rn(zr, J[2], __fma_rn(yr, J[1], __dmul_rn(xr, J[0])));
  const double rdet = __drcp_rn(det);           // == 1.0/det, correctly rounded
#pragma unroll
  for (int c = 0; c < 9; ++c) J[c] = __dmul_rn(J[c], rdet);
}

// compact geometry cache (every element extruded): per element
// kGeoCompactDoubles = 264 doubles, J0, J1, J3, J4 by in-plane node
// ij = i + 8j (4 x 64), then J8 by k (8).  The zeros are the +0 of jinv's
// block branch; the node phase keeps the general 27-FMA chain rule over all
// nine entries, so results are the full layout's bit for bit.
__device__ __forceinline__ void geo_compact_node(const double* g, int n, double* J) {
  const int ij = n & 63, k = n >> 6;
  J[0] = g[ij];
  J[1] = g[64 + ij];
  J[2] = 0.0;
  J[3] = g[128 + ij];
  J[4] = g[192 + ij];
  J[5] = 0.0;
  J[6] = 0.0;
  J[7] = 0.0;
  J[8] = g[256 + k];
}

struct McScratch {
  unsigned cases[2][kNC];       // by element parity: byte s = case of surface s
  unsigned char ntri[2][kNC];   // triangles of each cell (all surfaces)
  unsigned short coff[kNC];     // exclusive triangle offset of each cell
  unsigned short tri_cell[kMaxTriPerElem];   // cell of each triangle of the element
  int wtot[kMcThreads / 32];
  unsigned long long base;
  // marching-cubes tables, copied once per CTA
  unsigned char t_ntri[256];
  signed char t_tri[256][3 * NKB_MC_MAX_TRI];
  unsigned char t_edge[12][2];
};

}  // namespace

// mode: FUSED_FAST / FUSED_COUNT / FUSED_ORDERED (nkb_internal.h)
// kCached: the Jacobian inverse comes from the per-mesh geometry cache
// (p.geo: per element 9 arrays of 512 doubles, 36 KB contiguous) instead of
// x,y,z derivative pencils.  One thread moves element it+1's block into S_geo
// with a single bulk (TMA) copy as soon as the node phase of element it has
// consumed it; the node phase of it+1 waits on the mbarrier.  Warps 0-5 do
// the u,v,w pencils; warps 8-11 stage the next element.
// slot_xyz < 0: x,y,z are not staged (no slice plane; emission reads them via L2).
// kProf (debug, NKB_PROFILE_PHASES=1): lane 0 of warps 0 (pencils), 8
// (staging) and 12 (MC) accumulate clock64 cycles per loop phase.
template <bool kCached, bool kProf>
__global__ void __launch_bounds__(kThreads, 1) fused_kernel(const FusedParams p, int nin, int slot_sc,
                                                            int slot_vel, int slot_xyz) {
  constexpr int kD = kCached ? 9 : kNumD;              // derivative arrays held
  extern __shared__ __align__(16) double smem[];
  double* S_ring = smem;                               // kRing * nin * 512
  double* S_d = S_ring + kRing * nin * kArr;           // kD * 512 derivatives
  double* S_dv = S_d + (kD - 9) * kArr;                // u,v,w derivatives (9 arrays)
  double* S_geo = S_d + kD * kArr;                     // kCached: 9 * 512 d(r,s,t)/d(x,y,z), node order
  double* S_q = S_geo + (kCached ? 9 : 0) * kArr;      // 2 x (Q, |w|) * 512, by element parity
  unsigned char* S_bits = reinterpret_cast<unsigned char*>(S_q + 4 * kArr);   // 512 case bits
  __shared__ McScratch mc;
  __shared__ double s_mn[kThreads / 32], s_mx[kThreads / 32];
  __shared__ unsigned s_band, s_bor;                   // AND / OR of the element's case bits

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const bool is_mc = tid >= kPencilThreads;
  const int t = tid - kPencilThreads;                  // MC-warp thread index
  const long long E = p.n_elements;
  const long long G = gridDim.x;
  const long long n_it = (E > blockIdx.x) ? (E - blockIdx.x + G - 1) / G : 0;
  double cmin = INFINITY, cmax = -INFINITY;
  unsigned long long cta_fill = 0;     // FAST mode: triangles in this CTA's region (MC thread 0)

  // MC warps: coalesced 8-byte cp.async of element `e` into ring slot `b`
  int qn[4];                                          // swizzled slots of my 4 nodes
#pragma unroll
  for (int h = 0; h < 4; ++h) qn[h] = sw_node(t + kMcThreads * h);
  auto prefetch_mc = [&](long long e, int b) {
    double* dst = S_ring + b * nin * kArr;
    const long long g0 = e * (long long)kNN + t;
#pragma unroll
    for (int f = 0; f < kMaxIn; ++f) {
      if (f < nin) {
        const double* src = p.in_ptr[f] + g0;
        double* d = dst + f * kArr;
#pragma unroll
        for (int h = 0; h < 4; ++h) cp_async8(d + qn[h], src + kMcThreads * h);
      }
    }
  };
  // When the pencil warps have slack (cached geometry, or no gradients at
  // all) they stage the next element instead of the MC warps, which are on
  // the critical path: warps 8-11 with cached geometry, warps 0-7 without
  // gradients.
  const bool pw_prefetch = kCached || !p.need_grad;
  const int qp0 = sw_node(tid & 255), qp1 = sw_node((tid & 255) + 256);
  auto prefetch_pw = [&](long long e, int b) {
    double* dst = S_ring + b * nin * kArr;
    const long long g0 = e * (long long)kNN + tid;
#pragma unroll
    for (int f = 0; f < kMaxIn; ++f) {
      if (f < nin) {
        const double* src = p.in_ptr[f] + g0;
        double* d = dst + f * kArr;
        cp_async8(d + qp0, src);
        cp_async8(d + qp1, src + 256);
      }
    }
  };
  int qx[4];
#pragma unroll
  for (int h = 0; h < 4; ++h) qx[h] = sw_node((tid & 127) + kMcThreads * h);
  auto prefetch_w811 = [&](long long e, int b) {
    double* dst = S_ring + b * nin * kArr;
    const long long g0 = e * (long long)kNN + (tid & 127);
#pragma unroll
    for (int f = 0; f < kMaxIn; ++f) {
      if (f < nin) {
        const double* src = p.in_ptr[f] + g0;
        double* d = dst + f * kArr;
#pragma unroll
        for (int h = 0; h < 4; ++h) cp_async8(d + qx[h], src + kMcThreads * h);
      }
    }
  };
  auto prefetch = [&](long long e, int b) {
    if (kCached) {
      if (tid >= 256 && tid < 384) prefetch_w811(e, b);     // warps 8-11; 0-5 do the pencils
    } else if (pw_prefetch) {
      if (tid < 256) prefetch_pw(e, b);
    } else if (is_mc) {
      prefetch_mc(e, b);
    }
  };

  // MC warps: allocate and emit the triangles of element `e` (cases and
  // per-cell counts were classified by all warps at the end of its iteration)
  auto mc_element = [&](long long e, int par, const double* S_in, const double* Sq) {
    int cnt = 0, cc3[3] = {0, 0, 0};
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const int c = 3 * t + j;
      if (c < kNC) {
        cc3[j] = mc.ntri[par][c];
        cnt += cc3[j];
      }
    }
    // exclusive scan over the 128 MC threads (cell-major order)
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    const int mw = warp - kPencilThreads / 32;
    if (lane == 31) mc.wtot[mw] = incl;
    mc_bar();
    int before = 0, total = 0;
#pragma unroll
    for (int w = 0; w < kMcThreads / 32; ++w) {
      const int v = mc.wtot[w];
      before += (w < mw) ? v : 0;
      total += v;
    }
    int run = before + incl - cnt;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const int c = 3 * t + j;
      if (c < kNC) {
        mc.coff[c] = (unsigned short)run;
        for (int q = 0; q < cc3[j]; ++q) mc.tri_cell[run + q] = (unsigned short)c;
        run += cc3[j];
      }
    }
    if (t == 0) {
      unsigned long long base = 0;
      if (p.mode == FUSED_FAST) {
        // CTA-private region of the triangle buffer: no global atomics
        base = (unsigned long long)blockIdx.x * (unsigned long long)p.region_cap + cta_fill;
        cta_fill += (unsigned long long)total;
      } else if (p.mode == FUSED_COUNT) {
        p.elem_count[e] = total;
      } else {
        base = (unsigned long long)p.elem_offset[e];
      }
      mc.base = base;
    }
    mc_bar();
    if (p.mode == FUSED_COUNT || total == 0) return;
    const unsigned long long base = mc.base;
    // slot_xyz < 0 (no slice plane): coordinates are not staged; the few
    // active-cell corners are read through L2 from the global SoA arrays
    const bool xyz_staged = slot_xyz >= 0;
    const double* Sx = xyz_staged ? S_in + slot_xyz * kArr : p.x + e * (long long)kNN;
    const double* Sy = xyz_staged ? S_in + (slot_xyz + 1) * kArr : p.y + e * (long long)kNN;
    const double* Sz = xyz_staged ? S_in + (slot_xyz + 2) * kArr : p.z + e * (long long)kNN;
    const double* Su = S_in + slot_vel * kArr;
    auto value_at = [&](int src, int s, int q) -> double {
      if (src >= SRC_PLANE) return plane_dist(p.surf_n[s], Sx[q], Sy[q], Sz[q]);
      if (src == SRC_Q) return Sq[q];
      if (src == SRC_WMAG) return Sq[kArr + q];
      if (src == SRC_UMAG) return mag3(Su[q], Su[kArr + q], Su[2 * kArr + q]);
      return S_in[(slot_sc + src - SRC_SCALAR0) * kArr + q];
    };
    // triangle slot tt -> (cell, surface, case, table row)
    auto locate = [&](int tt, int& c, int& s, unsigned& cs, int& k) {
      c = mc.tri_cell[tt];
      int li = tt - (int)mc.coff[c];
      const unsigned packed = mc.cases[par][c];
      s = 0;
      cs = packed & 0xffu;
      for (;;) {
        const int nt = mc.t_ntri[cs];
        if (li < nt) break;
        li -= nt;
        ++s;
        cs = (packed >> (8 * s)) & 0xffu;
      }
      k = li;
    };
    auto overflow = [&](long long out) {   // counted, not written; the host grows the buffer and re-runs
      return p.mode == FUSED_FAST ? (out - (long long)blockIdx.x * p.region_cap >= p.region_cap)
                                  : (out >= p.tri_cap);
    };
    auto vertex = [&](int c, int s, unsigned cs, int k, int r) -> float4 {
      const int ca = c % kN, cb = (c / kN) % kN, ck = c / (kN * kN);
      const int src = p.surf_src[s];
      const double iso = p.surf_iso[s];
      const int ed = mc.t_tri[cs][3 * k + r];
      const int va = mc.t_edge[ed][0], vb = mc.t_edge[ed][1];
      const int ia = ca + voff_i(va), ja = cb + voff_j(va), ka = ck + voff_k(va);
      const int ib = ca + voff_i(vb), jb = cb + voff_j(vb), kb = ck + voff_k(vb);
      const int qa = sw(ia, ja, ka), qb = sw(ib, jb, kb);
      const double sa = value_at(src, s, qa), sb = value_at(src, s, qb);
      const double tv = __ddiv_rn(__dsub_rn(iso, sa), __dsub_rn(sb, sa));
      const double cla = value_at(p.color_src, 0, qa), clb = value_at(p.color_src, 0, qb);
      const int pa = xyz_staged ? qa : ia + kNP * ja + kNP * kNP * ka;
      const int pb = xyz_staged ? qb : ib + kNP * jb + kNP * kNP * kb;
      const double xa = Sx[pa], ya = Sy[pa], za = Sz[pa];
      const double xb = Sx[pb], yb = Sy[pb], zb = Sz[pb];
      float4 v;
      v.x = __double2float_rn(__fma_rn(tv, __dsub_rn(xb, xa), xa));
      v.y = __double2float_rn(__fma_rn(tv, __dsub_rn(yb, ya), ya));
      v.z = __double2float_rn(__fma_rn(tv, __dsub_rn(zb, za), za));
      v.w = __double2float_rn(__fma_rn(tv, __dsub_rn(clb, cla), cla));
      return v;
    };
    auto put_meta = [&](long long out, int c, int s, int k, unsigned cs) {
      if (p.meta)
        p.meta[out] = ((unsigned long long)e << 32) | ((unsigned long long)c << 16) |
                      ((unsigned long long)s << 12) | ((unsigned long long)k << 8) | cs;
    };
    if (3 * total <= kMcThreads) {
      // small element (the common case): one task per triangle VERTEX -- one
      // pass with a third of the dependent chain, consecutive float4 stores
      if (t < 3 * total) {
        const int tt = t / 3, r = t - 3 * tt;
        int c, s, k;
        unsigned cs;
        locate(tt, c, s, cs, k);
        const long long out = (long long)base + tt;
        if (!overflow(out)) {
          p.tri[3 * out + r] = vertex(c, s, cs, k, r);
          if (r == 0) put_meta(out, c, s, k, cs);
        }
      }
    } else {
      for (int tt = t; tt < total; tt += kMcThreads) {
        int c, s, k;
        unsigned cs;
        locate(tt, c, s, cs, k);
        const long long out = (long long)base + tt;
        if (overflow(out)) continue;
        float4 v[3];
#pragma unroll
        for (int r = 0; r < 3; ++r) v[r] = vertex(c, s, cs, k, r);
        float4* dst = p.tri + 3 * out;
        dst[0] = v[0];
        dst[1] = v[1];
        dst[2] = v[2];
        put_meta(out, c, s, k, cs);
      }
    }
  };

  for (int i = tid; i < 256; i += kThreads) mc.t_ntri[i] = g_mc_ntri[i];
  for (int i = tid; i < 256 * 3 * NKB_MC_MAX_TRI; i += kThreads) (&mc.t_tri[0][0])[i] = (&g_mc_tri[0][0])[i];
  if (tid < 24) (&mc.t_edge[0][0])[tid] = (&g_mc_edge_v[0][0])[tid];
  if (n_it > 0) prefetch(blockIdx.x, 0);
  __shared__ unsigned long long s_geo_bar;
  // geometry block per element: full (36 KB) or compact (2112 B)
  const long long geo_stride = p.geo_compact ? kGeoCompactDoubles : 9 * kNN;
  const unsigned geo_bytes = (unsigned)(geo_stride * sizeof(double));
  if (kCached && tid == 0) {
    mbar_init(&s_geo_bar, 1);
    if (n_it > 0) bulk_load(S_geo, p.geo + (long long)blockIdx.x * geo_stride, geo_bytes, &s_geo_bar);
  }
  cp_async_commit();
  int cls_any = 0;                                     // my sub-hex of the last element emits triangles
  long long pacc[6] = {0, 0, 0, 0, 0, 0}, pt = kProf ? clock64() : 0;
  auto tick = [&](int ph) {
    if (kProf) {
      const long long now = clock64();
      pacc[ph] += now - pt;
      pt = now;
    }
  };
  for (long long it = 0; it <= n_it; ++it) {
    const long long e = blockIdx.x + it * G;
    const int slot = (int)(it % kRing);
    const int par = (int)(it & 1);
    cp_async_wait_all();                               // my share of element `it` landed
    // element `it` staged; node phase it-1 done; does element it-1 emit anything?
    const int prev_emits = __syncthreads_or(cls_any);
    tick(0);
    cls_any = 0;
    if (tid == 0) {                                    // read by everyone before the barrier above
      s_band = ~0u;
      s_bor = 0u;
    }
    const double* S_in = S_ring + slot * nin * kArr;
    if (it + 1 < n_it) prefetch(e + G, (int)((it + 1) % kRing));
    cp_async_commit();
    if (is_mc) {
      if (it > 0 && p.n_surf > 0 && !prev_emits) {
        if (p.mode == FUSED_COUNT && t == 0) p.elem_count[e - G] = 0;   // empty element: skip the scan
      } else if (it > 0 && p.n_surf > 0) {
        const int ps = (int)((it - 1) % kRing), pp = (int)((it - 1) & 1);
        mc_element(e - G, pp, S_ring + ps * nin * kArr, S_q + pp * 2 * kArr);
      }
    } else if (it < n_it && p.need_grad) {
      // ---- pencils: thread = (group, dir, pencil); 3 fields share offsets ----
      const int g = tid / 192;                      // warp-uniform
      const int dir = (tid % 192) >> 6;             // warp-uniform
      int off[kNP];
      pencil_offsets(dir, tid & 7, (tid >> 3) & 7, off);
      if (kCached) {
        // u,v,w only, on warps 0-5 (warps 8-11 stage the next element)
        if (g == 0) {
          const double* su = S_in + slot_vel * kArr;
          double* d0 = S_dv + dir * kArr;
          pencil3(su, su + kArr, su + 2 * kArr, d0, d0 + 3 * kArr, d0 + 6 * kArr, off);
        }
      } else {
        // g = 0: x,y,z (constant-pencil rule)   1: u,v,w
        const int sf = (g == 0) ? slot_xyz : slot_vel;
        if (g == 0)
          pencil3<true>(S_in + (sf + 0) * kArr, S_in + (sf + 1) * kArr, S_in + (sf + 2) * kArr,
                        S_d + (3 * (3 * g + 0) + dir) * kArr, S_d + (3 * (3 * g + 1) + dir) * kArr,
                        S_d + (3 * (3 * g + 2) + dir) * kArr, off);
        else
          pencil3(S_in + (sf + 0) * kArr, S_in + (sf + 1) * kArr, S_in + (sf + 2) * kArr,
                  S_d + (3 * (3 * g + 0) + dir) * kArr, S_d + (3 * (3 * g + 1) + dir) * kArr,
                  S_d + (3 * (3 * g + 2) + dir) * kArr, off);
      }
    }
    if (it == n_it) break;
    tick(1);
    if (kCached) mbar_wait(&s_geo_bar, (unsigned)(it & 1));   // geometry of element `it` landed
    __syncthreads();                                   // derivatives of element `it` ready
    tick(2);

    // ---- node phase: one node per thread ----
    {
      const int n = tid;
      const int q = sw_node(n);
      const long long g0 = e * (long long)kNN;
      double* Sq = S_q + par * 2 * kArr;
      unsigned char* bits_out = S_bits;
      double vq = 0.0, vw = 0.0, vu = 0.0;
      if (p.need_grad) {
        double J[9];
        if (kCached && p.geo_compact) {
          geo_compact_node(S_geo, n, J);
        } else if (kCached) {
#pragma unroll
          for (int c = 0; c < 9; ++c) J[c] = S_geo[c * kArr + n];
        } else {
          double G9[9];
#pragma unroll
          for (int c = 0; c < 9; ++c) G9[c] = S_d[c * kArr + q];
          jinv(G9, J);
        }
        double U[9];
#pragma unroll
        for (int c = 0; c < 9; ++c) U[c] = S_dv[c * kArr + q];
        double A[9];
        chain_rule(U, J, A);
        const double off = __fma_rn(A[5], A[7], __fma_rn(A[2], A[6], __dmul_rn(A[1], A[3])));
        const double dia = __fma_rn(A[8], A[8], __fma_rn(A[4], A[4], __dmul_rn(A[0], A[0])));
        vq = -__fma_rn(0.5, dia, off);
        const double om0 = __dsub_rn(A[7], A[5]);
        const double om1 = __dsub_rn(A[2], A[6]);
        const double om2 = __dsub_rn(A[3], A[1]);
        Sq[q] = vq;
        if (p.need_wmag) {
          vw = mag3(om0, om1, om2);
          Sq[kArr + q] = vw;
        }
        if (p.q_out) p.q_out[g0 + n] = vq;
        if (p.wmag_out) p.wmag_out[g0 + n] = vw;
        if (p.vort_out) {
          p.vort_out[3 * (g0 + n) + 0] = om0;
          p.vort_out[3 * (g0 + n) + 1] = om1;
          p.vort_out[3 * (g0 + n) + 2] = om2;
        }
      }
      if (p.need_umag) vu = mag3(S_in[slot_vel * kArr + q], S_in[(slot_vel + 1) * kArr + q], S_in[(slot_vel + 2) * kArr + q]);
      unsigned bits = 0;
#pragma unroll
      for (int s = 0; s < NKB_MAX_SURFACES; ++s) {
        if (s >= p.n_surf) break;
        const int src = p.surf_src[s];
        double val;
        if (src >= SRC_PLANE)
          val = plane_dist(p.surf_n[s], S_in[slot_xyz * kArr + q], S_in[(slot_xyz + 1) * kArr + q],
                           S_in[(slot_xyz + 2) * kArr + q]);
        else if (src == SRC_Q) val = vq;
        else if (src == SRC_WMAG) val = vw;
        else if (src == SRC_UMAG) val = vu;
        else val = S_in[(slot_sc + src - SRC_SCALAR0) * kArr + q];
        bits |= (val >= p.surf_iso[s] ? 1u : 0u) << s;
      }
      bits_out[n] = (unsigned char)bits;
      {
        // per-warp AND / OR of the case bits: an element whose nodes all sit
        // on one side of every surface emits nothing and skips classification
        const unsigned wa = __reduce_and_sync(0xffffffffu, bits), wo = __reduce_or_sync(0xffffffffu, bits);
        if (lane == 0) {
          atomicAnd(&s_band, wa);
          atomicOr(&s_bor, wo);
        }
      }
      if (p.color_src >= 0) {
        const int src = p.color_src;
        const double c = (src == SRC_Q)      ? vq
                         : (src == SRC_WMAG) ? vw
                         : (src == SRC_UMAG) ? vu
                                             : S_in[(slot_sc + src - SRC_SCALAR0) * kArr + q];
        cmin = fmin(cmin, c);
        cmax = fmax(cmax, c);
      }
    }
    tick(3);
    if (p.n_surf == 0 && !kCached) continue;
    __syncthreads();                                   // case bits of element `it` ready
    tick(4);
    if (kCached && tid == 0 && it + 1 < n_it)          // S_geo consumed: fetch element it+1
      bulk_load(S_geo, p.geo + (e + G) * geo_stride, geo_bytes, &s_geo_bar);
    if (p.n_surf == 0) continue;
    if ((s_bor & ~s_band) == 0) continue;               // no surface crosses this element

    // ---- classify: one sub-hex per thread (all warps) ----
    if (tid < kNC) {
      const int c = tid;
      const int a = c % kN, b = (c / kN) % kN, k = c / (kN * kN);
      // the 8 corner bytes in VTK order from 4 node rows (8 bytes each):
      // row(b,k) -> v0 v1, row(b+1,k) -> v3 v2, row(b,k+1) -> v4 v5, row(b+1,k+1) -> v7 v6
      const unsigned long long* rows = reinterpret_cast<const unsigned long long*>(S_bits);
      const int sh = 8 * a;
      const unsigned r00 = (unsigned)(rows[b + kNP * k] >> sh), r10 = (unsigned)(rows[b + 1 + kNP * k] >> sh);
      const unsigned r01 = (unsigned)(rows[b + kNP * (k + 1)] >> sh);
      const unsigned r11 = (unsigned)(rows[b + 1 + kNP * (k + 1)] >> sh);
      const unsigned long long w = (unsigned long long)__byte_perm(r00, r10, 0x4510) |
                                   ((unsigned long long)__byte_perm(r01, r11, 0x4510) << 32);
      unsigned packed = 0;
      int nc = 0;
#pragma unroll
      for (int s = 0; s < NKB_MAX_SURFACES; ++s) {
        if (s >= p.n_surf) break;
        const unsigned cs = case_of(w, s);
        packed |= cs << (8 * s);
        nc += mc.t_ntri[cs];
      }
      mc.cases[par][c] = packed;
      mc.ntri[par][c] = (unsigned char)nc;
      cls_any = nc;
    }
    tick(5);
  }
  if (kProf && lane == 0 && (warp == 0 || warp == 8 || warp == 12)) {
    const int role = warp == 0 ? 0 : (warp == 8 ? 1 : 2);
#pragma unroll
    for (int ph = 0; ph < 6; ++ph) atomicAdd(p.prof + 6 * role + ph, (unsigned long long)pacc[ph]);
  }

  if (p.mode == FUSED_FAST && p.region_count != nullptr && tid == kPencilThreads) {
    p.region_count[blockIdx.x] = cta_fill;
    if (cta_fill) atomicAdd(&p.counters[0], cta_fill);
  }
  // colour range of all elements this CTA processed: one ordered atomic pair
  if (p.color_src >= 0 && p.mode != FUSED_ORDERED) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      cmin = fmin(cmin, __shfl_xor_sync(0xffffffffu, cmin, o));
      cmax = fmax(cmax, __shfl_xor_sync(0xffffffffu, cmax, o));
    }
    if (lane == 0) {
      s_mn[warp] = cmin;
      s_mx[warp] = cmax;
    }
    __syncthreads();
    if (tid == 0) {
      double mn = s_mn[0], mx = s_mx[0];
      for (int w = 1; w < kThreads / 32; ++w) {
        mn = fmin(mn, s_mn[w]);
        mx = fmax(mx, s_mx[w]);
      }
      if (mn <= mx) {
        atomicMin(&p.counters[1], enc_ordered(mn));
        atomicMax(&p.counters[2], enc_ordered(mx));
      }
    }
  }
}

// exclusive scan of per-element triangle counts (ordered mode); single CTA
__global__ void __launch_bounds__(1024) count_scan_kernel(const int* __restrict__ cnt, long long n,
                                                          long long* __restrict__ off,
                                                          unsigned long long* __restrict__ total) {
  __shared__ long long s_w[32];
  __shared__ long long s_carry;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_carry = 0;
  __syncthreads();
  for (long long base = 0; base < n; base += 1024) {
    const long long i = base + tid;
    const long long v = (i < n) ? cnt[i] : 0;
    long long x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_w[warp] = x;
    __syncthreads();
    if (warp == 0) {
      long long w = s_w[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const long long y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      s_w[lane] = w;
    }
    __syncthreads();
    const long long carry = s_carry;
    const long long excl = carry + (warp ? s_w[warp - 1] : 0) + x - v;
    if (i < n) off[i] = excl;
    __syncthreads();
    if (tid == 1023) s_carry = excl + v;
    __syncthreads();
  }
  if (tid == 0) *total = (unsigned long long)s_carry;
}

static int g_num_sms = 0;

int fused_grid(int64_t n_elements, int sm_reserve) {
  if (g_num_sms <= 0) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      g_num_sms = 148;
  }
  int64_t g = g_num_sms - (sm_reserve > 0 && sm_reserve < g_num_sms / 2 ? sm_reserve : 0);
  if (g > n_elements) g = n_elements;
  return (int)(g < 1 ? 1 : g);
}

// gather the CTA regions of a FAST-mode run into one contiguous array
__global__ void compact_kernel(const float4* __restrict__ tri, const unsigned long long* __restrict__ meta,
                               const unsigned long long* __restrict__ region_count, int n_regions,
                               long long region_cap, float4* __restrict__ out_tri,
                               unsigned long long* __restrict__ out_meta) {
  const int r = blockIdx.y;
  long long dst0 = 0;
  for (int i = 0; i < r; ++i) dst0 += (long long)min(region_count[i], (unsigned long long)region_cap);
  const long long n = (long long)min(region_count[r], (unsigned long long)region_cap);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long src = r * region_cap + i;
    out_tri[3 * (dst0 + i) + 0] = tri[3 * src + 0];
    out_tri[3 * (dst0 + i) + 1] = tri[3 * src + 1];
    out_tri[3 * (dst0 + i) + 2] = tri[3 * src + 2];
    if (meta && out_meta) out_meta[dst0 + i] = meta[src];
  }
}

int launch_compact(const float4* tri, const unsigned long long* meta, const unsigned long long* region_count,
                   int n_regions, int64_t region_cap, float4* out_tri, unsigned long long* out_meta,
                   int64_t n_total, cudaStream_t s) {
  if (n_regions <= 0 || n_total <= 0) return NKB_OK;
  compact_kernel<<<dim3(8, n_regions), 256, 0, s>>>(tri, meta, region_count, n_regions, region_cap, out_tri,
                                                    out_meta);
  NKB_CUDA(cudaGetLastError());
  return NKB_OK;
}

// ---- per-mesh geometry cache: d(r,s,t)/d(x,y,z) at every GLL node ----
// Same pencil3<true>/jinv code as the uncached fused kernel, so the cached
// values are bit-identical to what the fused kernel would recompute each step.
// Full layout (`full`): per element 9 arrays of 512 doubles (component c of
// node n of element e at geo[(9e + c) * 512 + n]), one 36 KB block per
// element.  Compact layout (`compact`, kGeoCompactDoubles doubles per element): the
// element's J0, J1, J3, J4 on the k = 0 plane and J8 along k; an element
// whose values do not have that structure (not extruded, so jinv took the
// general branch somewhere, or an entry varies where it must not) adds 1 to
// *n_general -- the host then builds the full layout instead.
__global__ void __launch_bounds__(kNN) geometry_kernel(const double* __restrict__ x, const double* __restrict__ y,
                                                       const double* __restrict__ z, long long E, double* full,
                                                       double* compact, unsigned long long* n_general) {
  __shared__ double S[12 * kArr];                  // x,y,z + 9 derivatives (48 KB); then J (node order)
  const int tid = threadIdx.x;
  const int q = sw_node(tid);
  for (long long e = blockIdx.x; e < E; e += gridDim.x) {
    const long long g = e * (long long)kNN + tid;
    S[q] = x[g];
    S[kArr + q] = y[g];
    S[2 * kArr + q] = z[g];
    __syncthreads();
    if (tid < 192) {
      const int dir = tid >> 6;
      int off[kNP];
      pencil_offsets(dir, tid & 7, (tid >> 3) & 7, off);
      double* D = S + 3 * kArr;
      pencil3<true>(S, S + kArr, S + 2 * kArr, D + dir * kArr, D + (3 + dir) * kArr, D + (6 + dir) * kArr, off);
    }
    __syncthreads();
    double G9[9], J[9];
#pragma unroll
    for (int c = 0; c < 9; ++c) G9[c] = S[(3 + c) * kArr + q];
    jinv(G9, J);
    if (full) {
#pragma unroll
      for (int c = 0; c < 9; ++c) full[(e * 9 + c) * kNN + tid] = J[c];
    }
    if (compact) {
      __syncthreads();                             // S is reused for J in node order
      const int cs[5] = {0, 1, 3, 4, 8};
#pragma unroll
      for (int u = 0; u < 5; ++u) S[u * kArr + tid] = J[cs[u]];
      __syncthreads();
      const int ij = tid & 63, k = tid >> 6;
      const auto bits = [](double v) { return __double_as_longlong(v); };
      bool ok = bits(J[2]) == 0 && bits(J[5]) == 0 && bits(J[6]) == 0 && bits(J[7]) == 0;
#pragma unroll
      for (int u = 0; u < 4; ++u) ok = ok && bits(S[u * kArr + ij]) == bits(J[cs[u]]);
      ok = ok && bits(S[4 * kArr + 64 * k]) == bits(J[8]);
      const int all_ok = __syncthreads_and(ok);
      double* dst = compact + e * kGeoCompactDoubles;
      if (tid < 256) dst[tid] = S[(tid >> 6) * kArr + (tid & 63)];
      else if (tid < 264) dst[tid] = S[4 * kArr + 64 * (tid - 256)];
      if (tid == 0 && !all_ok) atomicAdd(n_general, 1ULL);
    }
    __syncthreads();
  }
}

int launch_geometry(const double* x, const double* y, const double* z, int64_t E, double* full, double* compact,
                    unsigned long long* n_general, cudaStream_t s) {
  if (E <= 0) return NKB_OK;
  const long long grid = E < 148LL * 64 ? E : 148LL * 64;
  geometry_kernel<<<(unsigned)grid, kNN, 0, s>>>(x, y, z, (long long)E, full, compact, n_general);
  NKB_CUDA(cudaGetLastError());
  return NKB_OK;
}


// A/B switch (NKB_EMIT_PREFETCH=0): L2 prefetch of an emitting element's coordinates in K1g
__constant__ int g_emit_prefetch = 1;
__constant__ int g_emit_stage = 1;          // K1g: an emitting element's x,y,z copied into dead S_dv space

// ---- node programs: compile-time surface / colour sources of a pipeline ----
// The node phase's per-surface source dispatch (Q, |w|, |u|, a staged scalar
// or a plane distance, chosen per node from runtime codes) cost as many
// instructions as the velocity gradient itself (ncu, C2).  A node program
// fixes the source kind of every surface and of the colour at compile time;
// only the scalar slots, iso values and plane normals stay runtime.  Program 0
// is the generic runtime dispatch and runs every other pipeline.  The values
// and their operation order are the generic path's, so results are identical.
enum NodeKind : int { NK_NONE = 0, NK_Q, NK_W, NK_U, NK_SC, NK_PL };
struct NodeProg {
  int s[NKB_MAX_SURFACES];
  int c;
};
__host__ __device__ constexpr NodeProg node_prog(int k) {
  return k == 1   ? NodeProg{{NK_Q, NK_NONE, NK_NONE, NK_NONE}, NK_U}      // Q iso, colour |u|
         : k == 2 ? NodeProg{{NK_Q, NK_NONE, NK_NONE, NK_NONE}, NK_W}      // Q iso, colour |w|
         : k == 3 ? NodeProg{{NK_Q, NK_NONE, NK_NONE, NK_NONE}, NK_SC}     // Q iso, colour by a scalar
         : k == 4 ? NodeProg{{NK_SC, NK_Q, NK_PL, NK_NONE}, NK_SC}         // scalar iso + Q iso + slice, colour scalar
                  : NodeProg{{NK_NONE, NK_NONE, NK_NONE, NK_NONE}, NK_NONE};
}
constexpr int kNodeProgs = 5;
__host__ __device__ constexpr bool prog_uses(int k, int kind) {
  return node_prog(k).c == kind || node_prog(k).s[0] == kind || node_prog(k).s[1] == kind ||
         node_prog(k).s[2] == kind || node_prog(k).s[3] == kind;
}

static int node_kind_of(int src) {
  return src < 0             ? NK_NONE
         : src >= SRC_PLANE  ? NK_PL
         : src == SRC_Q      ? NK_Q
         : src == SRC_WMAG   ? NK_W
         : src == SRC_UMAG   ? NK_U
                             : NK_SC;
}

// the node program that runs pipeline `p` in K1g (0 = generic)
static int node_prog_of(const FusedParams& p) {
  const char* v = getenv("NKB_NODE_PROGS");            // A/B: NKB_NODE_PROGS=0 forces the generic program
  if (v && v[0] == '0') return 0;
  if (p.q_out || p.wmag_out || p.vort_out) return 0;
  for (int k = 1; k < kNodeProgs; ++k) {
    const NodeProg P = node_prog(k);
    bool ok = P.c == node_kind_of(p.color_src);
    for (int s = 0; s < NKB_MAX_SURFACES; ++s)
      ok = ok && P.s[s] == (s < p.n_surf ? node_kind_of(p.surf_src[s]) : NK_NONE);
    // |w| / |u| computed exactly when the program uses them
    ok = ok && (p.need_wmag != 0) == prog_uses(k, NK_W) && (p.need_umag != 0) == prog_uses(k, NK_U);
    if (ok) return k;
  }
  return 0;
}


// ---- K1g: the cached-geometry gradient pass, 2-3 independent CTAs per SM ----
// K1 runs one 512-thread CTA per SM whose phases (pencils | node | classify |
// emit) are serialised by CTA-wide barriers; its phase profile shows the SM
// waiting at them.  K1g runs two (or three, kOcc) 256-thread CTAs per SM,
// each owning one element at a time start to finish, so one CTA's barrier
// waits and load latency are covered by the others' work:
//   - inputs double-buffered (cp.async, 8 B per node, the swizzled layout of
//     K1), issued by warps 6-7 while warps 0-5 run the pencils; with the
//     compact cache the element's 2112-byte J^-1 block is staged alongside
//     (full cache: J^-1 read per node from global memory, pulled toward L2 one
//     element ahead by a bulk prefetch);
//   - u,v,w pencils on 192 threads (pencil3 of K1), then 2 nodes per thread
//     (node programs: compile-time sources, see node_prog), then
//     classification (2 sub-hexes per thread), one block scan of packed
//     (triangle, active-cell) counts, and emission with one task per triangle
//     vertex over all 256 threads -- all inside the element's iteration;
//   - three CTAs per SM when a CTA fits in 75 KB of shared memory (compact
//     cache, <= 3 staged arrays: C1, C3, C5) and 85 registers.  (C2 stages
//     5 arrays; reading its scalar and slice coordinate per node from global
//     memory instead, to fit three CTAs, was slower: 0.270 -> 0.309 ms.)
// Every value is computed by K1's device functions in K1's order, so the
// results are bit-identical to K1 and to the oracle.
constexpr int kG2Threads = 256;
constexpr int kG2MaxIn = 7;                 // 2 CTAs/SM of (2*nin + 11) * 4 KB shared memory

// static shared scratch of K1g; the per-element active-cell lists live in the
// derivative arrays' space (dead once the node phase has read them) and the
// triangle table is read through L1 (g_mc_tri), which keeps a CTA at <= 75 KB
// so that three fit on an SM when the staging is small (kOcc = 3)
struct G2Scratch {
  unsigned char t_ntri[256];
  unsigned char t_edge[12][2];
  int wsum[kG2Threads / 32];
  unsigned long long base;
  unsigned band, bor;
};

__device__ __forceinline__ void l2_prefetch(const void* g, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(g), "r"(bytes) : "memory");
}

// kCompact: the compact geometry cache (2112 B per element) is staged with
// the fields into shared memory; otherwise J^-1 is read from the full cache.
// kWmag: |vorticity| is used (surface, colour or export); kOut: some derived
// array is exported (q_out / wmag_out / vort_out).  Both are compile-time so
// the node phase carries no dead work for the common pipelines.
// kProg: node program (0 = generic runtime dispatch).
// kOcc: CTAs per SM the registers are budgeted for (2, or 3 for compact
// pipelines staging <= 3 arrays).
// kTma (A/B of the staging, NKB_K1G_TMA=1): the element's field arrays and
// J^-1 block arrive by TMA bulk copies (cp.async.bulk, one per 4 KB array,
// completion on an mbarrier per ring buffer) in natural node order instead of
// 8-byte cp.async into the XOR-swizzled layout; pencils, node phase and
// emission then index shared memory naturally.
template <bool kCompact, bool kWmag, bool kOut, int kProg, int kOcc, bool kTma = false>
__global__ void __launch_bounds__(kG2Threads, kOcc) fused2_kernel(const FusedParams p, int nin, int slot_sc,
                                                                 int slot_vel, int slot_xyz, int plane_slots) {
  extern __shared__ __align__(16) double smem[];
  double* S_ring = smem;                               // 2 * nin * 512
  double* S_dv = S_ring + 2 * nin * kArr;              // 9 * 512 u,v,w derivatives
  double* S_q = S_dv + 9 * kArr;                       // Q (and |w| with kWmag), swizzled
  // node programs colouring (or isosurfacing) by |u| keep it per node for the
  // emission: one load per corner instead of three loads and a square root
  constexpr bool kStoreU = prog_uses(kProg, NK_U);
  double* S_u = S_q + (kWmag ? 2 : 1) * kArr;          // kStoreU: |u| (swizzled)
  double* S_gc = S_u + (kStoreU ? 1 : 0) * kArr;       // kCompact: 2 x kGeoCompactDoubles
  // active-cell lists of the element being emitted: in S_dv's space, free
  // between the node-phase barrier and the next iteration's pencils
  unsigned* act_cases = reinterpret_cast<unsigned*>(S_dv);
  unsigned short* act_cell = reinterpret_cast<unsigned short*>(act_cases + kNC);
  unsigned short* act_off = act_cell + kNC;
  // triangle tt of the element -> its active cell (<= kMaxTriPerElem entries, 13.7 KB, also in S_dv's space)
  unsigned short* tri_act = act_off + kNC;
  unsigned char* S_bits = reinterpret_cast<unsigned char*>(S_gc + (kCompact ? 2 * kGeoCompactDoubles : 0));
  __shared__ G2Scratch mc;
  __shared__ double s_mn[kG2Threads / 32], s_mx[kG2Threads / 32];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long E = p.n_elements;
  const long long G = gridDim.x;
  const long long n_it = (E > blockIdx.x) ? (E - blockIdx.x + G - 1) / G : 0;
  double cmin = INFINITY, cmax = -INFINITY;
  unsigned long long cta_fill = 0;
  constexpr unsigned kGeoBytes = 9u * kNN * sizeof(double);

  for (int i = tid; i < 256; i += kG2Threads) mc.t_ntri[i] = g_mc_ntri[i];
  if (tid < 24) (&mc.t_edge[0][0])[tid] = (&g_mc_edge_v[0][0])[tid];

  const int q0 = kTma ? tid : sw_node(tid), q1 = kTma ? tid + kG2Threads : sw_node(tid + kG2Threads);
  // staging of the next element by warps 6-7 (idle during the u,v,w pencils):
  // 64 threads x 8 nodes per field, coalesced 8-byte cp.async
  int qs[8];
#pragma unroll
  for (int h = 0; h < 8; ++h) qs[h] = sw_node((tid & 63) + 64 * h);
  __shared__ unsigned long long s_tma_bar[2];
  if (kTma && tid == 192) {
    mbar_init(&s_tma_bar[0], 1);
    mbar_init(&s_tma_bar[1], 1);
  }
  if (kTma) __syncthreads();
  auto prefetch_tma = [&](long long e, int b) {      // one thread: nin + 1 bulk copies, one mbarrier
    if (tid != 192) return;
    double* dst = S_ring + b * nin * kArr;
    unsigned long long* bar = &s_tma_bar[b];
    const unsigned total = (unsigned)(nin * kArr * sizeof(double) + (kCompact ? kGeoCompactDoubles * sizeof(double) : 0));
    const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    // the buffer was last read through the generic proxy (previous element)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(total) : "memory");
    for (int f = 0; f < nin; ++f) {
      const unsigned d = (unsigned)__cvta_generic_to_shared(dst + f * kArr);
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(d), "l"(p.in_ptr[f] + e * (long long)kNN), "r"((unsigned)(kArr * sizeof(double))), "r"(a)
                   : "memory");
    }
    if (kCompact) {
      const unsigned d = (unsigned)__cvta_generic_to_shared(S_gc + b * kGeoCompactDoubles);
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(d), "l"(p.geo + e * kGeoCompactDoubles), "r"((unsigned)(kGeoCompactDoubles * sizeof(double))),
                   "r"(a)
                   : "memory");
    }
  };
  auto prefetch = [&](long long e, int b) {
    if (kTma) {
      prefetch_tma(e, b);
      return;
    }
    double* dst = S_ring + b * nin * kArr;
    const long long g0 = e * (long long)kNN + (tid & 63);
#pragma unroll
    for (int f = 0; f < kG2MaxIn; ++f) {
      if (f < nin) {
        const double* src = p.in_ptr[f] + g0;
        double* d = dst + f * kArr;
#pragma unroll
        for (int h = 0; h < 8; ++h) {
          NKB_DCHECK(qs[h] >= 0 && qs[h] < kArr && e >= 0 && e < E && f < nin && (b == 0 || b == 1));
          cp_async8(d + qs[h], src + 64 * h);
        }
      }
    }
    if (kCompact) {                                    // the element's compact J^-1 block
      const double* src = p.geo + e * kGeoCompactDoubles;
      double* d = S_gc + b * kGeoCompactDoubles;
#pragma unroll
      for (int h = 0; h < 5; ++h) {
        const int i = (tid & 63) + 64 * h;
        if (i < kGeoCompactDoubles) cp_async8(d + i, src + i);
      }
    }
  };
  if (n_it > 0) {
    if (tid >= 192) prefetch(blockIdx.x, 0);
    if (!kCompact && tid == 0) l2_prefetch(p.geo + (long long)blockIdx.x * 9 * kNN, kGeoBytes);
  }
  cp_async_commit();

  int off[kNP];                                        // pencil offsets (threads < 192)
  pencil_offsets(tid >> 6 < 3 ? tid >> 6 : 0, tid & 7, (tid >> 3) & 7, off);
  if (kTma) {                                          // natural node order
    const int dir = tid >> 6 < 3 ? tid >> 6 : 0, pa = tid & 7, pb = (tid >> 3) & 7;
#pragma unroll
    for (int m = 0; m < kNP; ++m)
      off[m] = dir == 0 ? m + 8 * pa + 64 * pb : dir == 1 ? pa + 8 * m + 64 * pb : pa + 8 * pb + 64 * m;
  }
  // staged slot of x, y, z for the slice planes (-1: no plane has a nonzero
  // normal component there, so the coordinate is not staged and enters the
  // node-phase distance as 0; only the case bits use it, and a zero of either
  // sign compares the same against the iso value)
  const int psx = (plane_slots & 0xff) == 0xff ? -1 : (plane_slots & 0xff);
  const int psy = ((plane_slots >> 8) & 0xff) == 0xff ? -1 : ((plane_slots >> 8) & 0xff);
  const int psz = ((plane_slots >> 16) & 0xff) == 0xff ? -1 : ((plane_slots >> 16) & 0xff);
  constexpr NodeProg NP = node_prog(kProg);
  const bool kEmitPrefetch = g_emit_prefetch;
  // an emitting element's coordinates (not staged): copied by 16-byte
  // cp.async into S_dv's space above the active-cell lists, which is dead
  // from the node-phase barrier to the next iteration's pencils
  // (two-CTA kernels only: the three-CTA ones have no registers to spare at 80)
  const bool emit_stage =
      kOcc == 2 && g_emit_stage && slot_xyz < 0 && ((plane_slots >> 24) & 1) && p.mode != FUSED_COUNT;
  double* const S_xyz = S_dv + 6 * kArr;
  static_assert(kNC * 8 + kMaxTriPerElem * 2 <= 6 * kArr * 8, "active-cell lists overlap the emission coordinates");
  // node programs: staged-array offset of each scalar surface and of a scalar colour
  int sc_off[NKB_MAX_SURFACES], sc_off_c = 0;
#pragma unroll
  for (int s = 0; s < NKB_MAX_SURFACES; ++s)
    sc_off[s] = (NP.s[s] == NK_SC) ? (slot_sc + p.surf_src[s] - SRC_SCALAR0) * kArr : 0;
  if (NP.c == NK_SC) sc_off_c = (slot_sc + p.color_src - SRC_SCALAR0) * kArr;
  // a scalar colour read from the array of the program's (single) scalar surface
  bool sc_col_same = false;
#pragma unroll
  for (int s = 0; s < NKB_MAX_SURFACES; ++s)
    if (NP.s[s] == NK_SC && NP.c == NK_SC && sc_off[s] == sc_off_c) sc_col_same = true;

  for (long long it = 0; it < n_it; ++it) {
    const long long e = blockIdx.x + it * G;
    const int b = (int)(it & 1);
    if (kTma) mbar_wait(&s_tma_bar[b], (unsigned)((it >> 1) & 1));
    else cp_async_wait_all();
    if (tid == 0) {
      mc.band = ~0u;
      mc.bor = 0u;
    }
    __syncthreads();                                   // element `it` staged; iteration it-1 finished
    if (it + 1 < n_it) {
      if (tid >= 192) prefetch(e + G, b ^ 1);
      if (!kCompact && tid == 0) l2_prefetch(p.geo + (e + G) * 9 * kNN, kGeoBytes);
    }
    cp_async_commit();
    const double* S_in = S_ring + b * nin * kArr;

    // J^-1 of my first node: loads in flight across the pencil phase
    double J0[9];
    if (!kCompact) {
#pragma unroll
      for (int c = 0; c < 9; ++c) J0[c] = __ldg(p.geo + (e * 9 + c) * kNN + tid);
    }

    // ---- u,v,w pencils: thread = (dir, pencil), 3 fields share offsets ----
    if (tid < 192) {
#pragma unroll
      for (int m = 0; m < kNP; ++m) NKB_DCHECK(off[m] >= 0 && off[m] < kArr);
      NKB_DCHECK(slot_vel >= 0 && slot_vel + 3 <= nin);
      const double* su = S_in + slot_vel * kArr;
      double* d0 = S_dv + (tid >> 6) * kArr;
      pencil3(su, su + kArr, su + 2 * kArr, d0, d0 + 3 * kArr, d0 + 6 * kArr, off);
    }
    __syncthreads();

    // ---- node phase: nodes tid and tid + 256 ----
    const long long g0 = e * (long long)kNN;
    unsigned wand = ~0u, wor = 0u;
    // compact: my two nodes share (i, j) -- their in-plane J^-1 entries are loaded once
    double Jij[4] = {0.0, 0.0, 0.0, 0.0};
    if (kCompact) {
      const double* g = S_gc + b * kGeoCompactDoubles;
      const int ij = tid & 63;
      Jij[0] = g[ij];
      Jij[1] = g[64 + ij];
      Jij[2] = g[128 + ij];
      Jij[3] = g[192 + ij];
    }
    // two-CTA kernels: the second node's derivatives are loaded before the
    // first node's arithmetic (both nodes' shared-memory loads in flight)
    // (two-CTA kernels and node program 2 (C3): measured faster; C5's program 1 slower)
    constexpr bool kPreU = kOcc == 2 || kProg == 2;
    double U1[9];
    if (kPreU) {
#pragma unroll
      for (int c = 0; c < 9; ++c) U1[c] = S_dv[c * kArr + q1];
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int n = tid + kG2Threads * h;
      const int q = h ? q1 : q0;
      NKB_DCHECK(n < kNN && q >= 0 && q < kArr);
      double J[9];
      if (kCompact) {                                  // geo_compact_node, with the shared (i, j) entries
        J[0] = Jij[0];
        J[1] = Jij[1];
        J[2] = 0.0;
        J[3] = Jij[2];
        J[4] = Jij[3];
        J[5] = 0.0;
        J[6] = 0.0;
        J[7] = 0.0;
        J[8] = S_gc[b * kGeoCompactDoubles + 256 + (n >> 6)];
      } else {
#pragma unroll
        for (int c = 0; c < 9; ++c) J[c] = h ? __ldg(p.geo + (e * 9 + c) * kNN + n) : J0[c];
      }
      double U[9];
#pragma unroll
      for (int c = 0; c < 9; ++c) U[c] = (kPreU && h) ? U1[c] : S_dv[c * kArr + q];
      double A[9];
      if (kCompact) chain_rule_block(U, J, A);           // every compact node is block diagonal
      else chain_rule(U, J, A);
      const double offd = __fma_rn(A[5], A[7], __fma_rn(A[2], A[6], __dmul_rn(A[1], A[3])));
      const double dia = __fma_rn(A[8], A[8], __fma_rn(A[4], A[4], __dmul_rn(A[0], A[0])));
      const double vq = -__fma_rn(0.5, dia, offd);
      const double om0 = __dsub_rn(A[7], A[5]);
      const double om1 = __dsub_rn(A[2], A[6]);
      const double om2 = __dsub_rn(A[3], A[1]);
      double vw = 0.0, vu = 0.0;
      S_q[q] = vq;
      if (kWmag) {
        vw = mag3(om0, om1, om2);
        S_q[kArr + q] = vw;
      }
      if (kOut) {
        if (p.q_out) p.q_out[g0 + n] = vq;
        if (p.wmag_out) p.wmag_out[g0 + n] = vw;
        if (p.vort_out) {
          p.vort_out[3 * (g0 + n) + 0] = om0;
          p.vort_out[3 * (g0 + n) + 1] = om1;
          p.vort_out[3 * (g0 + n) + 2] = om2;
        }
      }
      unsigned bits = 0;
      if (kProg == 0) {                               // generic: runtime source dispatch
        if (p.need_umag)
          vu = mag3(S_in[slot_vel * kArr + q], S_in[(slot_vel + 1) * kArr + q], S_in[(slot_vel + 2) * kArr + q]);
#pragma unroll
        for (int s = 0; s < NKB_MAX_SURFACES; ++s) {
          if (s >= p.n_surf) break;
          const int src = p.surf_src[s];
          double val;
          if (src >= SRC_PLANE)
            val = plane_dist(p.surf_n[s], psx >= 0 ? S_in[psx * kArr + q] : 0.0,
                             psy >= 0 ? S_in[psy * kArr + q] : 0.0, psz >= 0 ? S_in[psz * kArr + q] : 0.0);
          else if (src == SRC_Q) val = vq;
          else if (src == SRC_WMAG) val = vw;
          else if (src == SRC_UMAG) val = vu;
          else val = S_in[(slot_sc + src - SRC_SCALAR0) * kArr + q];
          bits |= (val >= p.surf_iso[s] ? 1u : 0u) << s;
        }
        if (p.color_src >= 0) {
          const int src = p.color_src;
          const double c = (src == SRC_Q)      ? vq
                           : (src == SRC_WMAG) ? vw
                           : (src == SRC_UMAG) ? vu
                                               : S_in[(slot_sc + src - SRC_SCALAR0) * kArr + q];
          cmin = fmin(cmin, c);
          cmax = fmax(cmax, c);
        }
      } else {                                        // node program: sources fixed at compile time
        if (prog_uses(kProg, NK_U)) {
          vu = mag3(S_in[slot_vel * kArr + q], S_in[(slot_vel + 1) * kArr + q], S_in[(slot_vel + 2) * kArr + q]);
          S_u[q] = vu;
        }
        double sc_val = 0.0;                            // the (last) scalar surface's value at this node
#pragma unroll
        for (int s = 0; s < NKB_MAX_SURFACES; ++s) {
          if (NP.s[s] == NK_NONE) continue;
          double val;
          if (NP.s[s] == NK_PL)
            val = plane_dist(p.surf_n[s], psx >= 0 ? S_in[psx * kArr + q] : 0.0,
                             psy >= 0 ? S_in[psy * kArr + q] : 0.0, psz >= 0 ? S_in[psz * kArr + q] : 0.0);
          else if (NP.s[s] == NK_Q) val = vq;
          else if (NP.s[s] == NK_W) val = vw;
          else if (NP.s[s] == NK_U) val = vu;
          else {
            NKB_DCHECK(sc_off[s] >= 0 && sc_off[s] + kArr <= nin * kArr);
            val = S_in[sc_off[s] + q];
            sc_val = val;
          }
          bits |= (val >= p.surf_iso[s] ? 1u : 0u) << s;
        }
        if (NP.c != NK_NONE) {
          double c;
          if (NP.c == NK_Q) c = vq;
          else if (NP.c == NK_W) c = vw;
          else if (NP.c == NK_U) c = vu;
          else if (sc_col_same) c = sc_val;              // the colour is the scalar surface's field
          else c = S_in[sc_off_c + q];
          cmin = fmin(cmin, c);
          cmax = fmax(cmax, c);
        }
      }
      S_bits[n] = (unsigned char)bits;
      wand &= bits;
      wor |= bits;
    }
    {
      const unsigned wa = __reduce_and_sync(0xffffffffu, wand), wo = __reduce_or_sync(0xffffffffu, wor);
      if (lane == 0) {
        atomicAnd(&mc.band, wa);
        atomicOr(&mc.bor, wo);
      }
    }
    __syncthreads();                                   // case bits, Q, |w| of element `it` ready
    if (p.n_surf == 0) continue;
    if ((mc.bor & ~mc.band) == 0) {                    // no surface crosses this element
      if (p.mode == FUSED_COUNT && tid == 0) p.elem_count[e] = 0;
      continue;
    }
    // the element emits: its corner coordinates (never staged unless a slice
    // uses them) are read by the emission a few hundred cycles from now --
    // copy them into shared memory (or pull them toward L2) while
    // classification runs
    if (emit_stage) {
      const long long gx = e * (long long)kNN;
      for (int i = tid; i < 3 * (kNN / 2); i += kG2Threads) {
        const int f = i / (kNN / 2), o = 2 * (i - f * (kNN / 2));
        NKB_DCHECK(f < 3 && o + 1 < kArr);
        cp_async16(S_xyz + f * kArr + o, (f == 0 ? p.x : f == 1 ? p.y : p.z) + gx + o);
      }
      cp_async_commit();
    } else if (kEmitPrefetch && tid == 0 && p.mode != FUSED_COUNT) {
      const long long gx = e * (long long)kNN;
      l2_prefetch(p.x + gx, kNN * sizeof(double));
      l2_prefetch(p.y + gx, kNN * sizeof(double));
      l2_prefetch(p.z + gx, kNN * sizeof(double));
    }

    // ---- classify: sub-hexes 2t, 2t+1; one block scan of (triangles, active cells) ----
    unsigned pk[2] = {0u, 0u};
    int nt[2] = {0, 0};
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int c = 2 * tid + u;
      if (c < kNC) {
        const unsigned long long w =
            corner_bytes(reinterpret_cast<const unsigned long long*>(S_bits), c % kN, (c / kN) % kN, c / (kN * kN));
#pragma unroll
        for (int s = 0; s < NKB_MAX_SURFACES; ++s) {
          if (s >= p.n_surf) break;
          const unsigned cs = case_of(w, s);
          pk[u] |= cs << (8 * s);
          nt[u] += mc.t_ntri[cs];
        }
      }
    }
    const int mine = ((nt[0] + nt[1]) << 10) | ((nt[0] > 0) + (nt[1] > 0));
    int incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    if (lane == 31) mc.wsum[warp] = incl;
    __syncthreads();
    int before = 0, all = 0;
#pragma unroll
    for (int w = 0; w < kG2Threads / 32; ++w) {
      const int v = mc.wsum[w];
      before += (w < warp) ? v : 0;
      all += v;
    }
    const int excl = before + incl - mine;
    int tri_off = excl >> 10, act = excl & 1023;
#pragma unroll
    for (int u = 0; u < 2; ++u)
      if (nt[u] > 0) {
        NKB_DCHECK(act >= 0 && act < kNC && 2 * tid + u < kNC);
        act_cell[act] = (unsigned short)(2 * tid + u);
        act_cases[act] = pk[u];
        act_off[act] = (unsigned short)tri_off;
        for (int t2 = 0; t2 < nt[u]; ++t2) tri_act[tri_off + t2] = (unsigned short)act;
        ++act;
        tri_off += nt[u];
      }
    const int total = all >> 10, n_act = all & 1023;
    if (tid == 0) {
      unsigned long long base = 0;
      if (p.mode == FUSED_FAST) {
        base = (unsigned long long)blockIdx.x * (unsigned long long)p.region_cap + cta_fill;
      } else if (p.mode == FUSED_COUNT) {
        p.elem_count[e] = total;
      } else {
        base = (unsigned long long)p.elem_offset[e];
      }
      mc.base = base;
    }
    cta_fill += (unsigned long long)total;             // every thread keeps the same count
    if (emit_stage) cp_async_wait_all();              // the element's coordinates have landed
    __syncthreads();
    if (p.mode == FUSED_COUNT || total == 0) continue;

    // ---- emit: one thread per active cell, (surface, table) order ----
    const bool xyz_staged = slot_xyz >= 0;
    const double* Sx = xyz_staged ? S_in + slot_xyz * kArr : emit_stage ? S_xyz : p.x + g0;
    const double* Sy = xyz_staged ? S_in + (slot_xyz + 1) * kArr : emit_stage ? S_xyz + kArr : p.y + g0;
    const double* Sz = xyz_staged ? S_in + (slot_xyz + 2) * kArr : emit_stage ? S_xyz + 2 * kArr : p.z + g0;
    const double* Su = S_in + slot_vel * kArr;
    // pn: the node's index in Sx/Sy/Sz (swizzled when staged, natural in global
    // memory otherwise); the edge's plane distances always use all three
    // coordinates, exactly as the oracle does
    auto value_at = [&](int src, int s, int q, int pn) -> double {
      if (src >= SRC_PLANE) return plane_dist(p.surf_n[s], Sx[pn], Sy[pn], Sz[pn]);
      if (src == SRC_Q) return S_q[q];
      if (src == SRC_WMAG) return S_q[kArr + q];
      if (src == SRC_UMAG) return kStoreU ? S_u[q] : mag3(Su[q], Su[kArr + q], Su[2 * kArr + q]);
      return S_in[(slot_sc + src - SRC_SCALAR0) * kArr + q];
    };
    // one task per triangle VERTEX over all 256 threads: triangle tt's
    // active cell from the per-triangle table the scan filled, then its
    // (surface, table row) by walking the cell's case bytes
    const unsigned long long base = mc.base;
    for (int task = tid; task < 3 * total; task += kG2Threads) {
      const int tt = task / 3, r = task - 3 * (task / 3);
      const int lo = tri_act[tt];                     // the active cell of triangle tt
      NKB_DCHECK(tt < kMaxTriPerElem && lo >= 0 && lo < n_act && n_act <= kNC);
      const int c = act_cell[lo];
      const unsigned packed = act_cases[lo];
      int li = tt - (int)act_off[lo], s = 0;
      unsigned cs = packed & 0xffu;
      for (;;) {
        const int nt = mc.t_ntri[cs];
        if (li < nt) break;
        li -= nt;
        ++s;
        cs = (packed >> (8 * s)) & 0xffu;
      }
      const int k = li;
      const long long out = (long long)base + tt;
      const bool over = p.mode == FUSED_FAST ? (out - (long long)blockIdx.x * p.region_cap >= p.region_cap)
                                             : (out >= p.tri_cap);
      if (over) continue;                              // counted, not written; the host grows and re-runs
      const int ca = c % kN, cb = (c / kN) % kN, ck = c / (kN * kN);
      const int src = p.surf_src[s];
      const double iso = p.surf_iso[s];
      const int ed = g_mc_tri[cs][3 * k + r];
      const int va = mc.t_edge[ed][0], vb = mc.t_edge[ed][1];
      const int ia = ca + voff_i(va), ja = cb + voff_j(va), ka = ck + voff_k(va);
      const int ib = ca + voff_i(vb), jb = cb + voff_j(vb), kb = ck + voff_k(vb);
      const int qa = kTma ? ia + kNP * ja + kNP * kNP * ka : sw(ia, ja, ka);
      const int qb = kTma ? ib + kNP * jb + kNP * kNP * kb : sw(ib, jb, kb);
      const int pa = xyz_staged ? qa : ia + kNP * ja + kNP * kNP * ka;
      const int pb = xyz_staged ? qb : ib + kNP * jb + kNP * kNP * kb;
      NKB_DCHECK(c >= 0 && c < kNC && s >= 0 && s < p.n_surf && k >= 0 && k < NKB_MC_MAX_TRI);
      NKB_DCHECK(qa >= 0 && qa < kArr && qb >= 0 && qb < kArr && pa >= 0 && pa < kNN && pb >= 0 && pb < kNN);
      NKB_DCHECK(out >= 0 && out < p.tri_cap);
      const double sa = value_at(src, s, qa, pa), sb = value_at(src, s, qb, pb);
      const double tv = __ddiv_rn(__dsub_rn(iso, sa), __dsub_rn(sb, sa));
      const double cla = value_at(p.color_src, 0, qa, pa), clb = value_at(p.color_src, 0, qb, pb);
      const double xa = Sx[pa], ya = Sy[pa], za = Sz[pa];
      const double xb = Sx[pb], yb = Sy[pb], zb = Sz[pb];
      float4 v;
      v.x = __double2float_rn(__fma_rn(tv, __dsub_rn(xb, xa), xa));
      v.y = __double2float_rn(__fma_rn(tv, __dsub_rn(yb, ya), ya));
      v.z = __double2float_rn(__fma_rn(tv, __dsub_rn(zb, za), za));
      v.w = __double2float_rn(__fma_rn(tv, __dsub_rn(clb, cla), cla));
      p.tri[3 * out + r] = v;
      if (p.meta && r == 0)
        p.meta[out] = ((unsigned long long)e << 32) | ((unsigned long long)c << 16) |
                      ((unsigned long long)s << 12) | ((unsigned long long)k << 8) | cs;
    }
  }

  if (p.mode == FUSED_FAST && p.region_count != nullptr && tid == 0) {
    p.region_count[blockIdx.x] = cta_fill;
    if (cta_fill) atomicAdd(&p.counters[0], cta_fill);
  }
  if (p.color_src >= 0 && p.mode != FUSED_ORDERED) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      cmin = fmin(cmin, __shfl_xor_sync(0xffffffffu, cmin, o));
      cmax = fmax(cmax, __shfl_xor_sync(0xffffffffu, cmax, o));
    }
    if (lane == 0) {
      s_mn[warp] = cmin;
      s_mx[warp] = cmax;
    }
    __syncthreads();
    if (tid == 0) {
      double mn = s_mn[0], mx = s_mx[0];
      for (int w = 1; w < kG2Threads / 32; ++w) {
        mn = fmin(mn, s_mn[w]);
        mx = fmax(mx, s_mx[w]);
      }
      if (mn <= mx) {
        atomicMin(&p.counters[1], enc_ordered(mn));
        atomicMax(&p.counters[2], enc_ordered(mx));
      }
    }
  }
}

static size_t fused2_smem_bytes(int nin, bool compact, bool wmag, bool umag = false) {
  return (size_t)(2 * nin + 10 + (wmag ? 1 : 0) + (umag ? 1 : 0)) * kArr * sizeof(double) +
         (compact ? 2 * kGeoCompactDoubles * sizeof(double) : 0) + kNN;
}

// K1g instantiations: generic program x (|w|, exports) and the node
// programs, budgeted for 2 CTAs per SM; compact pipelines whose CTA fits in
// 75 KB of shared memory (staging <= 3 arrays) also for 3 (kOcc = 3, <= 85
// registers)
using F2Kernel = void (*)(const FusedParams, int, int, int, int, int);
template <bool C, int O>
static F2Kernel f2_kernel_co(int wo, int prog) {
  switch (prog) {
    case 1: return fused2_kernel<C, prog_uses(1, NK_W), false, 1, O>;
    case 2: return fused2_kernel<C, prog_uses(2, NK_W), false, 2, O>;
    case 3: return fused2_kernel<C, prog_uses(3, NK_W), false, 3, O>;
    case 4: return fused2_kernel<C, prog_uses(4, NK_W), false, 4, O>;
    default: break;
  }
  switch (wo) {
    case 0: return fused2_kernel<C, false, false, 0, O>;
    case 1: return fused2_kernel<C, false, true, 0, O>;
    case 2: return fused2_kernel<C, true, false, 0, O>;
    default: return fused2_kernel<C, true, true, 0, O>;
  }
}
static bool fused2_tma() {
  static const bool on = getenv("NKB_K1G_TMA") && getenv("NKB_K1G_TMA")[0] == '1';
  return on;
}
static F2Kernel f2_kernel(bool compact, int wo, int prog, int occ = 2, bool tma = false) {
  if (tma && compact && prog == 4 && occ == 2) return fused2_kernel<true, false, false, 4, 2, true>;
  if (tma && compact && prog == 2 && occ == 3) return fused2_kernel<true, true, false, 2, 3, true>;
  if (tma && compact && prog == 1 && occ == 3) return fused2_kernel<true, false, false, 1, 3, true>;
  if (compact) return occ == 3 ? f2_kernel_co<true, 3>(wo, prog) : f2_kernel_co<true, 2>(wo, prog);
  return f2_kernel_co<false, 2>(wo, prog);
}
constexpr size_t kOcc3MaxSmem = 75u * 1024u - 512u;   // dynamic bytes per CTA that let 3 CTAs share an SM
static int fused2_occ(int nin, bool compact, bool wmag, bool umag) {
  static const int forced = [] {
    const char* v = getenv("NKB_K1G_OCC");               // A/B: NKB_K1G_OCC=2 forces two CTAs per SM
    return v ? atoi(v) : 0;
  }();
  if (!compact || forced == 2) return 2;
  return fused2_smem_bytes(nin, true, wmag, umag) <= kOcc3MaxSmem ? 3 : 2;
}
static int fused2_prepare() {
  const char* v = getenv("NKB_EMIT_PREFETCH");
  const int on = !(v && v[0] == '0');
  NKB_CUDA(cudaMemcpyToSymbol(g_emit_prefetch, &on, sizeof(on)));
  const char* vs = getenv("NKB_EMIT_STAGE");
  const int st = !(vs && vs[0] == '0');
  NKB_CUDA(cudaMemcpyToSymbol(g_emit_stage, &st, sizeof(st)));
  for (int c = 0; c < 2; ++c)
    for (int occ = 2; occ <= (c == 1 ? 3 : 2); ++occ) {
      const int bytes = (int)fused2_smem_bytes(occ == 3 ? 3 : kG2MaxIn, c == 1, true, true);
      for (int wo = 0; wo < 4; ++wo)
        NKB_CUDA(cudaFuncSetAttribute(f2_kernel(c == 1, wo, 0, occ), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      bytes));
      for (int k = 1; k < kNodeProgs; ++k)
        NKB_CUDA(cudaFuncSetAttribute(f2_kernel(c == 1, 0, k, occ), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      bytes));
    }
  NKB_CUDA(cudaFuncSetAttribute(f2_kernel(true, 0, 4, 2, true), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)fused2_smem_bytes(kG2MaxIn, true, true, true)));
  NKB_CUDA(cudaFuncSetAttribute(f2_kernel(true, 0, 2, 3, true), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)kOcc3MaxSmem));
  NKB_CUDA(cudaFuncSetAttribute(f2_kernel(true, 0, 1, 3, true), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)kOcc3MaxSmem));
  return NKB_OK;
}

// coordinates the slice planes use: bit c set when some plane's normal has a
// nonzero component c (K1g stages only those; emission reads x,y,z via L2)
static unsigned plane_axes(const FusedParams& p) {
  unsigned m = 0;
  for (int i = 0; i < p.n_surf; ++i)
    if (p.surf_src[i] >= SRC_PLANE)
      for (int c = 0; c < 3; ++c) m |= (p.surf_n[i][c] != 0.0 ? 1u : 0u) << c;
  return m;
}

// arrays K1g stages per element: the coordinates a slice normal uses, u,v,w, scalars
static int k1g_nin(const FusedParams& p) {
  const unsigned m = plane_axes(p);
  return (int)((m & 1) + ((m >> 1) & 1) + (m >> 2)) + (p.need_vel ? 3 : 0) + p.n_scalars;
}

static bool fused2_on(const FusedParams& p) {
  const char* v = getenv("NKB_FUSED2");               // A/B: NKB_FUSED2=0 forces K1
  if (v && v[0] == '0') return false;
  if (!(p.geo != nullptr && p.need_grad) || p.prof != nullptr) return false;
  // two CTAs per SM: (2 nin + 11) x 4 KB (+ 4 KB of compact geometry) each
  return k1g_nin(p) <= (p.geo_compact ? kG2MaxIn - 1 : kG2MaxIn);
}

static size_t fused_smem_bytes(int nin) {
  return (size_t)(kRing * nin + kNumD + 4) * kArr * sizeof(double) + 2 * kNN;
}

// one-time kernel attributes (outside any stream capture)
int launch_fused_prepare() {
  static bool done = false;
  if (done) return NKB_OK;
  const int mx = (int)fused_smem_bytes(kMaxIn);
  NKB_CUDA(cudaFuncSetAttribute(fused_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
  NKB_CUDA(cudaFuncSetAttribute(fused_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
  NKB_CUDA(cudaFuncSetAttribute(fused_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
  NKB_CUDA(cudaFuncSetAttribute(fused_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
  NKB_TRY(launch_stream_prepare());
  NKB_TRY(fused2_prepare());
  int dev = 0;
  NKB_CUDA(cudaGetDevice(&dev));
  NKB_CUDA(cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev));
  done = true;
  return NKB_OK;
}

// which pass runs the surfaces of `p`: 1 = the barrier-free warp-per-element
// pass (stream.cu) for pipelines without a velocity gradient, 0 = K1.
// NKB_STREAM=0 forces K1 (A/B runs); the phase profile is K1's.
int surface_pass_of(const FusedParams& p) {
  const char* v = getenv("NKB_STREAM");
  const bool on = v == nullptr || v[0] != '0';
  if (on && p.prof == nullptr && stream_eligible(p)) return 1;
  return fused2_on(p) ? 2 : 0;
}

// triangle regions (CTAs) of the pass that runs `p`
int fused_grid_for(const FusedParams& p, int64_t n_elements) {
  const int g = fused_grid(n_elements, p.sm_reserve);   // min(E, SMs - reserved)
  if (surface_pass_of(p) != 2) return g;
  const int64_t g2 = (int64_t)fused2_occ(k1g_nin(p), p.geo_compact != 0, p.need_wmag != 0, prog_uses(node_prog_of(p), NK_U)) * fused_grid(1LL << 40, p.sm_reserve);
  return (int)(n_elements < g2 ? (n_elements < 1 ? 1 : n_elements) : g2);
}

int launch_fused(const FusedParams& p, cudaStream_t s) {
  if (p.n_elements <= 0) return NKB_OK;
  const bool cached = p.geo != nullptr && p.need_grad;
  bool has_plane = false;
  for (int i = 0; i < p.n_surf; ++i) has_plane |= p.surf_src[i] >= SRC_PLANE;
  // staged inputs in slot order: [x, y, z], [u, v, w], [scalars]; with the
  // geometry cache x,y,z are staged only when a slice plane needs them
  const bool stage_xyz = !cached || has_plane;
  FusedParams q = p;
  int k = 0;
  int slot_xyz = -1, slot_vel = 0;
  if (stage_xyz) {
    slot_xyz = k;
    q.in_ptr[k++] = p.x;
    q.in_ptr[k++] = p.y;
    q.in_ptr[k++] = p.z;
  }
  if (p.need_vel) {
    slot_vel = k;
    for (int c = 0; c < 3; ++c) q.in_ptr[k++] = p.vel[c];
  }
  const int slot_sc = k;
  for (int c = 0; c < p.n_scalars; ++c) q.in_ptr[k++] = p.scalar[c];
  const int nin = k;
  if (nin > kMaxIn) return fail(NKB_EINVAL, "too many staged fields for one pass (coordinates, velocity and "
                                            "scalars exceed 8)");
  const size_t shm = fused_smem_bytes(nin);
  NKB_TRY(launch_fused_prepare());
  const int grid = fused_grid(p.n_elements, p.sm_reserve);
  const unsigned gx = (unsigned)grid;
  const int pass = surface_pass_of(p);
  if (pass == 1) return launch_stream(p, grid, s);
  if (pass == 2) {
    // K1g (always cached): stage only the coordinates a slice plane needs
    const unsigned m = plane_axes(p);
    FusedParams q2 = p;
    int k2 = 0, slot2_xyz = -1, slot2_vel = 0, ps = 0;
    if (m == 7u) {
      slot2_xyz = 0;
      for (int c = 0; c < 3; ++c) q2.in_ptr[k2++] = c == 0 ? p.x : c == 1 ? p.y : p.z;
      ps = 0 | (1 << 8) | (2 << 16);
    } else {
      for (int c = 0; c < 3; ++c) {
        if (m & (1u << c)) {
          ps |= k2 << (8 * c);
          q2.in_ptr[k2++] = c == 0 ? p.x : c == 1 ? p.y : p.z;
        } else {
          ps |= 0xff << (8 * c);
        }
      }
    }
    if (p.need_vel) {
      slot2_vel = k2;
      for (int c = 0; c < 3; ++c) q2.in_ptr[k2++] = p.vel[c];
    }
    const int slot2_sc = k2;
    for (int c = 0; c < p.n_scalars; ++c) q2.in_ptr[k2++] = p.scalar[c];
    if ((((uintptr_t)p.x | (uintptr_t)p.y | (uintptr_t)p.z) & 15u) == 0) ps |= 1 << 24;   // 16-byte copies allowed
    const unsigned g2 = (unsigned)fused_grid_for(p, p.n_elements);
    const bool compact = p.geo_compact != 0;
    const int prog = node_prog_of(p);
    const int wm = p.need_wmag != 0 ? 1 : 0;
    const int out = (p.q_out != nullptr || p.wmag_out != nullptr || p.vort_out != nullptr) ? 1 : 0;
    const size_t sh = fused2_smem_bytes(k2, compact, wm != 0, prog_uses(prog, NK_U));
    // TMA staging (A/B only): bulk copies need 16-byte aligned sources
    bool tma = fused2_tma();
    for (int f = 0; f < k2; ++f) tma = tma && ((uintptr_t)q2.in_ptr[f] & 15u) == 0;
    const F2Kernel k = f2_kernel(compact, prog == 0 ? 2 * wm + out : 0, prog,
                                 fused2_occ(k2, compact, wm != 0, prog_uses(prog, NK_U)), tma);
    k<<<g2, kG2Threads, sh, s>>>(q2, k2, slot2_sc, slot2_vel, slot2_xyz, ps);
    NKB_CUDA(cudaGetLastError());
    return NKB_OK;
  }
  if (p.prof) {
    if (cached) fused_kernel<true, true><<<gx, kThreads, shm, s>>>(q, nin, slot_sc, slot_vel, slot_xyz);
    else fused_kernel<false, true><<<gx, kThreads, shm, s>>>(q, nin, slot_sc, slot_vel, slot_xyz);
  } else {
    if (cached) fused_kernel<true, false><<<gx, kThreads, shm, s>>>(q, nin, slot_sc, slot_vel, slot_xyz);
    else fused_kernel<false, false><<<gx, kThreads, shm, s>>>(q, nin, slot_sc, slot_vel, slot_xyz);
  }
  NKB_CUDA(cudaGetLastError());
  return NKB_OK;
}

int launch_count_scan(const int* cnt, int64_t n, long long* off, unsigned long long* total, cudaStream_t s) {
  count_scan_kernel<<<1, 1024, 0, s>>>(cnt, n, off, total);
  NKB_CUDA(cudaGetLastError());
  return NKB_OK;
}

// the kernel variant a step runs (CUDA-graph cache key; env switches change it)
int fused_node_prog(const FusedParams& p) {
  return node_prog_of(p) + 16 * stream_prog_of(p) + 64 * fused2_occ(k1g_nin(p), p.geo_compact != 0, p.need_wmag != 0, prog_uses(node_prog_of(p), NK_U));
}

// CTAs per SM of the surface pass (K1g: 2 or 3; K1s and K1: 1)
int fused_ctas_per_sm(const FusedParams& p) {
  if (surface_pass_of(p) != 2) return 1;
  return fused2_occ(k1g_nin(p), p.geo_compact != 0, p.need_wmag != 0, prog_uses(node_prog_of(p), NK_U));
}

NKB_CHECKED_ACCESSOR(checked_read_fused)

}  // namespace nkb
