// K1: the fused in situ pass -- SEM->VTK adaptor gather, tensor-product
// derivatives, Jacobian inverse, velocity gradient, vorticity, Q-criterion,
// marching-cubes classification of every linear sub-hex and triangle
// emission, in ONE read of the element's GLL fields from HBM.
//
// Persistent, two ping-pong element pipelines per SM.  One CTA (512 threads)
// per SM walks the elements e_j = blockIdx.x + j*gridDim.x; warp group
// g = 0, 1 (8 warps each, own shared memory, own named barriers) takes the
// elements with j % 2 == g.  The groups never wait for each other, so one
// group's latency-bound node phase overlaps the other's FP64/shared-memory
// bound derivative phase.  Per element of a group:
//
//   6 pencil warps : even-odd 8-point derivatives of x,y,z | u,v,w along
//                    r,s,t (192 (dir, pencil) threads x 6 fields, smem
//                    offsets computed once, each coefficient feeds 3 DFMAs)
//   2 aux warps    : meanwhile node-local pre-pass of the element (plane /
//                    scalar / |u| case bits, colour range; via L2) and scan,
//                    allocate and emit the triangles of the group's previous
//                    element
//   -- group barrier --
//   aux warps      : cp.async prefetch of the group's next element
//   8 warps        : node phase (2 nodes / thread): Jacobian inverse, grad u,
//                    Q, |w|, Q / |w| case bits
//   -- group barrier --
//   8 warps        : classification (one sub-hex per thread)
//
// Only x,y,z,u,v,w are staged in shared memory (XOR-swizzled, bank-conflict
// free for node-parallel and r/s/t-pencil access).  Scalars, and the
// coordinates the node phase and the emission need after the prefetch has
// recycled the staging slot, are re-read through L2 (the element was streamed
// a few microseconds earlier), so HBM sees each field byte once.
//
// Output slots: FAST mode appends each element's triangles to a region of the
// triangle buffer private to the CTA (shared-memory counter, no global
// atomics); the raster walks the regions, an export compacts them.  The
// triangle order in the buffer therefore depends on the schedule -- the image
// does not (the raster is an order-independent min); inside an element the
// order is (cell, surface, table) always.  Deterministic global order
// (emit_meta) runs COUNT mode, an exclusive scan, then ORDERED mode.
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

#define NKB_MC_NO_HOST_TABLES
#include "mc_tables.h"
#include "nkb_internal.h"

namespace nkb {

__constant__ double c_D[kNP * kNP];
__constant__ double c_Ae[4][4];   // even half: 0.5*(D[i][m] + D[i][7-m])
__constant__ double c_Ao[4][4];   // odd half:  0.5*(D[i][m] - D[i][7-m])

// MC tables in global memory (copied to shared memory once per CTA)
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

constexpr int kThreads = 512;
constexpr int kGroupThreads = 256;     // one ping-pong pipeline
constexpr int kPencilThreads = 192;    // per group: 3 dirs x 64 pencils
constexpr int kAuxThreads = kGroupThreads - kPencilThreads;   // 64
constexpr int kArr = kNN;              // 512 doubles per staged array
constexpr int kNumD = 18;              // derivative arrays: d(f)/d(r,s,t) for x,y,z,u,v,w
constexpr int kStaged = 6;             // staged arrays: x,y,z,u,v,w
// per-group dynamic shared memory (doubles): staged + derivatives + (Q, |w|)
constexpr int kGroupDoubles = (kStaged + kNumD + 2) * kArr;
constexpr int kCellsPerAux = (kNC + kAuxThreads - 1) / kAuxThreads;   // 6

// node (i,j,k) -> shared-memory slot.  Within each 64 B line the 8 doubles
// are XOR-permuted by (j>>1 | (k&1)<<2); lines are XOR-permuted by (k&1).
// For every 16-lane half-warp pattern used below (node-parallel, r-, s- and
// t-pencils) the 16 accessed doubles fall in 16 distinct 8-byte bank pairs.
__device__ __forceinline__ int sw(int i, int j, int k) {
  return (i ^ ((j >> 1) | ((k & 1) << 2))) + 8 * (j ^ (k & 1)) + 64 * k;
}
__device__ __forceinline__ int sw_node(int n) { return sw(n & 7, (n >> 3) & 7, n >> 6); }

// VTK_HEXAHEDRON corner v -> lattice offset (matches NKB_MC_VERT_OFF_DATA)
__device__ __forceinline__ int voff_i(int v) { return (v ^ (v >> 1)) & 1; }
__device__ __forceinline__ int voff_j(int v) { return (v >> 1) & 1; }
__device__ __forceinline__ int voff_k(int v) { return v >> 2; }

__device__ __forceinline__ unsigned long long enc_ordered(double d) {
  unsigned long long b = (unsigned long long)__double_as_longlong(d);
  return (b & 0x8000000000000000ULL) ? ~b : (b | 0x8000000000000000ULL);
}

__device__ __forceinline__ void cp_async8(double* smem_dst, const double* gsrc) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
// named barriers: group g -> id 1+g over 256 threads; its aux warps -> id 3+g over 64
__device__ __forceinline__ void group_bar(int g) {
  asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "n"(kGroupThreads) : "memory");
}
__device__ __forceinline__ void aux_bar(int g) {
  asm volatile("bar.sync %0, %1;" ::"r"(3 + g), "n"(kAuxThreads) : "memory");
}

__device__ __forceinline__ double mag3(double a, double b, double c) {
  // reference ':mag' = sqrt(sum(v**2)) summed left to right (sinks.py:240-241)
  return __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(a, a), __dmul_rn(b, b)), __dmul_rn(c, c)));
}

__device__ __forceinline__ double plane_dist(const double* n, double x, double y, double z) {
  return __fma_rn(n[2], z, __fma_rn(n[1], y, __dmul_rn(n[0], x)));
}

__device__ __forceinline__ bool src_is_grad(int s) { return s == SRC_Q || s == SRC_WMAG; }

struct GroupScratch {
  unsigned cases[kNC];          // byte s = case of surface s
  unsigned char ntri[kNC];      // triangles of each cell (all surfaces)
  unsigned short coff[kNC];     // exclusive triangle offset of each cell
  int wtot[kAuxThreads / 32];
  unsigned long long base;      // output slot of the element's first triangle
  int total;                    // triangles to emit
};

struct Shared {
  GroupScratch grp[2];
  unsigned char t_ntri[256];
  signed char t_tri[256][3 * NKB_MC_MAX_TRI];
  unsigned char t_edge[12][2];
  unsigned long long cta_fill;  // FAST mode: triangles in this CTA's region
  double mn[kThreads / 32], mx[kThreads / 32];
};

}  // namespace

// mode: FUSED_FAST / FUSED_COUNT / FUSED_ORDERED (nkb_internal.h)
__global__ void __launch_bounds__(kThreads, 1) fused_kernel(const FusedParams p, int nst) {
  extern __shared__ __align__(16) double smem[];
  __shared__ Shared sh;

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int g = tid >> 8;                          // ping-pong group
  const int lt = tid & (kGroupThreads - 1);        // thread index within the group
  const bool is_pencil = lt < kPencilThreads;
  const int at = lt - kPencilThreads;              // aux thread index
  double* S_in = smem + g * kGroupDoubles;         // staged x,y,z,u,v,w (swizzled)
  double* S_d = S_in + kStaged * kArr;             // 18 derivative arrays
  double* S_q = S_d + kNumD * kArr;                // Q, |w| of the group's last node phase
  unsigned char* S_bits = reinterpret_cast<unsigned char*>(smem + 2 * kGroupDoubles) + g * kNN;
  GroupScratch& gs = sh.grp[g];

  for (int i = tid; i < 256; i += kThreads) sh.t_ntri[i] = g_mc_ntri[i];
  for (int i = tid; i < 256 * 3 * NKB_MC_MAX_TRI; i += kThreads) (&sh.t_tri[0][0])[i] = (&g_mc_tri[0][0])[i];
  if (tid < 24) (&sh.t_edge[0][0])[tid] = (&g_mc_edge_v[0][0])[tid];
  if (tid == 0) sh.cta_fill = 0;
  __syncthreads();

  const long long E = p.n_elements;
  const long long G = gridDim.x;
  const long long n_it = (E > blockIdx.x) ? (E - blockIdx.x + G - 1) / G : 0;
  const long long n_k = (n_it > g) ? (n_it - g + 1) / 2 : 0;   // elements of this group
  auto elem_of = [&](long long k) { return (long long)blockIdx.x + (2 * k + g) * G; };
  bool need_xyz = false, grad_surf = false;         // any slice plane / any Q or |w| surface
  for (int s = 0; s < p.n_surf; ++s) {
    need_xyz |= p.surf_src[s] >= SRC_PLANE;
    grad_surf |= src_is_grad(p.surf_src[s]);
  }
  const bool color_grad = src_is_grad(p.color_src);
  double cmin = INFINITY, cmax = -INFINITY;

  // aux warps: coalesced 8-byte cp.async of element e's staged arrays
  int qn[kArr / kAuxThreads];
#pragma unroll
  for (int h = 0; h < kArr / kAuxThreads; ++h) qn[h] = sw_node((at & (kAuxThreads - 1)) + kAuxThreads * h);
  auto prefetch = [&](long long e) {
    const long long g0 = e * (long long)kNN + at;
#pragma unroll
    for (int f = 0; f < kStaged; ++f) {
      if (f < nst) {
        const double* src = p.in_ptr[f] + g0;
        double* d = S_in + f * kArr;
#pragma unroll
        for (int h = 0; h < kArr / kAuxThreads; ++h) cp_async8(d + qn[h], src + kAuxThreads * h);
      }
    }
  };

  // global (L2-resident) per-node value of a source, by element-local node n
  auto gvalue = [&](int src, int s, long long g0, int n) -> double {
    if (src >= SRC_PLANE)
      return plane_dist(p.surf_n[s], __ldg(p.x + g0 + n), __ldg(p.y + g0 + n), __ldg(p.z + g0 + n));
    if (src == SRC_UMAG)
      return mag3(__ldg(p.vel[0] + g0 + n), __ldg(p.vel[1] + g0 + n), __ldg(p.vel[2] + g0 + n));
    return __ldg(p.scalar[src - SRC_SCALAR0] + g0 + n);
  };

  // aux warps: node-local classification bits (planes, scalars, |u|) and the
  // colour range of non-derived colour fields for element e, through L2
  auto prepass = [&](long long e) {
    const long long g0 = e * (long long)kNN;
#pragma unroll 1
    for (int hb = 0; hb < kArr / kAuxThreads; hb += 4) {
      double lx[4], ly[4], lz[4], ls0[4], ls1[4], lu[4], lv[4], lw[4];
#pragma unroll
      for (int h = 0; h < 4; ++h) {      // issue every load of the batch first
        const int n = at + kAuxThreads * (hb + h);
        lx[h] = ly[h] = lz[h] = ls0[h] = ls1[h] = lu[h] = lv[h] = lw[h] = 0.0;
        if (need_xyz) {
          lx[h] = __ldg(p.x + g0 + n);
          ly[h] = __ldg(p.y + g0 + n);
          lz[h] = __ldg(p.z + g0 + n);
        }
        if (p.n_scalars > 0) ls0[h] = __ldg(p.scalar[0] + g0 + n);
        if (p.n_scalars > 1) ls1[h] = __ldg(p.scalar[1] + g0 + n);
        if (p.need_umag) {
          lu[h] = __ldg(p.vel[0] + g0 + n);
          lv[h] = __ldg(p.vel[1] + g0 + n);
          lw[h] = __ldg(p.vel[2] + g0 + n);
        }
      }
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const int n = at + kAuxThreads * (hb + h);
        const double vu = p.need_umag ? mag3(lu[h], lv[h], lw[h]) : 0.0;
        auto local = [&](int src, int s) -> double {
          if (src >= SRC_PLANE) return plane_dist(p.surf_n[s], lx[h], ly[h], lz[h]);
          if (src == SRC_UMAG) return vu;
          return src == SRC_SCALAR0 ? ls0[h] : ls1[h];
        };
        unsigned bits = 0;
        for (int s = 0; s < p.n_surf; ++s)
          if (!src_is_grad(p.surf_src[s])) bits |= (local(p.surf_src[s], s) >= p.surf_iso[s] ? 1u : 0u) << s;
        S_bits[n] = (unsigned char)bits;
        if (p.color_src >= 0 && !color_grad) {
          const double c = local(p.color_src, 0);
          cmin = fmin(cmin, c);
          cmax = fmax(cmax, c);
        }
      }
    }
  };

  // aux warps: scan the per-cell counts of element e, allocate, emit
  auto scan_emit = [&](long long e) {
    int cc[kCellsPerAux], cnt = 0;
#pragma unroll
    for (int j = 0; j < kCellsPerAux; ++j) {
      const int c = kCellsPerAux * at + j;
      cc[j] = (c < kNC) ? gs.ntri[c] : 0;
      cnt += cc[j];
    }
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    const int aw = at >> 5;
    if (lane == 31) gs.wtot[aw] = incl;
    aux_bar(g);
    const int w0 = gs.wtot[0], w1 = gs.wtot[1];
    const int total = w0 + w1;
    int run = (aw ? w0 : 0) + incl - cnt;
#pragma unroll
    for (int j = 0; j < kCellsPerAux; ++j) {
      const int c = kCellsPerAux * at + j;
      if (c < kNC) gs.coff[c] = (unsigned short)run;
      run += cc[j];
    }
    if (at == 0) {
      unsigned long long base = 0;
      int emit_total = total;
      if (p.mode == FUSED_FAST) {
        // CTA-private region of the triangle buffer: shared counter only
        base = (unsigned long long)blockIdx.x * (unsigned long long)p.region_cap +
               (total ? atomicAdd(&sh.cta_fill, (unsigned long long)total) : 0ULL);
      } else if (p.mode == FUSED_COUNT) {
        p.elem_count[e] = total;
        emit_total = 0;
      } else {
        base = (unsigned long long)p.elem_offset[e];
      }
      gs.base = base;
      gs.total = emit_total;
    }
    aux_bar(g);
    const int emit_total = gs.total;
    if (emit_total == 0) return;
    const unsigned long long base = gs.base;
    const long long g0 = e * (long long)kNN;
    const double* Sq = S_q;
    auto value_at = [&](int src, int s, int n) -> double {
      if (src == SRC_Q) return Sq[sw_node(n)];
      if (src == SRC_WMAG) return Sq[kArr + sw_node(n)];
      return gvalue(src, s, g0, n);
    };
    for (int tt = at; tt < emit_total; tt += kAuxThreads) {
      int lo = 0, hi = kNC - 1;          // last cell with coff <= tt
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if ((int)gs.coff[mid] <= tt) lo = mid;
        else hi = mid - 1;
      }
      const int c = lo;
      int li = tt - (int)gs.coff[c];
      const unsigned packed = gs.cases[c];
      int s = 0;
      unsigned cs = packed & 0xffu;
      for (;;) {
        const int nt = sh.t_ntri[cs];
        if (li < nt) break;
        li -= nt;
        ++s;
        cs = (packed >> (8 * s)) & 0xffu;
      }
      const int k = li;
      const long long out = (long long)base + tt;
      if (p.mode == FUSED_FAST ? (out - (long long)blockIdx.x * p.region_cap >= p.region_cap)
                               : (out >= p.tri_cap))
        continue;   // overflow: counted, not written; the host grows the buffer and re-runs
      const int ca = c % kN, cb = (c / kN) % kN, ck = c / (kN * kN);
      const int src = p.surf_src[s];
      const double iso = p.surf_iso[s];
      float4 vtx[3];
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        const int ed = sh.t_tri[cs][3 * k + r];
        const int va = sh.t_edge[ed][0], vb = sh.t_edge[ed][1];
        const int na = (ca + voff_i(va)) + kNP * (cb + voff_j(va)) + kNP * kNP * (ck + voff_k(va));
        const int nb = (ca + voff_i(vb)) + kNP * (cb + voff_j(vb)) + kNP * kNP * (ck + voff_k(vb));
        const double sa = value_at(src, s, na), sb = value_at(src, s, nb);
        const double tv = __ddiv_rn(__dsub_rn(iso, sa), __dsub_rn(sb, sa));
        const double cla = value_at(p.color_src, 0, na), clb = value_at(p.color_src, 0, nb);
        const double xa = __ldg(p.x + g0 + na), xb = __ldg(p.x + g0 + nb);
        const double ya = __ldg(p.y + g0 + na), yb = __ldg(p.y + g0 + nb);
        const double za = __ldg(p.z + g0 + na), zb = __ldg(p.z + g0 + nb);
        vtx[r].x = __double2float_rn(__fma_rn(tv, __dsub_rn(xb, xa), xa));
        vtx[r].y = __double2float_rn(__fma_rn(tv, __dsub_rn(yb, ya), ya));
        vtx[r].z = __double2float_rn(__fma_rn(tv, __dsub_rn(zb, za), za));
        vtx[r].w = __double2float_rn(__fma_rn(tv, __dsub_rn(clb, cla), cla));
      }
      float4* dst = p.tri + 3 * out;
      dst[0] = vtx[0];
      dst[1] = vtx[1];
      dst[2] = vtx[2];
      if (p.meta)
        p.meta[out] = ((unsigned long long)e << 32) | ((unsigned long long)c << 16) |
                      ((unsigned long long)s << 12) | ((unsigned long long)k << 8) | cs;
    }
  };

  // optional phase profile (p.prof != nullptr): cycles per phase, lt == 0 and at == 0
  long long pf_t = clock64(), pf_acc[4] = {0, 0, 0, 0};
  auto pf = [&](int k) {
    if (p.prof && (lt == 0 || at == 0)) {
      const long long now = clock64();
      pf_acc[k] += now - pf_t;
      pf_t = now;
    }
  };

  if (!is_pencil && n_k > 0) prefetch(elem_of(0));
  cp_async_commit();
  for (long long k = 0; k <= n_k; ++k) {
    const long long e = elem_of(k);
    if (!is_pencil) cp_async_wait_all();
    group_bar(g);                                   // element k staged; classify k-1 done
    pf(0);
    if (is_pencil) {
      if (k < n_k && p.need_grad) {
        // ---- pencils: thread = (dir, pencil); 2 triples of fields share offsets ----
        const int dir = lt >> 6;                    // warp-uniform
        const int pa = lt & 7, pb = (lt >> 3) & 7;
        int off[kNP];
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
#pragma unroll 1
        for (int tg = 0; tg < 2; ++tg) {
          const double* s0 = S_in + (3 * tg + 0) * kArr;
          const double* s1 = S_in + (3 * tg + 1) * kArr;
          const double* s2 = S_in + (3 * tg + 2) * kArr;
          double* d0 = S_d + (3 * (3 * tg + 0) + dir) * kArr;
          double* d1 = S_d + (3 * (3 * tg + 1) + dir) * kArr;
          double* d2 = S_d + (3 * (3 * tg + 2) + dir) * kArr;
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
          // even-odd form (oracle deriv8): out[i] = E_i + O_i, out[7-i] = O_i - E_i
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
            d0[off[i]] = __dadd_rn(E0, O0);
            d1[off[i]] = __dadd_rn(E1, O1);
            d2[off[i]] = __dadd_rn(E2, O2);
            d0[off[kNP - 1 - i]] = __dsub_rn(O0, E0);
            d1[off[kNP - 1 - i]] = __dsub_rn(O1, E1);
            d2[off[kNP - 1 - i]] = __dsub_rn(O2, E2);
          }
        }
      }
    } else {
      if (k < n_k) prepass(e);                      // node-local bits + colour of element k
      if (k > 0 && p.n_surf > 0) scan_emit(elem_of(k - 1));   // the group's previous element
    }
    pf(1);
    group_bar(g);                                   // derivatives of element k ready
    if (k == n_k) break;
    pf(2);
    if (!is_pencil) {
      if (k + 1 < n_k) prefetch(elem_of(k + 1));    // staging slot free: pencils are done
      cp_async_commit();
    }

    // ---- node phase: nodes lt and lt + 256 ----
    const long long g0 = e * (long long)kNN;
#pragma unroll 1
    for (int n = lt; n < kNN; n += kGroupThreads) {
      const int q = sw_node(n);
      double vq = 0.0, vw = 0.0;
      if (p.need_grad) {
        double G9[9];
#pragma unroll
        for (int c = 0; c < 9; ++c) G9[c] = S_d[c * kArr + q];
        const double xr = G9[0], xs = G9[1], xt = G9[2];
        const double yr = G9[3], ys = G9[4], yt = G9[5];
        const double zr = G9[6], zs = G9[7], zt = G9[8];
        double J[9];
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
        double U[9];
#pragma unroll
        for (int c = 0; c < 9; ++c) U[c] = S_d[(9 + c) * kArr + q];
        double A[9];
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int b = 0; b < 3; ++b)
            A[3 * a + b] = __fma_rn(U[3 * a + 2], J[6 + b],
                                    __fma_rn(U[3 * a + 1], J[3 + b], __dmul_rn(U[3 * a + 0], J[0 + b])));
        const double off = __fma_rn(A[5], A[7], __fma_rn(A[2], A[6], __dmul_rn(A[1], A[3])));
        const double dia = __fma_rn(A[8], A[8], __fma_rn(A[4], A[4], __dmul_rn(A[0], A[0])));
        vq = -__fma_rn(0.5, dia, off);
        const double om0 = __dsub_rn(A[7], A[5]);
        const double om1 = __dsub_rn(A[2], A[6]);
        const double om2 = __dsub_rn(A[3], A[1]);
        S_q[q] = vq;
        if (p.need_wmag) {
          vw = mag3(om0, om1, om2);
          S_q[kArr + q] = vw;
        }
        if (p.q_out) p.q_out[g0 + n] = vq;
        if (p.wmag_out) p.wmag_out[g0 + n] = vw;
        if (p.vort_out) {
          p.vort_out[3 * (g0 + n) + 0] = om0;
          p.vort_out[3 * (g0 + n) + 1] = om1;
          p.vort_out[3 * (g0 + n) + 2] = om2;
        }
      }
      if (grad_surf) {                                // Q / |w| surfaces: OR into the pre-pass bits
        unsigned bits = 0;
        for (int s = 0; s < p.n_surf; ++s) {
          const int src = p.surf_src[s];
          if (src_is_grad(src)) bits |= ((src == SRC_Q ? vq : vw) >= p.surf_iso[s] ? 1u : 0u) << s;
        }
        S_bits[n] |= (unsigned char)bits;
      }
      if (color_grad) {
        const double c = (p.color_src == SRC_Q) ? vq : vw;
        cmin = fmin(cmin, c);
        cmax = fmax(cmax, c);
      }
    }
    pf(3);
    if (p.n_surf == 0) continue;
    group_bar(g);                                   // case bits of element k ready

    // ---- classify: cells lt and lt + 256 ----
    for (int c = lt; c < kNC; c += kGroupThreads) {
      const int a = c % kN, b = (c / kN) % kN, kk = c / (kN * kN);
      const int n0 = a + kNP * b + kNP * kNP * kk;
      unsigned cb[8];
#pragma unroll
      for (int v = 0; v < 8; ++v) cb[v] = S_bits[n0 + voff_i(v) + kNP * voff_j(v) + kNP * kNP * voff_k(v)];
      unsigned packed = 0;
      int nc = 0;
      for (int s = 0; s < p.n_surf; ++s) {
        unsigned cs = 0;
#pragma unroll
        for (int v = 0; v < 8; ++v) cs |= ((cb[v] >> s) & 1u) << v;
        packed |= cs << (8 * s);
        nc += sh.t_ntri[cs];
      }
      gs.cases[c] = packed;
      gs.ntri[c] = (unsigned char)nc;
    }
    pf(2);
  }

  if (p.prof && (lt == 0 || at == 0)) {
    long long* dst = p.prof + (long long)blockIdx.x * 16 + g * 8 + (lt == 0 ? 0 : 4);
    for (int k = 0; k < 4; ++k) dst[k] = pf_acc[k];
  }
  __syncthreads();
  if (p.mode == FUSED_FAST && p.region_count != nullptr && tid == 0) {
    p.region_count[blockIdx.x] = sh.cta_fill;
    if (sh.cta_fill) atomicAdd(&p.counters[0], sh.cta_fill);
  }
  // colour range of all elements this CTA processed: one ordered atomic pair
  if (p.color_src >= 0 && p.mode != FUSED_ORDERED) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      cmin = fmin(cmin, __shfl_xor_sync(0xffffffffu, cmin, o));
      cmax = fmax(cmax, __shfl_xor_sync(0xffffffffu, cmax, o));
    }
    if (lane == 0) {
      sh.mn[warp] = cmin;
      sh.mx[warp] = cmax;
    }
    __syncthreads();
    if (tid == 0) {
      double mn = sh.mn[0], mx = sh.mx[0];
      for (int w = 1; w < kThreads / 32; ++w) {
        mn = fmin(mn, sh.mn[w]);
        mx = fmax(mx, sh.mx[w]);
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

int fused_grid(int64_t n_elements) {
  if (g_num_sms <= 0) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      g_num_sms = 148;
  }
  int64_t g = g_num_sms;
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

static size_t fused_smem_bytes() {
  return (size_t)2 * kGroupDoubles * sizeof(double) + 2 * kNN;
}

int launch_fused(const FusedParams& p, cudaStream_t s) {
  if (p.n_elements <= 0) return NKB_OK;
  const int nst = p.need_vel ? 6 : 3;
  const size_t shm = fused_smem_bytes();
  static bool attr_set = false;
  if (!attr_set) {
    NKB_CUDA(cudaFuncSetAttribute(fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
    attr_set = true;
  }
  FusedParams q = p;   // staged inputs in slot order: x, y, z, [u, v, w]
  q.in_ptr[0] = p.x;
  q.in_ptr[1] = p.y;
  q.in_ptr[2] = p.z;
  if (p.need_vel)
    for (int c = 0; c < 3; ++c) q.in_ptr[3 + c] = p.vel[c];
  const int grid = fused_grid(p.n_elements);
  fused_kernel<<<(unsigned)grid, kThreads, shm, s>>>(q, nst);
  NKB_CUDA(cudaGetLastError());
  return NKB_OK;
}

int launch_count_scan(const int* cnt, int64_t n, long long* off, unsigned long long* total, cudaStream_t s) {
  count_scan_kernel<<<1, 1024, 0, s>>>(cnt, n, off, total);
  NKB_CUDA(cudaGetLastError());
  return NKB_OK;
}

}  // namespace nkb
