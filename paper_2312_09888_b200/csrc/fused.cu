// K1: the fused in situ pass -- SEM->VTK adaptor gather, tensor-product
// derivatives, Jacobian inverse, velocity gradient, vorticity, Q-criterion,
// marching-cubes classification of every linear sub-hex, and deterministic
// triangle emission through a single-pass decoupled look-back scan.
//
// One CTA (256 threads, 8 warps) per element; 2 CTAs per SM.  The element's
// GLL fields are read from HBM exactly once (coalesced) into XOR-swizzled
// shared-memory arrays (bank-conflict free for node-, r-, s- and t-pencil
// access), nothing but triangles (and optional AddArray exports) is written.
//
//   1. gather     : 7 fields (x,y,z,u,v,w,T) -> smem                 all warps
//   2. pencils    : 6 fields x 3 directions, one (dir, pencil) per   warps 0-5
//                   thread, smem offsets computed once, 6 fields
//      node-local : |u|, plane and scalar classification bits,       warps 6-7
//                   colour range of non-derived colour fields
//   3. node phase : Jacobian inverse, grad u, Q, |w|, Q/|w| bits      all warps
//   4. classify   : 343 sub-hexes x surfaces -> case bytes, counts
//   5. scan       : block scan + decoupled look-back across elements
//   6. emit       : vertices interpolated along canonical edges
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

// MC tables in global memory (read-only path; divergent indices)
__device__ const unsigned char g_mc_ntri[256] = {NKB_MC_NTRI_DATA};
__device__ const signed char g_mc_tri[256][3 * NKB_MC_MAX_TRI] = {NKB_MC_TRI_DATA};
__device__ const unsigned char g_mc_edge_v[12][2] = {NKB_MC_EDGE_V_DATA};

int set_dmat_constant(const double* dmat) {
  NKB_CUDA(cudaMemcpyToSymbol(c_D, dmat, sizeof(double) * kNP * kNP));
  return NKB_OK;
}

namespace {

constexpr int kThreads = 256;
constexpr int kArr = kNN;            // 512 doubles per staged array
constexpr int kNumD = 18;            // derivative arrays: d(f)/d(r,s,t) for x,y,z,u,v,w

// node (i,j,k) -> shared-memory slot.  Within each 64 B line the 8 doubles
// are XOR-permuted by (j>>1 | (k&1)<<2); lines are XOR-permuted by (k&1).
// For every 16-lane half-warp pattern used below (node-parallel, r-, s- and
// t-pencils) the 16 accessed doubles fall in 16 distinct 8-byte bank pairs:
// 2 wavefronts per 64-bit warp access, the minimum.
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

__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

constexpr unsigned long long kFlagAgg = 1ULL << 62;
constexpr unsigned long long kFlagPre = 2ULL << 62;
constexpr unsigned long long kValMask = (1ULL << 62) - 1;

// 8-point derivative of one pencil: out[i] = sum_m D[i][m] v[m], m ascending,
// first term a plain product then fma -- mirrored by oracle deriv8().
__device__ __forceinline__ void deriv8(const double* v, double* out) {
#pragma unroll
  for (int i = 0; i < kNP; ++i) {
    double acc = __dmul_rn(c_D[i * kNP + 0], v[0]);
#pragma unroll
    for (int m = 1; m < kNP; ++m) acc = __fma_rn(c_D[i * kNP + m], v[m], acc);
    out[i] = acc;
  }
}

__device__ __forceinline__ double mag3(double a, double b, double c) {
  // reference ':mag' = sqrt(sum(v**2)) summed left to right (sinks.py:240-241)
  return __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(a, a), __dmul_rn(b, b)), __dmul_rn(c, c)));
}

__device__ __forceinline__ double plane_dist(const double* n, double x, double y, double z) {
  return __fma_rn(n[2], z, __fma_rn(n[1], y, __dmul_rn(n[0], x)));
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ bool src_is_grad(int s) { return s == SRC_Q || s == SRC_WMAG; }

}  // namespace

// smem: nin staged inputs + 18 derivative arrays (4 KB each) + 512 case bits
__global__ void __launch_bounds__(kThreads, 2) fused_kernel(const FusedParams p, int nin,
                                                            int slot_vel, int slot_sc) {
  extern __shared__ __align__(16) double smem[];
  double* S_in = smem;                                 // nin * 512
  double* S_d = smem + nin * kArr;                     // 18 * 512
  unsigned char* S_bits = reinterpret_cast<unsigned char*>(S_d + kNumD * kArr);
  __shared__ unsigned s_tile;
  __shared__ long long s_warp[kThreads / 32];
  __shared__ long long s_base;
  __shared__ double s_mn[kThreads / 32], s_mx[kThreads / 32];

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_tile = atomicAdd(p.ticket, 1u);
  __syncthreads();
  const long long e = s_tile;
  const long long g0 = e * (long long)kNN;
  const bool color_grad = src_is_grad(p.color_src);

  // ---- 1. adaptor gather: element-local GLL fields -> shared (coalesced) ----
  // all loads are issued before any store so every thread keeps up to 16
  // independent 8-byte loads in flight (memory-level parallelism)
  {
    double r0[8], r1[8];
#pragma unroll
    for (int f = 0; f < 8; ++f) {
      if (f < nin) {
        r0[f] = __ldcs(p.in_ptr[f] + g0 + tid);
        r1[f] = __ldcs(p.in_ptr[f] + g0 + tid + kThreads);
      }
    }
    const int q0 = sw_node(tid), q1 = sw_node(tid + kThreads);
#pragma unroll
    for (int f = 0; f < 8; ++f) {
      if (f < nin) {
        S_in[f * kArr + q0] = r0[f];
        S_in[f * kArr + q1] = r1[f];
      }
    }
  }
  __syncthreads();

  double cmin = INFINITY, cmax = -INFINITY;
  if (warp < 6) {
    // ---- 2a. derivative pencils: thread = (dir, pencil); 6 fields ----
    if (p.need_grad) {
      const int dir = warp >> 1;               // warp-uniform
      const int pa = tid & 7, pb = (tid >> 3) & 7;
      int off[kNP];
#pragma unroll
      for (int m = 0; m < kNP; ++m)
        off[m] = (dir == 0) ? sw(m, pa, pb) : (dir == 1) ? sw(pa, m, pb) : sw(pa, pb, m);
#pragma unroll 1
      for (int f = 0; f < 6; ++f) {
        const double* src = S_in + (f < 3 ? f : slot_vel + f - 3) * kArr;
        double* dst = S_d + (3 * f + dir) * kArr;
        double v[kNP], o[kNP];
#pragma unroll
        for (int m = 0; m < kNP; ++m) v[m] = src[off[m]];
        deriv8(v, o);
#pragma unroll
        for (int m = 0; m < kNP; ++m) dst[off[m]] = o[m];
      }
    }
  } else {
    // ---- 2b. node-local work that needs no derivatives (64 threads) ----
    for (int n = tid - 192; n < kNN; n += 64) {
      const int q = sw_node(n);
      const double px = S_in[q], py = S_in[kArr + q], pz = S_in[2 * kArr + q];
      double vu = 0.0;
      if (p.need_vel)
        vu = mag3(S_in[slot_vel * kArr + q], S_in[(slot_vel + 1) * kArr + q], S_in[(slot_vel + 2) * kArr + q]);
      unsigned bits = 0;
      for (int s = 0; s < p.n_surf; ++s) {
        const int src = p.surf_src[s];
        if (src_is_grad(src)) continue;
        const double val = (src >= SRC_PLANE) ? plane_dist(p.surf_n[s], px, py, pz)
                           : (src == SRC_UMAG) ? vu
                                               : S_in[(slot_sc + src - SRC_SCALAR0) * kArr + q];
        bits |= (val >= p.surf_iso[s] ? 1u : 0u) << s;
      }
      S_bits[n] = (unsigned char)bits;
      if (p.color_src >= 0 && !color_grad) {
        const double c = (p.color_src == SRC_UMAG) ? vu : S_in[(slot_sc + p.color_src - SRC_SCALAR0) * kArr + q];
        cmin = fmin(cmin, c);
        cmax = fmax(cmax, c);
      }
    }
  }
  __syncthreads();

  // ---- 3. node phase: Jacobian inverse, grad u, Q, |w| (2 nodes / thread) ----
  if (p.need_grad) {
#pragma unroll 1
    for (int h = 0; h < 2; ++h) {
      const int n = tid + h * kThreads;
      const int q = sw_node(n);
      double G[9];
#pragma unroll
      for (int c = 0; c < 9; ++c) G[c] = S_d[c * kArr + q];
      const double xr = G[0], xs = G[1], xt = G[2];
      const double yr = G[3], ys = G[4], yt = G[5];
      const double zr = G[6], zs = G[7], zt = G[8];
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
      const double rdet = __ddiv_rn(1.0, det);
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
      const double vq = -__fma_rn(0.5, dia, off);
      const double om0 = __dsub_rn(A[7], A[5]);
      const double om1 = __dsub_rn(A[2], A[6]);
      const double om2 = __dsub_rn(A[3], A[1]);
      const double vw = mag3(om0, om1, om2);
      // this thread owns node q's derivative slots: overwrite d0 <- Q, d1 <- |w|
      S_d[0 * kArr + q] = vq;
      S_d[1 * kArr + q] = vw;
      if (p.q_out) p.q_out[g0 + n] = vq;
      if (p.wmag_out) p.wmag_out[g0 + n] = vw;
      if (p.vort_out) {
        p.vort_out[3 * (g0 + n) + 0] = om0;
        p.vort_out[3 * (g0 + n) + 1] = om1;
        p.vort_out[3 * (g0 + n) + 2] = om2;
      }
      unsigned bits = 0;
      for (int s = 0; s < p.n_surf; ++s) {
        const int src = p.surf_src[s];
        if (!src_is_grad(src)) continue;
        bits |= ((src == SRC_Q ? vq : vw) >= p.surf_iso[s] ? 1u : 0u) << s;
      }
      if (bits) S_bits[n] |= (unsigned char)bits;
      if (color_grad) {
        const double c = (p.color_src == SRC_Q) ? vq : vw;
        cmin = fmin(cmin, c);
        cmax = fmax(cmax, c);
      }
    }
  }
  if (p.n_surf == 0 && p.color_src < 0) return;   // export-only run (AddArray)

  // colour range: block reduce -> one ordered atomic per CTA
  if (p.color_src >= 0) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      cmin = fmin(cmin, __shfl_xor_sync(0xffffffffu, cmin, o));
      cmax = fmax(cmax, __shfl_xor_sync(0xffffffffu, cmax, o));
    }
    if (lane == 0) {
      s_mn[warp] = cmin;
      s_mx[warp] = cmax;
    }
  }
  __syncthreads();
  if (p.color_src >= 0 && tid == 0) {
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
  if (p.n_surf == 0) return;

  // ---- 4. classify sub-hexes: thread t owns cells 2t, 2t+1 ----
  unsigned cases[2] = {0u, 0u};   // byte s = case of surface s
  int cnt = 0;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int c = 2 * tid + h;
    if (c < kNC) {
      const int a = c % kN, b = (c / kN) % kN, cc = c / (kN * kN);
      const int n0 = a + kNP * b + kNP * kNP * cc;
      unsigned cb[8];
#pragma unroll
      for (int v = 0; v < 8; ++v) cb[v] = S_bits[n0 + voff_i(v) + kNP * voff_j(v) + kNP * kNP * voff_k(v)];
      unsigned packed = 0;
      for (int s = 0; s < p.n_surf; ++s) {
        unsigned cs = 0;
#pragma unroll
        for (int v = 0; v < 8; ++v) cs |= ((cb[v] >> s) & 1u) << v;
        packed |= cs << (8 * s);
        cnt += g_mc_ntri[cs];
      }
      cases[h] = packed;
    }
  }

  // ---- 5. block exclusive scan + decoupled look-back across elements ----
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    long long wv = (lane < kThreads / 32) ? s_warp[lane] : 0;
    long long wi = wv;
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      long long t = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += t;
    }
    const long long total = __shfl_sync(0xffffffffu, wi, 7);
    if (lane < kThreads / 32) s_warp[lane] = wi - wv;   // exclusive warp offsets
    const long long tile = e;
    if (lane == 0) {
      if (tile == 0) st_release(&p.tile_status[0], kFlagPre | (unsigned long long)total);
      else st_release(&p.tile_status[tile], kFlagAgg | (unsigned long long)total);
      if (total) atomicAdd(&p.counters[0], (unsigned long long)total);
    }
    long long excl = 0;
    if (tile > 0) {
      long long j = tile - 1;
      while (true) {
        const long long idx = j - lane;
        unsigned long long st = kFlagPre;   // before element 0: prefix 0
        if (idx >= 0) {
          do {
            st = ld_acquire(&p.tile_status[idx]);
          } while ((st >> 62) == 0);
        }
        const unsigned pre = __ballot_sync(0xffffffffu, (st >> 62) == 2);
        const int stop = pre ? (__ffs(pre) - 1) : 32;
        long long val = (lane <= stop) ? (long long)(st & kValMask) : 0;
        excl += warp_sum(val);
        if (pre) break;
        j -= 32;
      }
      if (lane == 0) st_release(&p.tile_status[tile], kFlagPre | (unsigned long long)(excl + total));
    }
    if (lane == 0) s_base = excl;
  }
  __syncthreads();
  long long out = s_base + s_warp[warp] + (incl - cnt);

  // ---- 6. emit triangles (vertex interpolation along canonical edges) ----
  if (cnt == 0) return;
  const double* Sx = S_in;
  const double* Sy = S_in + kArr;
  const double* Sz = S_in + 2 * kArr;
  const double* Su = S_in + slot_vel * kArr;
  // per-node scalar of a source, recomputed where it is not stored
  auto value_at = [&](int src, int s, int q) -> double {
    if (src >= SRC_PLANE) return plane_dist(p.surf_n[s], Sx[q], Sy[q], Sz[q]);
    if (src == SRC_Q) return S_d[q];
    if (src == SRC_WMAG) return S_d[kArr + q];
    if (src == SRC_UMAG) return mag3(Su[q], Su[kArr + q], Su[2 * kArr + q]);
    return S_in[(slot_sc + src - SRC_SCALAR0) * kArr + q];
  };
#pragma unroll 1
  for (int h = 0; h < 2; ++h) {
    const int c = 2 * tid + h;
    if (c >= kNC) break;
    const int a = c % kN, b = (c / kN) % kN, cc = c / (kN * kN);
    for (int s = 0; s < p.n_surf; ++s) {
      const unsigned cs = (cases[h] >> (8 * s)) & 0xffu;
      const int nt = g_mc_ntri[cs];
      if (nt == 0) continue;
      const int src = p.surf_src[s];
      const double iso = p.surf_iso[s];
      for (int k = 0; k < nt; ++k, ++out) {
        if (out >= p.tri_cap) continue;
        float4 vtx[3];
#pragma unroll
        for (int r = 0; r < 3; ++r) {
          const int ed = g_mc_tri[cs][3 * k + r];
          const int va = g_mc_edge_v[ed][0], vb = g_mc_edge_v[ed][1];
          const int qa = sw(a + voff_i(va), b + voff_j(va), cc + voff_k(va));
          const int qb = sw(a + voff_i(vb), b + voff_j(vb), cc + voff_k(vb));
          const double sa = value_at(src, s, qa), sb = value_at(src, s, qb);
          const double t = __ddiv_rn(__dsub_rn(iso, sa), __dsub_rn(sb, sa));
          const double ca = value_at(p.color_src, 0, qa), cb = value_at(p.color_src, 0, qb);
          vtx[r].x = __double2float_rn(__fma_rn(t, __dsub_rn(Sx[qb], Sx[qa]), Sx[qa]));
          vtx[r].y = __double2float_rn(__fma_rn(t, __dsub_rn(Sy[qb], Sy[qa]), Sy[qa]));
          vtx[r].z = __double2float_rn(__fma_rn(t, __dsub_rn(Sz[qb], Sz[qa]), Sz[qa]));
          vtx[r].w = __double2float_rn(__fma_rn(t, __dsub_rn(cb, ca), ca));
        }
        float4* dst = p.tri + 3 * out;
        dst[0] = vtx[0];
        dst[1] = vtx[1];
        dst[2] = vtx[2];
        if (p.meta)
          p.meta[out] = ((unsigned long long)e << 32) | ((unsigned long long)c << 16) |
                        ((unsigned long long)s << 12) | ((unsigned long long)k << 8) | cs;
      }
    }
  }
}

int launch_fused(const FusedParams& p, cudaStream_t s) {
  if (p.n_elements <= 0) return NKB_OK;
  int nin = 3 + (p.need_vel ? 3 : 0) + p.n_scalars;
  int slot_vel = 3;
  int slot_sc = 3 + (p.need_vel ? 3 : 0);
  size_t shm = (size_t)(nin + kNumD) * kArr * sizeof(double) + kNN;
  static bool attr_set = false;
  if (!attr_set) {
    NKB_CUDA(cudaFuncSetAttribute(fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)((3 + 3 + kMaxScalars + kNumD) * kArr * sizeof(double) + kNN)));
    attr_set = true;
  }
  FusedParams q = p;   // staged inputs in slot order: x, y, z, [u, v, w], [scalars]
  int k = 0;
  q.in_ptr[k++] = p.x;
  q.in_ptr[k++] = p.y;
  q.in_ptr[k++] = p.z;
  if (p.need_vel)
    for (int c = 0; c < 3; ++c) q.in_ptr[k++] = p.vel[c];
  for (int c = 0; c < p.n_scalars; ++c) q.in_ptr[k++] = p.scalar[c];
  fused_kernel<<<(unsigned)p.n_elements, kThreads, shm, s>>>(q, nin, slot_vel, slot_sc);
  NKB_CUDA(cudaGetLastError());
  return NKB_OK;
}

}  // namespace nkb
