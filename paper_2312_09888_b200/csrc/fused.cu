// K1: the fused in situ pass -- SEM->VTK adaptor gather, tensor-product
// derivatives, Jacobian inverse, velocity gradient, vorticity, Q-criterion,
// marching-cubes classification of every linear sub-hex, and deterministic
// triangle emission through a single-pass decoupled look-back scan.
//
// One CTA (256 threads) per element; the element's GLL fields are read from
// HBM exactly once (coalesced, element-local order i fastest) into a
// swizzled, plane-padded shared-memory layout, and nothing but triangles (and
// optional AddArray exports) is written back.
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
constexpr int kPlane = 72;              // 64 doubles + 8 pad per k-plane
constexpr int kArr = kNP * kPlane;      // 576 doubles per staged array

// node (i,j,k) -> shared-memory slot.  XOR swizzle inside each 8-double line
// plus plane padding makes r-, s-, t-pencil reads and node-parallel accesses
// all bank-conflict free (2 wavefronts per 64-bit warp access).
__device__ __forceinline__ int sw(int i, int j, int k) {
  return (i ^ ((j >> 1) | ((k & 1) << 2))) + 8 * j + kPlane * k;
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

// derivatives of three staged arrays in[f0..f0+2] along r,s,t into d[0..8]
// (d[3*f + dir]).  576 pencils over 256 threads; (field, dir) warp-uniform.
__device__ __forceinline__ void pencils3(const double* __restrict__ in0, double* __restrict__ d,
                                         int tid) {
#pragma unroll 1
  for (int task = tid; task < 9 * 64; task += kThreads) {
    const int f = task / 192;
    const int rem = task - f * 192;
    const int dir = rem >> 6;
    const int p = rem & 63;
    const int a = p & 7, b = p >> 3;
    const double* src = in0 + f * kArr;
    double* dst = d + (3 * f + dir) * kArr;
    double v[kNP], o[kNP];
    if (dir == 0) {
#pragma unroll
      for (int m = 0; m < kNP; ++m) v[m] = src[sw(m, a, b)];
      deriv8(v, o);
#pragma unroll
      for (int m = 0; m < kNP; ++m) dst[sw(m, a, b)] = o[m];
    } else if (dir == 1) {
#pragma unroll
      for (int m = 0; m < kNP; ++m) v[m] = src[sw(a, m, b)];
      deriv8(v, o);
#pragma unroll
      for (int m = 0; m < kNP; ++m) dst[sw(a, m, b)] = o[m];
    } else {
#pragma unroll
      for (int m = 0; m < kNP; ++m) v[m] = src[sw(a, b, m)];
      deriv8(v, o);
#pragma unroll
      for (int m = 0; m < kNP; ++m) dst[sw(a, b, m)] = o[m];
    }
  }
}

__device__ __forceinline__ double mag3(double a, double b, double c) {
  // reference ':mag' = sqrt(sum(v**2)) summed left to right (sinks.py:240-241)
  return __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(a, a), __dmul_rn(b, b)), __dmul_rn(c, c)));
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace

// Shared memory: nin staged input arrays + 9 scratch arrays (kArr doubles
// each) + the 9-component Jacobian inverse per node + 512 classification
// bytes.  ~111 KB at nin=7 -> 2 CTAs (16 warps) per SM.
__global__ void __launch_bounds__(kThreads, 2) fused_kernel(const FusedParams p, int nin,
                                                            int slot_vel, int slot_sc) {
  extern __shared__ __align__(16) double smem[];
  double* S_in = smem;                 // nin * kArr
  double* S_d = smem + nin * kArr;     // 9 * kArr
  double* S_j = S_d + 9 * kArr;        // 9 * kNN: Jacobian inverse, compact [c][node]
  unsigned char* S_bits = reinterpret_cast<unsigned char*>(S_j + 9 * kNN);  // 512
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

  // ---- 1. adaptor gather: element-local GLL fields -> shared (coalesced) ----
  {
    const int q0 = sw_node(tid), q1 = sw_node(tid + kThreads);
    auto stage = [&](const double* __restrict__ src, int slot) {
      const double a0 = __ldcs(src + g0 + tid);
      const double a1 = __ldcs(src + g0 + tid + kThreads);
      S_in[slot * kArr + q0] = a0;
      S_in[slot * kArr + q1] = a1;
    };
    stage(p.x, 0);
    stage(p.y, 1);
    stage(p.z, 2);
    if (p.need_vel) {
      stage(p.vel[0], slot_vel);
      stage(p.vel[1], slot_vel + 1);
      stage(p.vel[2], slot_vel + 2);
    }
    if (p.n_scalars > 0) stage(p.scalar[0], slot_sc);
    if (p.n_scalars > 1) stage(p.scalar[1], slot_sc + 1);
  }
  __syncthreads();

  // per-node derived scalars are written into scratch slots after phase 5
  // slot map: Q -> d0, |w| -> d1, |u| -> d2, plane k -> d(3+k)
  double cmin = INFINITY, cmax = -INFINITY;

  if (p.need_grad) {
    // ---- 2. geometric derivatives x,y,z along r,s,t ----
    pencils3(S_in, S_d, tid);
    __syncthreads();
    // ---- 3. Jacobian inverse per node ----
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int q = sw_node(tid + h * kThreads);
      const double xr = S_d[0 * kArr + q], xs = S_d[1 * kArr + q], xt = S_d[2 * kArr + q];
      const double yr = S_d[3 * kArr + q], ys = S_d[4 * kArr + q], yt = S_d[5 * kArr + q];
      const double zr = S_d[6 * kArr + q], zs = S_d[7 * kArr + q], zt = S_d[8 * kArr + q];
      double K[9];
      K[0] = __fma_rn(ys, zt, -__dmul_rn(yt, zs));
      K[1] = __fma_rn(xt, zs, -__dmul_rn(xs, zt));
      K[2] = __fma_rn(xs, yt, -__dmul_rn(xt, ys));
      K[3] = __fma_rn(yt, zr, -__dmul_rn(yr, zt));
      K[4] = __fma_rn(xr, zt, -__dmul_rn(xt, zr));
      K[5] = __fma_rn(xt, yr, -__dmul_rn(xr, yt));
      K[6] = __fma_rn(yr, zs, -__dmul_rn(ys, zr));
      K[7] = __fma_rn(xs, zr, -__dmul_rn(xr, zs));
      K[8] = __fma_rn(xr, ys, -__dmul_rn(xs, yr));
      const double det = __fma_rn(zr, K[2], __fma_rn(yr, K[1], __dmul_rn(xr, K[0])));
      const double rdet = __ddiv_rn(1.0, det);
#pragma unroll
      for (int c = 0; c < 9; ++c) S_j[c * kNN + tid + h * kThreads] = __dmul_rn(K[c], rdet);
    }
    __syncthreads();
    // ---- 4. velocity derivatives u,v,w along r,s,t ----
    pencils3(S_in + slot_vel * kArr, S_d, tid);
    __syncthreads();
  }

  // ---- 5. per-node derived fields, classification bits, colour range ----
  {
#pragma unroll 1
    for (int h = 0; h < 2; ++h) {
      const int n = tid + h * kThreads;
      const int q = sw_node(n);
      double vq = 0.0, vw = 0.0, vu = 0.0;
      double om0 = 0.0, om1 = 0.0, om2 = 0.0;
      if (p.need_grad) {
        double U[9], J[9];
#pragma unroll
        for (int c = 0; c < 9; ++c) U[c] = S_d[c * kArr + q];
#pragma unroll
        for (int c = 0; c < 9; ++c) J[c] = S_j[c * kNN + n];
        double A[9];
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int b = 0; b < 3; ++b)
            A[3 * a + b] = __fma_rn(U[3 * a + 2], J[6 + b],
                                    __fma_rn(U[3 * a + 1], J[3 + b],
                                             __dmul_rn(U[3 * a + 0], J[0 + b])));
        const double off = __fma_rn(A[5], A[7], __fma_rn(A[2], A[6], __dmul_rn(A[1], A[3])));
        const double dia = __fma_rn(A[8], A[8], __fma_rn(A[4], A[4], __dmul_rn(A[0], A[0])));
        vq = -__fma_rn(0.5, dia, off);
        om0 = __dsub_rn(A[7], A[5]);
        om1 = __dsub_rn(A[2], A[6]);
        om2 = __dsub_rn(A[3], A[1]);
        vw = mag3(om0, om1, om2);
        S_d[0 * kArr + q] = vq;
        S_d[1 * kArr + q] = vw;
        if (p.q_out) p.q_out[g0 + n] = vq;
        if (p.wmag_out) p.wmag_out[g0 + n] = vw;
        if (p.vort_out) {
          p.vort_out[3 * (g0 + n) + 0] = om0;
          p.vort_out[3 * (g0 + n) + 1] = om1;
          p.vort_out[3 * (g0 + n) + 2] = om2;
        }
      }
      if (p.need_vel) {
        vu = mag3(S_in[slot_vel * kArr + q], S_in[(slot_vel + 1) * kArr + q],
                  S_in[(slot_vel + 2) * kArr + q]);
        S_d[2 * kArr + q] = vu;
      }
      const double px = S_in[0 * kArr + q], py = S_in[1 * kArr + q], pz = S_in[2 * kArr + q];
      unsigned bits = 0;
      for (int s = 0; s < p.n_surf; ++s) {
        const int src = p.surf_src[s];
        double val;
        if (src >= SRC_PLANE) {
          val = __fma_rn(p.surf_n[s][2], pz, __fma_rn(p.surf_n[s][1], py, __dmul_rn(p.surf_n[s][0], px)));
          S_d[(3 + (src - SRC_PLANE)) * kArr + q] = val;
        } else if (src == SRC_Q) {
          val = vq;
        } else if (src == SRC_WMAG) {
          val = vw;
        } else if (src == SRC_UMAG) {
          val = vu;
        } else {
          val = S_in[(slot_sc + src - SRC_SCALAR0) * kArr + q];
        }
        bits |= (val >= p.surf_iso[s] ? 1u : 0u) << s;
      }
      S_bits[n] = (unsigned char)bits;
      if (p.color_src >= 0) {
        const int src = p.color_src;
        double c = (src == SRC_Q)      ? vq
                   : (src == SRC_WMAG) ? vw
                   : (src == SRC_UMAG) ? vu
                                       : S_in[(slot_sc + src - SRC_SCALAR0) * kArr + q];
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
    atomicMin(&p.counters[1], enc_ordered(mn));
    atomicMax(&p.counters[2], enc_ordered(mx));
  }
  if (p.n_surf == 0) return;

  // ---- 6. classify sub-hexes: thread t owns cells 2t, 2t+1 ----
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
      for (int v = 0; v < 8; ++v)
        cb[v] = S_bits[n0 + voff_i(v) + kNP * voff_j(v) + kNP * kNP * voff_k(v)];
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

  // ---- 7. block exclusive scan + decoupled look-back across elements ----
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
    // publish aggregate, then look back
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

  // ---- 8. emit triangles (vertex interpolation along canonical edges) ----
  if (cnt == 0) return;
  const double* Sx = S_in;
  const double* Sy = S_in + kArr;
  const double* Sz = S_in + 2 * kArr;
  const double* Sc;
  {
    const int src = p.color_src;
    Sc = (src == SRC_Q)      ? S_d
         : (src == SRC_WMAG) ? S_d + kArr
         : (src == SRC_UMAG) ? S_d + 2 * kArr
                             : S_in + (slot_sc + src - SRC_SCALAR0) * kArr;
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int c = 2 * tid + h;
    if (c >= kNC) break;
    const int a = c % kN, b = (c / kN) % kN, cc = c / (kN * kN);
    for (int s = 0; s < p.n_surf; ++s) {
      const unsigned cs = (cases[h] >> (8 * s)) & 0xffu;
      const int nt = g_mc_ntri[cs];
      if (nt == 0) continue;
      const int src = p.surf_src[s];
      const double* Ss = (src >= SRC_PLANE) ? S_d + (3 + src - SRC_PLANE) * kArr
                         : (src == SRC_Q)   ? S_d
                         : (src == SRC_WMAG) ? S_d + kArr
                         : (src == SRC_UMAG) ? S_d + 2 * kArr
                                             : S_in + (slot_sc + src - SRC_SCALAR0) * kArr;
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
          const double sa = Ss[qa], sb = Ss[qb];
          const double t = __ddiv_rn(__dsub_rn(iso, sa), __dsub_rn(sb, sa));
          vtx[r].x = __double2float_rn(__fma_rn(t, __dsub_rn(Sx[qb], Sx[qa]), Sx[qa]));
          vtx[r].y = __double2float_rn(__fma_rn(t, __dsub_rn(Sy[qb], Sy[qa]), Sy[qa]));
          vtx[r].z = __double2float_rn(__fma_rn(t, __dsub_rn(Sz[qb], Sz[qa]), Sz[qa]));
          vtx[r].w = __double2float_rn(__fma_rn(t, __dsub_rn(Sc[qb], Sc[qa]), Sc[qa]));
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
  size_t shm = (size_t)(nin + 9) * kArr * sizeof(double) + 9 * kNN * sizeof(double) + kNN;
  static bool attr_set = false;
  if (!attr_set) {
    NKB_CUDA(cudaFuncSetAttribute(fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)((3 + 3 + kMaxScalars + 9) * kArr * sizeof(double) +
                                        9 * kNN * sizeof(double) + kNN)));
    attr_set = true;
  }
  fused_kernel<<<(unsigned)p.n_elements, kThreads, shm, s>>>(p, nin, slot_vel, slot_sc);
  NKB_CUDA(cudaGetLastError());
  return NKB_OK;
}

}  // namespace nkb
