// GetMesh / AddArray export kernels: the explicit VTK form of the SEM
// adaptor (R11).  Pure data movement, HBM-bound.
//
// Reference anchors: component-fastest AoS layout `flat = c + comps*point`
// (data_model.py:8-14), FieldArray export (data_model.py:27-55),
// scalar_field ':mag' (sinks.py:227-242).  VTK_HEXAHEDRON corner order
// (0,0,0),(1,0,0),(1,1,0),(0,1,0) then the same at +k is the VTK convention
// (SURVEY.md §8a R11 [ext]); point ids are element-local GLL ids
// e*(N+1)^3 + i + (N+1)*(j + (N+1)*k).
#include <cuda_runtime.h>

#include "nkb_internal.h"

namespace nkb {

namespace {

inline unsigned grid_for(long long n, int threads) {
  long long b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > 148 * 32) b = 148 * 32;
  return (unsigned)b;
}

// Connectivity, CELLS and field AoS exports are written OUTPUT-major: thread
// o stores output word o (item o / K, word o % K), so every warp store is
// one contiguous run instead of K-word strides the L2 has to merge (C2:
// connectivity 2.8 -> 4.3 TB/s, velocity AoS 3.8 -> 4.6 TB/s).  The points
// (3 coalesced loads, 3 strided stores per thread) measured faster as is
// (5.1 vs 4.6 TB/s).
__global__ void points_aos_kernel(const double* __restrict__ x, const double* __restrict__ y,
                                  const double* __restrict__ z, long long n, double* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double a = __ldcs(x + i), b = __ldcs(y + i), c = __ldcs(z + i);
    out[3 * i + 0] = a;
    out[3 * i + 1] = b;
    out[3 * i + 2] = c;
  }
}

// first point id of sub-hex c, and the id of its VTK_HEXAHEDRON corner v
__device__ __forceinline__ long long cell_n0(long long c) {
  const long long e = c / kNC;
  const int l = (int)(c - e * kNC);
  const int a = l % kN, b = (l / kN) % kN, k = l / (kN * kN);
  return e * kNN + a + kNP * b + kNP * kNP * k;
}
__device__ __forceinline__ int corner_off(int v) {   // (0,0,0),(1,0,0),(1,1,0),(0,1,0), then +k
  return ((v ^ (v >> 1)) & 1) + kNP * ((v >> 1) & 1) + kNP * kNP * (v >> 2);
}

__global__ void connectivity_kernel(long long ncells, long long* __restrict__ conn,
                                    long long* __restrict__ offsets, unsigned char* __restrict__ types) {
  const long long stride = (long long)gridDim.x * blockDim.x, t0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (conn)
    for (long long o = t0; o < 8 * ncells; o += stride)   // output-major: word o = corner o%8 of cell o/8
      conn[o] = cell_n0(o >> 3) + corner_off((int)(o & 7));
  for (long long c = t0; c < ncells; c += stride) {
    if (offsets) {
      offsets[c] = 8 * c;
      if (c == ncells - 1) offsets[ncells] = 8 * ncells;
    }
    if (types) types[c] = NKB_VTK_HEXAHEDRON;
  }
}

template <int kComp>   // 0: runtime ncomp
__global__ void field_aos_kernel(const double* __restrict__ base, long long stride, int ncomp,
                                 long long n, double* __restrict__ out) {
  const int nc = kComp ? kComp : ncomp;
  for (long long o = blockIdx.x * (long long)blockDim.x + threadIdx.x; o < nc * n;
       o += (long long)gridDim.x * blockDim.x) {
    const long long i = o / nc;
    const int c = (int)(o - nc * i);
    out[o] = __ldcs(base + c * stride + i);
  }
}

__global__ void field_mag_kernel(const double* __restrict__ base, long long stride, int ncomp,
                                 long long n, double* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double v0 = __ldcs(base + i);
    double acc = __dmul_rn(v0, v0);
    for (int c = 1; c < ncomp; ++c) {
      const double v = __ldcs(base + c * stride + i);
      acc = __dadd_rn(acc, __dmul_rn(v, v));
    }
    out[i] = __dsqrt_rn(acc);
  }
}

// ---- big-endian sections of a legacy-VTK UNSTRUCTURED_GRID (checkpoint) ----
__device__ __forceinline__ unsigned long long bswap64(unsigned long long v) {
  const unsigned lo = (unsigned)v, hi = (unsigned)(v >> 32);
  return ((unsigned long long)__byte_perm(lo, 0, 0x0123) << 32) | __byte_perm(hi, 0, 0x0123);
}
__device__ __forceinline__ unsigned bswap32(unsigned v) { return __byte_perm(v, 0, 0x0123); }

__global__ void be_points_kernel(const double* __restrict__ x, const double* __restrict__ y,
                                 const double* __restrict__ z, long long n, unsigned long long* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    out[3 * i + 0] = bswap64((unsigned long long)__double_as_longlong(__ldcs(x + i)));
    out[3 * i + 1] = bswap64((unsigned long long)__double_as_longlong(__ldcs(y + i)));
    out[3 * i + 2] = bswap64((unsigned long long)__double_as_longlong(__ldcs(z + i)));
  }
}

// CELLS section: per cell int32 {8, 8 point ids} (VTK_HEXAHEDRON corner order)
__global__ void be_cells_kernel(long long ncells, unsigned* __restrict__ out) {
  for (long long o = blockIdx.x * (long long)blockDim.x + threadIdx.x; o < 9 * ncells;
       o += (long long)gridDim.x * blockDim.x) {   // output-major: word o%9 of cell o/9
    const long long c = o / 9;
    const int w = (int)(o - 9 * c);
    out[o] = bswap32(w == 0 ? 8u : (unsigned)(cell_n0(c) + corner_off(w - 1)));
  }
}

__global__ void be_types_kernel(long long ncells, unsigned* __restrict__ out) {
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < ncells;
       c += (long long)gridDim.x * blockDim.x)
    out[c] = bswap32((unsigned)NKB_VTK_HEXAHEDRON);
}

__global__ void bswap64_kernel(unsigned long long* p, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    p[i] = bswap64(p[i]);
}

__device__ __forceinline__ unsigned long long enc_ordered(double d) {
  unsigned long long b = (unsigned long long)__double_as_longlong(d);
  return (b & 0x8000000000000000ULL) ? ~b : (b | 0x8000000000000000ULL);
}

// enc6 = {enc(min x), enc(min y), enc(min z), ~enc(max x), ~enc(max y), ~enc(max z)}:
// every word is a running minimum, so ranks combine with one ncclMin.
__global__ void bounds_kernel(const double* __restrict__ x, const double* __restrict__ y,
                              const double* __restrict__ z, long long n, unsigned long long* enc6) {
  double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double v[3] = {x[i], y[i], z[i]};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      mn[a] = fmin(mn[a], v[a]);
      mx[a] = fmax(mx[a], v[a]);
    }
  }
#pragma unroll
  for (int a = 0; a < 3; ++a) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      mn[a] = fmin(mn[a], __shfl_xor_sync(0xffffffffu, mn[a], o));
      mx[a] = fmax(mx[a], __shfl_xor_sync(0xffffffffu, mx[a], o));
    }
  }
  if ((threadIdx.x & 31) == 0 && mn[0] <= mx[0]) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      atomicMin(&enc6[a], enc_ordered(mn[a]));
      atomicMin(&enc6[3 + a], ~enc_ordered(mx[a]));
    }
  }
}

}  // namespace

int launch_bounds_kernel(const double* x, const double* y, const double* z, int64_t n,
                         unsigned long long* enc6, cudaStream_t s) {
  if (n <= 0) return NKB_OK;
  bounds_kernel<<<grid_for(n, 256), 256, 0, s>>>(x, y, z, n, enc6);
  NKB_CUDA(cudaGetLastError());
  return NKB_OK;
}

int launch_be_points(const double* x, const double* y, const double* z, int64_t npts, void* out, cudaStream_t s) {
  if (npts <= 0) return NKB_OK;
  be_points_kernel<<<grid_for(npts, 256), 256, 0, s>>>(x, y, z, npts, reinterpret_cast<unsigned long long*>(out));
  NKB_CUDA(cudaGetLastError());
  return NKB_OK;
}

int launch_be_cells(int64_t ncells, void* out, cudaStream_t s) {
  if (ncells <= 0) return NKB_OK;
  be_cells_kernel<<<grid_for(9 * ncells, 256), 256, 0, s>>>(ncells, reinterpret_cast<unsigned*>(out));
  NKB_CUDA(cudaGetLastError());
  return NKB_OK;
}

int launch_be_types(int64_t ncells, void* out, cudaStream_t s) {
  if (ncells <= 0) return NKB_OK;
  be_types_kernel<<<grid_for(ncells, 256), 256, 0, s>>>(ncells, reinterpret_cast<unsigned*>(out));
  NKB_CUDA(cudaGetLastError());
  return NKB_OK;
}

int launch_bswap64(void* p, int64_t n, cudaStream_t s) {
  if (n <= 0) return NKB_OK;
  bswap64_kernel<<<grid_for(n, 256), 256, 0, s>>>(reinterpret_cast<unsigned long long*>(p), n);
  NKB_CUDA(cudaGetLastError());
  return NKB_OK;
}

int launch_points_aos(const double* x, const double* y, const double* z, int64_t npts, double* out,
                      cudaStream_t s) {
  points_aos_kernel<<<grid_for(npts, 256), 256, 0, s>>>(x, y, z, npts, out);
  NKB_CUDA(cudaGetLastError());
  return NKB_OK;
}

int launch_connectivity(int64_t ncells, int64_t* conn, int64_t* offsets, unsigned char* types,
                        cudaStream_t s) {
  connectivity_kernel<<<grid_for(8 * ncells, 256), 256, 0, s>>>(
      ncells, reinterpret_cast<long long*>(conn), reinterpret_cast<long long*>(offsets), types);
  NKB_CUDA(cudaGetLastError());
  return NKB_OK;
}

int launch_field_aos(const double* base, int64_t stride, int ncomp, int64_t npts, double* out,
                     cudaStream_t s) {
  const unsigned g = grid_for(npts * ncomp, 256);
  if (ncomp == 1) field_aos_kernel<1><<<g, 256, 0, s>>>(base, stride, ncomp, npts, out);
  else if (ncomp == 3) field_aos_kernel<3><<<g, 256, 0, s>>>(base, stride, ncomp, npts, out);
  else field_aos_kernel<0><<<g, 256, 0, s>>>(base, stride, ncomp, npts, out);
  NKB_CUDA(cudaGetLastError());
  return NKB_OK;
}

int launch_field_mag(const double* base, int64_t stride, int ncomp, int64_t npts, double* out,
                     cudaStream_t s) {
  field_mag_kernel<<<grid_for(npts, 256), 256, 0, s>>>(base, stride, ncomp, npts, out);
  NKB_CUDA(cudaGetLastError());
  return NKB_OK;
}

}  // namespace nkb
