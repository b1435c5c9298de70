// Device helpers shared by the in situ passes (fused.cu: K1 with gradients,
// stream.cu: K1s without).  Every floating-point operation here is restated
// in the same order by the CPU oracle (oracle/sem_oracle.c), so both kernels
// give bit-identical node values, case indices and triangle vertices.
#pragma once

#include <cuda_runtime.h>

namespace nkb {
namespace dev {

__device__ __forceinline__ double mag3(double a, double b, double c) {
  // reference ':mag' = sqrt(sum(v**2)) summed left to right (sinks.py:240-241)
  return __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(a, a), __dmul_rn(b, b)), __dmul_rn(c, c)));
}

__device__ __forceinline__ double plane_dist(const double* n, double x, double y, double z) {
  return __fma_rn(n[2], z, __fma_rn(n[1], y, __dmul_rn(n[0], x)));
}

// Velocity gradient A[3a + b] = sum_d U[3a + d] J[3d + b] (U[3a + d] =
// du_a/dr_d, J = d(r,s,t)/d(x,y,z)), oracle chain_rule.  When J is block
// diagonal -- J2 = J5 = J6 = J7 = +0 exactly, jinv's block branch and every
// node of the compact cache -- the zero terms are skipped; otherwise the
// 3-term fma chain in d order.
__device__ __forceinline__ bool jinv_is_block(const double* J) {
  return (__double_as_longlong(J[2]) | __double_as_longlong(J[5]) | __double_as_longlong(J[6]) |
          __double_as_longlong(J[7])) == 0;
}
__device__ __forceinline__ void chain_rule_block(const double* U, const double* J, double* A) {
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    A[3 * a + 0] = __fma_rn(U[3 * a + 1], J[3], __dmul_rn(U[3 * a + 0], J[0]));
    A[3 * a + 1] = __fma_rn(U[3 * a + 1], J[4], __dmul_rn(U[3 * a + 0], J[1]));
    A[3 * a + 2] = __dmul_rn(U[3 * a + 2], J[8]);
  }
}
__device__ __forceinline__ void chain_rule(const double* U, const double* J, double* A) {
  if (jinv_is_block(J)) {
    chain_rule_block(U, J, A);
    return;
  }
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b)
      A[3 * a + b] = __fma_rn(U[3 * a + 2], J[6 + b], __fma_rn(U[3 * a + 1], J[3 + b], __dmul_rn(U[3 * a + 0], J[0 + b])));
}

// VTK_HEXAHEDRON corner v -> lattice offset (matches NKB_MC_VERT_OFF_DATA)
__device__ __forceinline__ int voff_i(int v) { return (v ^ (v >> 1)) & 1; }
__device__ __forceinline__ int voff_j(int v) { return (v >> 1) & 1; }
__device__ __forceinline__ int voff_k(int v) { return v >> 2; }

// case byte of surface s from the 8 corner bit-bytes packed in w (byte v =
// bits of corner v): gather bit s of every byte into one byte (bit v)
__device__ __forceinline__ unsigned case_of(unsigned long long w, int s) {
  return (unsigned)((((w >> s) & 0x0101010101010101ULL) * 0x0102040810204080ULL) >> 56);
}

// the 8 corner bytes of sub-hex (a,b,k) in VTK order from 4 node rows of
// case bits (8 bytes each, node order): row(b,k) -> v0 v1, row(b+1,k) ->
// v3 v2, row(b,k+1) -> v4 v5, row(b+1,k+1) -> v7 v6
__device__ __forceinline__ unsigned long long corner_bytes(const unsigned long long* rows, int a, int b, int k) {
  const int sh = 8 * a;
  const unsigned r00 = (unsigned)(rows[b + 8 * k] >> sh), r10 = (unsigned)(rows[b + 1 + 8 * k] >> sh);
  const unsigned r01 = (unsigned)(rows[b + 8 * (k + 1)] >> sh);
  const unsigned r11 = (unsigned)(rows[b + 1 + 8 * (k + 1)] >> sh);
  return (unsigned long long)__byte_perm(r00, r10, 0x4510) | ((unsigned long long)__byte_perm(r01, r11, 0x4510) << 32);
}

// order-preserving double -> u64 encoding (min/max via integer atomics)
__device__ __forceinline__ unsigned long long enc_ordered(double d) {
  unsigned long long b = (unsigned long long)__double_as_longlong(d);
  return (b & 0x8000000000000000ULL) ? ~b : (b | 0x8000000000000000ULL);
}

}  // namespace dev
}  // namespace nkb
