// Sort-last depth composite fused with the colormap resolve, over NVLink peer
// memory (R16 of SURVEY.md §8a).
//
// Every rank rasterises its element partition into a packed-key buffer
// (depth bits << 32 | scalar bits, + 2 colour-range words).  Instead of an
// ncclReduce to rank 0 followed by a resolve on rank 0, each rank owns a band
// of image rows and, in ONE kernel,
//   - min-reduces that band straight out of every peer's key buffer (P2P
//     loads through CUDA IPC mappings over NVLink/NVSwitch),
//   - resolves the colormap (global range = min/max of all peers' range words),
//   - stores RGBA8 + depth directly into rank 0's image (P2P stores).
// Bytes crossing NVLink per rank: (N-1)/N of the key buffer in, (N-1)/N of
// the RGBA+depth band out -- the same as a reduce-scatter + gather, with no
// separate resolve pass and no host round trip.
//
// Ordering uses per-rank epoch flags in peer memory with system-scope
// release / acquire; every spin has a globaltimer timeout so a lost peer
// cannot hang the GPU (the host reports NKB_ENCCL instead).  Key buffers are
// double-buffered by epoch parity; before a rank clears a buffer it waits
// until every peer has finished reading it (epoch - 2).
//
// The result is identical to the NCCL path and to one GPU: min over packed
// keys is associative and commutative (tests/test_gpu_multi.py).
//
// Two kernels do the same work.  p2p_composite_kernel: every thread loads a
// pixel pair from every rank (many CTAs, latency hidden by parallelism).
// p2p_composite_bulk_kernel: tiles of the band move into shared memory by
// bulk copies (cp.async.bulk, one per rank and tile, from peer memory over
// NVLink), two tiles in flight per CTA on mbarriers, so a few CTAs on the
// SMs a split step leaves free (run_step) sustain the band while the next
// step's surface pass holds the rest of the GPU.
#include <cuda_runtime.h>
#include <math.h>

#include "checked.cuh"
#include "nkb_internal.h"
#include "raster_dev.cuh"

namespace nkb {

namespace {

constexpr unsigned long long kTimeoutNs = 2000000000ULL;   // 2 s

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// wait until flags[first .. first+n) >= target (all peers); 0 = ok, 1 = timeout
__device__ int wait_flags(const unsigned long long* flags, int first, int n, unsigned long long target,
                          int* err) {
  const unsigned long long t0 = gtimer();
  for (int p = 0; p < n; ++p) {
    while (ld_acquire_sys(flags + first + p) < target) {
      if (gtimer() - t0 > kTimeoutNs) {
        atomicExch(err, 1);
        return 1;
      }
    }
  }
  return 0;
}

// ---- bulk-copy composite ----
constexpr int kBulkStages = 2;         // 64 KB per CTA: fits beside two three-CTA K1g CTAs (146 KB)
constexpr int kBulkStageBytes = 32768;
inline __host__ __device__ int bulk_tile_px(int nranks) { return (kBulkStageBytes / 8 / nranks) & ~255; }

__device__ __forceinline__ void mbar_init(unsigned long long* bar) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(a) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect(unsigned long long* bar, unsigned bytes) {
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(d), "l"(src), "r"(bytes), "r"(b) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n"
      ".reg .pred P;\n"
      "W_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
      "@!P bra W_%=;\n"
      "}\n" ::"r"(b), "r"(parity) : "memory");
}

__global__ void epoch_kernel(P2PParams p) {
  const unsigned long long e = *p.dev_epoch + 1ULL;
  *p.dev_epoch = e;
  if (p.ep_slot) *p.ep_slot = e;
}

__global__ void signal_kernel(P2PParams p, int which, const unsigned long long* count) {
  // which 0: "keys ready", 1: "done reading peers' keys" (+ this rank's triangle count)
  const unsigned long long epoch = *p.dev_epoch;
  const int q = threadIdx.x;
  if (q < p.nranks) {
    if (count) p.peer_flags[q][2 * kMaxRanks + p.rank] = *count;
    if (which == 0) p.peer_flags[q][3 * kMaxRanks + p.rank] = *p.overflow;
    __threadfence_system();
    st_release_sys(p.peer_flags[q] + which * kMaxRanks + p.rank, epoch);
  }
}

// wait until every rank reached (this step's epoch - back)
__global__ void wait_kernel(P2PParams p, int which, unsigned long long back) {
  const unsigned long long ep = *p.dev_epoch;
  if (threadIdx.x == 0 && ep > back) wait_flags(p.flags, which * kMaxRanks, p.nranks, ep - back, p.err);
}

__global__ void __launch_bounds__(256) p2p_composite_kernel(P2PParams p) {
  const unsigned long long epoch = *p.dev_epoch;
  __shared__ int s_ok;
  __shared__ double s_lo, s_hi;
  if (threadIdx.x == 0) {
    s_ok = !wait_flags(p.flags, 0, p.nranks, epoch, p.err);
    // global colour range from every rank's range words
    unsigned long long wmin = ~0ULL, wmax = ~0ULL;
    for (int q = 0; q < p.nranks; ++q) {
      const unsigned long long* z = p.peer_keys[q];
      wmin = min(wmin, z[p.npx]);
      wmax = min(wmax, z[p.npx + 1]);
    }
    double lo = p.vmin, hi = p.vmax;
    if (!(lo == lo)) lo = (wmin == ~0ULL) ? 0.0 : rdev::dec_ordered(wmin);
    if (!(hi == hi)) hi = (~wmax == 0ULL) ? 0.0 : rdev::dec_ordered(~wmax);
    s_lo = lo;
    s_hi = hi;
    if (blockIdx.x == 0 && p.range_out) {
      p.range_out[0] = lo;
      p.range_out[1] = hi;
    }
  }
  __syncthreads();
  if (!s_ok) return;
  const double lo = s_lo, hi = s_hi, span = __dsub_rn(hi, lo);
  const long long r0 = (long long)p.height * p.rank / p.nranks, r1 = (long long)p.height * (p.rank + 1) / p.nranks;
  const long long i0 = r0 * p.width, i1 = r1 * p.width;
  auto resolve = [&](unsigned long long key, long long i) {
    uchar4 o;
    float dep;
    if (key == ~0ULL) {
      o = make_uchar4(p.bg[0], p.bg[1], p.bg[2], p.bg[3]);
      dep = INFINITY;
    } else {
      const double s = (double)__uint_as_float((unsigned)(key & 0xffffffffULL));
      dep = __uint_as_float((unsigned)(key >> 32));
      double t = hi > lo ? __ddiv_rn(__dsub_rn(s, lo), span) : 0.0;
      t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
      o = rdev::cmap_rgba(p.cmap, t);
    }
    NKB_DCHECK(i >= i0 && i < i1 && i < p.npx);
    reinterpret_cast<uchar4*>(p.root_rgba)[i] = o;
    p.root_depth[i] = dep;
  };
  // pairs of pixels: one 16-byte load per peer, all peers' loads in flight
  // before the min (remote NVLink loads are latency-bound, not bandwidth-bound)
  const long long j0 = (i0 + 1) >> 1, j1 = i1 >> 1;   // whole pairs [2*j0, 2*j1)
  const long long stride = (long long)gridDim.x * blockDim.x, t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  for (long long j = j0 + t; j < j1; j += stride) {
    ulonglong2 v[kMaxRanks];
#pragma unroll
    for (int q = 0; q < kMaxRanks; ++q)
      if (q < p.nranks) v[q] = reinterpret_cast<const ulonglong2*>(p.peer_keys[q])[j];
    unsigned long long a = ~0ULL, b = ~0ULL;
#pragma unroll
    for (int q = 0; q < kMaxRanks; ++q)
      if (q < p.nranks) {
        a = min(a, v[q].x);
        b = min(b, v[q].y);
      }
    resolve(a, 2 * j);
    resolve(b, 2 * j + 1);
  }
  // an odd pixel at either end of the band
  if (t < 2) {
    const long long i = t == 0 ? i0 : i1 - 1;
    if ((t == 0 && (i0 & 1) && i0 < i1) || (t == 1 && (i1 & 1) && i1 - 1 >= i0)) {
      unsigned long long key = ~0ULL;
      for (int q = 0; q < p.nranks; ++q) key = min(key, p.peer_keys[q][i]);
      resolve(key, i);
    }
  }
}

// the band's 16-byte aligned part in tiles of T pixels: tile t at
// a0 + t*T, CTA blockIdx.x takes tiles blockIdx.x, + gridDim.x, ...
__global__ void __launch_bounds__(256) p2p_composite_bulk_kernel(P2PParams p) {
  extern __shared__ __align__(128) unsigned long long s_keys[];   // [stage][rank][T]
  __shared__ __align__(8) unsigned long long bar[kBulkStages];
  __shared__ int s_ok;
  __shared__ double s_lo, s_hi;
  const unsigned long long epoch = *p.dev_epoch;
  const int R = p.nranks, T = bulk_tile_px(R), tid = threadIdx.x;
  const long long r0 = (long long)p.height * p.rank / R, r1 = (long long)p.height * (p.rank + 1) / R;
  const long long i0 = r0 * p.width, i1 = r1 * p.width;
  const long long a0 = (i0 + 1) & ~1LL, a1 = i1 & ~1LL;
  const long long ntiles = a1 > a0 ? (a1 - a0 + T - 1) / T : 0;
  auto tile_len = [&](long long t) { return (int)min((long long)T, a1 - (a0 + t * T)); };
  auto issue = [&](long long t, int st) {
    const int L = tile_len(t);
    mbar_expect(&bar[st], (unsigned)(L * 8 * R));
    for (int q = 0; q < R; ++q)
      bulk_g2s(s_keys + ((long long)st * R + q) * T, p.peer_keys[q] + a0 + t * T, (unsigned)(L * 8), &bar[st]);
  };
  if (tid == 0) {
    s_ok = !wait_flags(p.flags, 0, R, epoch, p.err);
    unsigned long long wmin = ~0ULL, wmax = ~0ULL;
    for (int q = 0; q < R; ++q) {
      const unsigned long long* z = p.peer_keys[q];
      wmin = min(wmin, z[p.npx]);
      wmax = min(wmax, z[p.npx + 1]);
    }
    double lo = p.vmin, hi = p.vmax;
    if (!(lo == lo)) lo = (wmin == ~0ULL) ? 0.0 : rdev::dec_ordered(wmin);
    if (!(hi == hi)) hi = (~wmax == 0ULL) ? 0.0 : rdev::dec_ordered(~wmax);
    s_lo = lo;
    s_hi = hi;
    if (blockIdx.x == 0 && p.range_out) {
      p.range_out[0] = lo;
      p.range_out[1] = hi;
    }
    if (s_ok) {
      for (int st = 0; st < kBulkStages; ++st) mbar_init(&bar[st]);
      // peers' keys were acquired through the generic proxy; the bulk copies read through the async proxy
      asm volatile("fence.proxy.async.global;" ::: "memory");
      for (int j = 0; j < kBulkStages; ++j) {
        const long long t = blockIdx.x + (long long)j * gridDim.x;
        if (t < ntiles) issue(t, j);
      }
    }
  }
  __syncthreads();
  if (!s_ok) return;
  const double lo = s_lo, hi = s_hi, span = __dsub_rn(hi, lo);
  auto resolve = [&](unsigned long long key, long long i) {
    uchar4 o;
    float dep;
    if (key == ~0ULL) {
      o = make_uchar4(p.bg[0], p.bg[1], p.bg[2], p.bg[3]);
      dep = INFINITY;
    } else {
      const double s = (double)__uint_as_float((unsigned)(key & 0xffffffffULL));
      dep = __uint_as_float((unsigned)(key >> 32));
      double t = hi > lo ? __ddiv_rn(__dsub_rn(s, lo), span) : 0.0;
      t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
      o = rdev::cmap_rgba(p.cmap, t);
    }
    NKB_DCHECK(i >= i0 && i < i1 && i < p.npx);
    reinterpret_cast<uchar4*>(p.root_rgba)[i] = o;
    p.root_depth[i] = dep;
  };
  for (long long j = 0;; ++j) {
    const long long t = blockIdx.x + j * gridDim.x;
    if (t >= ntiles) break;
    const int st = (int)(j % kBulkStages);
    mbar_wait(&bar[st], (unsigned)((j / kBulkStages) & 1));
    const int L = tile_len(t);
    const unsigned long long* S = s_keys + (long long)st * R * T;
    for (int i = tid; i < L; i += blockDim.x) {
      unsigned long long k = S[i];
      for (int q = 1; q < R; ++q) k = min(k, S[q * T + i]);
      resolve(k, a0 + t * T + i);
    }
    __syncthreads();                                  // stage st consumed
    if (tid == 0) {
      const long long tn = blockIdx.x + (j + kBulkStages) * gridDim.x;
      if (tn < ntiles) issue(tn, st);
    }
  }
  // the band's odd end pixels (outside the aligned part)
  if (blockIdx.x == 0 && tid < 2) {
    const long long i = tid == 0 ? i0 : i1 - 1;
    if ((tid == 0 && (i0 & 1) && i0 < i1) || (tid == 1 && (i1 & 1) && i1 - 1 >= i0 && i1 - 1 != i0)) {
      unsigned long long key = ~0ULL;
      for (int q = 0; q < R; ++q) key = min(key, p.peer_keys[q][i]);
      resolve(key, i);
    }
  }
}

}  // namespace

int launch_p2p_epoch(const P2PParams& p, cudaStream_t s) {
  epoch_kernel<<<1, 1, 0, s>>>(p);
  NKB_CUDA(cudaGetLastError());
  return NKB_OK;
}

int launch_p2p_signal(const P2PParams& p, int which, const unsigned long long* count, cudaStream_t s) {
  signal_kernel<<<1, 32, 0, s>>>(p, which, count);
  NKB_CUDA(cudaGetLastError());
  return NKB_OK;
}

int launch_p2p_wait(const P2PParams& p, int which, unsigned long long back, cudaStream_t s) {
  wait_kernel<<<1, 32, 0, s>>>(p, which, back);
  NKB_CUDA(cudaGetLastError());
  return NKB_OK;
}

int launch_p2p_composite(const P2PParams& p, cudaStream_t s) {
  const long long band = (long long)p.width * ((long long)p.height / p.nranks + 1);
  if (p.bulk) {
    const int T = bulk_tile_px(p.nranks);
    const size_t shm = (size_t)kBulkStages * p.nranks * T * sizeof(unsigned long long);
    static bool attr = false;
    if (!attr) {
      NKB_CUDA(cudaFuncSetAttribute(p2p_composite_bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    kBulkStages * kBulkStageBytes));
      attr = true;
    }
    long long blocks = (band + T - 1) / T;
    if (blocks > 148 * 2) blocks = 148 * 2;
    if (p.max_blocks > 0 && blocks > p.max_blocks) blocks = p.max_blocks;
    if (blocks < 1) blocks = 1;
    p2p_composite_bulk_kernel<<<(unsigned)blocks, 256, shm, s>>>(p);
    NKB_CUDA(cudaGetLastError());
    return NKB_OK;
  }
  long long blocks = (band / 2 + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (p.max_blocks > 0 && blocks > p.max_blocks) blocks = p.max_blocks;
  if (blocks < 1) blocks = 1;
  p2p_composite_kernel<<<(unsigned)blocks, 256, 0, s>>>(p);
  NKB_CUDA(cudaGetLastError());
  return NKB_OK;
}

NKB_CHECKED_ACCESSOR(checked_read_composite)

}  // namespace nkb
