// Direct stiffness summation (DSSUM) of element-local SEM fields -- the
// gather-scatter that makes derived fields C0-continuous across element
// faces.  NekRS does this with its gs handles over
// mesh->globalIds; here the caller hands in the same global node ids.
//
// Value of a global node g with copies on ranks r0 < r1 < ...:
//   P_r   = left fold of rank r's copies in increasing local GLL index,
//   total = ((P_r0 + P_r1) + P_r2) + ...,       avg = total / (number of copies)
// and every copy is overwritten with avg.  One rank: avg = left fold / count.
//
// Setup (once per mesh): CUB radix sort of (gid, local index) gives, per
// unique gid u, the CSR run of its local copies (stable sort: increasing
// local index).  Across ranks, unique gids are hashed to an owner rank
// (gid % R), which learns every gid's copy count and rank set and answers
// each rank with its shared gids; each pair of ranks then shares a list in
// increasing gid order.  Per call: sum kernel -> pack/exchange partials with
// the neighbour ranks (grouped ncclSend/Recv, in abi.cu) -> combine in rank
// order -> scatter.
//
// One rank (gs_average_local): the runs are regrouped once by copy count.
// Runs of K = 2..kGroupMax copies are stored per K as K structure-of-arrays
// rows of local indices (row j = every run's j-th copy, runs in gid order),
// so one thread averages one run with K coalesced index loads, K independent
// gathers, a left fold and K stores; single-copy runs are never touched
// (v / 1 == v) and longer runs go through the CSR.  One launch covers every
// group.
#include <cub/cub.cuh>
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

constexpr int kRunBlock = 256;

__global__ void run_key_kernel(const int* cnt, long long U, unsigned char* key, int* u_of, int* hist) {
  __shared__ int h[kGroupMax + 2];                  // block histogram: one global atomic per bin per block
  if (threadIdx.x < kGroupMax + 2) h[threadIdx.x] = 0;
  __syncthreads();
  for (long long u = blockIdx.x * (long long)blockDim.x + threadIdx.x; u < U; u += (long long)gridDim.x * blockDim.x) {
    const int c = cnt[u];
    const int k = c > kGroupMax ? kGroupMax + 1 : c;
    key[u] = (unsigned char)k;
    u_of[u] = (int)u;
    atomicAdd(&h[k], 1);
  }
  __syncthreads();
  if (threadIdx.x < kGroupMax + 2 && h[threadIdx.x]) atomicAdd(&hist[threadIdx.x], h[threadIdx.x]);
}

// sorted run p (stable by key): run u = order[p] of K = key copies -> its group rows
__global__ void run_fill_kernel(const unsigned char* key, const int* order, long long U, const int* idx,
                                const int* off, GsGroups gr, int* lrun) {
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < U; p += (long long)gridDim.x * blockDim.x) {
    const int k = key[p], u = order[p];
    if (k < 2) continue;
    const long long r = p - gr.first[k];
    if (k > kGroupMax) {
      lrun[r] = u;
      continue;
    }
    int* rows = gr.idx + gr.base[k];
    for (int j = 0; j < k; ++j) rows[(long long)j * gr.n[k] + r] = idx[off[u] + j];
  }
}

// runs per thread for K copies: about eight gathers in flight per thread
__host__ __device__ constexpr int runs_per_thread(int k) { return k <= 2 ? 4 : k <= 4 ? 2 : 1; }

// runs r0 + i * kRunBlock (i < R) of group K: every index load, then every
// gather, issued before the first use
template <int K>
__device__ __forceinline__ void avg_runs(double* __restrict__ v, const int* __restrict__ rows, long long nk,
                                         long long r0) {
  constexpr int R = runs_per_thread(K);
  int id[R][K];
  double x[R][K];
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int j = 0; j < K; ++j) {
      const long long r = r0 + (long long)i * kRunBlock;
      id[i][j] = r < nk ? __ldg(rows + j * nk + r) : -1;
    }
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int j = 0; j < K; ++j) x[i][j] = id[i][j] >= 0 ? v[id[i][j]] : 0.0;
#pragma unroll
  for (int i = 0; i < R; ++i) {
    double t = x[i][0];
#pragma unroll
    for (int j = 1; j < K; ++j) t = __dadd_rn(t, x[i][j]);
    const double a = __ddiv_rn(t, (double)K);
    if (id[i][0] >= 0)
#pragma unroll
      for (int j = 0; j < K; ++j) v[id[i][j]] = a;
  }
}

// block b belongs to group k with gr.block[k] <= b < gr.block[k+1]; k = kGroupMax + 1: CSR runs
__global__ void __launch_bounds__(kRunBlock) gs_avg_kernel(double* __restrict__ v, GsGroups gr,
                                                           const int* __restrict__ lrun, const int* __restrict__ idx,
                                                           const int* __restrict__ off) {
  const int b = blockIdx.x;
  int k = 2;
#pragma unroll
  for (int q = 3; q <= kGroupMax + 1; ++q) k += b >= gr.block[q];
  const long long r = (long long)(b - gr.block[k]) * kRunBlock * runs_per_thread(k) + threadIdx.x;
  if (r >= gr.n[k]) return;
  const int* rows = gr.idx + (k <= kGroupMax ? gr.base[k < kGroupMax ? k : kGroupMax] : 0);
  switch (k) {
    case 2: avg_runs<2>(v, rows, gr.n[2], r); break;
    case 3: avg_runs<3>(v, rows, gr.n[3], r); break;
    case 4: avg_runs<4>(v, rows, gr.n[4], r); break;
    case 5: avg_runs<5>(v, rows, gr.n[5], r); break;
    case 6: avg_runs<6>(v, rows, gr.n[6], r); break;
    case 7: avg_runs<7>(v, rows, gr.n[7], r); break;
    case 8: avg_runs<8>(v, rows, gr.n[8], r); break;
    default: {
      const int u = lrun[r], a = off[u], e = off[u + 1];
      double t = v[idx[a]];
      for (int j = a + 1; j < e; ++j) t = __dadd_rn(t, v[idx[j]]);
      const double m = __ddiv_rn(t, (double)(e - a));
      for (int j = a; j < e; ++j) v[idx[j]] = m;
    }
  }
}

__global__ void iota_kernel(int* v, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    v[i] = (int)i;
}

__global__ void head_kernel(const long long* k, long long n, int* head) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    head[i] = (i == 0 || k[i] != k[i - 1]) ? 1 : 0;
}

// seg = inclusive scan of head: sorted position i belongs to run seg[i] - 1
__global__ void runs_kernel(const long long* k, const int* head, const int* seg, long long n, int* off,
                            long long* ugid) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    if (head[i]) {
      off[seg[i] - 1] = (int)i;
      ugid[seg[i] - 1] = k[i];
    }
}

__global__ void count_kernel(const int* off, long long U, int* cnt) {
  for (long long u = blockIdx.x * (long long)blockDim.x + threadIdx.x; u < U; u += (long long)gridDim.x * blockDim.x)
    cnt[u] = off[u + 1] - off[u];
}

__global__ void gs_sum_kernel(const double* __restrict__ v, const int* __restrict__ idx, const int* __restrict__ off,
                              long long U, double* __restrict__ part) {
  for (long long u = blockIdx.x * (long long)blockDim.x + threadIdx.x; u < U; u += (long long)gridDim.x * blockDim.x) {
    const int a = off[u], b = off[u + 1];
    double s = v[idx[a]];
    for (int k = a + 1; k < b; ++k) s = __dadd_rn(s, v[idx[k]]);
    part[u] = s;
  }
}

__global__ void gs_scatter_kernel(double* __restrict__ v, const int* __restrict__ idx, const int* __restrict__ off,
                                  long long U, const double* __restrict__ total, const int* __restrict__ mult) {
  for (long long u = blockIdx.x * (long long)blockDim.x + threadIdx.x; u < U; u += (long long)gridDim.x * blockDim.x) {
    const double avg = __ddiv_rn(total[u], (double)mult[u]);
    for (int k = off[u]; k < off[u + 1]; ++k) v[idx[k]] = avg;
  }
}

__global__ void gs_pack_kernel(const double* __restrict__ part, const int* __restrict__ list, int m,
                               double* __restrict__ buf) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < m; j += gridDim.x * blockDim.x) buf[j] = part[list[j]];
}

// shared gid j (local unique index su[j]): fold the partials of its ranks in
// rank order; pos[j*R + q] = position in the buffer received from rank q
__global__ void gs_combine_kernel(double* __restrict__ part, const int* __restrict__ su,
                                  const unsigned char* __restrict__ mask, const int* __restrict__ pos, int n_shared,
                                  int R, int me, const double* const* __restrict__ recv) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n_shared; j += gridDim.x * blockDim.x) {
    const int u = su[j];
    const unsigned m = mask[j];
    double t = 0.0;
    bool first = true;
    for (int q = 0; q < R; ++q) {
      if (!(m & (1u << q))) continue;
      const double v = (q == me) ? part[u] : recv[q][pos[(long long)j * R + q]];
      t = first ? v : __dadd_rn(t, v);
      first = false;
    }
    part[u] = t;
  }
}

// ---- multi-rank discovery helpers ----

__global__ void dest_hist_kernel(const long long* ugid, long long U, int R, int* hist) {
  __shared__ int h[kMaxRanks];                      // block histogram: one global atomic per rank per block
  if (threadIdx.x < kMaxRanks) h[threadIdx.x] = 0;
  __syncthreads();
  for (long long u = blockIdx.x * (long long)blockDim.x + threadIdx.x; u < U; u += (long long)gridDim.x * blockDim.x)
    atomicAdd(&h[(int)(ugid[u] % R)], 1);
  __syncthreads();
  if (threadIdx.x < R && h[threadIdx.x]) atomicAdd(&hist[threadIdx.x], h[threadIdx.x]);
}

// bucket (gid, count) pairs by owner rank; cursor[q] starts at the bucket offset
__global__ void dest_scatter_kernel(const long long* ugid, const int* cnt, long long U, int R, int* cursor,
                                    long long* out) {
  for (long long u = blockIdx.x * (long long)blockDim.x + threadIdx.x; u < U; u += (long long)gridDim.x * blockDim.x) {
    const int q = (int)(ugid[u] % R);
    const int at = atomicAdd(&cursor[q], 1);
    out[2LL * at] = ugid[u];
    out[2LL * at + 1] = cnt[u];
  }
}

}  // namespace

// sort (gid, local index) and build the CSR of unique gids
int gs_build_local(const long long* gid, long long n, GsLocal& g, cudaStream_t s) {
  g.n = n;
  g.U = 0;
  if (n <= 0) return NKB_OK;
  if (n > 0x7fffffffLL) return fail(NKB_EINVAL, "too many GLL points for one rank");
  long long* kout = nullptr;
  int *iota = nullptr, *head = nullptr, *seg = nullptr;
  void* tmp = nullptr;
  size_t tb = 0, tb2 = 0;
  NKB_CUDA(cudaMallocAsync(&kout, sizeof(long long) * n, s));
  NKB_CUDA(cudaMallocAsync(&iota, sizeof(int) * n, s));
  NKB_CUDA(cudaMallocAsync(&head, sizeof(int) * n, s));
  NKB_CUDA(cudaMallocAsync(&seg, sizeof(int) * n, s));
  NKB_CUDA(cudaMalloc(&g.idx, sizeof(int) * n));
  iota_kernel<<<grid_for(n, 256), 256, 0, s>>>(iota, n);
  NKB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, gid, kout, iota, g.idx, (int)n, 0, 64, s));
  NKB_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb2, head, seg, (int)n, s));
  NKB_CUDA(cudaMallocAsync(&tmp, tb > tb2 ? tb : tb2, s));
  // stable: copies of one gid stay in increasing local index order
  NKB_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, gid, kout, iota, g.idx, (int)n, 0, 64, s));
  head_kernel<<<grid_for(n, 256), 256, 0, s>>>(kout, n, head);
  NKB_CUDA(cub::DeviceScan::InclusiveSum(tmp, tb2, head, seg, (int)n, s));
  int last = 0;
  NKB_CUDA(cudaMemcpyAsync(&last, seg + n - 1, sizeof(int), cudaMemcpyDeviceToHost, s));
  NKB_CUDA(cudaStreamSynchronize(s));
  g.U = last;
  NKB_CUDA(cudaMalloc(&g.off, sizeof(int) * (g.U + 1)));
  NKB_CUDA(cudaMalloc(&g.ugid, sizeof(long long) * g.U));
  NKB_CUDA(cudaMalloc(&g.mult, sizeof(int) * g.U));
  NKB_CUDA(cudaMalloc(&g.part, sizeof(double) * g.U));
  runs_kernel<<<grid_for(n, 256), 256, 0, s>>>(kout, head, seg, n, g.off, g.ugid);
  const int nn = (int)n;
  NKB_CUDA(cudaMemcpyAsync(g.off + g.U, &nn, sizeof(int), cudaMemcpyHostToDevice, s));
  count_kernel<<<grid_for(g.U, 256), 256, 0, s>>>(g.off, g.U, g.mult);
  NKB_CUDA(cudaGetLastError());
  NKB_TRY(gs_build_groups(g, s));
  NKB_CUDA(cudaFreeAsync(kout, s));
  NKB_CUDA(cudaFreeAsync(iota, s));
  NKB_CUDA(cudaFreeAsync(head, s));
  NKB_CUDA(cudaFreeAsync(seg, s));
  NKB_CUDA(cudaFreeAsync(tmp, s));
  NKB_CUDA(cudaStreamSynchronize(s));
  return NKB_OK;
}

// regroup the runs by copy count for the one-rank kernel (see the header)
int gs_build_groups(GsLocal& g, cudaStream_t s) {
  GsGroups& gr = g.groups;
  gr = GsGroups();
  if (g.U == 0) return NKB_OK;
  unsigned char *key = nullptr, *key_s = nullptr;
  int *u_of = nullptr, *order = nullptr, *hist = nullptr;
  void* tmp = nullptr;
  size_t tb = 0;
  NKB_CUDA(cudaMallocAsync(&key, g.U, s));
  NKB_CUDA(cudaMallocAsync(&key_s, g.U, s));
  NKB_CUDA(cudaMallocAsync(&u_of, sizeof(int) * g.U, s));
  NKB_CUDA(cudaMallocAsync(&order, sizeof(int) * g.U, s));
  NKB_CUDA(cudaMallocAsync(&hist, sizeof(int) * (kGroupMax + 2), s));
  NKB_CUDA(cudaMemsetAsync(hist, 0, sizeof(int) * (kGroupMax + 2), s));
  run_key_kernel<<<grid_for(g.U, 256), 256, 0, s>>>(g.mult, g.U, key, u_of, hist);
  NKB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, key, key_s, u_of, order, (int)g.U, 0, 4, s));
  NKB_CUDA(cudaMallocAsync(&tmp, tb, s));
  NKB_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, key, key_s, u_of, order, (int)g.U, 0, 4, s));  // stable
  int h[kGroupMax + 2];
  NKB_CUDA(cudaMemcpyAsync(h, hist, sizeof(h), cudaMemcpyDeviceToHost, s));
  NKB_CUDA(cudaStreamSynchronize(s));
  long long first = 0, base = 0, blocks = 0;
  for (int k = 0; k <= kGroupMax + 1; ++k) {
    gr.first[k] = first;
    gr.n[k] = h[k];
    first += h[k];
    if (k >= 2) {
      gr.block[k] = (int)blocks;
      const long long per = (long long)kRunBlock * runs_per_thread(k);
      blocks += (h[k] + per - 1) / per;
      if (k <= kGroupMax) {
        gr.base[k] = base;
        base += (long long)k * h[k];
      }
    }
  }
  if (blocks > 0x7fffffffLL) return fail(NKB_EINVAL, "too many shared GLL nodes for one rank");
  gr.blocks = (int)blocks;
  if (base) NKB_CUDA(cudaMalloc(&gr.idx, sizeof(int) * base));
  if (h[kGroupMax + 1]) NKB_CUDA(cudaMalloc(&g.lrun, sizeof(int) * h[kGroupMax + 1]));
  run_fill_kernel<<<grid_for(g.U, 256), 256, 0, s>>>(key_s, order, g.U, g.idx, g.off, gr, g.lrun);
  NKB_CUDA(cudaGetLastError());
  NKB_CUDA(cudaFreeAsync(key, s));
  NKB_CUDA(cudaFreeAsync(key_s, s));
  NKB_CUDA(cudaFreeAsync(u_of, s));
  NKB_CUDA(cudaFreeAsync(order, s));
  NKB_CUDA(cudaFreeAsync(hist, s));
  NKB_CUDA(cudaFreeAsync(tmp, s));
  return NKB_OK;
}

int gs_average_local(const GsLocal& g, double* v, cudaStream_t s) {
  if (g.groups.blocks == 0) return NKB_OK;
  gs_avg_kernel<<<g.groups.blocks, kRunBlock, 0, s>>>(v, g.groups, g.lrun, g.idx, g.off);
  NKB_CUDA(cudaGetLastError());
  return NKB_OK;
}

void gs_free(GsLocal& g) {
  cudaFree(g.groups.idx);
  cudaFree(g.lrun);
  cudaFree(g.idx);
  cudaFree(g.off);
  cudaFree(g.ugid);
  cudaFree(g.mult);
  cudaFree(g.part);
  cudaFree(g.su);
  cudaFree(g.smask);
  cudaFree(g.spos);
  cudaFree(g.slist);
  cudaFree(g.sbuf);
  cudaFree(g.rbuf);
  cudaFree(g.rptr);
  g = GsLocal();
}

int gs_sum(const GsLocal& g, const double* v, cudaStream_t s) {
  if (g.U == 0) return NKB_OK;
  gs_sum_kernel<<<grid_for(g.U, 256), 256, 0, s>>>(v, g.idx, g.off, g.U, g.part);
  NKB_CUDA(cudaGetLastError());
  return NKB_OK;
}

int gs_pack(const GsLocal& g, int q, cudaStream_t s) {
  const int m = g.ncount[q];
  if (m == 0) return NKB_OK;
  gs_pack_kernel<<<grid_for(m, 256), 256, 0, s>>>(g.part, g.slist + g.noff[q], m, g.sbuf + g.noff[q]);
  NKB_CUDA(cudaGetLastError());
  return NKB_OK;
}

int gs_combine(const GsLocal& g, int R, int me, cudaStream_t s) {
  if (g.n_shared == 0) return NKB_OK;
  gs_combine_kernel<<<grid_for(g.n_shared, 256), 256, 0, s>>>(g.part, g.su, g.smask, g.spos, g.n_shared, R, me,
                                                              g.rptr);
  NKB_CUDA(cudaGetLastError());
  return NKB_OK;
}

int gs_scatter(const GsLocal& g, double* v, cudaStream_t s) {
  if (g.U == 0) return NKB_OK;
  gs_scatter_kernel<<<grid_for(g.U, 256), 256, 0, s>>>(v, g.idx, g.off, g.U, g.part, g.mult);
  NKB_CUDA(cudaGetLastError());
  return NKB_OK;
}

// bucket my unique (gid, count) pairs by owner rank gid % R into out[2*U]
// (int64 pairs); counts[q] = entries for rank q (host)
int gs_bucket_by_owner(const GsLocal& g, int R, long long* out, std::vector<int>& counts, cudaStream_t s) {
  counts.assign(R, 0);
  if (g.U == 0) return NKB_OK;
  int* d = nullptr;
  NKB_CUDA(cudaMallocAsync(&d, sizeof(int) * 2 * R, s));
  NKB_CUDA(cudaMemsetAsync(d, 0, sizeof(int) * 2 * R, s));
  dest_hist_kernel<<<grid_for(g.U, 256), 256, 0, s>>>(g.ugid, g.U, R, d);
  NKB_CUDA(cudaMemcpyAsync(counts.data(), d, sizeof(int) * R, cudaMemcpyDeviceToHost, s));
  NKB_CUDA(cudaStreamSynchronize(s));
  std::vector<int> start(R, 0);
  for (int q = 1; q < R; ++q) start[q] = start[q - 1] + counts[q - 1];
  NKB_CUDA(cudaMemcpyAsync(d + R, start.data(), sizeof(int) * R, cudaMemcpyHostToDevice, s));
  dest_scatter_kernel<<<grid_for(g.U, 256), 256, 0, s>>>(g.ugid, g.mult, g.U, R, d + R, out);
  NKB_CUDA(cudaGetLastError());
  NKB_CUDA(cudaFreeAsync(d, s));
  NKB_CUDA(cudaStreamSynchronize(s));
  return NKB_OK;
}

}  // namespace nkb
