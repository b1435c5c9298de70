// Collective and auxiliary ABI entry points: DSSUM
// over global node ids, in transit N:1 staging, and numpy-exact field
// statistics.  Kernels live in dssum.cu / stats.cu; this file is the host
// orchestration over NCCL.
#include <cuda_runtime.h>
#include <math.h>
#include <stdlib.h>
#include <nccl.h>
#include <string.h>

#include <algorithm>
#include <array>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "ctx.h"

namespace nkb {

static int shape_id(StatsTables& T, long long len) {
  auto it = T.shape_of_len.find(len);
  if (it != T.shape_of_len.end()) return it->second;
  StatShapeHost sh;
  pairwise_shape(len, sh);
  if ((int)sh.leaves.size() > kMaxChunkLeaves) return -1;
  T.shapes.push_back(std::move(sh));
  const int id = (int)T.shapes.size() - 1;
  T.shape_of_len[len] = id;
  return id;
}

void stats_tables_free(StatsTables& T) {
  cudaFree(T.d_chunks);
  cudaFree(T.d_shapes);
  cudaFree(T.d_leaves);
  cudaFree(T.d_nodes);
  cudaFree(T.d_levels);
  cudaFree(T.d_out);
  cudaFreeHost(T.h_out);
  T.h_out = nullptr;
  T.d_chunks = nullptr;
  T.d_shapes = nullptr;
  T.d_leaves = nullptr;
  T.d_nodes = nullptr;
  T.d_levels = nullptr;
  T.d_out = nullptr;
}

}  // namespace nkb

// ---- DSSUM: global node ids and the gather-scatter -----------------------------

int nkb_mesh_set_global_ids(nkb_ctx* ctx, const int64_t* gid, void* stream) {
  NKB_TRY(ctx_check(ctx));
  if (!ctx->x) return fail(NKB_ESTATE, "global ids before mesh_set");
  const int64_t n = ctx->E * kNN;
  if (n > 0 && !gid) return fail(NKB_EINVAL, "null global id pointer");
  cudaStream_t s = (cudaStream_t)stream;
  ctx->gs_ready = false;
  gs_free(ctx->gs);
  GsLocal& g = ctx->gs;
  NKB_TRY(gs_build_local(reinterpret_cast<const long long*>(gid), n, g, s));
  if (g.U > 0) {
    long long first = 0;
    NKB_CUDA(cudaMemcpy(&first, g.ugid, sizeof(first), cudaMemcpyDeviceToHost));
    if (first < 0) return fail(NKB_EINVAL, "global ids must be non-negative");
  }
  const int R = (ctx->comm && ctx->nranks > 1) ? ctx->nranks : 1, me = ctx->rank;
  g.ncount.assign(R, 0);
  g.noff.assign(R + 1, 0);
  if (R == 1) {
    ctx->gs_ready = true;
    return NKB_OK;
  }
  // (1) every unique (gid, local count) to its owner rank gid % R
  long long* sendb = nullptr;
  NKB_CUDA(cudaMalloc(&sendb, sizeof(long long) * 2 * std::max<long long>(g.U, 1)));
  std::vector<int> scount;
  NKB_TRY(gs_bucket_by_owner(g, R, sendb, scount, s));
  auto all_counts = [&](const std::vector<int>& mine, std::vector<int>& recv_from) -> int {
    // recv_from[q] = what rank q sends to me
    long long* d = nullptr;
    NKB_CUDA(cudaMalloc(&d, sizeof(long long) * R * (R + 1)));
    std::vector<long long> m(mine.begin(), mine.end());
    NKB_CUDA(cudaMemcpy(d + (size_t)R * R, m.data(), sizeof(long long) * R, cudaMemcpyHostToDevice));
    NKB_NCCL(g_nccl.AllGather(d + (size_t)R * R, d, R, ncclInt64, ctx->comm, s));
    std::vector<long long> all((size_t)R * R);
    NKB_CUDA(cudaMemcpyAsync(all.data(), d, sizeof(long long) * R * R, cudaMemcpyDeviceToHost, s));
    NKB_CUDA(cudaStreamSynchronize(s));
    cudaFree(d);
    recv_from.assign(R, 0);
    for (int q = 0; q < R; ++q) recv_from[q] = (int)all[(size_t)q * R + me];
    return NKB_OK;
  };
  auto alltoallv = [&](const long long* sb, const std::vector<int>& sc, long long* rb, const std::vector<int>& rc,
                       int width) -> int {
    size_t so = 0, ro = 0;
    NKB_NCCL(g_nccl.GroupStart());
    for (int q = 0; q < R; ++q) {
      if (sc[q]) NKB_NCCL(g_nccl.Send(sb + so, (size_t)sc[q] * width, ncclInt64, q, ctx->comm, s));
      if (rc[q]) NKB_NCCL(g_nccl.Recv(rb + ro, (size_t)rc[q] * width, ncclInt64, q, ctx->comm, s));
      so += (size_t)sc[q] * width;
      ro += (size_t)rc[q] * width;
    }
    NKB_NCCL(g_nccl.GroupEnd());
    NKB_CUDA(cudaStreamSynchronize(s));
    return NKB_OK;
  };
  std::vector<int> rcount;
  NKB_TRY(all_counts(scount, rcount));
  long long nrecv = 0;
  for (int q = 0; q < R; ++q) nrecv += rcount[q];
  long long* recvb = nullptr;
  NKB_CUDA(cudaMalloc(&recvb, sizeof(long long) * 2 * std::max<long long>(nrecv, 1)));
  NKB_TRY(alltoallv(sendb, scount, recvb, rcount, 2));
  cudaFree(sendb);
  // (2) owner: per gid, total copies and the set of ranks (host; setup only)
  std::vector<long long> rec((size_t)2 * nrecv);
  if (nrecv) NKB_CUDA(cudaMemcpy(rec.data(), recvb, sizeof(long long) * 2 * nrecv, cudaMemcpyDeviceToHost));
  cudaFree(recvb);
  std::vector<std::pair<long long, int>> ent;   // (gid, entry index)
  ent.reserve(nrecv);
  std::vector<int> src(nrecv);
  {
    long long k = 0;
    for (int q = 0; q < R; ++q)
      for (int i = 0; i < rcount[q]; ++i, ++k) {
        src[k] = q;
        ent.emplace_back(rec[2 * k], (int)k);
      }
  }
  std::sort(ent.begin(), ent.end());
  std::vector<std::vector<long long>> reply(R);   // per source rank: (gid, total, mask) triplets
  for (size_t a = 0; a < ent.size();) {
    size_t b = a;
    long long total = 0;
    unsigned mask = 0;
    while (b < ent.size() && ent[b].first == ent[a].first) {
      total += rec[2 * ent[b].second + 1];
      mask |= 1u << src[ent[b].second];
      ++b;
    }
    if (__builtin_popcount(mask) > 1)
      for (size_t c = a; c < b; ++c) {
        auto& r = reply[src[ent[c].second]];
        r.push_back(ent[a].first);
        r.push_back(total);
        r.push_back(mask);
      }
    a = b;
  }
  // (3) answers back to the ranks that hold each shared gid
  std::vector<int> rep_count(R), got_count;
  std::vector<long long> rep_flat;
  for (int q = 0; q < R; ++q) {
    rep_count[q] = (int)(reply[q].size() / 3);
    rep_flat.insert(rep_flat.end(), reply[q].begin(), reply[q].end());
  }
  NKB_TRY(all_counts(rep_count, got_count));
  long long ngot = 0;
  for (int q = 0; q < R; ++q) ngot += got_count[q];
  long long *d_rep = nullptr, *d_got = nullptr;
  NKB_CUDA(cudaMalloc(&d_rep, sizeof(long long) * std::max<size_t>(rep_flat.size(), 1)));
  NKB_CUDA(cudaMalloc(&d_got, sizeof(long long) * 3 * std::max<long long>(ngot, 1)));
  if (!rep_flat.empty())
    NKB_CUDA(cudaMemcpy(d_rep, rep_flat.data(), sizeof(long long) * rep_flat.size(), cudaMemcpyHostToDevice));
  NKB_TRY(alltoallv(d_rep, rep_count, d_got, got_count, 3));
  std::vector<long long> got((size_t)3 * ngot);
  if (ngot) NKB_CUDA(cudaMemcpy(got.data(), d_got, sizeof(long long) * 3 * ngot, cudaMemcpyDeviceToHost));
  cudaFree(d_rep);
  cudaFree(d_got);
  // (4) my shared gids in increasing gid order; neighbour lists; global counts
  std::vector<std::array<long long, 3>> sh((size_t)ngot);
  for (long long k = 0; k < ngot; ++k) sh[k] = {got[3 * k], got[3 * k + 1], got[3 * k + 2]};
  std::sort(sh.begin(), sh.end());
  std::vector<long long> ug(g.U);
  if (g.U) NKB_CUDA(cudaMemcpy(ug.data(), g.ugid, sizeof(long long) * g.U, cudaMemcpyDeviceToHost));
  std::vector<int> mult(g.U);
  if (g.U) NKB_CUDA(cudaMemcpy(mult.data(), g.mult, sizeof(int) * g.U, cudaMemcpyDeviceToHost));
  const int ns = (int)sh.size();
  std::vector<int> su(ns), spos((size_t)ns * R, -1);
  std::vector<unsigned char> smask(ns);
  std::vector<std::vector<int>> lists(R);
  for (int j = 0; j < ns; ++j) {
    const long long gg = sh[j][0];
    const auto it = std::lower_bound(ug.begin(), ug.end(), gg);
    if (it == ug.end() || *it != gg) return fail(NKB_EINVAL, "internal: shared gid not found locally");
    const int u = (int)(it - ug.begin());
    su[j] = u;
    mult[u] = (int)sh[j][1];
    smask[j] = (unsigned char)sh[j][2];
    for (int q = 0; q < R; ++q)
      if (q != me && (sh[j][2] & (1LL << q))) {
        spos[(size_t)j * R + q] = (int)lists[q].size();
        lists[q].push_back(u);
      }
  }
  std::vector<int> flat;
  for (int q = 0; q < R; ++q) {
    g.noff[q] = (int)flat.size();
    g.ncount[q] = (int)lists[q].size();
    flat.insert(flat.end(), lists[q].begin(), lists[q].end());
  }
  g.noff[R] = (int)flat.size();
  g.n_shared = ns;
  if (g.U) NKB_CUDA(cudaMemcpy(g.mult, mult.data(), sizeof(int) * g.U, cudaMemcpyHostToDevice));
  const size_t nf = std::max<size_t>(flat.size(), 1);
  NKB_CUDA(cudaMalloc(&g.su, sizeof(int) * std::max(ns, 1)));
  NKB_CUDA(cudaMalloc(&g.smask, std::max(ns, 1)));
  NKB_CUDA(cudaMalloc(&g.spos, sizeof(int) * std::max<size_t>(spos.size(), 1)));
  NKB_CUDA(cudaMalloc(&g.slist, sizeof(int) * nf));
  NKB_CUDA(cudaMalloc(&g.sbuf, sizeof(double) * nf));
  NKB_CUDA(cudaMalloc(&g.rbuf, sizeof(double) * nf));
  NKB_CUDA(cudaMalloc(&g.rptr, sizeof(double*) * R));
  if (ns) {
    NKB_CUDA(cudaMemcpy(g.su, su.data(), sizeof(int) * ns, cudaMemcpyHostToDevice));
    NKB_CUDA(cudaMemcpy(g.smask, smask.data(), ns, cudaMemcpyHostToDevice));
    NKB_CUDA(cudaMemcpy(g.spos, spos.data(), sizeof(int) * spos.size(), cudaMemcpyHostToDevice));
  }
  if (!flat.empty()) NKB_CUDA(cudaMemcpy(g.slist, flat.data(), sizeof(int) * flat.size(), cudaMemcpyHostToDevice));
  std::vector<const double*> rp(R);
  for (int q = 0; q < R; ++q) rp[q] = g.rbuf + g.noff[q];
  NKB_CUDA(cudaMemcpy(g.rptr, rp.data(), sizeof(double*) * R, cudaMemcpyHostToDevice));
  ctx->gs_ready = true;
  return NKB_OK;
}

// ---- in transit: N:1 GPU-direct staging of SEM partitions ---------------------

static unsigned long long fnv1a(const std::string& t, unsigned long long h = 1469598103934665603ULL) {
  for (unsigned char c : t) h = (h ^ c) * 1099511628211ULL;
  return h;
}

int nkb_transit_gather(nkb_ctx* ctx, int root, void* stream) {
  NKB_TRY(ctx_check(ctx));
  if (!ctx->x) return fail(NKB_ESTATE, "transit before mesh_set");
  if (!ctx->comm || ctx->nranks < 2) return fail(NKB_ESTATE, "transit needs a communicator with >= 2 ranks");
  const int R = ctx->nranks, me = ctx->rank;
  if (root < 0 || root >= R) return fail(NKB_EINVAL, "root out of range");
  cudaStream_t s = (cudaStream_t)stream;
  // schema check + partition sizes: (E, element offset, #fields, hash of names/components)
  std::string sig;
  for (auto& f : ctx->fields) sig += f.name + ":" + std::to_string(f.ncomp) + ";";
  const long long mine[4] = {(long long)ctx->E, (long long)ctx->elem_off, (long long)ctx->fields.size(),
                             (long long)(fnv1a(sig) & 0x7fffffffffffffffULL)};
  long long* d = nullptr;
  NKB_CUDA(cudaMalloc(&d, sizeof(long long) * 4 * (R + 1)));
  NKB_CUDA(cudaMemcpy(d + 4 * R, mine, sizeof(mine), cudaMemcpyHostToDevice));
  NKB_NCCL(g_nccl.AllGather(d + 4 * R, d, 4, ncclInt64, ctx->comm, s));
  std::vector<long long> all(4 * R);
  NKB_CUDA(cudaMemcpyAsync(all.data(), d, sizeof(long long) * 4 * R, cudaMemcpyDeviceToHost, s));
  NKB_CUDA(cudaStreamSynchronize(s));
  cudaFree(d);
  std::vector<long long> lo(R + 1, 0);
  for (int q = 0; q < R; ++q) {
    if (all[4 * q + 2] != mine[2] || all[4 * q + 3] != mine[3])
      return fail(NKB_EINVAL, "transit: ranks carry different field schemas");
    if (q > 0 && all[4 * q + 1] != all[4 * (q - 1) + 1] + all[4 * (q - 1)])
      return fail(NKB_EINVAL, "transit: partitions are not contiguous in rank order");
    lo[q + 1] = lo[q] + all[4 * q];
  }
  const int64_t Et = lo[R], nt = Et * kNN;
  // arrays in order: x, y, z, then every component of every field (SoA)
  std::vector<std::pair<const double*, int64_t>> arrs;   // (local base, stride unused)
  arrs.push_back({ctx->x, 0});
  arrs.push_back({ctx->y, 0});
  arrs.push_back({ctx->z, 0});
  for (auto& f : ctx->fields)
    for (int c = 0; c < f.ncomp; ++c) arrs.push_back({f.base + (int64_t)c * f.comp_stride, 0});
  const int na = (int)arrs.size();
  const int64_t nloc = ctx->E * kNN;
  if (me == root && ctx->tr_cap < (int64_t)na * nt) {
    cudaFree(ctx->tr_buf);
    ctx->tr_buf = nullptr;
    ctx->tr_cap = 0;
    NKB_CUDA(cudaMalloc(&ctx->tr_buf, sizeof(double) * std::max<int64_t>((int64_t)na * nt, 1)));
    ctx->tr_cap = (int64_t)na * nt;
  }
  NKB_NCCL(g_nccl.GroupStart());
  for (int a = 0; a < na; ++a) {
    if (me == root) {
      double* dst = ctx->tr_buf + (int64_t)a * nt;
      for (int q = 0; q < R; ++q) {
        const int64_t cnt = all[4 * q] * kNN;
        if (cnt == 0) continue;
        if (q == root)
          NKB_CUDA(cudaMemcpyAsync(dst + lo[q] * kNN, arrs[a].first, sizeof(double) * cnt, cudaMemcpyDeviceToDevice, s));
        else
          NKB_NCCL(g_nccl.Recv(dst + lo[q] * kNN, (size_t)cnt, ncclFloat64, q, ctx->comm, s));
      }
    } else if (nloc > 0) {
      NKB_NCCL(g_nccl.Send(arrs[a].first, (size_t)nloc, ncclFloat64, root, ctx->comm, s));
    }
  }
  NKB_NCCL(g_nccl.GroupEnd());
  NKB_CUDA(cudaStreamSynchronize(s));
  if (me != root) return NKB_OK;
  // the endpoint's context now describes the assembled mesh (producer order)
  std::vector<Field> nf;
  int a = 3;
  for (auto& f : ctx->fields) {
    Field g = f;
    g.base = ctx->tr_buf + (int64_t)a * nt;
    g.comp_stride = nt;
    a += f.ncomp;
    nf.push_back(g);
  }
  const double* tb = ctx->tr_buf;
  NKB_TRY(nkb_mesh_set(ctx, Et, kN, tb, tb + nt, tb + 2 * nt, 0, Et));
  ctx->fields = nf;
  return NKB_OK;
}

namespace nkb {
int gs_apply(nkb_ctx* ctx, double* field, cudaStream_t s) {
  GsLocal& g = ctx->gs;
  const int R = (ctx->comm && ctx->nranks > 1) ? ctx->nranks : 1;
  if (R == 1 && !getenv("NKB_DSSUM_TWO_PASS")) return gs_average_local(g, field, s);
  NKB_TRY(gs_sum(g, field, s));
  if (R > 1 && g.n_shared > 0) {
    for (int q = 0; q < R; ++q) NKB_TRY(gs_pack(g, q, s));
    NKB_NCCL(g_nccl.GroupStart());
    for (int q = 0; q < R; ++q)
      if (g.ncount[q]) {
        NKB_NCCL(g_nccl.Send(g.sbuf + g.noff[q], g.ncount[q], ncclFloat64, q, ctx->comm, s));
        NKB_NCCL(g_nccl.Recv(g.rbuf + g.noff[q], g.ncount[q], ncclFloat64, q, ctx->comm, s));
      }
    NKB_NCCL(g_nccl.GroupEnd());
    NKB_TRY(gs_combine(g, R, ctx->rank, s));
  }
  return gs_scatter(g, field, s);
}
}  // namespace nkb

int nkb_dssum(nkb_ctx* ctx, double* field, void* stream) {
  NKB_TRY(ctx_check(ctx));
  if (!ctx->gs_ready) return fail(NKB_ESTATE, "dssum needs nkb_mesh_set_global_ids");
  if (ctx->E > 0 && !field) return fail(NKB_EINVAL, "null field");
  return gs_apply(ctx, field, (cudaStream_t)stream);
}

// ---- field statistics (stats sink) --------------------------------------------

static double dec_ordered_stats(unsigned long long e) {
  const unsigned long long b = (e & 0x8000000000000000ULL) ? (e & ~0x8000000000000000ULL) : ~e;
  double d;
  memcpy(&d, &b, sizeof(d));
  return d;
}

static void stats_bind(const StatsTables& T, StatsParams& P) {
  P.chunks = T.d_chunks;
  P.n_chunks = T.n_dev;
  P.shapes = T.d_shapes;
  P.leaves = T.d_leaves;
  P.nodes = T.d_nodes;
  P.level_start = T.d_levels;
  P.out_sum = T.d_out;
  P.out_mm = reinterpret_cast<unsigned long long*>(T.d_out + T.n_dev);
}

// upload chunk list + shape tables; returns the kernel parameters
static int stats_upload(StatsTables& T, const std::vector<StatChunk>& chunks, StatsParams& P) {
  std::vector<StatShape> shp;
  std::vector<int2> lv, nd;
  std::vector<int> ls;
  for (auto& sh : T.shapes) {
    StatShape d;
    d.leaf0 = (int)lv.size();
    d.n_leaves = (int)sh.leaves.size();
    d.node0 = (int)nd.size();
    d.n_nodes = (int)sh.nodes.size();
    d.level0 = (int)ls.size();
    d.n_levels = sh.n_levels;
    lv.insert(lv.end(), sh.leaves.begin(), sh.leaves.end());
    nd.insert(nd.end(), sh.nodes.begin(), sh.nodes.end());
    ls.insert(ls.end(), sh.level_start.begin(), sh.level_start.end());
    shp.push_back(d);
  }
  if (nd.empty()) nd.push_back(make_int2(0, 0));
  if (ls.empty()) ls.push_back(0);
  stats_tables_free(T);
  const int n = (int)chunks.size();
  NKB_CUDA(cudaMalloc(&T.d_chunks, sizeof(StatChunk) * std::max(n, 1)));
  NKB_CUDA(cudaMalloc(&T.d_shapes, sizeof(StatShape) * std::max<size_t>(shp.size(), 1)));
  NKB_CUDA(cudaMalloc(&T.d_leaves, sizeof(int2) * std::max<size_t>(lv.size(), 1)));
  NKB_CUDA(cudaMalloc(&T.d_nodes, sizeof(int2) * nd.size()));
  NKB_CUDA(cudaMalloc(&T.d_levels, sizeof(int) * ls.size()));
  NKB_CUDA(cudaMalloc(&T.d_out, sizeof(double) * (n + 3)));
  NKB_CUDA(cudaMallocHost(&T.h_out, sizeof(double) * (n + 3)));
  if (n) NKB_CUDA(cudaMemcpy(T.d_chunks, chunks.data(), sizeof(StatChunk) * n, cudaMemcpyHostToDevice));
  if (!shp.empty()) NKB_CUDA(cudaMemcpy(T.d_shapes, shp.data(), sizeof(StatShape) * shp.size(), cudaMemcpyHostToDevice));
  if (!lv.empty()) NKB_CUDA(cudaMemcpy(T.d_leaves, lv.data(), sizeof(int2) * lv.size(), cudaMemcpyHostToDevice));
  NKB_CUDA(cudaMemcpy(T.d_nodes, nd.data(), sizeof(int2) * nd.size(), cudaMemcpyHostToDevice));
  NKB_CUDA(cudaMemcpy(T.d_levels, ls.data(), sizeof(int) * ls.size(), cudaMemcpyHostToDevice));
  T.n_dev = n;
  stats_bind(T, P);
  return NKB_OK;
}

int nkb_stats(nkb_ctx* ctx, const nkb_segment* segs, int nseg, int collective, double out[3], void* stream) {
  NKB_TRY(ctx_check(ctx));
  if (!out || (nseg > 0 && !segs)) return fail(NKB_EINVAL, "null argument");
  if (nseg < 0 || nseg > kMaxSeg) return fail(NKB_EINVAL, "between 0 and 16 segments");
  cudaStream_t s = (cudaStream_t)stream;
  StatsParams P;
  memset(&P, 0, sizeof(P));
  long long n = 0;
  for (int i = 0; i < nseg; ++i) {
    const nkb_segment& g = segs[i];
    if (g.n_tuples < 0 || g.ncomp < 1) return fail(NKB_EINVAL, "bad segment shape");
    if (g.n_tuples > 0 && !g.base) return fail(NKB_EINVAL, "null segment pointer");
    if (g.ncomp > 1 && g.comp_stride < g.n_tuples) return fail(NKB_EINVAL, "comp_stride smaller than the tuple count");
    if (g.n_tuples == 0) continue;
    StatSeg& d = P.seg[P.nseg++];
    d.base = g.base;
    d.n_tuples = g.n_tuples;
    d.ncomp = g.ncomp;
    d.comp_stride = g.ncomp > 1 ? g.comp_stride : g.n_tuples;
    d.start = n;
    n += g.n_tuples * g.ncomp;
  }
  P.n = n;
  // global layout: rank r holds values [lo[r], lo[r+1])
  const bool coll = collective && ctx->comm && ctx->nranks > 1;
  const int R = coll ? ctx->nranks : 1, me = coll ? ctx->rank : 0;
  std::vector<long long> lo(R + 1, 0);
  if (coll) {
    unsigned long long* d = nullptr;
    NKB_CUDA(cudaMallocAsync(&d, sizeof(unsigned long long) * (R + 1), s));
    const unsigned long long mine = (unsigned long long)n;
    NKB_CUDA(cudaMemcpyAsync(d + R, &mine, sizeof(mine), cudaMemcpyHostToDevice, s));
    NKB_NCCL(g_nccl.AllGather(d + R, d, 1, ncclUint64, ctx->comm, s));
    std::vector<unsigned long long> cnt(R);
    NKB_CUDA(cudaMemcpyAsync(cnt.data(), d, sizeof(unsigned long long) * R, cudaMemcpyDeviceToHost, s));
    NKB_CUDA(cudaFreeAsync(d, s));
    NKB_CUDA(cudaStreamSynchronize(s));
    for (int r = 0; r < R; ++r) lo[r + 1] = lo[r] + (long long)cnt[r];
  } else {
    lo[1] = n;
  }
  const long long N = lo[R];
  if (N == 0) return fail(NKB_EINVAL, "zero-size array to reduction operation minimum which has no identity");

  // the plan and its device tables depend only on the rank layout: cached
  auto key = lo;
  key.push_back(me);
  auto& slot = ctx->stats_cache[key];
  const bool fresh = !slot;
  if (fresh) {
    if (ctx->stats_cache.size() > 32) {           // bounded: drop the others
      for (auto& kv : ctx->stats_cache)
        if (kv.second && kv.first != key) stats_tables_free(*kv.second);
      auto keep = std::move(slot);
      ctx->stats_cache.clear();
      ctx->stats_cache[key] = std::move(keep);
    }
    ctx->stats_cache[key].reset(new StatsTables());
  }
  StatsTables& T = *ctx->stats_cache[key];
  std::vector<int> boundary;
  const int nc_plan = fresh ? -1 : (int)T.plan.size();
  if (fresh) {
    pairwise_plan(N, lo, T.plan);
    T.owned_count.assign(R, 0);
  }
  const int nc = (int)T.plan.size();
  for (int i = 0; i < nc; ++i) {
    const PlanChunk& c = T.plan[i];
    if (c.owner < 0) {
      boundary.push_back(i);
      continue;
    }
    if (!fresh) continue;
    ++T.owned_count[c.owner];
    if (c.owner == me) {
      const int sid = shape_id(T, c.n);
      if (sid < 0) return fail(NKB_EINVAL, "internal: chunk shape too large");
      T.mine.push_back({c.off - lo[me], sid});
      T.mine_idx.push_back(i);
    }
  }
  (void)nc_plan;
  std::vector<double> sums(nc, 0.0);
  double mn = INFINITY, mx = -INFINITY;
  bool nan = false;
  // one launch over `chunks`: hs = chunk sums, hm = {min, max, NaN flag} of all their values
  auto run = [&](StatsTables& TT, const std::vector<StatChunk>& chunks, bool upload, StatsParams& Q,
                 std::vector<double>& hs, std::vector<double>& hm) -> int {
    if (upload) NKB_TRY(stats_upload(TT, chunks, Q));
    else stats_bind(TT, Q);
    const int m = (int)chunks.size();
    NKB_CUDA(cudaMemsetAsync(Q.out_mm, 0xff, sizeof(unsigned long long), s));       // enc(min) <- max
    NKB_CUDA(cudaMemsetAsync(Q.out_mm + 1, 0, 2 * sizeof(unsigned long long), s));  // enc(max), NaN <- 0
    NKB_TRY(launch_pairwise_chunks(Q, s));
    NKB_CUDA(cudaMemcpyAsync(TT.h_out, TT.d_out, sizeof(double) * (m + 3), cudaMemcpyDeviceToHost, s));
    NKB_CUDA(cudaStreamSynchronize(s));
    hs.assign(TT.h_out, TT.h_out + m);
    unsigned long long w[3];
    memcpy(w, TT.h_out + m, sizeof(w));
    hm = {w[0] == ~0ULL ? INFINITY : dec_ordered_stats(w[0]), w[1] == 0ULL ? -INFINITY : dec_ordered_stats(w[1]),
          w[2] ? 1.0 : 0.0};
    return NKB_OK;
  };
  std::vector<double> hs, hm;
  NKB_TRY(run(T, T.mine, fresh, P, hs, hm));
  const double lmn = hm[0], lmx = hm[1], lnan = hm[2];
  if (!coll) {
    for (size_t k = 0; k < T.mine.size(); ++k) sums[T.mine_idx[k]] = hs[k];
    mn = lmn;
    mx = lmx;
    nan = lnan != 0.0;
  } else {
    // every rank's owned chunk sums (contiguous in plan order) + min / max
    int maxo = 0;
    for (int r = 0; r < R; ++r) maxo = std::max(maxo, T.owned_count[r]);
    const int w = maxo + 3;
    std::vector<double> send(w, 0.0), all((size_t)w * R);
    for (size_t k = 0; k < T.mine.size(); ++k) send[k] = hs[k];
    send[maxo] = lmn;
    send[maxo + 1] = lmx;
    send[maxo + 2] = lnan;
    double* d = nullptr;
    NKB_CUDA(cudaMallocAsync(&d, sizeof(double) * (size_t)w * (R + 1), s));
    NKB_CUDA(cudaMemcpyAsync(d + (size_t)w * R, send.data(), sizeof(double) * w, cudaMemcpyHostToDevice, s));
    NKB_NCCL(g_nccl.AllGather(d + (size_t)w * R, d, w, ncclFloat64, ctx->comm, s));
    NKB_CUDA(cudaMemcpyAsync(all.data(), d, sizeof(double) * (size_t)w * R, cudaMemcpyDeviceToHost, s));
    // boundary windows: first / last kWin values of every rank
    std::vector<double> win((size_t)2 * kWin * R);
    double* dw = nullptr;
    if (!boundary.empty()) {
      NKB_CUDA(cudaMallocAsync(&dw, sizeof(double) * 2 * kWin * (R + 1), s));
      NKB_TRY(launch_stat_windows(P, dw + (size_t)2 * kWin * R, s));
      NKB_NCCL(g_nccl.AllGather(dw + (size_t)2 * kWin * R, dw, 2 * kWin, ncclFloat64, ctx->comm, s));
      NKB_CUDA(cudaMemcpyAsync(win.data(), dw, sizeof(double) * 2 * kWin * R, cudaMemcpyDeviceToHost, s));
    }
    NKB_CUDA(cudaStreamSynchronize(s));
    NKB_CUDA(cudaFreeAsync(d, s));
    if (dw) NKB_CUDA(cudaFreeAsync(dw, s));
    std::vector<int> seen(R, 0);
    for (int i = 0; i < nc; ++i) {
      const int o = T.plan[i].owner;
      if (o >= 0) sums[i] = all[(size_t)w * o + seen[o]++];
    }
    for (int r = 0; r < R; ++r) {
      if (lo[r + 1] == lo[r]) continue;
      mn = fmin(mn, all[(size_t)w * r + maxo]);
      mx = fmax(mx, all[(size_t)w * r + maxo + 1]);
      if (all[(size_t)w * r + maxo + 2] != 0.0) nan = true;
    }
    if (!boundary.empty()) {
      // the leaves across rank boundaries, rebuilt from the windows and
      // summed on the GPU like any other chunk (every rank, same result)
      std::vector<double> vals;
      std::vector<StatChunk> bch;
      StatsTables TB;
      for (int i : boundary) {
        const PlanChunk& c = T.plan[i];
        bch.push_back({(long long)vals.size(), shape_id(TB, c.n)});
        for (long long g = c.off; g < c.off + c.n; ++g) {
          const int r = (int)(std::upper_bound(lo.begin(), lo.end(), g) - lo.begin()) - 1;
          const long long l = g - lo[r], nr = lo[r + 1] - lo[r];
          vals.push_back(l < kWin ? win[(size_t)2 * kWin * r + l]
                                  : win[(size_t)2 * kWin * r + kWin + (l - (nr - kWin))]);
        }
      }
      double* dv = nullptr;
      NKB_CUDA(cudaMalloc(&dv, sizeof(double) * vals.size()));
      NKB_CUDA(cudaMemcpy(dv, vals.data(), sizeof(double) * vals.size(), cudaMemcpyHostToDevice));
      StatsParams B;
      memset(&B, 0, sizeof(B));
      B.nseg = 1;
      B.seg[0] = {dv, (long long)vals.size(), 1, (long long)vals.size(), 0};
      B.n = (long long)vals.size();
      std::vector<double> bs, bm;
      const int rc = run(TB, bch, true, B, bs, bm);
      cudaFree(dv);
      stats_tables_free(TB);
      NKB_TRY(rc);
      for (size_t k = 0; k < boundary.size(); ++k) sums[boundary[k]] = bs[k];
      mn = fmin(mn, bm[0]);
      mx = fmax(mx, bm[1]);
      if (bm[2] != 0.0) nan = true;
    }
  }
  if (T.comb.empty()) pairwise_combine_program(N, lo, T.comb);
  const double total = 0.0 + pairwise_combine(T.comb, sums);     // np.add.reduce: identity + pairwise
  out[0] = nan ? NAN : mn;
  out[1] = nan ? NAN : mx;
  out[2] = total / (double)N;                                    // np.mean: sum / count
  return NKB_OK;
}

