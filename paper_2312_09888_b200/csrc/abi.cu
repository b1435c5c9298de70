// C ABI of libnekb200.so (see include/nekb200.h for the contract and the
// reference interface each entry point replaces).
//
// Host-side orchestration of one in situ step:
//   reset scan state -> K1 fused (adaptor+grad+Q+classify+emit) -> K2 raster
//   -> [NCCL min-reduce of packed keys + range words] -> K3 resolve -> report
// The step is stream-ordered; nkb_execute synchronises once at the end to fill
// the report (SENSEI's Execute returns after the analysis ran).
#include <cuda_runtime.h>
#include <cstdio>
#include <dlfcn.h>
#include <math.h>
#include <nccl.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <array>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "ctx.h"

namespace nkb {

static thread_local std::string g_err;

void set_error(const std::string& msg) { g_err = msg; }
int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

NcclApi g_nccl;

int load_nccl() {
  if (g_nccl.ok) return NKB_OK;
  const char* names[] = {"libnccl.so.2", "libnccl.so"};
  for (const char* n : names) {
    g_nccl.h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
    if (g_nccl.h) break;
  }
  if (!g_nccl.h) return fail(NKB_ENCCL, "cannot dlopen libnccl.so.2");
#define NKB_SYM(field, name)                                             \
  g_nccl.field = reinterpret_cast<decltype(g_nccl.field)>(dlsym(g_nccl.h, name)); \
  if (!g_nccl.field) return fail(NKB_ENCCL, std::string("missing NCCL symbol ") + name);
  NKB_SYM(GetUniqueId, "ncclGetUniqueId");
  NKB_SYM(CommInitRank, "ncclCommInitRank");
  NKB_SYM(CommDestroy, "ncclCommDestroy");
  NKB_SYM(Reduce, "ncclReduce");
  NKB_SYM(AllReduce, "ncclAllReduce");
  NKB_SYM(AllGather, "ncclAllGather");
  NKB_SYM(Send, "ncclSend");
  NKB_SYM(Recv, "ncclRecv");
  NKB_SYM(GroupStart, "ncclGroupStart");
  NKB_SYM(GroupEnd, "ncclGroupEnd");
  NKB_SYM(GetErrorString, "ncclGetErrorString");
#undef NKB_SYM
  g_nccl.ok = true;
  return NKB_OK;
}



constexpr int kMaxRegions = 1024;   // >= SM count: one triangle region per fused CTA

// mesh bounds reduction (defined in mesh_export.cu)
int launch_bounds_kernel(const double* x, const double* y, const double* z, int64_t n,
                         unsigned long long* enc6, cudaStream_t s);

}  // namespace nkb

using namespace nkb;


static void p2p_release(nkb_ctx* ctx) {
  if (ctx->comp_stream) cudaStreamSynchronize(ctx->comp_stream);   // composite halves still reading the buffers
  for (void* q : ctx->p2p.opened) cudaIpcCloseMemHandle(q);
  ctx->p2p.opened.clear();
  cudaFree(ctx->p2p.keys[0]);
  cudaFree(ctx->p2p.keys[1]);
  cudaFree(ctx->p2p.flags);
  cudaFree(ctx->p2p.err);
  cudaFree(ctx->p2p.dev_epoch);
  cudaFreeHost(ctx->p2p.h_res);
  ctx->p2p.keys[0] = ctx->p2p.keys[1] = nullptr;
  ctx->p2p.flags = nullptr;
  ctx->p2p.err = nullptr;
  ctx->p2p.dev_epoch = nullptr;
  ctx->p2p.h_res = nullptr;
  ctx->p2p.h_res_dev = nullptr;
  ctx->p2p.ready = false;
  for (int k = 0; k < 2; ++k) {                       // captured steps reference these buffers
    if (ctx->graph_exec[k]) cudaGraphExecDestroy(ctx->graph_exec[k]);
    ctx->graph_exec[k] = nullptr;
    ctx->graph_key[k].clear();
    if (ctx->graph_exec_a[k]) cudaGraphExecDestroy(ctx->graph_exec_a[k]);
    ctx->graph_exec_a[k] = nullptr;
    ctx->graph_key_a[k].clear();
    if (ctx->graph_exec_b[k]) cudaGraphExecDestroy(ctx->graph_exec_b[k]);
    ctx->graph_exec_b[k] = nullptr;
    ctx->graph_key_b[k].clear();
  }
}

// collective: every rank calls it with the same image size.  Allocates the two
// key buffers and the flag array, then exchanges CUDA IPC handles (keys x2,
// flags, and the image of every rank) with one ncclAllGather.
static int p2p_setup(nkb_ctx* ctx, int W, int H, cudaStream_t s) {
  auto& P = ctx->p2p;
  if (P.ready && P.W == W && P.H == H) return NKB_OK;
  if (P.ready) {
    NKB_CUDA(cudaStreamSynchronize(s));
    p2p_release(ctx);
  }
  const size_t npx = (size_t)W * H;
  NKB_CUDA(cudaMalloc(&P.keys[0], (npx + 2) * sizeof(unsigned long long)));
  NKB_CUDA(cudaMalloc(&P.keys[1], (npx + 2) * sizeof(unsigned long long)));
  NKB_CUDA(cudaMalloc(&P.flags, 4 * kMaxRanks * sizeof(unsigned long long)));
  NKB_CUDA(cudaMemset(P.flags, 0, 4 * kMaxRanks * sizeof(unsigned long long)));
  NKB_CUDA(cudaMalloc(&P.err, sizeof(int)));
  NKB_CUDA(cudaMemset(P.err, 0, sizeof(int)));
  NKB_CUDA(cudaMalloc(&P.dev_epoch, 3 * sizeof(unsigned long long)));
  NKB_CUDA(cudaMemset(P.dev_epoch, 0, 3 * sizeof(unsigned long long)));
  NKB_CUDA(cudaMallocHost(&P.h_res, (2 + kMaxRanks) * sizeof(unsigned long long)));
  memset(P.h_res, 0, (2 + kMaxRanks) * sizeof(unsigned long long));
  NKB_CUDA(cudaHostGetDevicePointer((void**)&P.h_res_dev, P.h_res, 0));
  constexpr int kH = 5;
  cudaIpcMemHandle_t mine[kH];
  void* ptrs[kH] = {P.keys[0], P.keys[1], P.flags, ctx->rgba, ctx->depth};
  for (int i = 0; i < kH; ++i) NKB_CUDA(cudaIpcGetMemHandle(&mine[i], ptrs[i]));
  const size_t hb = sizeof(mine);
  char *d_send = nullptr, *d_recv = nullptr;
  NKB_CUDA(cudaMalloc(&d_send, hb));
  NKB_CUDA(cudaMalloc(&d_recv, hb * ctx->nranks));
  NKB_CUDA(cudaMemcpy(d_send, mine, hb, cudaMemcpyHostToDevice));
  NKB_NCCL(g_nccl.AllGather(d_send, d_recv, hb, ncclChar, ctx->comm, s));
  std::vector<cudaIpcMemHandle_t> all((size_t)kH * ctx->nranks);
  NKB_CUDA(cudaMemcpyAsync(all.data(), d_recv, hb * ctx->nranks, cudaMemcpyDeviceToHost, s));
  NKB_CUDA(cudaStreamSynchronize(s));
  cudaFree(d_recv);
  int ok = 1;
  for (int q = 0; q < ctx->nranks && ok; ++q) {
    void* mapped[kH];
    for (int i = 0; i < kH; ++i) {
      if (q == ctx->rank) {
        mapped[i] = ptrs[i];
        continue;
      }
      cudaError_t e = cudaIpcOpenMemHandle(&mapped[i], all[(size_t)q * kH + i], cudaIpcMemLazyEnablePeerAccess);
      if (e != cudaSuccess) {
        cudaGetLastError();
        ok = 0;
        break;
      }
      P.opened.push_back(mapped[i]);
    }
    if (!ok) break;
    P.peer_keys[0][q] = (const unsigned long long*)mapped[0];
    P.peer_keys[1][q] = (const unsigned long long*)mapped[1];
    P.peer_flags[q] = (unsigned long long*)mapped[2];
    if (q == 0) {
      P.root_rgba = (unsigned char*)mapped[3];
      P.root_depth = (float*)mapped[4];
    }
  }
  // every rank takes the same path: one rank that cannot map a peer (partial
  // peer-access topology) sends all of them to the NCCL composite
  int* d_ok = reinterpret_cast<int*>(d_send);
  NKB_CUDA(cudaMemcpyAsync(d_ok, &ok, sizeof(int), cudaMemcpyHostToDevice, s));
  NKB_NCCL(g_nccl.AllReduce(d_ok, d_ok, 1, ncclInt32, ncclMin, ctx->comm, s));
  int all_ok = 0;
  NKB_CUDA(cudaMemcpyAsync(&all_ok, d_ok, sizeof(int), cudaMemcpyDeviceToHost, s));
  NKB_CUDA(cudaStreamSynchronize(s));
  cudaFree(d_send);
  if (!all_ok) {
    p2p_release(ctx);           // closes the mappings this rank did open
    P.unavailable = true;       // no peer mapping somewhere: the NCCL composite is used instead
    return NKB_OK;
  }
  P.W = W;
  P.H = H;
  P.epoch = 0;
  P.ready = true;
  return NKB_OK;
}

// checked build (NKB_CHECKED): device bounds-check violations of the last
// kernels, per source file; the product build's accessors return 0
int nkb::checked_violations() {
  struct {
    const char* file;
    unsigned long long (*read)(int*);
  } src[] = {{"fused.cu", checked_read_fused},
             {"stream.cu", checked_read_stream},
             {"raster.cu", checked_read_raster},
             {"composite.cu", checked_read_composite}};
  for (auto& f : src) {
    int line = 0;
    const unsigned long long n = f.read(&line);
    if (n) return fail(NKB_ECUDA, std::string("device bounds check failed ") + std::to_string(n) + "x, first at " +
                                      f.file + ":" + std::to_string(line));
  }
  return NKB_OK;
}

int nkb::ctx_check(nkb_ctx* ctx) {
  if (!ctx) return fail(NKB_EINVAL, "null context");
  NKB_CUDA(cudaSetDevice(ctx->device));
  return NKB_OK;
}

extern "C" {

int nkb_abi_version(void) { return NKB_ABI_VERSION; }
const char* nkb_last_error(void) { return g_err.c_str(); }

int nkb_device_count(int* out) {
  if (!out) return fail(NKB_EINVAL, "null out");
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    *out = 0;
    return fail(NKB_ECUDA, std::string("cudaGetDeviceCount: ") + cudaGetErrorString(e));
  }
  *out = n;
  return NKB_OK;
}

int nkb_gll(int order, double* nodes, double* dmat) {
  if (order < 1 || order > 30) return fail(NKB_EINVAL, "order must be in [1, 30]");
  std::vector<double> x(order + 1), D((order + 1) * (order + 1));
  gll_nodes_dmat(order, x.data(), D.data());
  if (nodes) memcpy(nodes, x.data(), sizeof(double) * x.size());
  if (dmat) memcpy(dmat, D.data(), sizeof(double) * D.size());
  return NKB_OK;
}

int nkb_ctx_create(int cuda_device, nkb_ctx** out) {
  if (!out) return fail(NKB_EINVAL, "null out");
  *out = nullptr;
  int n = 0;
  NKB_CUDA(cudaGetDeviceCount(&n));
  if (cuda_device < 0 || cuda_device >= n)
    return fail(NKB_EINVAL, "cuda_device " + std::to_string(cuda_device) + " out of range (" +
                                std::to_string(n) + " devices)");
  NKB_CUDA(cudaSetDevice(cuda_device));
  nkb_ctx* c = new nkb_ctx();
  c->device = cuda_device;
  gll_nodes_dmat(kN, c->gll, c->D);
  NKB_CUDA(cudaMalloc(&c->counters, 64));
  c->ticket = reinterpret_cast<unsigned int*>(c->counters + 4);
  NKB_CUDA(cudaMalloc(&c->range_dev, 2 * sizeof(double)));
  NKB_CUDA(cudaMallocHost(&c->h_counters, (8 + kMaxRegions) * sizeof(unsigned long long)));
  memset(c->h_counters, 0, (8 + kMaxRegions) * sizeof(unsigned long long));
  NKB_CUDA(cudaHostGetDevicePointer((void**)&c->h_counters_dev, c->h_counters, 0));
  NKB_CUDA(cudaMalloc(&c->region_count, kMaxRegions * sizeof(unsigned long long)));
  for (auto& e : c->ev) NKB_CUDA(cudaEventCreate(&e));
  if (const char* g = getenv("NKB_GEOM_CACHE")) c->geo_enabled = strcmp(g, "0") == 0 ? 0 : (strcmp(g, "full") == 0 ? 2 : 1);
  *out = c;
  return NKB_OK;
}

int nkb_ctx_destroy(nkb_ctx* ctx) {
  if (!ctx) return NKB_OK;
  cudaSetDevice(ctx->device);
  cudaDeviceSynchronize();
  p2p_release(ctx);
  if (ctx->comm && g_nccl.ok) g_nccl.CommDestroy(ctx->comm);
  cudaFree(ctx->elem_count);
  cudaFree(ctx->elem_offset);
  cudaFree(ctx->counters);
  cudaFree(ctx->tri);
  cudaFree(ctx->meta);
  cudaFree(ctx->region_count);
  cudaFree(ctx->tri_export);
  cudaFree(ctx->meta_export);
  cudaFree(ctx->zbufs[0]);
  cudaFree(ctx->rticket);
  cudaFree(ctx->rgba);
  cudaFree(ctx->depth);
  cudaFree(ctx->range_dev);
  cudaFree(ctx->geo);
  cudaFree(ctx->geo_flag);
  cudaFree(ctx->prof);
  for (auto& kv : ctx->stats_cache)
    if (kv.second) stats_tables_free(*kv.second);
  gs_free(ctx->gs);
  cudaFree(ctx->tr_buf);
  for (int k = 0; k < 2; ++k) {
    if (ctx->graph_exec[k]) cudaGraphExecDestroy(ctx->graph_exec[k]);
    if (ctx->graph_exec_a[k]) cudaGraphExecDestroy(ctx->graph_exec_a[k]);
    if (ctx->graph_exec_b[k]) cudaGraphExecDestroy(ctx->graph_exec_b[k]);
    if (ctx->ev_a[k]) cudaEventDestroy(ctx->ev_a[k]);
    if (ctx->ev_b[k]) cudaEventDestroy(ctx->ev_b[k]);
  }
  if (ctx->cap_stream) cudaStreamDestroy(ctx->cap_stream);
  if (ctx->comp_stream) cudaStreamDestroy(ctx->comp_stream);
  cudaFree(ctx->csnap);
  cudaFree(ctx->dq);
  cudaFree(ctx->dw);
  cudaFree(ctx->rgb_dev);
  cudaFreeHost(ctx->h_ppm);
  cudaFree(ctx->s_ptrs);
  cudaFree(ctx->s_col0);
  cudaFree(ctx->s_minmax);
  cudaFreeHost(ctx->h_counters);
  for (auto& e : ctx->ev)
    if (e) cudaEventDestroy(e);
  delete ctx;
  return NKB_OK;
}

// ---- DataAdaptor -------------------------------------------------------------

int nkb_mesh_set(nkb_ctx* ctx, int64_t n_elements, int order, const double* x, const double* y,
                 const double* z, int64_t element_offset, int64_t n_elements_global) {
  NKB_TRY(ctx_check(ctx));
  if (order != kN)
    return fail(NKB_EINVAL, "unsupported polynomial order " + std::to_string(order) +
                                " (this build supports N=" + std::to_string(kN) + ")");
  if (n_elements < 0) return fail(NKB_EINVAL, "negative element count");
  if (n_elements > 0 && (!x || !y || !z)) return fail(NKB_EINVAL, "null coordinate pointer");
  if (n_elements > (int64_t)0x7fffffff) return fail(NKB_EINVAL, "too many elements for one rank");
  const bool same = ctx->E == n_elements && ctx->N == order && ctx->x == x && ctx->y == y && ctx->z == z;
  if (!same) {
    ctx->geo_valid = false;                // a different mesh: rebuild the geometry cache on demand
    ctx->gs_ready = false;                 // ... and the global-id gather-scatter must be set again
  }
  ctx->E = n_elements;
  ctx->N = order;
  ctx->x = x;
  ctx->y = y;
  ctx->z = z;
  ctx->elem_off = element_offset;
  ctx->E_global = n_elements_global > 0 ? n_elements_global : n_elements;
  NKB_TRY(set_dmat_constant(ctx->D));
  ctx->image_valid = false;
  return NKB_OK;
}

int nkb_field_set(nkb_ctx* ctx, const char* name, int ncomp, const double* base, int64_t comp_stride) {
  NKB_TRY(ctx_check(ctx));
  if (!name || !*name) return fail(NKB_EINVAL, "empty field name");
  if (strchr(name, ':')) return fail(NKB_EINVAL, "field names may not contain ':'");
  if (ncomp < 1 || ncomp > 9) return fail(NKB_EINVAL, "components must be in [1, 9]");
  if (!base && ctx->E > 0) return fail(NKB_EINVAL, "null field pointer");
  int64_t npts = ctx->E * kNN;
  if (ncomp > 1 && comp_stride < npts)
    return fail(NKB_EINVAL, "comp_stride smaller than the point count");
  for (auto& f : ctx->fields)
    if (f.name == name) {
      f.ncomp = ncomp;
      f.base = base;
      f.comp_stride = comp_stride;
      return NKB_OK;
    }
  Field f;
  f.name = name;
  f.ncomp = ncomp;
  f.base = base;
  f.comp_stride = comp_stride;
  ctx->fields.push_back(f);
  return NKB_OK;
}

int nkb_field_clear(nkb_ctx* ctx) {
  NKB_TRY(ctx_check(ctx));
  ctx->fields.clear();
  return NKB_OK;
}

int nkb_mesh_modified(nkb_ctx* ctx) {
  NKB_TRY(ctx_check(ctx));
  ctx->geo_valid = false;
  return NKB_OK;
}

static void geo_release(nkb_ctx* ctx) {
  cudaFree(ctx->geo);
  ctx->geo = nullptr;
  ctx->geo_bytes = 0;
  ctx->geo_layout = NKB_GEO_NONE;
  ctx->geo_valid = false;
}

int nkb_set_geometry_cache(nkb_ctx* ctx, int enable) {
  NKB_TRY(ctx_check(ctx));
  if (enable < 0 || enable > 2) return fail(NKB_EINVAL, "geometry cache mode must be 0 (off), 1 (on) or 2 (full layout)");
  if (enable != ctx->geo_enabled) geo_release(ctx);   // give the memory back / rebuild in the new layout
  ctx->geo_enabled = enable;
  return NKB_OK;
}

int nkb_geometry_info(nkb_ctx* ctx, int* layout, int64_t* bytes) {
  NKB_TRY(ctx_check(ctx));
  const bool built = ctx->geo_valid && ctx->geo != nullptr;
  if (layout) *layout = built ? ctx->geo_layout : NKB_GEO_NONE;
  if (bytes) *bytes = built ? ctx->geo_bytes : 0;
  return NKB_OK;
}

// Attach the geometry cache to a gradient step, building it first when the
// mesh changed: the compact layout when every element is extruded (one host
// read of the build's flag, once per mesh), else the full layout.  On
// allocation failure the step runs uncached (the other GPU kernel variant --
// same results), never on the CPU.
}  // extern "C"

int nkb::geo_attach(nkb_ctx* ctx, FusedParams& fp, cudaStream_t s) {
  fp.geo = nullptr;
  fp.geo_compact = 0;
  if (!fp.need_grad || !ctx->geo_enabled || ctx->E <= 0) return NKB_OK;
  if (!ctx->geo_valid) {
    geo_release(ctx);
    const int64_t E = ctx->E;
    if (ctx->geo_enabled == 1) {
      if (!ctx->geo_flag) NKB_CUDA(cudaMalloc(&ctx->geo_flag, sizeof(unsigned long long)));
      double* c = nullptr;
      const size_t cb = (size_t)E * kGeoCompactDoubles * sizeof(double);
      if (cudaMalloc(&c, cb) == cudaSuccess) {
        NKB_CUDA(cudaMemsetAsync(ctx->geo_flag, 0, sizeof(unsigned long long), s));
        NKB_TRY(launch_geometry(ctx->x, ctx->y, ctx->z, E, nullptr, c, ctx->geo_flag, s));
        unsigned long long n_general = 0;
        NKB_CUDA(cudaMemcpyAsync(&n_general, ctx->geo_flag, sizeof(n_general), cudaMemcpyDeviceToHost, s));
        NKB_CUDA(cudaStreamSynchronize(s));
        if (n_general == 0) {
          ctx->geo = c;
          ctx->geo_bytes = (int64_t)cb;
          ctx->geo_layout = NKB_GEO_COMPACT;
        } else {
          cudaFree(c);
        }
      } else {
        cudaGetLastError();
      }
    }
    if (!ctx->geo) {
      const size_t fb = (size_t)E * kNN * 9 * sizeof(double);
      if (cudaMalloc(&ctx->geo, fb) != cudaSuccess) {
        cudaGetLastError();
        ctx->geo = nullptr;
        return NKB_OK;
      }
      NKB_TRY(launch_geometry(ctx->x, ctx->y, ctx->z, E, ctx->geo, nullptr, nullptr, s));
      ctx->geo_bytes = (int64_t)fb;
      ctx->geo_layout = NKB_GEO_FULL;
    }
    ctx->geo_valid = true;
    ctx->geo_built = true;
  }
  fp.geo = ctx->geo;
  fp.geo_compact = ctx->geo_layout == NKB_GEO_COMPACT ? 1 : 0;
  ctx->geo_used = true;
  return NKB_OK;
}

extern "C" {


int nkb_set_velocity_name(nkb_ctx* ctx, const char* name) {
  NKB_TRY(ctx_check(ctx));
  if (!name || !*name) return fail(NKB_EINVAL, "empty velocity name");
  ctx->vel_name = name;
  return NKB_OK;
}

int nkb_get_mesh_metadata(nkb_ctx* ctx, nkb_mesh_metadata* out) {
  NKB_TRY(ctx_check(ctx));
  if (!out) return fail(NKB_EINVAL, "null out");
  out->n_elements = ctx->E;
  out->order = ctx->N;
  out->n_points = ctx->E * kNN;
  out->n_cells = ctx->E * kNC;
  out->cell_type = NKB_VTK_HEXAHEDRON;
  out->element_offset = ctx->elem_off;
  out->n_elements_global = ctx->E_global;
  out->n_fields = (int)ctx->fields.size();
  out->rank = ctx->rank;
  out->nranks = ctx->nranks;
  return NKB_OK;
}

int nkb_get_mesh(nkb_ctx* ctx, double* points, int64_t* conn, int64_t* offsets, unsigned char* types,
                 void* stream) {
  NKB_TRY(ctx_check(ctx));
  if (!ctx->x) return fail(NKB_ESTATE, "GetMesh before mesh_set");
  cudaStream_t s = (cudaStream_t)stream;
  if (ctx->E == 0) return NKB_OK;
  if (points) NKB_TRY(launch_points_aos(ctx->x, ctx->y, ctx->z, ctx->E * kNN, points, s));
  if (conn || offsets || types) NKB_TRY(launch_connectivity(ctx->E * kNC, conn, offsets, types, s));
  return NKB_OK;
}

int nkb_encode_be(nkb_ctx* ctx, const char* what, void* dst, int64_t cap, int64_t* nbytes, void* stream) {
  NKB_TRY(ctx_check(ctx));
  if (!what || !nbytes) return fail(NKB_EINVAL, "null argument");
  if (!ctx->x) return fail(NKB_ESTATE, "encode before mesh_set");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t npts = ctx->E * kNN, ncells = ctx->E * kNC;
  const std::string w(what);
  int64_t need;
  int ncomp = 0;
  if (w == "POINTS") {
    need = 24 * npts;
  } else if (w == "CELLS") {
    if (npts > 0x7fffffffLL) return fail(NKB_ERANGE, "legacy VTK CELLS hold int32 point ids: too many points");
    need = 36 * ncells;
  } else if (w == "CELL_TYPES") {
    need = 4 * ncells;
  } else {
    NKB_TRY(nkb_array_components(ctx, what, &ncomp));
    need = 8 * (int64_t)ncomp * npts;
  }
  *nbytes = need;
  if (!dst) return NKB_OK;                                     // size query
  if (cap < need) return fail(NKB_ERANGE, "destination too small: need " + std::to_string(need) + " bytes");
  if (w == "POINTS") return launch_be_points(ctx->x, ctx->y, ctx->z, npts, dst, s);
  if (w == "CELLS") return launch_be_cells(ncells, dst, s);
  if (w == "CELL_TYPES") return launch_be_types(ncells, dst, s);
  int nc = 0;
  NKB_TRY(nkb_add_array(ctx, what, 0, reinterpret_cast<double*>(dst), &nc, stream));   // AoS f64
  return launch_bswap64(dst, (int64_t)nc * npts, s);
}

int nkb_mesh_bounds(nkb_ctx* ctx, double* out6, void* stream) {
  NKB_TRY(ctx_check(ctx));
  if (!out6) return fail(NKB_EINVAL, "null out");
  if (!ctx->x) return fail(NKB_ESTATE, "bounds before mesh_set");
  cudaStream_t s = (cudaStream_t)stream;
  unsigned long long* d6 = nullptr;
  NKB_CUDA(cudaMallocAsync(&d6, 6 * sizeof(unsigned long long), s));
  NKB_CUDA(cudaMemsetAsync(d6, 0xff, 6 * sizeof(unsigned long long), s));
  NKB_TRY(launch_bounds_kernel(ctx->x, ctx->y, ctx->z, ctx->E * kNN, d6, s));
  if (ctx->comm && ctx->nranks > 1) {
    NKB_NCCL(g_nccl.AllReduce(d6, d6, 6, ncclUint64, ncclMin, ctx->comm, s));
  }
  unsigned long long h6[6];
  NKB_CUDA(cudaMemcpyAsync(h6, d6, sizeof(h6), cudaMemcpyDeviceToHost, s));
  NKB_CUDA(cudaFreeAsync(d6, s));
  NKB_CUDA(cudaStreamSynchronize(s));
  // words: enc(min x,y,z), ~enc(max x,y,z)
  for (int a = 0; a < 3; ++a) {
    out6[2 * a] = dec_ordered_h(h6[a]);
    out6[2 * a + 1] = dec_ordered_h(~h6[3 + a]);
  }
  return NKB_OK;
}

}  // extern "C"

const Field* nkb::find_field(nkb_ctx* ctx, const std::string& name) {
  for (auto& f : ctx->fields)
    if (f.name == name) return &f;
  return nullptr;
}

extern "C" {


int nkb_array_components(nkb_ctx* ctx, const char* name, int* ncomp_out) {
  NKB_TRY(ctx_check(ctx));
  if (!name || !ncomp_out) return fail(NKB_EINVAL, "null argument");
  std::string n(name);
  if (n == "Q" || n == "vorticity:mag") {
    *ncomp_out = 1;
    return NKB_OK;
  }
  if (n == "vorticity") {
    *ncomp_out = 3;
    return NKB_OK;
  }
  auto colon = n.find(':');
  std::string base = n.substr(0, colon);
  const Field* f = find_field(ctx, base);
  if (!f) return fail(NKB_EINVAL, "no field named '" + base + "'");
  if (colon == std::string::npos) {
    *ncomp_out = f->ncomp;
    return NKB_OK;
  }
  if (n.substr(colon + 1) != "mag") return fail(NKB_EINVAL, "unknown derived scalar '" + n.substr(colon + 1) + "'");
  *ncomp_out = 1;
  return NKB_OK;
}

// forward

int nkb_add_array(nkb_ctx* ctx, const char* name, int association, double* out, int* ncomp_out,
                  void* stream) {
  NKB_TRY(ctx_check(ctx));
  if (!name || !out) return fail(NKB_EINVAL, "null argument");
  if (association != NKB_ASSOC_POINT)
    return fail(NKB_EINVAL, "only point arrays exist on the SEM mesh");
  if (!ctx->x) return fail(NKB_ESTATE, "AddArray before mesh_set");
  cudaStream_t s = (cudaStream_t)stream;
  std::string n(name);
  int nc = 0;
  NKB_TRY(nkb_array_components(ctx, name, &nc));
  if (ncomp_out) *ncomp_out = nc;
  const int64_t npts = ctx->E * kNN;
  if (npts == 0) return NKB_OK;
  if (n == "Q" || n == "vorticity" || n == "vorticity:mag") {
    const Field* v = find_field(ctx, ctx->vel_name);
    if (!v || v->ncomp != 3)
      return fail(NKB_EINVAL, "derived array '" + n + "' needs a 3-component field '" + ctx->vel_name + "'");
    FusedParams fp;
    NKB_TRY(fused_params_base(ctx, fp));
    fp.need_grad = 1;
    fp.need_vel = 1;
    fp.vel[0] = v->base;
    fp.vel[1] = v->base + v->comp_stride;
    fp.vel[2] = v->base + 2 * v->comp_stride;
    fp.color_src = -1;
    fp.n_surf = 0;
    if (n == "Q") fp.q_out = out;
    if (n == "vorticity") fp.vort_out = out;
    if (n == "vorticity:mag") {
      fp.wmag_out = out;
      fp.need_wmag = 1;
    }
    NKB_CUDA(cudaMemsetAsync(ctx->counters, 0, 64, s));
    NKB_TRY(geo_attach(ctx, fp, s));
    NKB_TRY(launch_fused(fp, s));
    return NKB_OK;
  }
  auto colon = n.find(':');
  const Field* f = find_field(ctx, n.substr(0, colon));
  if (colon == std::string::npos) return launch_field_aos(f->base, f->comp_stride, f->ncomp, npts, out, s);
  return launch_field_mag(f->base, f->comp_stride, f->ncomp, npts, out, s);
}

// ---- AnalysisAdaptor::Execute ---------------------------------------------------

}  // extern "C"

int nkb::fused_params_base(nkb_ctx* ctx, FusedParams& fp) {
  memset(&fp, 0, sizeof(fp));
  fp.n_elements = ctx->E;
  fp.x = ctx->x;
  fp.y = ctx->y;
  fp.z = ctx->z;
  fp.mode = FUSED_FAST;
  fp.counters = ctx->counters;
  fp.color_src = -1;
  return NKB_OK;
}

extern "C" {


struct Resolved {
  FusedParams fp;
  Colormap cm;
};

// map a pipeline field name onto a per-node source of the fused kernel
static int resolve_src(nkb_ctx* ctx, const char* name, FusedParams& fp, int* src) {
  std::string n(name);
  if (n.empty()) return fail(NKB_EINVAL, "empty field name in pipeline");
  auto need_velocity = [&]() -> int {
    const Field* v = find_field(ctx, ctx->vel_name);
    if (!v) return fail(NKB_EINVAL, "no field named '" + ctx->vel_name + "' (needed for '" + n + "')");
    if (v->ncomp != 3)
      return fail(NKB_EINVAL, "velocity field '" + ctx->vel_name + "' must have 3 components");
    fp.need_vel = 1;
    fp.vel[0] = v->base;
    fp.vel[1] = v->base + v->comp_stride;
    fp.vel[2] = v->base + 2 * v->comp_stride;
    return NKB_OK;
  };
  if (n == "Q" || n == "vorticity:mag") {
    NKB_TRY(need_velocity());
    fp.need_grad = 1;
    *src = (n == "Q") ? SRC_Q : SRC_WMAG;
    if (n != "Q") fp.need_wmag = 1;
    return NKB_OK;
  }
  auto colon = n.find(':');
  std::string base = n.substr(0, colon);
  const Field* f = find_field(ctx, base);
  if (!f) return fail(NKB_EINVAL, "no field named '" + base + "'");
  if (colon != std::string::npos) {
    std::string suf = n.substr(colon + 1);
    if (suf != "mag") return fail(NKB_EINVAL, "unknown derived scalar '" + suf + "'");
    if (base != ctx->vel_name)
      return fail(NKB_EINVAL, "':mag' in the fused path is supported for the velocity field '" +
                                  ctx->vel_name + "' only");
    NKB_TRY(need_velocity());
    fp.need_umag = 1;
    *src = SRC_UMAG;
    return NKB_OK;
  }
  if (f->ncomp != 1)  // mirrors sinks.scalar_field (sinks.py:234-238)
    return fail(NKB_EINVAL, "field '" + base + "' has " + std::to_string(f->ncomp) +
                                " components; request a derived scalar such as '" + base + ":mag'");
  for (int k = 0; k < fp.n_scalars; ++k)
    if (fp.scalar[k] == f->base) {
      *src = SRC_SCALAR0 + k;
      return NKB_OK;
    }
  if (fp.n_scalars >= kMaxScalars)
    return fail(NKB_EINVAL, "at most " + std::to_string(kMaxScalars) + " distinct scalar fields per pipeline");
  fp.scalar[fp.n_scalars] = f->base;
  *src = SRC_SCALAR0 + fp.n_scalars;
  fp.n_scalars++;
  return NKB_OK;
}

// per-segment slopes of np.interp, computed once on the host with the same
// IEEE operations the kernels used per pixel (-ffp-contract=off): bit-identical
static void colormap_slopes(Colormap& cm) {
  for (int j = 0; j + 1 < cm.n; ++j)
    for (int ch = 0; ch < 3; ++ch) cm.slope[j][ch] = (cm.rgb[j + 1][ch] - cm.rgb[j][ch]) / (cm.t[j + 1] - cm.t[j]);
}

static int build_colormap(const nkb_pipeline* p, Colormap& cm) {
  memset(&cm, 0, sizeof(cm));
  if (p->n_anchors == 0) {  // DEFAULT_COLORMAP (sinks.py:213)
    cm.n = 3;
    const double t[3] = {0.0, 0.5, 1.0};
    const double c[3][3] = {{59, 76, 192}, {255, 255, 255}, {180, 4, 38}};
    for (int i = 0; i < 3; ++i) {
      cm.t[i] = t[i];
      for (int ch = 0; ch < 3; ++ch) cm.rgb[i][ch] = c[i][ch];
    }
    colormap_slopes(cm);
    return NKB_OK;
  }
  if (p->n_anchors < 2 || p->n_anchors > NKB_MAX_ANCHORS)
    return fail(NKB_EINVAL, "colormap needs 2..8 anchors");
  // ColorMap.__post_init__ (sinks.py:196-199)
  if (p->anchor_t[0] != 0.0 || p->anchor_t[p->n_anchors - 1] != 1.0)
    return fail(NKB_EINVAL, "anchor positions must strictly increase from 0 to 1");
  for (int i = 1; i < p->n_anchors; ++i)
    if (!(p->anchor_t[i] > p->anchor_t[i - 1]))
      return fail(NKB_EINVAL, "anchor positions must strictly increase from 0 to 1");
  cm.n = p->n_anchors;
  for (int i = 0; i < cm.n; ++i) {
    cm.t[i] = p->anchor_t[i];
    for (int ch = 0; ch < 3; ++ch) cm.rgb[i][ch] = (double)p->anchor_rgb[i][ch];
  }
  colormap_slopes(cm);
  return NKB_OK;
}

static int ensure_image(nkb_ctx* ctx, int W, int H) {
  if (ctx->W == W && ctx->H == H && ctx->zbuf) return NKB_OK;
  cudaFree(ctx->zbufs[0]);
  cudaFree(ctx->rgba);
  cudaFree(ctx->depth);
  ctx->zbuf = ctx->zbufs[0] = ctx->zbufs[1] = nullptr;
  ctx->rgba = nullptr;
  ctx->depth = nullptr;
  const size_t npx = (size_t)W * H;
  // the second buffer starts 256-byte aligned whatever W*H is (bulk copies of
  // a key buffer -- the partition composite -- need 16-byte alignment)
  const size_t zstride = (npx + 2 + 31) & ~size_t(31);
  NKB_CUDA(cudaMalloc(&ctx->zbufs[0], 2 * zstride * sizeof(unsigned long long)));
  NKB_CUDA(cudaMemset(ctx->zbufs[0], 0xff, 2 * zstride * sizeof(unsigned long long)));
  ctx->zbufs[1] = ctx->zbufs[0] + zstride;
  ctx->zbuf = ctx->zbufs[0];
  ctx->zpar_next = 0;
  ctx->znext_clean = true;
  if (!ctx->rticket) {
    NKB_CUDA(cudaMalloc(&ctx->rticket, sizeof(unsigned int)));
    NKB_CUDA(cudaMemset(ctx->rticket, 0, sizeof(unsigned int)));
  }
  NKB_CUDA(cudaMalloc(&ctx->rgba, npx * 4));
  NKB_CUDA(cudaMalloc(&ctx->depth, npx * sizeof(float)));
  ctx->W = W;
  ctx->H = H;
  return NKB_OK;
}

// threads per triangle in K2: four when the image has >= 256 pixels per
// element of the whole mesh -- few, large triangles (C1: 2048 px per element,
// raster 0.051 -> 0.027 ms) -- else one (C2-C5: 1-32 px per element, where
// splitting rows only adds set-up work; profiles/r2/raster_lanes_ab.txt).
// NKB_RASTER_LANES=1|2|4 overrides.
static int raster_lanes(const nkb_ctx* ctx, const nkb_pipeline* p) {
  static const int forced = [] {
    const char* v = getenv("NKB_RASTER_LANES");
    const int k = v ? atoi(v) : 0;
    return k == 1 || k == 2 || k == 4 ? k : 0;
  }();
  if (forced) return forced;
  const long long e = ctx->E_global > 0 ? ctx->E_global : ctx->E;
  return e > 0 && (long long)p->width * p->height >= 256 * e ? 4 : 1;
}

static int ensure_tri(nkb_ctx* ctx, int64_t cap, bool meta) {
  if (cap <= ctx->tri_cap && (!meta || ctx->meta_alloc)) return NKB_OK;
  cap = std::max(cap, ctx->tri_cap);
  cudaFree(ctx->tri);
  cudaFree(ctx->meta);
  ctx->tri = nullptr;
  ctx->meta = nullptr;
  ctx->meta_alloc = false;
  NKB_CUDA(cudaMalloc(&ctx->tri, (size_t)cap * 3 * sizeof(float4)));
  if (meta || ctx->meta_alloc) {
    NKB_CUDA(cudaMalloc(&ctx->meta, (size_t)cap * sizeof(unsigned long long)));
    ctx->meta_alloc = true;
  }
  ctx->tri_cap = cap;
  return NKB_OK;
}

// Enqueue one step on stream s (no host synchronisation): memsets -> K1
// (or count/scan/ordered emit) -> zbuf clear -> raster -> range words ->
// composite -> resolve -> D2H of the report words.
// part 3: the whole step on `s`.  P2P steps may be enqueued in two halves
// (run_step): part 1 = surface pass .. raster .. "keys ready" + the counter
// report, part 2 = composite .. "done reading" + the range / P2P report on
// the composite stream; part 2 then reads the step's epoch and counters from
// their parity slots, which the next step's part 1 does not touch.
static int enqueue_step(nkb_ctx* ctx, const nkb_pipeline* p, FusedParams fp, const Colormap& cm, cudaStream_t s,
                        bool composite, bool ordered, unsigned long long ep, int part = 3) {
  const bool timing = p->timing != 0;
  const int64_t npx = (int64_t)p->width * p->height;
  const bool split = part != 3;
  const int par = (int)(ep & 1);
  if (part & 1) {
  fp.tri = ctx->tri;
  fp.meta = p->emit_meta ? ctx->meta : nullptr;
  fp.tri_cap = ctx->tri_cap;
  ctx->n_regions = fused_grid_for(fp, ctx->E);
  ctx->region_cap = ctx->tri_cap / ctx->n_regions;
  fp.region_cap = ctx->region_cap;
  fp.region_count = ctx->region_count;
  // every surface-pass CTA assigns its region's count (FAST mode); only an
  // empty partition (no launch) needs the zero
  if (ctx->E <= 0) NKB_CUDA(cudaMemsetAsync(ctx->region_count, 0, sizeof(unsigned long long) * ctx->n_regions, s));
  // counters {0, enc(+max), 0, 0}
  NKB_TRY(launch_init_counters(ctx->counters, s));
  if (timing) NKB_CUDA(cudaEventRecord(ctx->ev[0], s));
  if (ordered) {
    // deterministic (element, cell, surface, table) order: count, scan, emit
    if (ctx->elem_cap < ctx->E) {
      cudaFree(ctx->elem_count);
      cudaFree(ctx->elem_offset);
      ctx->elem_count = nullptr;
      ctx->elem_offset = nullptr;
      NKB_CUDA(cudaMalloc(&ctx->elem_count, sizeof(int) * ctx->E));
      NKB_CUDA(cudaMalloc(&ctx->elem_offset, sizeof(long long) * ctx->E));
      ctx->elem_cap = ctx->E;
    }
    FusedParams fc = fp;
    fc.mode = FUSED_COUNT;
    fc.elem_count = ctx->elem_count;
    NKB_TRY(launch_fused(fc, s));
    NKB_TRY(launch_count_scan(ctx->elem_count, ctx->E, ctx->elem_offset, ctx->counters, s));
    FusedParams fo = fp;
    fo.mode = FUSED_ORDERED;
    fo.elem_offset = ctx->elem_offset;
    NKB_TRY(launch_fused(fo, s));
  } else {
    NKB_TRY(launch_fused(fp, s));
  }
  if (timing) NKB_CUDA(cudaEventRecord(ctx->ev[1], s));
  }
  const bool p2p = composite && ctx->p2p.ready;
  unsigned long long* zbuf = ctx->zbuf;
  P2PParams pp;
  if (p2p) {
    auto& P = ctx->p2p;
    memset(&pp, 0, sizeof(pp));
    pp.rank = ctx->rank;
    pp.nranks = ctx->nranks;
    pp.flags = P.flags;
    for (int q = 0; q < ctx->nranks; ++q) {
      pp.peer_flags[q] = P.peer_flags[q];
      pp.peer_keys[q] = P.peer_keys[ep & 1][q];
    }
    pp.npx = npx;
    pp.width = p->width;
    pp.height = p->height;
    pp.vmin = p->vmin;
    pp.vmax = p->vmax;
    pp.cmap = cm;
    memcpy(pp.bg, p->background, 4);
    pp.root_rgba = P.root_rgba;
    pp.root_depth = P.root_depth;
    pp.range_out = ctx->range_dev;
    pp.err = P.err;
    pp.dev_epoch = P.dev_epoch;
    pp.overflow = ctx->counters + 6;
    zbuf = P.keys[ep & 1];
    {
      const char* v = getenv("NKB_COMPOSITE_BULK");         // 0: the per-thread load kernel
      pp.bulk = !(v && v[0] == '0');
    }
    if (split) {
      if (part == 1) pp.ep_slot = P.dev_epoch + 1 + par;
      else pp.dev_epoch = P.dev_epoch + 1 + par;
      if (fp.sm_reserve > 0) pp.max_blocks = 2 * fp.sm_reserve;   // two bulk CTAs (96 KB smem each) per SM
      pp.bulk = 1;
    }
    if (part & 1) {
      NKB_TRY(launch_p2p_epoch(pp, s));              // device epoch := ep
      // every peer has finished reading this key buffer (epoch ep-2) before it is cleared
      NKB_TRY(launch_p2p_wait(pp, 1, 2, s));
    }
  }
  if (part & 1) {
  // (a one-GPU step's key buffer was cleared by the previous step's resolve)
  if (composite || ctx->step_clear) NKB_TRY(launch_zbuf_clear(zbuf, npx, s));
  RasterParams rp;
  rp.tri = ctx->tri;
  if (ordered) {          // one contiguous region; its count is the scan total
    rp.region_count = ctx->counters;
    rp.n_regions = 1;
    rp.region_cap = ctx->tri_cap;
  } else {
    rp.region_count = ctx->region_count;
    rp.n_regions = ctx->n_regions;
    rp.region_cap = ctx->region_cap;
  }
  memcpy(rp.view, p->view, 12 * sizeof(double));
  memcpy(rp.view + 12, p->persp, 4 * sizeof(double));
  rp.width = p->width;
  rp.height = p->height;
  rp.zbuf = zbuf;
  rp.lanes_per_tri = raster_lanes(ctx, p);
  NKB_TRY(launch_raster(rp, s));
  if (composite)                                   // (one GPU: in the resolve tail)
    NKB_TRY(launch_range_words(ctx->counters, zbuf + npx, rp.region_count == ctx->counters ? nullptr : rp.region_count,
                               rp.n_regions, rp.region_cap, ctx->tri_cap, s,
                               split ? ctx->csnap + 8 * par : nullptr));
  if (timing) NKB_CUDA(cudaEventRecord(ctx->ev[2], s));
  if (p2p) NKB_TRY(launch_p2p_signal(pp, 0, nullptr, s));   // "keys ready" (+ this rank's overflow word)
  if (timing) NKB_CUDA(cudaEventRecord(ctx->ev[6], s));
  }
  if (p2p && (part & 2)) {
    // fused sort-last composite + resolve over NVLink peer memory
    NKB_TRY(launch_p2p_composite(pp, s));
    if (timing) NKB_CUDA(cudaEventRecord(ctx->ev[7], s));
    NKB_TRY(launch_p2p_signal(pp, 1, split ? ctx->csnap + 8 * par : ctx->counters, s));
    if (timing) NKB_CUDA(cudaEventRecord(ctx->ev[8], s));
    if (ctx->rank == 0) NKB_TRY(launch_p2p_wait(pp, 1, 0, s));
  } else if (composite && !p2p) {
    NKB_NCCL(g_nccl.GroupStart());
    NKB_NCCL(g_nccl.Reduce(ctx->zbuf, ctx->zbuf, (size_t)npx + 2, ncclUint64, ncclMin, 0, ctx->comm, s));
    NKB_NCCL(g_nccl.AllReduce(ctx->counters, ctx->counters + 3, 1, ncclUint64, ncclSum, ctx->comm, s));
    // any rank overflowed -> every rank re-runs (counters[7])
    NKB_NCCL(g_nccl.AllReduce(ctx->counters + 6, ctx->counters + 7, 1, ncclUint64, ncclMax, ctx->comm, s));
    NKB_NCCL(g_nccl.GroupEnd());
  }
  if (timing) NKB_CUDA(cudaEventRecord(ctx->ev[3], s));
  ReportParams rep;
  rep.counters = ctx->counters;
  rep.range = ctx->range_dev;
  rep.region_count = ordered ? nullptr : ctx->region_count;
  rep.n_regions = ordered ? 0 : ctx->n_regions;
  rep.h_counters = ctx->h_counters_dev;
  rep.err = p2p ? ctx->p2p.err : nullptr;
  rep.peer_counts = p2p ? ctx->p2p.flags + 2 * kMaxRanks : nullptr;
  rep.peer_overflow = p2p ? ctx->p2p.flags + 3 * kMaxRanks : nullptr;
  rep.nranks = ctx->nranks;
  rep.h_res = p2p ? ctx->p2p.h_res_dev : nullptr;
  rep.part = part;
  if (!composite) {
    // one GPU: resolve, clear the other key buffer for the next step, and
    // (last CTA) range words + overflow word + report -- one launch
    ResolveParams rs;
    rs.zbuf = zbuf;
    rs.width = p->width;
    rs.height = p->height;
    rs.lo = rs.hi = 0.0;
    rs.range_words = nullptr;
    rs.vmin = p->vmin;
    rs.vmax = p->vmax;
    rs.cmap = cm;
    memcpy(rs.bg, p->background, 4);
    rs.rgba = ctx->rgba;
    rs.depth = ctx->depth;
    rs.range_out = ctx->range_dev;
    rs.counters = ctx->counters;
    rs.clear_next = zbuf == ctx->zbufs[0] ? ctx->zbufs[1] : ctx->zbufs[0];
    rs.words = zbuf + npx;
    rs.region_count = ordered ? nullptr : ctx->region_count;
    rs.n_regions = ctx->n_regions;
    rs.region_cap = ctx->region_cap;
    rs.tri_cap = ctx->tri_cap;
    rs.ticket = ctx->rticket;
    NKB_TRY(launch_resolve_tail(rs, rep, s));
    if (timing) NKB_CUDA(cudaEventRecord(ctx->ev[4], s));
    return NKB_OK;
  }
  if (!p2p && ctx->rank == 0) {
    ResolveParams rs;
    rs.zbuf = ctx->zbuf;
    rs.width = p->width;
    rs.height = p->height;
    rs.lo = rs.hi = 0.0;
    rs.range_words = ctx->zbuf + npx;
    rs.vmin = p->vmin;
    rs.vmax = p->vmax;
    rs.cmap = cm;
    memcpy(rs.bg, p->background, 4);
    rs.rgba = ctx->rgba;
    rs.depth = ctx->depth;
    rs.range_out = ctx->range_dev;
    NKB_TRY(launch_resolve(rs, s));
  }
  if (timing) NKB_CUDA(cudaEventRecord(ctx->ev[4], s));
  NKB_TRY(launch_report(rep, s));
  return NKB_OK;
}

// the launch parameters a captured step depends on (graph cache key)
static std::string step_key(nkb_ctx* ctx, const nkb_pipeline* p, const FusedParams& fp, const Colormap& cm,
                            bool ordered) {
  std::string k;
  auto add = [&](const void* d, size_t n) { k.append(reinterpret_cast<const char*>(d), n); };
  add(p, sizeof(*p));
  add(&fp, sizeof(fp));
  add(&cm, sizeof(cm));
  const void* ptrs[] = {ctx->tri, ctx->meta, ctx->zbuf, ctx->rgba, ctx->depth, ctx->counters, ctx->region_count,
                        ctx->elem_count, ctx->elem_offset, ctx->range_dev, ctx->h_counters};
  add(ptrs, sizeof(ptrs));
  const int64_t v[] = {ctx->tri_cap, ctx->E, ordered ? 1 : 0, surface_pass_of(fp), fused_node_prog(fp),
                       raster_lanes(ctx, p)};
  add(v, sizeof(v));
  return k;
}

// after the step's report words have landed (stream synchronised): the P2P
// timeout flag and the global triangle count
static int collect_step(nkb_ctx* ctx, bool p2p) {
  if (p2p) {
    if (*reinterpret_cast<const int*>(ctx->p2p.h_res)) {
      cudaMemset(ctx->p2p.err, 0, sizeof(int));   // report once; a later step starts clean
      return fail(NKB_ENCCL, "P2P composite: timed out waiting for a peer rank");
    }
    unsigned long long tot = 0;
    for (int q = 0; q < ctx->nranks; ++q) tot += ctx->p2p.h_res[1 + q];
    ctx->h_counters[3] = tot;   // meaningful on rank 0 (every rank reports to every rank)
  }
  return NKB_OK;
}

// the step's second half on the composite stream (P2P, NKB_COMPOSITE_OVERLAP != 0)
static bool composite_overlap() {
  static const bool on = !(getenv("NKB_COMPOSITE_OVERLAP") && strcmp(getenv("NKB_COMPOSITE_OVERLAP"), "0") == 0);
  return on;
}

// SMs the surface pass of a split step leaves to the previous step's
// composite (persistent K1g / K1s grids would otherwise hold every SM)
static bool composite_overlap_forced() {            // NKB_COMPOSITE_OVERLAP=2: also beside 3-CTA K1g
  static const bool on = getenv("NKB_COMPOSITE_OVERLAP") && strcmp(getenv("NKB_COMPOSITE_OVERLAP"), "2") == 0;
  return on;
}

static int composite_sms() {
  static const int n = [] {
    const char* v = getenv("NKB_COMPOSITE_SMS");
    return v ? atoi(v) : 4;
  }();
  return n;
}

static int ensure_comp_stream(nkb_ctx* ctx) {
  if (ctx->comp_stream) return NKB_OK;
  NKB_CUDA(cudaStreamCreateWithFlags(&ctx->comp_stream, cudaStreamNonBlocking));
  for (int k = 0; k < 2; ++k) {
    NKB_CUDA(cudaEventCreateWithFlags(&ctx->ev_a[k], cudaEventDisableTiming));
    NKB_CUDA(cudaEventCreateWithFlags(&ctx->ev_b[k], cudaEventDisableTiming));
  }
  if (!ctx->csnap) NKB_CUDA(cudaMalloc(&ctx->csnap, 16 * sizeof(unsigned long long)));
  return NKB_OK;
}

// order `s` after the last composite half (image, range and report words)
static int join_composite(nkb_ctx* ctx, cudaStream_t s) {
  if (ctx->last_b >= 0) NKB_CUDA(cudaStreamWaitEvent(s, ctx->ev_b[ctx->last_b], 0));
  return NKB_OK;
}

// NKB_SPLIT_TRACE=1: per-step event times of the two halves of split steps
// (A start / end on the caller's stream, B start / end on the composite
// stream), printed to stderr at the next synchronisation
struct SplitTrace {
  std::vector<cudaEvent_t> ev;   // 4 per step
  int n = 0;
};
static SplitTrace g_trace;
static bool split_trace() {
  static const bool on = getenv("NKB_SPLIT_TRACE") != nullptr;
  return on;
}
static void trace_mark(int k, cudaStream_t s) {
  const size_t i = (size_t)g_trace.n * 4 + k;
  while (g_trace.ev.size() <= i) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    g_trace.ev.push_back(e);
  }
  cudaEventRecord(g_trace.ev[i], s);
}
static void trace_flush(int rank) {
  if (g_trace.n == 0) return;
  float t[4];
  for (int j = 0; j < g_trace.n; ++j) {
    for (int k = 0; k < 4; ++k) cudaEventElapsedTime(&t[k], g_trace.ev[0], g_trace.ev[4 * j + k]);
    fprintf(stderr, "[nkb split rank %d] step %d A %.4f-%.4f B %.4f-%.4f (A %.4f, B %.4f ms)\n", rank, j, t[0], t[1],
            t[2], t[3], t[1] - t[0], t[3] - t[2]);
  }
  g_trace.n = 0;
}

static int sync_step(nkb_ctx* ctx, cudaStream_t s) {
  NKB_CUDA(cudaStreamSynchronize(s));
  if (ctx->last_b >= 0) NKB_CUDA(cudaStreamSynchronize(ctx->comp_stream));
  if (split_trace()) trace_flush(ctx->rank);
  return NKB_OK;
}

// the sticky overflow words the report kernel ORs into (no device work pending)
static void clear_overflow_words(nkb_ctx* ctx) {
  ctx->h_counters[6] = ctx->h_counters[7] = 0;
  if (ctx->p2p.h_res) ctx->p2p.h_res[1 + kMaxRanks] = 0;
}

static int run_step(nkb_ctx* ctx, const nkb_pipeline* p, FusedParams fp, const Colormap& cm,
                    cudaStream_t s, bool composite, bool ordered, bool sync = true) {
  const bool p2p = composite && ctx->p2p.ready;
  if (sync) clear_overflow_words(ctx);
  const unsigned long long ep = p2p ? ++ctx->p2p.epoch : 0;   // the device counter follows in-stream
  int slot = (int)(ep & 1);
  if (!composite) {
    // one GPU: alternate the two key buffers (graph slot = buffer); the
    // step's resolve clears the other one for the next step
    slot = ctx->zpar_next;
    ctx->zbuf = ctx->zbufs[slot];
    ctx->step_clear = !ctx->znext_clean;
    ctx->zpar_next = slot ^ 1;
    ctx->znext_clean = true;
  } else {
    ctx->step_clear = true;
    // the NCCL composite reduces into ctx->zbuf: the next one-GPU step must clear it first
    if (!p2p && ctx->zbuf == ctx->zbufs[ctx->zpar_next]) ctx->znext_clean = false;
  }
  // P2P: the composite half of step k runs on ctx->comp_stream while step
  // k+1's surface pass runs on `s`.  Step k+2 (same parity slots) waits for
  // step k's composite half; the cross-GPU order stays with the epoch flags.
  // (stream-ordered steps only: a synchronous step waits for its composite
  // anyway; and not beside three-CTA K1g grids, whose SMs have no room left
  // for the composite's CTAs -- measured unstable / slower)
  const bool split = !sync && p2p && composite_overlap() && fp.prof == nullptr && !p->timing &&
                     (composite_overlap_forced() || fused_ctas_per_sm(fp) <= 2);
  if (split) {
    fp.sm_reserve = composite_sms();
    NKB_TRY(ensure_comp_stream(ctx));
    if (ctx->ev_b_live[slot]) NKB_CUDA(cudaStreamWaitEvent(s, ctx->ev_b[slot], 0));
  } else {
    NKB_TRY(join_composite(ctx, s));               // a one-stream step after split ones
  }
  // Steps replay a CUDA graph of the whole launch sequence (one launch
  // instead of ~10-14), re-captured whenever a parameter changes.  With the
  // P2P composite the epoch lives on the device and only the key-buffer
  // parity alternates, so two graphs (two pairs when split) cover every
  // step; the NCCL composite path stays eager.
  static const bool graphs = !(getenv("NKB_GRAPHS") && strcmp(getenv("NKB_GRAPHS"), "0") == 0);
  // (per-stage timing keeps the eager path: its events bracket the stages)
  const int parts[2] = {split ? 1 : 3, 2};
  for (int h = 0; h < (split ? 2 : 1); ++h) {
    const int part = parts[h];
    cudaStream_t hs = h == 0 ? s : ctx->comp_stream;
    if (h == 1) {
      if (split_trace()) trace_mark(1, s);
      NKB_CUDA(cudaEventRecord(ctx->ev_a[slot], s));
      NKB_CUDA(cudaStreamWaitEvent(hs, ctx->ev_a[slot], 0));
      if (split_trace()) trace_mark(2, hs);
    } else if (split && split_trace()) {
      trace_mark(0, s);
    }
    if (graphs && (!composite || p2p) && fp.prof == nullptr && !p->timing) {
      if (ordered && ctx->elem_cap < ctx->E) {       // (allocation happens outside the capture)
        cudaFree(ctx->elem_count);
        cudaFree(ctx->elem_offset);
        ctx->elem_count = nullptr;
        ctx->elem_offset = nullptr;
        NKB_CUDA(cudaMalloc(&ctx->elem_count, sizeof(int) * ctx->E));
        NKB_CUDA(cudaMalloc(&ctx->elem_offset, sizeof(long long) * ctx->E));
        ctx->elem_cap = ctx->E;
      }
      NKB_TRY(launch_fused_prepare());
      std::string key = step_key(ctx, p, fp, cm, ordered);
      if (p2p) {
        const void* pk[] = {ctx->p2p.keys[0], ctx->p2p.keys[1], ctx->p2p.flags, ctx->p2p.dev_epoch, ctx->p2p.h_res,
                            ctx->csnap};
        key.append(reinterpret_cast<const char*>(pk), sizeof(pk));
        key.push_back((char)slot);
        key.push_back((char)part);
      }
      key.push_back(ctx->step_clear ? 'c' : 'n');
      // whole steps, first halves and second halves keep separate graphs
      // (synchronous and stream-ordered steps alternate without re-capture)
      cudaGraphExec_t& gx = part == 3 ? ctx->graph_exec[slot] : part == 1 ? ctx->graph_exec_a[slot]
                                                                          : ctx->graph_exec_b[slot];
      std::string& gk = part == 3 ? ctx->graph_key[slot] : part == 1 ? ctx->graph_key_a[slot] : ctx->graph_key_b[slot];
      if (!gx || key != gk) {
        if (gx) cudaGraphExecDestroy(gx);
        gx = nullptr;
        if (!ctx->cap_stream) NKB_CUDA(cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking));
        NKB_CUDA(cudaStreamBeginCapture(ctx->cap_stream, cudaStreamCaptureModeRelaxed));
        const int rc = enqueue_step(ctx, p, fp, cm, ctx->cap_stream, composite, ordered, ep, part);
        cudaGraph_t g = nullptr;
        const cudaError_t ce = cudaStreamEndCapture(ctx->cap_stream, &g);
        NKB_TRY(rc);
        NKB_CUDA(ce);
        const cudaError_t ie = cudaGraphInstantiate(&gx, g, 0);
        cudaGraphDestroy(g);
        NKB_CUDA(ie);
        gk = key;
      }
      NKB_CUDA(cudaGraphLaunch(gx, hs));
    } else {
      NKB_TRY(enqueue_step(ctx, p, fp, cm, hs, composite, ordered, ep, part));
    }
  }
  if (split) {
    if (split_trace()) {
      trace_mark(3, ctx->comp_stream);
      ++g_trace.n;
    }
    NKB_CUDA(cudaEventRecord(ctx->ev_b[slot], ctx->comp_stream));
    ctx->ev_b_live[slot] = true;
    ctx->last_b = slot;
  } else {
    ctx->last_b = -1;
  }
  ctx->last_fast = !ordered;
  if (!sync) return NKB_OK;                        // stream-ordered (nkb_execute_async): collected at the wait
  NKB_TRY(sync_step(ctx, s));
  return collect_step(ctx, p2p);
}

// capacity the step needed (per-region maximum in FAST mode; the region
// counts are read from the device only here, after an overflow -- the step
// report carries the 8 counter words alone)
static int64_t needed_capacity(nkb_ctx* ctx, bool ordered) {
  const int64_t total = (int64_t)ctx->h_counters[0];
  if (ordered) return total;
  std::vector<unsigned long long> rc(ctx->n_regions > 0 ? ctx->n_regions : 1, 0ULL);
  if (ctx->n_regions > 0 &&
      cudaMemcpy(rc.data(), ctx->region_count, sizeof(unsigned long long) * ctx->n_regions,
                 cudaMemcpyDeviceToHost) != cudaSuccess)
    return 2 * ctx->tri_cap;                           // (unreachable in practice) grow generously
  int64_t mx = 0;
  for (int r = 0; r < ctx->n_regions; ++r) mx = std::max<int64_t>(mx, (int64_t)rc[r]);
  return mx * ctx->n_regions;
}

// Continuous derived fields: compute Q / |w| for every node in one gradient
// pass, DSSUM-average them, and let the main pass read them as scalar
// fields (no gradients there).
static int continuous_prepass(nkb_ctx* ctx, const nkb_pipeline* p, FusedParams& fp, cudaStream_t s) {
  bool uq = fp.color_src == SRC_Q, uw = fp.color_src == SRC_WMAG;
  for (int k = 0; k < fp.n_surf; ++k) {
    uq |= fp.surf_src[k] == SRC_Q;
    uw |= fp.surf_src[k] == SRC_WMAG;
  }
  if (!uq && !uw) return NKB_OK;
  if (!ctx->gs_ready) return fail(NKB_ESTATE, "continuous derived fields need nkb_mesh_set_global_ids");
  const int64_t npts = ctx->E * kNN;
  if (ctx->dcap < npts) {
    cudaFree(ctx->dq);
    cudaFree(ctx->dw);
    ctx->dq = ctx->dw = nullptr;
    ctx->dcap = 0;
    NKB_CUDA(cudaMalloc(&ctx->dq, sizeof(double) * std::max<int64_t>(npts, 1)));
    NKB_CUDA(cudaMalloc(&ctx->dw, sizeof(double) * std::max<int64_t>(npts, 1)));
    ctx->dcap = npts;
  }
  if (npts > 0) {
    FusedParams fq;
    NKB_TRY(fused_params_base(ctx, fq));
    fq.need_grad = 1;
    fq.need_vel = 1;
    for (int c = 0; c < 3; ++c) fq.vel[c] = fp.vel[c];
    fq.need_wmag = uw ? 1 : 0;
    fq.color_src = -1;
    fq.n_surf = 0;
    fq.q_out = uq ? ctx->dq : nullptr;
    fq.wmag_out = uw ? ctx->dw : nullptr;
    NKB_CUDA(cudaMemsetAsync(ctx->counters, 0, 64, s));
    NKB_TRY(geo_attach(ctx, fq, s));
    NKB_TRY(launch_fused(fq, s));
  }
  if (uq) NKB_TRY(gs_apply(ctx, ctx->dq, s));
  if (uw) NKB_TRY(gs_apply(ctx, ctx->dw, s));
  // the main pass reads the averaged fields as scalars
  auto slot = [&](const double* base, int* src) -> int {
    for (int k = 0; k < fp.n_scalars; ++k)
      if (fp.scalar[k] == base) {
        *src = SRC_SCALAR0 + k;
        return NKB_OK;
      }
    if (fp.n_scalars >= kMaxScalars) return fail(NKB_EINVAL, "too many scalar fields for a continuous pipeline");
    fp.scalar[fp.n_scalars] = base;
    *src = SRC_SCALAR0 + fp.n_scalars++;
    return NKB_OK;
  };
  int sq = -1, sw = -1;
  if (uq) NKB_TRY(slot(ctx->dq, &sq));
  if (uw) NKB_TRY(slot(ctx->dw, &sw));
  for (int k = 0; k < fp.n_surf; ++k) {
    if (fp.surf_src[k] == SRC_Q) fp.surf_src[k] = sq;
    else if (fp.surf_src[k] == SRC_WMAG) fp.surf_src[k] = sw;
  }
  if (fp.color_src == SRC_Q) fp.color_src = sq;
  else if (fp.color_src == SRC_WMAG) fp.color_src = sw;
  fp.need_grad = 0;
  fp.need_wmag = 0;
  if (!fp.need_umag) fp.need_vel = 0;
  return NKB_OK;
}

// one step's parameters, validated and resolved (shared by the synchronous
// and the stream-ordered Execute)
struct StepPlan {
  FusedParams fp;
  Colormap cm;
  bool composite = false, ordered = false;
};

static int prepare_step(nkb_ctx* ctx, const nkb_pipeline* p, cudaStream_t s, StepPlan& plan) {
  NKB_TRY(ctx_check(ctx));
  if (!p) return fail(NKB_EINVAL, "null pipeline");
  if (!ctx->x) return fail(NKB_ESTATE, "Execute before mesh_set");
  if (p->width < 1 || p->height < 1 || p->width > 16384 || p->height > 16384)
    return fail(NKB_EINVAL, "image size must be in [1, 16384]");
  if (p->n_surfaces < 0 || p->n_surfaces > NKB_MAX_SURFACES)
    return fail(NKB_EINVAL, "n_surfaces must be in [0, 4]");
  for (int i = 0; i < 12; ++i)
    if (!isfinite(p->view[i])) return fail(NKB_EINVAL, "view matrix must be finite");
  for (int i = 0; i < 4; ++i)
    if (!isfinite(p->persp[i])) return fail(NKB_EINVAL, "perspective row must be finite");
  FusedParams& fp = plan.fp;
  NKB_TRY(fused_params_base(ctx, fp));
  fp.n_surf = p->n_surfaces;
  for (int k = 0; k < p->n_surfaces; ++k) {
    const nkb_surface& sf = p->surfaces[k];
    char fname[NKB_NAME_MAX + 1];
    memcpy(fname, sf.field, NKB_NAME_MAX);
    fname[NKB_NAME_MAX] = 0;
    if (sf.kind == NKB_SURF_ISO) {
      NKB_TRY(resolve_src(ctx, fname, fp, &fp.surf_src[k]));
      if (!isfinite(sf.value)) return fail(NKB_EINVAL, "iso value must be finite");
      fp.surf_iso[k] = sf.value;
    } else if (sf.kind == NKB_SURF_SLICE) {
      if (!(isfinite(sf.normal[0]) && isfinite(sf.normal[1]) && isfinite(sf.normal[2]) &&
            isfinite(sf.value)))
        return fail(NKB_EINVAL, "slice plane must be finite");
      if (sf.normal[0] == 0.0 && sf.normal[1] == 0.0 && sf.normal[2] == 0.0)
        return fail(NKB_EINVAL, "slice normal must be non-zero");
      fp.surf_src[k] = SRC_PLANE + k;
      fp.surf_iso[k] = sf.value;
      for (int a = 0; a < 3; ++a) fp.surf_n[k][a] = sf.normal[a];
    } else {
      return fail(NKB_EINVAL, "unknown surface kind " + std::to_string(sf.kind));
    }
  }
  {
    char cname[NKB_NAME_MAX + 1];
    memcpy(cname, p->color_field, NKB_NAME_MAX);
    cname[NKB_NAME_MAX] = 0;
    NKB_TRY(resolve_src(ctx, cname, fp, &fp.color_src));
  }
  Colormap& cm = plan.cm;
  NKB_TRY(build_colormap(p, cm));

  const bool composite = plan.composite = p->composite && ctx->comm && ctx->nranks > 1;
  if (p->composite && ctx->nranks > 1 && !ctx->comm) return fail(NKB_ENCCL, "composite without comm");

  NKB_TRY(ensure_image(ctx, p->width, p->height));
  if (ctx->tri_cap == 0) {
    // initial capacity; NKB_TRI_CAP0 overrides it (tests force an overflow on one rank)
    const char* c0 = getenv("NKB_TRI_CAP0");
    const int64_t cap0 = c0 ? std::max<int64_t>(1, atoll(c0)) : std::max<int64_t>(1 << 16, ctx->E * 16);
    NKB_TRY(ensure_tri(ctx, cap0, p->emit_meta));
  }
  else NKB_TRY(ensure_tri(ctx, ctx->tri_cap, p->emit_meta));

  const bool ordered = plan.ordered = p->emit_meta && ctx->E > 0 && p->n_surfaces > 0;
  if (composite && !ctx->p2p.unavailable) {
    const char* mode = getenv("NKB_COMPOSITE");
    if (!(mode && strcmp(mode, "nccl") == 0)) NKB_TRY(p2p_setup(ctx, p->width, p->height, s));
  }
  ctx->geo_used = ctx->geo_built = false;
  if (p->timing) NKB_CUDA(cudaEventRecord(ctx->ev[5], s));
  if (p->continuous) NKB_TRY(continuous_prepass(ctx, p, fp, s));
  NKB_TRY(geo_attach(ctx, fp, s));
  return NKB_OK;
}

int nkb_execute(nkb_ctx* ctx, const nkb_pipeline* p, nkb_report* out, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (ctx && ctx->async_pending) return fail(NKB_ESTATE, "an nkb_execute_async step is pending: nkb_execute_wait first");
  StepPlan plan;
  NKB_TRY(prepare_step(ctx, p, s, plan));
  FusedParams& fp = plan.fp;
  const Colormap& cm = plan.cm;
  const bool composite = plan.composite, ordered = plan.ordered;
  const bool prof = getenv("NKB_PROFILE_PHASES") != nullptr && !ordered;
  if (prof) {
    if (!ctx->prof) NKB_CUDA(cudaMalloc(&ctx->prof, 18 * sizeof(unsigned long long)));
    NKB_CUDA(cudaMemsetAsync(ctx->prof, 0, 18 * sizeof(unsigned long long), s));
    fp.prof = ctx->prof;
  }
  NKB_TRY(run_step(ctx, p, fp, cm, s, composite, ordered));
  if (prof) {
    unsigned long long h[18];
    NKB_CUDA(cudaMemcpy(h, ctx->prof, sizeof(h), cudaMemcpyDeviceToHost));
    static const char* ph[6] = {"top-barrier", "role-work", "pre-node-wait", "node", "post-node-wait", "classify"};
    static const char* role[3] = {"pencil(w0)", "stage(w8)", "mc(w12)"};
    for (int r = 0; r < 3; ++r) {
      fprintf(stderr, "[nkb phases] %-11s", role[r]);
      for (int k = 0; k < 6; ++k)
        fprintf(stderr, " %s=%.0f", ph[k], ctx->E ? (double)h[6 * r + k] / (double)ctx->E : 0.0);
      fprintf(stderr, " (cycles/element)\n");
    }
    fp.prof = nullptr;
  }
  // Overflow: the step's triangles did not fit (counted, not written).  The
  // decision is collective -- every rank sees whether ANY rank overflowed
  // (P2P flags / NCCL max) -- so all ranks grow (those that overflowed) and
  // re-run together, and the composite is redone from complete triangle sets.
  int reran = 0;
  int64_t ntri = (int64_t)ctx->h_counters[0];
  for (int attempt = 0; attempt < 2; ++attempt) {
    const bool own_over = ctx->h_counters[6] != 0;
    bool any_over = own_over;
    if (composite) any_over = ctx->p2p.ready ? ctx->p2p.h_res[1 + kMaxRanks] != 0 : ctx->h_counters[7] != 0;
    if (!any_over) break;
    if (own_over) {
      const int64_t need = needed_capacity(ctx, ordered);
      NKB_TRY(ensure_tri(ctx, std::max(need + need / 4 + 1024 * ctx->n_regions, ctx->tri_cap + ctx->tri_cap / 4),
                         p->emit_meta));
    }
    NKB_TRY(run_step(ctx, p, fp, cm, s, composite, ordered));
    ntri = (int64_t)ctx->h_counters[0];
    reran = 1;
  }
  ctx->last_ntri = ntri;
  if (getenv("NKB_CHECKED_SELFTEST")) {
    NKB_TRY(checked_selftest(s));
    NKB_CUDA(cudaStreamSynchronize(s));
  }
  NKB_TRY(checked_violations());
  ctx->image_valid = (!composite || ctx->rank == 0);
  if (out) {
    memset(out, 0, sizeof(*out));
    out->n_triangles = ntri;
    out->n_triangles_global = composite ? (int64_t)ctx->h_counters[3] : ntri;
    out->tri_capacity = ctx->tri_cap;
    double r[2];
    memcpy(r, ctx->h_counters + 4, sizeof(r));
    out->range[0] = r[0];
    out->range[1] = r[1];
    out->data_range[0] = ctx->h_counters[1] == ~0ULL ? NAN : dec_ordered_h(ctx->h_counters[1]);
    out->data_range[1] = ctx->h_counters[2] == 0ULL ? NAN : dec_ordered_h(ctx->h_counters[2]);
    out->reran = reran;
    out->geometry_cached = ctx->geo_used ? 1 : 0;
    out->surface_pass = surface_pass_of(fp);
    if (p->timing) {
      if (ctx->geo_built) cudaEventElapsedTime(&out->ms_geometry, ctx->ev[5], ctx->ev[0]);
      cudaEventElapsedTime(&out->ms_fused, ctx->ev[0], ctx->ev[1]);
      cudaEventElapsedTime(&out->ms_raster, ctx->ev[1], ctx->ev[2]);
      cudaEventElapsedTime(&out->ms_composite, ctx->ev[2], ctx->ev[3]);
      if (ctx->p2p.ready && p->composite && ctx->nranks > 1 && getenv("NKB_TIMING_DETAIL")) {
        float a = 0, b = 0, c = 0, d = 0;              // signal(ready) | composite (incl. peer wait) | signal(done) | done wait
        cudaEventElapsedTime(&a, ctx->ev[2], ctx->ev[6]);
        cudaEventElapsedTime(&b, ctx->ev[6], ctx->ev[7]);
        cudaEventElapsedTime(&c, ctx->ev[7], ctx->ev[8]);
        cudaEventElapsedTime(&d, ctx->ev[8], ctx->ev[3]);
        fprintf(stderr, "[nkb composite rank %d] signal %.4f composite %.4f signal %.4f wait %.4f ms\n", ctx->rank, a,
                b, c, d);
      }
      cudaEventElapsedTime(&out->ms_resolve, ctx->ev[3], ctx->ev[4]);
    }
  }
  return NKB_OK;
}

int nkb_execute_async(nkb_ctx* ctx, const nkb_pipeline* p, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (!p) return fail(NKB_EINVAL, "null pipeline");
  if (p->timing) return fail(NKB_EINVAL, "nkb_execute_async: pipeline.timing must be 0 (use nkb_execute)");
  // No host synchronisation with a step still pending: its report is
  // superseded, while its overflow and P2P timeout words stay sticky until
  // nkb_execute_wait reports them.  The first step of a sequence starts
  // from clear overflow words (nothing is in flight then).
  if (ctx && !ctx->async_pending && ctx->h_counters) clear_overflow_words(ctx);
  StepPlan plan;
  NKB_TRY(prepare_step(ctx, p, s, plan));
  NKB_TRY(run_step(ctx, p, plan.fp, plan.cm, s, plan.composite, plan.ordered, false));
  ctx->async_pending = true;
  ctx->async_composite = plan.composite;
  ctx->async_ordered = plan.ordered;
  ctx->async_emit_meta = p->emit_meta != 0;
  ctx->async_surface_pass = surface_pass_of(plan.fp);
  ctx->image_valid = (!plan.composite || ctx->rank == 0);
  return NKB_OK;
}

int nkb_execute_wait(nkb_ctx* ctx, nkb_report* out, void* stream) {
  NKB_TRY(ctx_check(ctx));
  if (!ctx->async_pending) return fail(NKB_ESTATE, "nkb_execute_wait without a pending nkb_execute_async");
  cudaStream_t s = (cudaStream_t)stream;
  NKB_TRY(sync_step(ctx, s));
  ctx->async_pending = false;
  const bool composite = ctx->async_composite;
  NKB_TRY(collect_step(ctx, composite && ctx->p2p.ready));
  const bool own_over = ctx->h_counters[6] != 0;
  bool any_over = own_over;
  if (composite) any_over = ctx->p2p.ready ? ctx->p2p.h_res[1 + kMaxRanks] != 0 : ctx->h_counters[7] != 0;
  clear_overflow_words(ctx);
  if (own_over) {                                  // grow for the next steps (this one stays incomplete)
    const int64_t need = needed_capacity(ctx, ctx->async_ordered);
    NKB_TRY(ensure_tri(ctx, std::max(need + need / 4 + 1024 * ctx->n_regions, ctx->tri_cap + ctx->tri_cap / 4),
                       ctx->async_emit_meta));
  }
  const int64_t ntri = (int64_t)ctx->h_counters[0];
  ctx->last_ntri = ntri;
  NKB_TRY(checked_violations());
  if (out) {
    memset(out, 0, sizeof(*out));
    out->n_triangles = ntri;
    out->n_triangles_global = composite ? (int64_t)ctx->h_counters[3] : ntri;
    out->tri_capacity = ctx->tri_cap;
    double r[2];
    memcpy(r, ctx->h_counters + 4, sizeof(r));
    out->range[0] = r[0];
    out->range[1] = r[1];
    out->data_range[0] = ctx->h_counters[1] == ~0ULL ? NAN : dec_ordered_h(ctx->h_counters[1]);
    out->data_range[1] = ctx->h_counters[2] == 0ULL ? NAN : dec_ordered_h(ctx->h_counters[2]);
    out->geometry_cached = ctx->geo_used ? 1 : 0;
    out->surface_pass = ctx->async_surface_pass;
    out->overflowed = any_over ? 1 : 0;
    out->composite_overlapped = ctx->last_b >= 0 ? 1 : 0;
  }
  return NKB_OK;
}

int nkb_composite_partitions(nkb_ctx* root, nkb_ctx* const* parts, int n, const nkb_pipeline* p, void* stream) {
  NKB_TRY(ctx_check(root));
  if (!p || !parts) return fail(NKB_EINVAL, "null pipeline or partition list");
  if (n < 1 || n > kMaxRanks) return fail(NKB_EINVAL, "partition count must be in [1, 8]");
  const int W = p->width, H = p->height;
  for (int q = 0; q < n; ++q) {
    if (!parts[q] || parts[q]->device != root->device)
      return fail(NKB_EINVAL, "every partition context must live on the root's device");
    if (!parts[q]->zbuf || parts[q]->W != W || parts[q]->H != H)
      return fail(NKB_ESTATE, "partition " + std::to_string(q) + " has no key buffer of this image size "
                              "(execute it with the same pipeline and composite = 0 first)");
  }
  Colormap cm;
  NKB_TRY(build_colormap(p, cm));
  NKB_TRY(ensure_image(root, W, H));
  cudaStream_t s = (cudaStream_t)stream;
  for (int q = 0; q < n; ++q)            // the partitions' steps ran on their own streams
    if (parts[q] != root) NKB_CUDA(cudaDeviceSynchronize());
  // the flag protocol is satisfied up front: every "keys ready" word at epoch 1
  unsigned long long* flags = nullptr;
  int* err = nullptr;
  NKB_CUDA(cudaMalloc(&flags, (4 * kMaxRanks + 1) * sizeof(unsigned long long)));
  NKB_CUDA(cudaMalloc(&err, sizeof(int)));
  std::vector<unsigned long long> h(4 * kMaxRanks + 1, 0ULL);
  for (int q = 0; q < n; ++q) h[q] = 1ULL;
  h[4 * kMaxRanks] = 1ULL;               // the device epoch
  NKB_CUDA(cudaMemcpyAsync(flags, h.data(), h.size() * sizeof(unsigned long long), cudaMemcpyHostToDevice, s));
  NKB_CUDA(cudaMemsetAsync(err, 0, sizeof(int), s));
  P2PParams pp;
  memset(&pp, 0, sizeof(pp));
  pp.nranks = n;
  pp.flags = flags;
  for (int q = 0; q < n; ++q) {
    pp.peer_flags[q] = flags;
    pp.peer_keys[q] = parts[q]->zbuf;
  }
  pp.npx = (long long)W * H;
  pp.width = W;
  pp.height = H;
  pp.vmin = p->vmin;
  pp.vmax = p->vmax;
  pp.cmap = cm;
  memcpy(pp.bg, p->background, 4);
  pp.root_rgba = root->rgba;
  pp.root_depth = root->depth;
  pp.range_out = root->range_dev;
  pp.err = err;
  {
    const char* v = getenv("NKB_COMPOSITE_BULK");           // 0: the per-thread load kernel
    pp.bulk = !(v && v[0] == '0');
  }
  pp.dev_epoch = flags + 4 * kMaxRanks;
  int rc = NKB_OK;
  for (int r = 0; r < n && rc == NKB_OK; ++r) {   // each "rank" resolves its band of rows
    pp.rank = r;
    rc = launch_p2p_composite(pp, s);
  }
  int h_err = 0;
  if (rc == NKB_OK) {
    cudaMemcpyAsync(&h_err, err, sizeof(int), cudaMemcpyDeviceToHost, s);
    if (cudaStreamSynchronize(s) != cudaSuccess) rc = fail(NKB_ECUDA, cudaGetErrorString(cudaGetLastError()));
  }
  cudaFree(flags);
  cudaFree(err);
  NKB_TRY(rc);
  if (h_err) return fail(NKB_ECUDA, "partition composite: flag wait failed");
  NKB_TRY(checked_violations());
  root->image_valid = true;
  return NKB_OK;
}

int nkb_image_device(nkb_ctx* ctx, const unsigned char** rgba, const float** depth,
                     const uint64_t** zbuf) {
  NKB_TRY(ctx_check(ctx));
  if (!ctx->image_valid) return fail(NKB_ESTATE, "no image (execute not run, or not the composite root)");
  if (rgba) *rgba = ctx->rgba;
  if (depth) *depth = ctx->depth;
  if (zbuf) *zbuf = reinterpret_cast<const uint64_t*>(ctx->zbuf);
  return NKB_OK;
}

int nkb_image_copy(nkb_ctx* ctx, unsigned char* rgba, float* depth, void* stream) {
  NKB_TRY(ctx_check(ctx));
  if (!ctx->image_valid) return fail(NKB_ESTATE, "no image (execute not run, or not the composite root)");
  cudaStream_t s = (cudaStream_t)stream;
  const size_t npx = (size_t)ctx->W * ctx->H;
  NKB_TRY(join_composite(ctx, s));
  if (rgba) NKB_CUDA(cudaMemcpyAsync(rgba, ctx->rgba, npx * 4, cudaMemcpyDeviceToHost, s));
  if (depth) NKB_CUDA(cudaMemcpyAsync(depth, ctx->depth, npx * sizeof(float), cudaMemcpyDeviceToHost, s));
  NKB_CUDA(cudaStreamSynchronize(s));
  return NKB_OK;
}

int nkb_image_ppm(nkb_ctx* ctx, const unsigned char** ppm, int64_t* nbytes, void* stream) {
  NKB_TRY(ctx_check(ctx));
  if (!ppm || !nbytes) return fail(NKB_EINVAL, "null out");
  if (!ctx->image_valid) return fail(NKB_ESTATE, "no image (execute not run, or not the composite root)");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t npx = (int64_t)ctx->W * ctx->H;
  char hdr[64];
  const int hn = snprintf(hdr, sizeof(hdr), "P6\n%d %d\n255\n", ctx->W, ctx->H);
  const int64_t total = hn + 3 * npx;
  if (ctx->ppm_cap < total) {
    cudaFree(ctx->rgb_dev);
    cudaFreeHost(ctx->h_ppm);
    ctx->rgb_dev = nullptr;
    ctx->h_ppm = nullptr;
    ctx->ppm_cap = 0;
    NKB_CUDA(cudaMalloc(&ctx->rgb_dev, (size_t)std::max<int64_t>(3 * npx, 16)));
    NKB_CUDA(cudaMallocHost(&ctx->h_ppm, (size_t)total));
    ctx->ppm_cap = total;
  }
  memcpy(ctx->h_ppm, hdr, hn);
  NKB_TRY(join_composite(ctx, s));
  NKB_TRY(launch_pack_rgb(ctx->rgba, ctx->rgb_dev, npx, s));
  NKB_CUDA(cudaMemcpyAsync(ctx->h_ppm + hn, ctx->rgb_dev, (size_t)(3 * npx), cudaMemcpyDeviceToHost, s));
  NKB_CUDA(cudaStreamSynchronize(s));
  *ppm = ctx->h_ppm;
  *nbytes = total;
  return NKB_OK;
}

int nkb_triangles_device(nkb_ctx* ctx, const float** tri, const uint64_t** meta, int64_t* n) {
  NKB_TRY(ctx_check(ctx));
  const int64_t cnt = std::min<int64_t>(ctx->last_ntri, ctx->tri_cap);
  if (!ctx->last_fast) {
    if (tri) *tri = reinterpret_cast<const float*>(ctx->tri);
    if (meta) *meta = reinterpret_cast<const uint64_t*>(ctx->meta);
    if (n) *n = cnt;
    return NKB_OK;
  }
  // FAST mode wrote per-CTA regions: compact them into one array
  if (ctx->export_cap < cnt) {
    cudaFree(ctx->tri_export);
    cudaFree(ctx->meta_export);
    ctx->tri_export = nullptr;
    ctx->meta_export = nullptr;
    NKB_CUDA(cudaMalloc(&ctx->tri_export, (size_t)std::max<int64_t>(cnt, 1) * 3 * sizeof(float4)));
    NKB_CUDA(cudaMalloc(&ctx->meta_export, (size_t)std::max<int64_t>(cnt, 1) * sizeof(unsigned long long)));
    ctx->export_cap = cnt;
  }
  NKB_TRY(launch_compact(ctx->tri, ctx->meta_alloc ? ctx->meta : nullptr, ctx->region_count, ctx->n_regions,
                         ctx->region_cap, ctx->tri_export, ctx->meta_alloc ? ctx->meta_export : nullptr, cnt,
                         nullptr));
  NKB_CUDA(cudaStreamSynchronize(nullptr));
  if (tri) *tri = reinterpret_cast<const float*>(ctx->tri_export);
  if (meta) *meta = ctx->meta_alloc ? reinterpret_cast<const uint64_t*>(ctx->meta_export) : nullptr;
  if (n) *n = cnt;
  return NKB_OK;
}

// ---- composite communicator ------------------------------------------------------

int nkb_nccl_unique_id(unsigned char id_out[128]) {
  if (!id_out) return fail(NKB_EINVAL, "null out");
  NKB_TRY(load_nccl());
  ncclUniqueId id;
  NKB_NCCL(g_nccl.GetUniqueId(&id));
  memcpy(id_out, id.internal, 128);
  return NKB_OK;
}

int nkb_comm_init(nkb_ctx* ctx, const unsigned char id[128], int nranks, int rank) {
  NKB_TRY(ctx_check(ctx));
  if (!id) return fail(NKB_EINVAL, "null id");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(NKB_EINVAL, "bad rank / nranks");
  NKB_TRY(load_nccl());
  if (ctx->comm) {
    g_nccl.CommDestroy(ctx->comm);
    ctx->comm = nullptr;
  }
  ncclUniqueId uid;
  memcpy(uid.internal, id, 128);
  NKB_NCCL(g_nccl.CommInitRank(&ctx->comm, nranks, uid, rank));
  ctx->rank = rank;
  ctx->nranks = nranks;
  return NKB_OK;
}

int nkb_comm_destroy(nkb_ctx* ctx) {
  NKB_TRY(ctx_check(ctx));
  cudaDeviceSynchronize();
  p2p_release(ctx);
  if (ctx->comm && g_nccl.ok) g_nccl.CommDestroy(ctx->comm);
  ctx->comm = nullptr;
  ctx->rank = 0;
  ctx->nranks = 1;
  return NKB_OK;
}

// ---- reference 2D renderer -------------------------------------------------------

int nkb_render_structured(nkb_ctx* ctx, int n_blocks, const double* const* values, const int64_t* ni,
                          int64_t rows, int comps, int mode, int width, int height, double vmin,
                          double vmax, unsigned char* rgb_out, double* range_out, void* stream) {
  NKB_TRY(ctx_check(ctx));
  if (n_blocks < 1 || !values || !ni) return fail(NKB_EINVAL, "no blocks to assemble");
  if (rows < 1 || comps < 1) return fail(NKB_EINVAL, "empty block");
  if (mode == 0 && comps != 1)
    return fail(NKB_EINVAL, "field has " + std::to_string(comps) +
                                " components; request a derived scalar such as 'field:mag'");
  if (mode != 0 && mode != 1) return fail(NKB_EINVAL, "unknown derived scalar mode");
  if (width < 1 || height < 1) return fail(NKB_EINVAL, "image size must be positive");
  if (!rgb_out) return fail(NKB_EINVAL, "null output");
  cudaStream_t s = (cudaStream_t)stream;
  NKB_TRY(join_composite(ctx, s));                // a composite half may still write the image / range
  if (ctx->s_cap < n_blocks) {
    cudaFree(ctx->s_ptrs);
    cudaFree(ctx->s_col0);
    ctx->s_ptrs = nullptr;
    ctx->s_col0 = nullptr;
    NKB_CUDA(cudaMalloc(&ctx->s_ptrs, sizeof(double*) * n_blocks));
    NKB_CUDA(cudaMalloc(&ctx->s_col0, sizeof(int64_t) * (n_blocks + 1)));
    ctx->s_cap = n_blocks;
  }
  if (!ctx->s_minmax) NKB_CUDA(cudaMalloc(&ctx->s_minmax, 4 * sizeof(unsigned long long)));
  std::vector<int64_t> col0(n_blocks + 1, 0);
  for (int b = 0; b < n_blocks; ++b) {
    if (ni[b] < 1 || !values[b]) return fail(NKB_EINVAL, "empty block " + std::to_string(b));
    col0[b + 1] = col0[b] + ni[b];
  }
  NKB_CUDA(cudaMemcpyAsync(ctx->s_ptrs, values, sizeof(double*) * n_blocks, cudaMemcpyHostToDevice, s));
  NKB_CUDA(cudaMemcpyAsync(ctx->s_col0, col0.data(), sizeof(int64_t) * (n_blocks + 1),
                           cudaMemcpyHostToDevice, s));
  unsigned long long init[2] = {~0ULL, 0ULL};
  NKB_CUDA(cudaMemcpyAsync(ctx->s_minmax, init, sizeof(init), cudaMemcpyHostToDevice, s));
  StructuredParams sp;
  sp.n_blocks = n_blocks;
  sp.values = ctx->s_ptrs;
  sp.col0 = ctx->s_col0;
  sp.ni_total = col0[n_blocks];
  sp.rows = rows;
  sp.comps = comps;
  sp.mode = mode;
  sp.width = width;
  sp.height = height;
  nkb_pipeline dummy;
  memset(&dummy, 0, sizeof(dummy));
  NKB_TRY(build_colormap(&dummy, sp.cmap));
  sp.minmax = ctx->s_minmax;
  sp.vmin = vmin;
  sp.vmax = vmax;
  sp.rgb = rgb_out;
  sp.range_out = ctx->range_dev;
  if (!(vmin == vmin) || !(vmax == vmax)) NKB_TRY(launch_structured_minmax(sp, s));
  NKB_TRY(launch_structured_render(sp, s));
  if (range_out)
    NKB_CUDA(cudaMemcpyAsync(range_out, ctx->range_dev, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
  NKB_CUDA(cudaStreamSynchronize(s));
  return NKB_OK;
}

// ---- memory helpers ------------------------------------------------------------------

int nkb_device_alloc(nkb_ctx* ctx, int64_t bytes, void** out) {
  NKB_TRY(ctx_check(ctx));
  if (!out || bytes < 0) return fail(NKB_EINVAL, "bad allocation request");
  *out = nullptr;
  NKB_CUDA(cudaMalloc(out, (size_t)std::max<int64_t>(bytes, 1)));
  return NKB_OK;
}
int nkb_device_free(nkb_ctx* ctx, void* p) {
  NKB_TRY(ctx_check(ctx));
  NKB_CUDA(cudaFree(p));
  return NKB_OK;
}
int nkb_host_alloc(int64_t bytes, void** out) {
  if (!out || bytes < 0) return fail(NKB_EINVAL, "bad allocation request");
  *out = nullptr;
  NKB_CUDA(cudaMallocHost(out, (size_t)std::max<int64_t>(bytes, 1)));
  return NKB_OK;
}
int nkb_host_free(void* p) {
  NKB_CUDA(cudaFreeHost(p));
  return NKB_OK;
}
int nkb_memcpy(void* dst, const void* src, int64_t bytes, int kind, void* stream) {
  if (bytes < 0 || kind < 1 || kind > 3) return fail(NKB_EINVAL, "bad memcpy request");
  if (bytes == 0) return NKB_OK;
  NKB_CUDA(cudaMemcpyAsync(dst, src, (size_t)bytes, (cudaMemcpyKind)kind, (cudaStream_t)stream));
  return NKB_OK;
}
int nkb_stream_sync(void* stream) {
  NKB_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  return NKB_OK;
}
int nkb_device_sync(void) {
  NKB_CUDA(cudaDeviceSynchronize());
  return NKB_OK;
}

}  // extern "C"
