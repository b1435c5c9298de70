// Library context shared by the ABI translation units (abi.cu: context,
// mesh, Execute; abi_collective.cu: DSSUM, in transit staging, statistics).
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <map>
#include <memory>
#include <string>
#include <vector>

#include "nkb_internal.h"

namespace nkb {

// ---- NCCL, resolved at runtime so the library loads without it -------------
struct NcclApi {
  bool ok = false;
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, int, ncclComm_t,
                         cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
extern NcclApi g_nccl;
int load_nccl();

#define NKB_NCCL(call)                                                                  \
  do {                                                                                  \
    ncclResult_t _r = (call);                                                           \
    if (_r != ncclSuccess)                                                              \
      return ::nkb::fail(NKB_ENCCL, std::string(#call) + ": " + g_nccl.GetErrorString(_r)); \
  } while (0)

// inverse of the kernels' ordered encoding of doubles (monotone as unsigned
// 64-bit: sign set -> flip all bits, else set the sign bit)
static inline double dec_ordered_h(unsigned long long u) {
  unsigned long long b = (u & 0x8000000000000000ULL) ? (u & 0x7fffffffffffffffULL) : ~u;
  double d;
  memcpy(&d, &b, 8);
  return d;
}

// device copies of one pairwise plan (tables for the chunks this rank owns)
struct StatsTables {
  std::vector<PlanChunk> plan;
  std::vector<StatChunk> mine;                 // owned chunks, local offsets
  std::vector<int> mine_idx;                   // their plan indices
  std::vector<int> owned_count;                // per rank
  std::vector<StatShapeHost> shapes;
  std::map<long long, int> shape_of_len;
  StatChunk* d_chunks = nullptr;
  StatShape* d_shapes = nullptr;
  int2* d_leaves = nullptr;
  int2* d_nodes = nullptr;
  int* d_levels = nullptr;
  double* d_out = nullptr;                     // sums [n] + 3 reduced words (min, max, NaN)
  double* h_out = nullptr;                     // pinned copy of d_out
  std::vector<int> comb;                       // postfix program of the tree above the chunks
  int n_dev = 0;
};

void stats_tables_free(StatsTables& T);

}  // namespace nkb

// the context is the opaque `nkb_ctx` of the C ABI (global scope); its
// members use the internal types
using namespace nkb;  // internal header, included by the ABI translation units only

struct nkb_ctx {
  int device = 0;
  // mesh (borrowed)
  int64_t E = 0;
  int N = 0;
  const double *x = nullptr, *y = nullptr, *z = nullptr;
  int64_t elem_off = 0, E_global = 0;
  std::vector<Field> fields;
  std::string vel_name = "velocity";
  double gll[kNP], D[kNP * kNP];
  // step scratch (library-owned)
  int* elem_count = nullptr;                  // ordered mode: per-element triangle counts
  long long* elem_offset = nullptr;           // ordered mode: exclusive scan
  int64_t elem_cap = 0;
  unsigned long long* counters = nullptr;   // [0] ntri [1] enc min [2] enc max [3] ntri global; then ticket
  unsigned int* ticket = nullptr;
  float4* tri = nullptr;
  unsigned long long* meta = nullptr;
  int64_t tri_cap = 0;                      // = n_regions * region_cap in FAST mode
  bool meta_alloc = false;
  unsigned long long* region_count = nullptr;   // [kMaxRegions] FAST-mode per-CTA fill
  int64_t region_cap = 0;
  int n_regions = 0;
  bool last_fast = false;
  float4* tri_export = nullptr;             // compacted FAST-mode triangles (on request)
  unsigned long long* meta_export = nullptr;
  int64_t export_cap = 0;
  unsigned long long* zbuf = nullptr;       // W*H + 2 range words: the last step's key buffer
  // one-GPU steps alternate two key buffers: each step's resolve clears the
  // other one for the next step (launch_resolve_tail)
  unsigned long long* zbufs[2] = {nullptr, nullptr};   // one allocation
  int zpar_next = 0;
  bool znext_clean = false;                 // zbufs[zpar_next] is all ~0
  unsigned int* rticket = nullptr;          // the tail's last-CTA ticket
  bool step_clear = true;                   // the step being enqueued clears its key buffer first
  unsigned char* rgba = nullptr;
  float* depth = nullptr;
  unsigned char* rgb_dev = nullptr;         // packed RGB for the PPM payload
  unsigned char* h_ppm = nullptr;           // pinned: PPM header + RGB
  int64_t ppm_cap = 0;
  double* range_dev = nullptr;
  int W = 0, H = 0;
  bool image_valid = false;
  int64_t last_ntri = 0;
  // pinned host staging
  unsigned long long* h_counters = nullptr;  // 4 + 2 (range)
  unsigned long long* h_counters_dev = nullptr;  // mapped device pointer of h_counters
  // structured renderer scratch
  const double** s_ptrs = nullptr;
  int64_t* s_col0 = nullptr;
  unsigned long long* s_minmax = nullptr;
  int s_cap = 0;
  // comm
  ncclComm_t comm = nullptr;
  int rank = 0, nranks = 1;
  cudaEvent_t ev[9] = {};                   // stage events; 6-8: P2P composite detail (timing)
  // geometry cache of d(r,s,t)/d(x,y,z) (fused.cu geometry_kernel): compact
  // (all elements extruded, kGeoCompact doubles per element) or full (9 SoA
  // arrays of 512 doubles per element)
  int geo_enabled = 1;                       // 0 off, 1 compact when possible, 2 full layout only
  bool geo_valid = false;
  double* geo = nullptr;
  int geo_layout = 0;                        // NKB_GEO_NONE / FULL / COMPACT
  int64_t geo_bytes = 0;
  unsigned long long* geo_flag = nullptr;    // device counter of non-extruded elements (build only)
  bool geo_used = false;                     // last step used it
  bool geo_built = false;                    // last step (re)built it
  unsigned long long* prof = nullptr;        // debug phase profile (NKB_PROFILE_PHASES=1)
  // nkb_execute_async: the enqueued step whose report nkb_execute_wait collects
  bool async_pending = false;
  bool async_composite = false, async_ordered = false, async_emit_meta = false;
  int async_surface_pass = 0;
  std::map<std::vector<long long>, std::unique_ptr<StatsTables>> stats_cache;   // nkb_stats plans
  GsLocal gs;                                // DSSUM gather-scatter plan (nkb_mesh_set_global_ids)
  bool gs_ready = false;
  // in transit staging (nkb_transit_gather): the assembled mesh on the endpoint
  double* tr_buf = nullptr;
  int64_t tr_cap = 0;                        // doubles
  cudaGraphExec_t graph_exec[2] = {nullptr, nullptr};   // captured steps (by key-buffer parity)
  std::string graph_key[2];
  cudaStream_t cap_stream = nullptr;
  // P2P steps in two halves (run_step): A = surface pass .. raster .. "keys
  // ready" on the caller's stream, B = composite .. report on comp_stream,
  // so step k's composite overlaps step k+1's surface pass
  cudaStream_t comp_stream = nullptr;
  cudaEvent_t ev_a[2] = {}, ev_b[2] = {};    // by key-buffer parity
  bool ev_b_live[2] = {false, false};
  int last_b = -1;                           // parity of the last B enqueued (image / range writer)
  cudaGraphExec_t graph_exec_a[2] = {nullptr, nullptr}, graph_exec_b[2] = {nullptr, nullptr};
  std::string graph_key_a[2], graph_key_b[2];
  unsigned long long* csnap = nullptr;       // [2][8] counters of the step, by parity (range_words_kernel)
  double* dq = nullptr;                      // continuous pipeline: DSSUM'd Q / |w| scratch
  double* dw = nullptr;
  int64_t dcap = 0;
  // P2P composite state (composite.cu)
  struct {
    bool ready = false, unavailable = false;
    int W = 0, H = 0;
    unsigned long long* keys[2] = {nullptr, nullptr};
    unsigned long long* flags = nullptr;
    int* err = nullptr;
    std::vector<void*> opened;
    const unsigned long long* peer_keys[2][kMaxRanks] = {};
    unsigned long long* peer_flags[kMaxRanks] = {};
    unsigned char* root_rgba = nullptr;
    float* root_depth = nullptr;
    unsigned long long epoch = 0;            // host copy of the step epoch
    unsigned long long* dev_epoch = nullptr; // [0] device counter, [1 + parity] the composite stream's copy
    unsigned long long* h_res = nullptr;     // pinned: [0] timeout flag, [1..] per-rank triangles
    unsigned long long* h_res_dev = nullptr; // its mapped device pointer (report_kernel writes it)
  } p2p;
};

namespace nkb {
int ctx_check(nkb_ctx* ctx);
const Field* find_field(nkb_ctx* ctx, const std::string& name);
int geo_attach(nkb_ctx* ctx, FusedParams& fp, cudaStream_t s);
int fused_params_base(nkb_ctx* ctx, FusedParams& fp);
int gs_apply(nkb_ctx* ctx, double* field, cudaStream_t s);
}  // namespace nkb
