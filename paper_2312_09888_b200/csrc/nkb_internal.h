// Internal declarations shared by the libnekb200 translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/nekb200.h"

namespace nkb {

// ---- error plumbing ------------------------------------------------------
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);

#ifndef NKB_TRY
#define NKB_TRY(expr)            \
  do {                           \
    int _rc = (expr);            \
    if (_rc != NKB_OK) return _rc; \
  } while (0)
#endif

#define NKB_CUDA(call)                                                              \
  do {                                                                              \
    cudaError_t _e = (call);                                                        \
    if (_e != cudaSuccess)                                                          \
      return ::nkb::fail(NKB_ECUDA, std::string(#call) + ": " + cudaGetErrorString(_e)); \
  } while (0)

#define NKB_CHECK(cond, code, msg) \
  do {                             \
    if (!(cond)) return ::nkb::fail((code), (msg)); \
  } while (0)

// ---- compile-time geometry of the supported element order ------------------
constexpr int kN = 7;              // polynomial order
constexpr int kNP = kN + 1;        // GLL nodes per direction
constexpr int kNN = kNP * kNP * kNP;   // 512 nodes per element
constexpr int kNC = kN * kN * kN;      // 343 sub-hexes per element

// ---- field registry --------------------------------------------------------
struct Field {
  std::string name;
  int ncomp = 0;
  const double* base = nullptr;
  int64_t comp_stride = 0;
};

// ---- sources of a per-node scalar inside the fused kernel ------------------
enum Src : int {
  SRC_Q = 0,        // Q-criterion
  SRC_WMAG = 1,     // |vorticity|
  SRC_UMAG = 2,     // |velocity|
  SRC_SCALAR0 = 3,  // loaded scalar field slot 0
  SRC_SCALAR1 = 4,  // loaded scalar field slot 1
  SRC_PLANE = 8,    // plane distance of surface k: SRC_PLANE + k
};
constexpr int kMaxScalars = 4;

struct FusedParams {
  int64_t n_elements;
  const double* x;
  const double* y;
  const double* z;
  const double* vel[3];
  const double* scalar[kMaxScalars];
  const double* in_ptr[8];          // filled by launch_fused: staged inputs in slot order
  int need_grad;                    // compute velocity gradient (Q / vorticity)
  int need_vel;                     // load velocity
  int need_wmag;                    // |vorticity| used (surface, colour or export)
  int need_umag;                    // |velocity| used (surface or colour)
  int n_scalars;
  int n_surf;
  int surf_src[NKB_MAX_SURFACES];
  double surf_iso[NKB_MAX_SURFACES];
  double surf_n[NKB_MAX_SURFACES][3];
  int color_src;                    // -1: no colour (export-only run)
  // exports (may be null)
  double* q_out;
  double* wmag_out;
  double* vort_out;                 // AoS 3 comps
  // triangle output
  float4* tri;                      // 3 float4 per triangle
  unsigned long long* meta;         // may be null
  int64_t tri_cap;
  // output slot allocation
  int mode;                         // FUSED_FAST | FUSED_COUNT | FUSED_ORDERED
  long long region_cap;             // FAST: triangles per CTA region (CTA b owns [b*cap, (b+1)*cap))
  unsigned long long* region_count; // FAST: [gridDim.x] triangles each CTA produced
  int* elem_count;                  // [n_elements] (COUNT mode)
  const long long* elem_offset;     // [n_elements] exclusive scan (ORDERED mode)
  unsigned long long* counters;     // [0] total triangles, [1] enc(min colour), [2] enc(max colour)
  const double* geo;                // optional geometry cache d(r,s,t)/d(x,y,z): [E][9][512] (full)
  int geo_compact;                  // 1: geo is the compact layout [E][kGeoCompactDoubles]
  unsigned long long* prof;         // debug: [role 3][phase 6] cycle sums (NKB_PROFILE_PHASES=1)
  int sm_reserve;                   // SMs the surface pass leaves free (the previous step's composite)
};
enum FusedMode : int { FUSED_FAST = 0, FUSED_COUNT = 1, FUSED_ORDERED = 2 };

struct RasterParams {
  const float4* tri;
  const unsigned long long* region_count;   // [n_regions] triangles in each region
  int n_regions;
  int64_t region_cap;               // region r = tri[r*region_cap, r*region_cap + count)
  double view[16];                  // 3x4 view rows + perspective row (all zero: orthographic)
  int width, height;
  unsigned long long* zbuf;
  int lanes_per_tri = 1;            // 1, 2 or 4 threads per triangle (pixel rows split)
};

struct Colormap {
  int n;
  double t[NKB_MAX_ANCHORS];
  double rgb[NKB_MAX_ANCHORS][3];
  double slope[NKB_MAX_ANCHORS][3];   // (rgb[j+1]-rgb[j]) / (t[j+1]-t[j]), IEEE on the host
};

// ---- P2P sort-last composite (composite.cu) ----------------------------------
constexpr int kMaxRanks = 8;
struct P2PParams {
  int rank, nranks;
  unsigned long long* flags;                          // local [4*kMaxRanks]: ready | done | tri count | overflow
  const unsigned long long* overflow;                 // local counters[6]: this step overflowed
  unsigned long long* peer_flags[kMaxRanks];          // every rank's flags (IPC-mapped)
  const unsigned long long* peer_keys[kMaxRanks];     // every rank's key buffer of this epoch
  long long npx;
  int width, height;
  double vmin, vmax;                                  // NaN => global data range
  Colormap cmap;
  unsigned char bg[4];
  unsigned char* root_rgba;                           // rank 0's image (IPC-mapped)
  float* root_depth;
  double* range_out;                                  // local [2]
  int max_blocks = 0;                                 // composite grid cap (0: fill the GPU)
  int bulk = 0;                                       // 1: bulk-copy (TMA) composite kernel
  int* err;                                           // local: 1 = peer timeout
  unsigned long long* dev_epoch;                      // local: step epoch (device counter, graph-safe)
  unsigned long long* ep_slot = nullptr;              // epoch_kernel also stores the new epoch here: the
                                                      // parity slot the composite stream's kernels read
};
// the epoch lives on the device, so a step's launches are identical every
// step (CUDA-graph replayable); only the key-buffer parity alternates
int launch_p2p_epoch(const P2PParams& p, cudaStream_t s);
int launch_p2p_signal(const P2PParams& p, int which, const unsigned long long* count, cudaStream_t s);
int launch_p2p_wait(const P2PParams& p, int which, unsigned long long back, cudaStream_t s);
int launch_p2p_composite(const P2PParams& p, cudaStream_t s);

// step report -> mapped pinned host words (device pointers of cudaMallocHost memory)
struct ReportParams {
  const unsigned long long* counters;       // [4]
  const double* range;                      // [2]
  const unsigned long long* region_count;   // [n_regions] or null (ordered mode)
  int n_regions;
  unsigned long long* h_counters;           // host words [0..3] counters, [4..5] range bits, [6..7] overflow
  const int* err;                           // P2P: timeout flag, or null
  const unsigned long long* peer_counts;    // P2P: [kMaxRanks] per-rank triangle counts
  const unsigned long long* peer_overflow;  // P2P: [kMaxRanks] per-rank overflow words
  int nranks;
  unsigned long long* h_res;                // P2P host words [0] timeout, [1..kMaxRanks] counts,
                                            // [1+kMaxRanks] any rank overflowed; or null
  int part = 3;                             // 1: counters + regions, 2: range + P2P words, 3: both
};
int launch_report(const ReportParams& p, cudaStream_t s);

struct ResolveParams {
  const unsigned long long* zbuf;
  int width, height;
  double lo, hi;          // resolved on host when known, else read from range_words
  const unsigned long long* range_words;  // [2]: enc(lo), ~enc(hi) (after composite), may be null
  double vmin, vmax;      // NaN => from range_words
  Colormap cmap;
  unsigned char bg[4];
  unsigned char* rgba;
  float* depth;
  double* range_out;      // [2] device, range used
  // one-GPU step tail (all null otherwise): the range from the step's
  // counters, the next step's key buffer cleared in the same pass, and the
  // range words + overflow word + report done by the last CTA (ticket)
  unsigned long long* counters = nullptr;     // [1] enc(min) [2] enc(max); [6] := overflow
  unsigned long long* clear_next = nullptr;   // [W*H + 2] := ~0
  unsigned long long* words = nullptr;        // this step's range words (zbuf + W*H)
  const unsigned long long* region_count = nullptr;
  int n_regions = 0;
  long long region_cap = 0, tri_cap = 0;
  unsigned int* ticket = nullptr;             // zero between launches
};

// ---- kernel launchers (defined in .cu files) --------------------------------
int set_dmat_constant(const double* dmat);
int fused_grid(int64_t n_elements, int sm_reserve = 0);       // CTAs (= triangle regions) of launch_fused
int launch_fused(const FusedParams& p, cudaStream_t s);
int launch_fused_prepare();
// K1s (stream.cu): pipelines without a velocity gradient (no exports, fields
// 16-byte aligned); launch_fused dispatches to it when surface_pass_of == 1
bool stream_eligible(const FusedParams& p);
// checked build: per-file device bounds-check counters (checked.cuh)
unsigned long long checked_read_fused(int* line);
unsigned long long checked_read_stream(int* line);
unsigned long long checked_read_raster(int* line);
unsigned long long checked_read_composite(int* line);
int checked_violations();
int checked_selftest(cudaStream_t s);          // NKB_CHECKED_SELFTEST=1: one failing check
int fused_ctas_per_sm(const FusedParams& p);   // surface pass CTAs per SM (composite overlap policy)
int fused_node_prog(const FusedParams& p);   // K1g + 16 x K1s node program (graph key)
int stream_prog_of(const FusedParams& p);    // K1s node program
int surface_pass_of(const FusedParams& p);     // 0 K1, 1 K1s (stream.cu), 2 K1g (2-3 CTAs per SM)
int fused_grid_for(const FusedParams& p, int64_t n_elements);   // triangle regions of that pass
int launch_stream(const FusedParams& p, int grid, cudaStream_t s);
int launch_stream_prepare();
// geometry cache build: full layout (9 x 512 doubles per element) and/or the
// compact one (kGeoCompactDoubles per element; *n_general counts elements
// that do not fit it)
constexpr int kGeoCompactDoubles = 4 * 64 + 8;
int launch_geometry(const double* x, const double* y, const double* z, int64_t E, double* full, double* compact,
                    unsigned long long* n_general, cudaStream_t s);
int launch_compact(const float4* tri, const unsigned long long* meta, const unsigned long long* region_count,
                   int n_regions, int64_t region_cap, float4* out_tri, unsigned long long* out_meta,
                   int64_t n_total, cudaStream_t s);
int launch_count_scan(const int* cnt, int64_t n, long long* off, unsigned long long* total, cudaStream_t s);
int launch_zbuf_clear(unsigned long long* zbuf, int64_t n, cudaStream_t s);
int launch_init_counters(unsigned long long* counters, cudaStream_t s);   // [8] step counters
int launch_raster(const RasterParams& p, cudaStream_t s);
int launch_range_words(unsigned long long* counters, unsigned long long* words,
                       const unsigned long long* region_count, int n_regions, int64_t region_cap, int64_t tri_cap,
                       cudaStream_t s, unsigned long long* snap = nullptr);   // snap: copy of counters[0..7]
int launch_resolve(const ResolveParams& p, cudaStream_t s);
// the one-GPU tail: resolve + next key-buffer clear + range words + report in one launch
int launch_resolve_tail(const ResolveParams& p, const ReportParams& rep, cudaStream_t s);
// ---- stats.cu: numpy-exact min / max / mean ----
constexpr long long kChunk = 32768;      // values per CTA subtree (<= 640 leaves of 57..128)
constexpr int kWin = 128;                // boundary window (one pairwise leaf)
constexpr int kMaxChunkLeaves = 640;
constexpr int kMaxSeg = 16;
struct StatSeg {
  const double* base;
  long long n_tuples;
  int ncomp;
  long long comp_stride;
  long long start;                       // first AoS index of this segment
};
struct StatChunk {
  long long off;                         // first AoS index (in the segments' numbering)
  int shape;
};
struct StatShape {
  int leaf0, n_leaves, node0, n_nodes, level0, n_levels;
};
struct StatsParams {
  StatSeg seg[kMaxSeg];
  int nseg;
  long long n;                           // values in the segments
  const StatChunk* chunks;
  int n_chunks;
  const StatShape* shapes;
  const int2* leaves;                    // (offset in chunk, length)
  const int2* nodes;                     // children as slots of the value array
  const int* level_start;
  double* out_sum;                       // [n_chunks]
  unsigned long long* out_mm;            // [3]: enc(min) (atomicMin), enc(max) (atomicMax), NaN flag
};
struct PlanChunk {
  long long off, n;
  int owner;                             // rank, or -1 for a leaf across a rank boundary
};
struct StatShapeHost {
  std::vector<int2> leaves, nodes;
  std::vector<int> level_start;
  int n_levels = 0;
};
void pairwise_plan(long long n, const std::vector<long long>& rank_lo, std::vector<PlanChunk>& out);
void pairwise_combine_program(long long n, const std::vector<long long>& rank_lo, std::vector<int>& prog);
double pairwise_combine(const std::vector<int>& prog, const std::vector<double>& chunk_sums);
void pairwise_shape(long long n, StatShapeHost& sh);
int launch_pairwise_chunks(const StatsParams& p, cudaStream_t s);
int launch_stat_windows(const StatsParams& p, double* out, cudaStream_t s);

int launch_be_points(const double* x, const double* y, const double* z, int64_t npts, void* out, cudaStream_t s);
int launch_be_cells(int64_t ncells, void* out, cudaStream_t s);
int launch_be_types(int64_t ncells, void* out, cudaStream_t s);
int launch_bswap64(void* p, int64_t n, cudaStream_t s);
// ---- dssum.cu: gather-scatter (direct stiffness summation) ----
constexpr int kGroupMax = 8;          // one-rank DSSUM: runs of 2..8 copies grouped by count
struct GsGroups {                     // (kernel parameter: passed by value)
  int* idx = nullptr;                 // per K: K rows of n[K] local indices (SoA) at base[K]
  long long base[kGroupMax + 1] = {};
  long long n[kGroupMax + 2] = {};    // runs per copy count; [kGroupMax + 1] = longer runs (CSR)
  long long first[kGroupMax + 2] = {};  // first position of count k in the count-sorted run order
  int block[kGroupMax + 2] = {};      // first block of each group (k >= 2)
  int blocks = 0;
};
struct GsLocal {
  long long n = 0, U = 0;            // local GLL copies, unique global ids
  int* idx = nullptr;                // [n] local indices sorted by gid (stable)
  int* off = nullptr;                // [U+1] CSR runs
  long long* ugid = nullptr;         // [U] sorted unique gids
  int* mult = nullptr;               // [U] copies over all ranks
  double* part = nullptr;            // [U] partial / total sums
  GsGroups groups;                   // one rank: runs grouped by copy count
  int* lrun = nullptr;               // runs longer than kGroupMax (unique indices)
  // shared with other ranks (multi-rank only)
  int n_shared = 0;
  int* su = nullptr;                 // [n_shared] unique index of each shared gid (increasing gid)
  unsigned char* smask = nullptr;    // [n_shared] ranks holding it
  int* spos = nullptr;               // [n_shared * R] position in rank q's buffer
  int* slist = nullptr;              // per neighbour q: unique indices to send, at noff[q]
  double* sbuf = nullptr;            // send buffers (same layout)
  double* rbuf = nullptr;            // receive buffers (same layout: list lengths match)
  const double** rptr = nullptr;     // [R] device pointers into rbuf (mine unused)
  std::vector<int> ncount, noff;     // per neighbour list length / offset (host)
};
int gs_build_local(const long long* gid, long long n, GsLocal& g, cudaStream_t s);
void gs_free(GsLocal& g);
int gs_sum(const GsLocal& g, const double* v, cudaStream_t s);
int gs_build_groups(GsLocal& g, cudaStream_t s);
int gs_average_local(const GsLocal& g, double* v, cudaStream_t s);   // one rank: sum + scatter in one pass
int gs_pack(const GsLocal& g, int q, cudaStream_t s);
int gs_combine(const GsLocal& g, int R, int me, cudaStream_t s);
int gs_scatter(const GsLocal& g, double* v, cudaStream_t s);
int gs_bucket_by_owner(const GsLocal& g, int R, long long* out, std::vector<int>& counts, cudaStream_t s);

int launch_pack_rgb(const unsigned char* rgba, unsigned char* rgb, int64_t npx, cudaStream_t s);
int launch_points_aos(const double* x, const double* y, const double* z, int64_t npts,
                      double* out, cudaStream_t s);
int launch_connectivity(int64_t ncells, int64_t* conn, int64_t* offsets, unsigned char* types,
                        cudaStream_t s);
int launch_field_aos(const double* base, int64_t stride, int ncomp, int64_t npts, double* out,
                     cudaStream_t s);
int launch_field_mag(const double* base, int64_t stride, int ncomp, int64_t npts, double* out,
                     cudaStream_t s);
struct StructuredParams {
  int n_blocks;
  const double* const* values;  // device array of device pointers
  const int64_t* col0;          // device [n_blocks+1] prefix of ni
  int64_t ni_total, rows;
  int comps, mode;
  int width, height;
  Colormap cmap;
  unsigned long long* minmax;   // device [2] ordered encodings
  double vmin, vmax;
  unsigned char* rgb;
  double* range_out;
};
int launch_structured_minmax(const StructuredParams& p, cudaStream_t s);
int launch_structured_render(const StructuredParams& p, cudaStream_t s);

// GLL nodes / derivative matrix (host, deterministic; see gll.cpp)
void gll_nodes_dmat(int order, double* nodes, double* dmat);

}  // namespace nkb
