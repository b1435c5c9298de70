/*
 * nekb200.h -- C ABI of libnekb200.so, the B200-native in situ analysis hot
 * path (SEM adaptor -> velocity gradient / vorticity / Q-criterion ->
 * marching-cubes isosurface + slice -> raster to RGBA+depth -> sort-last
 * depth composite), plus the drop-in GPU path for the reference's 2D
 * pseudocolor renderer.
 *
 * The reference (`/root/reference/pkg/src/nekmini`, pure Python) has no FFI:
 * its hot path is the in-process sink protocol
 *     cls(params) / consume(snapshot) -> int / finalize()
 * (`sinks.py:310-418`) driven by `Bridge.update` (`bridge.py:145-177`), and the
 * paper's SENSEI surface `DataAdaptor{Initialize, GetNumberOfMeshes,
 * GetMeshMetadata, GetMesh, AddArray}` / `AnalysisAdaptor::Execute`
 * (`PAPER.md:141-150`, `:158-168`).  Each entry point below names the
 * reference interface it replaces.  The Python package binds these with
 * ctypes (paper_2312_09888_b200/_native.py); INTEGRATION.md shows the stub a
 * maintainer of the reference would add.
 *
 * Conventions
 *  - every function returns an int status (NKB_OK == 0); the message of the
 *    last failure on the calling thread is nkb_last_error().
 *  - device pointers are BORROWED for the duration of the call (the library
 *    never frees caller memory).  Library-owned outputs (image, depth,
 *    triangles) stay valid until the next nkb_execute on the same context.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default).
 *  - layout of every SEM field (NekRS convention): element-major, then the
 *    (N+1)^3 GLL nodes of the element with i (r-direction) fastest:
 *        value(e, i, j, k) = f[e*(N+1)^3 + i + (N+1)*(j + (N+1)*k)]
 *    A multi-component field is `ncomp` such arrays, comp_stride doubles apart
 *    (NekRS `fieldOffset`).  Exported VTK arrays are component-fastest AoS,
 *    `flat = c + comps*point` (reference data_model.py:8-14).
 *  - a context is confined to one host thread at a time (bridge.py:132-137).
 */
#ifndef NEKB200_H
#define NEKB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NKB_ABI_VERSION 1

/* status codes -> Python exceptions (see _native.py) */
#define NKB_OK      0
#define NKB_EINVAL  1   /* ValueError: bad argument / unknown field / schema */
#define NKB_ERANGE  2   /* ValueError: buffer too small (needed size reported) */
#define NKB_EIO     3   /* OSError */
#define NKB_ECUDA   4   /* RuntimeError: CUDA runtime failure */
#define NKB_ENCCL   5   /* RuntimeError: NCCL failure / comm not initialised */
#define NKB_ESTATE  6   /* RuntimeError: call order (e.g. execute before mesh_set) */

/* VTK cell type of every sub-hex (VTK_HEXAHEDRON) */
#define NKB_VTK_HEXAHEDRON 12

#define NKB_MAX_SURFACES 4
#define NKB_MAX_ANCHORS  8
#define NKB_NAME_MAX     64

#define NKB_SURF_ISO    0   /* marching cubes on a field:   inside = f >= value */
#define NKB_SURF_SLICE  1   /* marching cubes on n.x - value: inside = n.x >= value */

#define NKB_ASSOC_POINT 0
#define NKB_ASSOC_CELL  1

typedef struct nkb_ctx nkb_ctx;

typedef struct {
    int     kind;                    /* NKB_SURF_ISO | NKB_SURF_SLICE */
    char    field[NKB_NAME_MAX];     /* iso field: "Q", "vorticity:mag", "<vec>:mag", or a registered scalar */
    double  value;                   /* iso value, or plane offset c in n.x = c */
    double  normal[3];               /* slice plane normal (any length) */
} nkb_surface;

/* One in situ analysis (the Catalyst pipeline stand-in).  The colormap
 * semantics are the reference's: range = global data min/max of the colour
 * field unless vmin/vmax are finite (sinks.py:264-265), t=(d-lo)/(hi-lo) or 0
 * when hi<=lo (sinks.py:266-269), piecewise-linear anchors evaluated like
 * np.interp then floor(v+0.5) (sinks.py:201-209).  Row 0 is the top of the
 * image (sinks.py:256-257). */
typedef struct {
    int          n_surfaces;                       /* 0..NKB_MAX_SURFACES */
    nkb_surface  surfaces[NKB_MAX_SURFACES];
    char         color_field[NKB_NAME_MAX];        /* scalar used for colour */
    int          width, height;
    /* (col, row, depth) = view * (x, y, z, 1), row-major 3x4, pixel units;
       pixel (c, r) is sampled at its centre (c+0.5, r+0.5); depth must land
       in [0, 1] (outside = clipped). */
    double       view[12];
    double       vmin, vmax;                       /* NaN => global data range */
    int          n_anchors;                        /* 0 => reference DEFAULT_COLORMAP */
    double       anchor_t[NKB_MAX_ANCHORS];
    unsigned char anchor_rgb[NKB_MAX_ANCHORS][3];
    unsigned char background[4];                   /* RGBA of uncovered pixels */
    int          emit_meta;                        /* 1: record per-triangle (element, cell, surface, case) */
    int          composite;                        /* 1: depth-composite across the comm (nkb_comm_init) */
    int          timing;                           /* 1: fill per-stage CUDA-event times in nkb_report */
    int          continuous;                       /* 1: DSSUM-average derived sources (Q, vorticity:mag)
                                                      before surfaces / colour (C0 across element faces);
                                                      needs nkb_mesh_set_global_ids */
    /* perspective: w = persp . (x, y, z, 1) and (col, row, depth) = view * (x, y, z, 1) / w
       (vertices with w <= 0 drop their triangle); all zero = orthographic (no division) */
    double       persp[4];
} nkb_pipeline;

typedef struct {
    int64_t n_triangles;          /* this rank */
    int64_t n_triangles_global;   /* all ranks when composite (else == n_triangles) */
    int64_t tri_capacity;         /* current triangle buffer capacity */
    double  range[2];             /* colour range actually used (global when composite) */
    double  data_range[2];        /* colour-field min/max over this rank's points */
    float   ms_fused, ms_raster, ms_composite, ms_resolve;   /* when timing */
    int     reran;                /* 1 if the triangle buffer grew and the step re-ran */
    int     geometry_cached;      /* 1 if the step used the geometry cache */
    float   ms_geometry;          /* time spent (re)building the cache this step (when timing) */
    int     surface_pass;         /* surface pass that ran: 0 = K1 fused (velocity gradient),
                                     1 = K1s stream (no gradient; NKB_STREAM=0 forces K1),
                                     2 = K1g gradient pass, 2-3 CTAs per SM (geometry cache; NKB_FUSED2=0 forces K1) */
    int     overflowed;           /* nkb_execute_wait only: the step's triangles overflowed on some
                                     rank (its triangle set and image are incomplete; the buffer
                                     has grown for the steps enqueued from now on) */
    int     composite_overlapped; /* nkb_execute_wait only: the last step's P2P composite ran
                                     on the library's stream beside the next surface pass */
} nkb_report;

typedef struct {
    int64_t n_elements;           /* local E */
    int     order;                /* N */
    int64_t n_points;             /* E*(N+1)^3 element-local GLL points */
    int64_t n_cells;              /* E*N^3 linear sub-hexes */
    int     cell_type;            /* NKB_VTK_HEXAHEDRON */
    int64_t element_offset;       /* global id of local element 0 (partition) */
    int64_t n_elements_global;
    int     n_fields;
    int     rank, nranks;
} nkb_mesh_metadata;

/* ---- library / context ------------------------------------------------- */
int         nkb_abi_version(void);
const char* nkb_last_error(void);
int         nkb_ctx_create(int cuda_device, nkb_ctx** out);
int         nkb_ctx_destroy(nkb_ctx* ctx);

/* GLL nodes (N+1) and differentiation matrix D ((N+1)^2, row-major,
 * D[i][m] = dl_m/dr at r_i) exactly as the kernels use them. */
int nkb_gll(int order, double* nodes, double* dmat);

/* ---- DataAdaptor (nek_sensei::DataAdaptor) ----------- */
/* Initialize(nek_data): borrow the device-resident element coordinates.
 * replaces: solver.snapshot_of -> Block(...) construction (solver.py:282-305) */
int nkb_mesh_set(nkb_ctx* ctx, int64_t n_elements, int order,
                 const double* x, const double* y, const double* z,
                 int64_t element_offset, int64_t n_elements_global);
/* Geometry cache.  The first step that needs velocity gradients computes the
 * Jacobian inverse d(r,s,t)/d(x,y,z) at every GLL node (72 B/point, the SEM
 * "geometric factors" NekRS keeps in mesh->vgeo) and later steps reuse it;
 * values are bit-identical to recomputing them.  Calling nkb_mesh_set again
 * with the same pointers, sizes and offsets keeps the cache (static mesh);
 * after editing coordinates in place (moving mesh) call nkb_mesh_modified.
 * nkb_set_geometry_cache(ctx, 0) disables it; 1 (default) keeps it in the
 * compact layout when every element is extruded (x, y independent of t, z of
 * r and s: 2 KB per element instead of 36 KB) and the full one otherwise; 2
 * forces the full layout.  Env NKB_GEOM_CACHE=0 / full sets the default. */
/* Global GLL node ids (NekRS mesh->globalIds), DEVICE int64[E*(N+1)^3],
 * read during the call: builds the gather-scatter of nkb_dssum.  Collective
 * when a communicator is initialised (finds the ids shared with other ranks).
 * Dropped by nkb_mesh_set with a different mesh.  SURVEY.md §8f row 1. */
int nkb_mesh_set_global_ids(nkb_ctx* ctx, const int64_t* gid, void* stream);
/* Direct stiffness average, in place, of a DEVICE point field (E*(N+1)^3
 * doubles): every copy of a global node gets
 *   ((P_r0 + P_r1) + ...) / count,  P_r = sum of rank r's copies in
 * increasing local index order (ranks in increasing order).  Collective. */
int nkb_dssum(nkb_ctx* ctx, double* field, void* stream);
/* In transit (the paper's staging mode, reference transport.py:358-376):
 * collective N:1 gather of every rank's mesh and registered fields to `root`
 * over NCCL send/recv (GPU-direct, no host copy), concatenated in rank order
 * (partitions must be contiguous and share one field schema).  Afterwards
 * root's context describes the assembled mesh (library-owned buffers, valid
 * until the next gather) and root can run nkb_execute on it alone. */
int nkb_transit_gather(nkb_ctx* ctx, int root, void* stream);
int nkb_mesh_modified(nkb_ctx* ctx);
int nkb_set_geometry_cache(nkb_ctx* ctx, int enable);
/* Geometry-cache introspection: *layout = NKB_GEO_NONE (not built / off),
 * NKB_GEO_FULL (9 doubles per GLL point) or NKB_GEO_COMPACT (every element
 * extruded: 4 x 64 in-plane entries + 8 axial entries per element);
 * *bytes = device bytes the cache holds (either pointer may be NULL). */
#define NKB_GEO_NONE    0
#define NKB_GEO_FULL    1
#define NKB_GEO_COMPACT 2
int nkb_geometry_info(nkb_ctx* ctx, int* layout, int64_t* bytes);
/* register (or re-point) a device-resident point field, borrowed.
 * replaces: FieldArray(name, POINT, comps, values) (data_model.py:27-55) */
int nkb_field_set(nkb_ctx* ctx, const char* name, int ncomp,
                  const double* base, int64_t comp_stride);
int nkb_field_clear(nkb_ctx* ctx);
/* GetNumberOfMeshes == 1; GetMeshMetadata (data_model.py:111-128 metadata_of) */
int nkb_get_mesh_metadata(nkb_ctx* ctx, nkb_mesh_metadata* out);
/* bounding box of the local mesh (global over the comm when initialised):
 * out6 = {xmin, xmax, ymin, ymax, zmin, zmax} (host). */
int nkb_mesh_bounds(nkb_ctx* ctx, double* out6, void* stream);
/* GetMesh: VTK unstructured grid of linear sub-hexes, into caller DEVICE
 * buffers sized from the metadata (any may be NULL to skip):
 *   points   [n_points*3]  double AoS (x,y,z)
 *   conn     [n_cells*8]   int64 point ids, VTK_HEXAHEDRON corner order
 *   offsets  [n_cells+1]   int64 (8*c)
 *   types    [n_cells]     uint8 (12) */
int nkb_get_mesh(nkb_ctx* ctx, double* points, int64_t* conn, int64_t* offsets,
                 unsigned char* types, void* stream);
/* AddArray: point array `name` as VTK AoS doubles into a caller DEVICE
 * buffer of n_points*ncomp.  name is a registered field, "<vec>:mag",
 * "Q", "vorticity" (3 comps) or "vorticity:mag".  *ncomp_out may be NULL.
 * replaces: scalar_field (sinks.py:227-242) / FieldArray export */
int nkb_add_array(nkb_ctx* ctx, const char* name, int association,
                  double* out, int* ncomp_out, void* stream);
/* Checkpoint export (legacy-VTK UNSTRUCTURED_GRID, the SEM analogue of the
 * reference's _encode_vtk, sinks.py:58-102): one BINARY section, big-endian
 * as the legacy format requires, encoded on the GPU into the caller's DEVICE
 * buffer `dst` (cap bytes).  what = "POINTS" (f64 x,y,z per point),
 * "CELLS" (int32 {8, ids...} per sub-hex, VTK_HEXAHEDRON order), "CELL_TYPES"
 * (int32 12) or any AddArray name (f64, components fastest).  dst == NULL:
 * *nbytes = the size only.  NKB_ERANGE when cap is too small or the point ids
 * do not fit int32. */
int nkb_encode_be(nkb_ctx* ctx, const char* what, void* dst, int64_t cap, int64_t* nbytes, void* stream);
int nkb_array_components(nkb_ctx* ctx, const char* name, int* ncomp_out);
/* name of the vector field derived quantities are computed from (default "velocity") */
int nkb_set_velocity_name(nkb_ctx* ctx, const char* name);

/* ---- AnalysisAdaptor::Execute (RenderSink.consume, sinks.py:342-348) --- */
int nkb_execute(nkb_ctx* ctx, const nkb_pipeline* p, nkb_report* out, void* stream);
/* Stream-ordered Execute: enqueue the step on `stream` and return without
 * a host synchronisation, so consecutive steps (and, across ranks, the P2P
 * composite) are ordered on the device only and host jitter does not couple
 * the ranks.  nkb_execute_wait synchronises and fills the report of the
 * last enqueued step.  The triangle buffer cannot grow behind an enqueued
 * step: a step that overflows is reported (overflowed = 1 if any step of the
 * sequence overflowed on any rank; triangles and image incomplete) and the
 * buffer grows for later steps; nkb_execute (which re-runs an overflowing
 * step) guarantees a complete result.  pipeline.timing must be 0.  With the
 * P2P composite each step's composite runs on a library stream beside the
 * next step's surface pass (NKB_COMPOSITE_OVERLAP=0: one stream). */
int nkb_execute_async(nkb_ctx* ctx, const nkb_pipeline* p, void* stream);
int nkb_execute_wait(nkb_ctx* ctx, nkb_report* out, void* stream);
/* results of the last execute (device pointers, library-owned; after
 * nkb_execute_async, valid once nkb_execute_wait returned) */
int nkb_image_device(nkb_ctx* ctx, const unsigned char** rgba, const float** depth,
                     const uint64_t** zbuf);
/* copy the last image to host memory (rgba: W*H*4, depth: W*H floats, either may be NULL) */
int nkb_image_copy(nkb_ctx* ctx, unsigned char* rgba, float* depth, void* stream);
/* The image as a complete binary PPM (P6 header + RGB rows, top row first),
 * byte-identical to write_ppm(ImageRGB(...)) (sinks.py:298-303), in
 * library-owned PINNED host memory valid until the next call on this ctx:
 * the RGBA->RGB pack runs on the GPU and only 3 B/pixel cross PCIe.
 * replaces: ImageRGB(w, h, rgba[..., :3].tobytes()) + write_ppm's encode */
int nkb_image_ppm(nkb_ctx* ctx, const unsigned char** ppm, int64_t* nbytes, void* stream);

/* ---- field statistics (StatsSink, sinks.py:366-393) ------------------------ */
/* One borrowed DEVICE array run: n_tuples tuples of ncomp components, the
 * components comp_stride values apart (SoA), read in the reference's AoS
 * order (component fastest, data_model.py:8-14). */
typedef struct nkb_segment {
    const double* base;
    int64_t       n_tuples;
    int           ncomp;
    int64_t       comp_stride;   /* ignored when ncomp == 1 */
} nkb_segment;
/* min, max and mean of the concatenated segments -- and, with collective != 0
 * and a communicator, of all ranks' concatenations in rank order -- with
 * numpy's arithmetic: out = {vals.min(), vals.max(), vals.mean()}, the mean
 * being np.add.reduce's pairwise summation divided by the count, bit for bit.
 * NaN anywhere gives NaN min/max/mean.  Zero values: NKB_EINVAL (numpy raises).
 * replaces: np.concatenate(...) + min/max/mean in StatsSink.consume (sinks.py:381-386) */
int nkb_stats(nkb_ctx* ctx, const nkb_segment* segs, int nseg, int collective, double out[3], void* stream);
/* triangles of the last execute, in deterministic (element, cell, surface, table) order:
 *   tri  [n*12] float: per vertex (x, y, z, colour scalar), 3 vertices
 *   meta [n]    uint64: element<<32 | cell<<16 | surface<<12 | tri_in_case<<8 | case
 *               (only when pipeline.emit_meta) */
int nkb_triangles_device(nkb_ctx* ctx, const float** tri, const uint64_t** meta, int64_t* n);

/* ---- sort-last composite over NCCL (assemble_global analogue,
 *      data_model.py:188-225 / transport.py:358-376) -------------------- */
/* In-process sort-last composite of n <= 8 partition contexts on ONE device
 * (e.g. R element ranges of one mesh, each executed with the same pipeline
 * and composite = 0): runs the P2P composite kernel (min over the partitions'
 * key buffers, global colour range, colormap resolve) once per band of rows,
 * exactly as n ranks would over NVLink, into root's image.  root may be one
 * of the partitions.  Lets a one-GPU box check R16's kernel bit for bit. */
int nkb_composite_partitions(nkb_ctx* root, nkb_ctx* const* parts, int n, const nkb_pipeline* p, void* stream);
int nkb_nccl_unique_id(unsigned char id_out[128]);
int nkb_comm_init(nkb_ctx* ctx, const unsigned char id[128], int nranks, int rank);
int nkb_comm_destroy(nkb_ctx* ctx);

/* ---- reference 2D pseudocolor renderer on the GPU (drop-in for
 *      sinks.render, sinks.py:245-295) ---------------------------------- */
/* Blocks tiled along x in producer order (assemble_global, data_model.py:188-225):
 * block b has ni[b] columns and `rows` = nk*nj rows, `comps` components, AoS
 * component-fastest, DEVICE pointer values[b].  mode 0: scalar (comps must be
 * 1), mode 1: ':mag'.  vmin/vmax NaN => data range.  rgb_out: DEVICE buffer
 * width*height*3, row 0 = top. */
int nkb_render_structured(nkb_ctx* ctx, int n_blocks, const double* const* values,
                          const int64_t* ni, int64_t rows, int comps, int mode,
                          int width, int height, double vmin, double vmax,
                          unsigned char* rgb_out, double* range_out, void* stream);

/* ---- memory helpers so the Python host layer needs no other CUDA binding */
int nkb_device_alloc(nkb_ctx* ctx, int64_t bytes, void** out);
int nkb_device_free(nkb_ctx* ctx, void* p);
int nkb_host_alloc(int64_t bytes, void** out);      /* pinned */
int nkb_host_free(void* p);
/* kind: 1 H2D, 2 D2H, 3 D2D (cudaMemcpyKind) */
int nkb_memcpy(void* dst, const void* src, int64_t bytes, int kind, void* stream);
int nkb_stream_sync(void* stream);
int nkb_device_sync(void);
int nkb_device_count(int* out);

#ifdef __cplusplus
}
#endif
#endif /* NEKB200_H */
