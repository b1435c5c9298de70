/* The in situ step driven from plain C through libnekb200's ABI -- what a
 * NekRS / SENSEI bridge (C++) would do with its device-resident fields:
 *
 *   nkb_ctx_create -> nkb_mesh_set (x, y, z) -> nkb_field_set (velocity,
 *   temperature) -> nkb_execute (iso Q, iso T, slice) -> nkb_image_ppm
 *
 * The mesh is a 3 x 2 x 2 box of order-7 elements with analytic fields;
 * tests/test_c_api.py feeds the dumped arrays to the Python path and to the
 * CPU oracle and checks the image byte for byte.
 *
 *   gcc -O2 -I include examples/insitu_c_api.c -L <lib dir> -lnekb200 -lm
 *   ./insitu_c_api out.ppm [fields.bin]     (fields.bin: the 7 host arrays, for the test)
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "nekb200.h"

#define CHECK(call)                                                        \
  do {                                                                     \
    int rc_ = (call);                                                      \
    if (rc_ != NKB_OK) {                                                   \
      fprintf(stderr, "%s failed (%d): %s\n", #call, rc_, nkb_last_error()); \
      return 1;                                                            \
    }                                                                      \
  } while (0)

enum { NX = 3, NY = 2, NZ = 2, NP = 8, NN = NP * NP * NP };

int main(int argc, char** argv) {
  const char* out = argc > 1 ? argv[1] : "insitu_c_api.ppm";
  const int64_t E = NX * NY * NZ, npts = E * NN;
  double nodes[NP];
  CHECK(nkb_gll(7, nodes, NULL));

  /* host fields: element-major, i fastest (NekRS layout); velocity SoA */
  double* h = (double*)malloc(sizeof(double) * (size_t)npts * 7);
  double *x = h, *y = h + npts, *z = h + 2 * npts, *u = h + 3 * npts, *t = h + 6 * npts;
  for (int64_t e = 0; e < E; ++e) {
    const int ex = (int)(e % NX), ey = (int)((e / NX) % NY), ez = (int)(e / (NX * NY));
    for (int k = 0; k < NP; ++k)
      for (int j = 0; j < NP; ++j)
        for (int i = 0; i < NP; ++i) {
          const int64_t g = e * NN + i + NP * (j + NP * k);
          x[g] = (ex + 0.5 * (nodes[i] + 1.0)) / NX * 2.0;
          y[g] = (ey + 0.5 * (nodes[j] + 1.0)) / NY * 1.5;
          z[g] = (ez + 0.5 * (nodes[k] + 1.0)) / NZ;
          u[g] = sin(2.0 * x[g]) * cos(3.0 * y[g]);
          u[npts + g] = -cos(2.0 * x[g]) * sin(3.0 * y[g]) + 0.3 * z[g];
          u[2 * npts + g] = sin(4.0 * z[g]) * cos(x[g] + y[g]);
          t[g] = cos(1.3 * x[g] + 0.4) * sin(2.1 * y[g] - 0.3) + z[g];
        }
  }

  if (argc > 2) {                                   /* the exact inputs, for the Python comparison */
    FILE* fb = fopen(argv[2], "wb");
    if (!fb || fwrite(h, sizeof(double), (size_t)npts * 7, fb) != (size_t)npts * 7) return 1;
    fclose(fb);
  }

  nkb_ctx* ctx = NULL;
  CHECK(nkb_ctx_create(0, &ctx));
  void* d = NULL;                                   /* device copy (a solver would own these) */
  CHECK(nkb_device_alloc(ctx, (int64_t)sizeof(double) * npts * 7, &d));
  CHECK(nkb_memcpy(d, h, (int64_t)sizeof(double) * npts * 7, 1, NULL));
  const double* dd = (const double*)d;
  CHECK(nkb_mesh_set(ctx, E, 7, dd, dd + npts, dd + 2 * npts, 0, E));
  CHECK(nkb_field_set(ctx, "velocity", 3, dd + 3 * npts, npts));
  CHECK(nkb_field_set(ctx, "temperature", 1, dd + 6 * npts, npts));

  nkb_pipeline p;
  memset(&p, 0, sizeof(p));
  p.n_surfaces = 3;
  p.surfaces[0].kind = NKB_SURF_ISO;
  strcpy(p.surfaces[0].field, "Q");
  p.surfaces[0].value = 0.5;
  p.surfaces[1].kind = NKB_SURF_ISO;
  strcpy(p.surfaces[1].field, "temperature");
  p.surfaces[1].value = 0.6;
  p.surfaces[2].kind = NKB_SURF_SLICE;
  p.surfaces[2].value = 0.75;
  p.surfaces[2].normal[0] = 0.0;
  p.surfaces[2].normal[1] = 1.0;
  p.surfaces[2].normal[2] = 0.0;
  strcpy(p.color_field, "temperature");
  p.width = 160;
  p.height = 120;
  /* top-down orthographic camera: col = 70 x + 10, row = 110 - 70 y, depth = 1 - z / 2 */
  const double view[12] = {70.0, 0.0, 0.0, 10.0, 0.0, -70.0, 0.0, 110.0, 0.0, 0.0, -0.5, 1.0};
  memcpy(p.view, view, sizeof(view));
  p.vmin = NAN;
  p.vmax = NAN;
  p.n_anchors = 0;                                  /* reference DEFAULT_COLORMAP */

  nkb_report rep;
  CHECK(nkb_execute(ctx, &p, &rep, NULL));
  const unsigned char* ppm = NULL;
  int64_t n = 0;
  CHECK(nkb_image_ppm(ctx, &ppm, &n, NULL));
  FILE* f = fopen(out, "wb");
  if (!f || fwrite(ppm, 1, (size_t)n, f) != (size_t)n) {
    fprintf(stderr, "cannot write %s\n", out);
    return 1;
  }
  fclose(f);
  printf("triangles %lld range %.17g %.17g bytes %lld\n", (long long)rep.n_triangles, rep.range[0], rep.range[1],
         (long long)n);
  CHECK(nkb_device_free(ctx, d));
  CHECK(nkb_ctx_destroy(ctx));
  free(h);
  return 0;
}
