// Gauss-Lobatto-Legendre nodes and the nodal differentiation matrix.
//
// No reference anchor exists (the reference has no spectral elements,
// SPEC.md:8, :169); this is the standard construction used by Nek5000/NekRS
// (nodes = roots of (1-r^2) P_N'(r), D[i][m] = d l_m / dr at r_i).  Built with
// -ffp-contract=off so the CPU oracle (oracle/sem_oracle.c) reproduces every
// bit.  Nodes are symmetrised (x[N-i] = -x[i] exactly) so that D is exactly
// centro-antisymmetric (D[N-i][N-m] == -D[i][m]).
#include <math.h>

#include "nkb_internal.h"

namespace nkb {

static double legendre(int n, double x) {
  double p0 = 1.0, p1 = x;
  if (n == 0) return p0;
  for (int k = 2; k <= n; ++k) {
    double p2 = ((double)(2 * k - 1) * x * p1 - (double)(k - 1) * p0) / (double)k;
    p0 = p1;
    p1 = p2;
  }
  return p1;
}

void gll_nodes_dmat(int N, double* x, double* D) {
  const int np = N + 1;
  for (int i = 0; i < np; ++i) x[i] = -cos(M_PI * (double)i / (double)N);
  // Newton on the Lobatto polynomial (lglnodes recurrence form)
  for (int it = 0; it < 100; ++it) {
    double maxd = 0.0;
    for (int i = 0; i < np; ++i) {
      double pn = legendre(N, x[i]);
      double pm = legendre(N - 1, x[i]);
      double dx = (x[i] * pn - pm) / ((double)np * pn);
      x[i] = x[i] - dx;
      if (fabs(dx) > maxd) maxd = fabs(dx);
    }
    if (maxd < 1e-15) break;
  }
  for (int i = 0; i < np / 2; ++i) {
    double a = 0.5 * (x[N - i] - x[i]);
    x[i] = -a;
    x[N - i] = a;
  }
  x[0] = -1.0;
  x[N] = 1.0;
  if (N % 2 == 0) x[N / 2] = 0.0;

  double LN[32];
  for (int i = 0; i < np; ++i) LN[i] = legendre(N, x[i]);
  for (int i = 0; i < np; ++i)
    for (int m = 0; m < np; ++m)
      D[i * np + m] = (i == m) ? 0.0 : LN[i] / (LN[m] * (x[i] - x[m]));
  D[0] = -(double)(N * (N + 1)) / 4.0;
  D[N * np + N] = (double)(N * (N + 1)) / 4.0;
}

}  // namespace nkb
