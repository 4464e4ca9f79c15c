// krylov.cu -- dispatch of run_solve to the per-(K, field) instantiations.
#include <cstdio>

#include "krylov.cuh"

namespace mpk {

template <int K, bool CX>
int run_typed(DMat &A, const SolveParams &p, const double *d_b, double *d_x,
              double *d_hist, SolveOut *out, cudaStream_t st, char *errbuf);

int run_solve(DMat &A, const SolveParams &p, const double *d_b, double *d_x,
              double *d_hist, SolveOut *out, cudaStream_t st, char *errbuf) {
  const bool cx = A.cx;
  switch (p.k) {
    case 2:
      return cx ? run_typed<2, true>(A, p, d_b, d_x, d_hist, out, st, errbuf)
                : run_typed<2, false>(A, p, d_b, d_x, d_hist, out, st, errbuf);
    case 3:
      return cx ? run_typed<3, true>(A, p, d_b, d_x, d_hist, out, st, errbuf)
                : run_typed<3, false>(A, p, d_b, d_x, d_hist, out, st, errbuf);
    case 4:
      return cx ? run_typed<4, true>(A, p, d_b, d_x, d_hist, out, st, errbuf)
                : run_typed<4, false>(A, p, d_b, d_x, d_hist, out, st, errbuf);
    default:
      snprintf(errbuf, 256, "unsupported component count k=%d (need 2..4)",
               p.k);
      return 3;
  }
}

}  // namespace mpk
