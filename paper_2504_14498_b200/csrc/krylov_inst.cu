// krylov_inst.cu -- one (K, complex) instantiation of the device solver per
// object file (compiled once per -DMPK_K/-DMPK_CX pair, in parallel).
#include "krylov_impl.cuh"

namespace mpk {
template int run_typed<MPK_K, MPK_CX>(DMat &, const SolveParams &,
                                      const double *, double *, double *,
                                      SolveOut *, cudaStream_t, char *);
}  // namespace mpk
