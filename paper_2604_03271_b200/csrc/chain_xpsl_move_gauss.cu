// chain_xpsl_move_gauss.cu -- instantiates k_chain<FAM_XPSL, *, *, false, NZ_GAUSS> (see chain.cuh):
// xps with the Lorentzian basis pinned (eta prior Uniform(0, <= 1e-7)).
#include "chain.cuh"

namespace smc {
cudaError_t launch_chain_xpsl_move_gauss(const Shape& s, int dmax, const GroupDesc* gds, const int* list, const int* prefix,
                                        int n_list, int total_ctas, cudaStream_t st) {
  return launch_chain_fam<FAM_XPSL, false, NZ_GAUSS>(s, dmax, gds, list, prefix, n_list, total_ctas, st);
}
}  // namespace smc
