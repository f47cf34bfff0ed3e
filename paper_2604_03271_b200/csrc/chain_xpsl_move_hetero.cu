// chain_xpsl_move_hetero.cu -- instantiates k_chain<FAM_XPSL, *, *, false, NZ_HETERO> (see chain.cuh):
// xps with the Lorentzian basis pinned (eta prior Uniform(0, <= 1e-7)).
#include "chain.cuh"

namespace smc {
cudaError_t launch_chain_xpsl_move_hetero(const Shape& s, int dmax, const GroupDesc* gds, const int* list, const int* prefix,
                                        int n_list, int total_ctas, cudaStream_t st) {
  return launch_chain_fam<FAM_XPSL, false, NZ_HETERO>(s, dmax, gds, list, prefix, n_list, total_ctas, st);
}
}  // namespace smc
