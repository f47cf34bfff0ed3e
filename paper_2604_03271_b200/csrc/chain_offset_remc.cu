// chain_offset_remc.cu -- instantiates k_chain<FAM_OFFSET, *, *, false, NZ_DYN, REMC = true> (see chain.cuh):
// replica-exchange sweeps of the conjugate test family (the closed-form check of the REMC comparator).
#include "chain.cuh"

namespace smc {
cudaError_t launch_chain_offset_remc(const Shape& s, int dmax, const GroupDesc* gds, const int* list,
                                     const int* prefix, int n_list, int total_ctas, cudaStream_t st) {
  return launch_chain_fam<FAM_OFFSET, false, NZ_DYN, true>(s, dmax, gds, list, prefix, n_list, total_ctas, st);
}
}  // namespace smc
