// chain_offset_move_dyn.cu -- instantiates k_chain<FAM_OFFSET, *, *, false, NZ_DYN> (see chain.cuh).
#include "chain.cuh"

namespace smc {
cudaError_t launch_chain_offset_move_dyn(const Shape& s, int dmax, const GroupDesc* gds, const int* list, const int* prefix,
                                         int n_list, int total_ctas, cudaStream_t st) {
  return launch_chain_fam<FAM_OFFSET, false, NZ_DYN>(s, dmax, gds, list, prefix, n_list, total_ctas, st);
}
}  // namespace smc
