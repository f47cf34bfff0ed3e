// chain_gm_remc.cu -- instantiates k_chain<FAM_GM, *, *, false, NZ_DYN, REMC = true> (see chain.cuh):
// one replica-exchange sweep per replica (the REMC comparator, remc.cpp:125-133).
#include "chain.cuh"

namespace smc {
cudaError_t launch_chain_gm_remc(const Shape& s, int dmax, const GroupDesc* gds, const int* list, const int* prefix,
                                   int n_list, int total_ctas, cudaStream_t st) {
  return launch_chain_fam<FAM_GM, false, NZ_DYN, true>(s, dmax, gds, list, prefix, n_list, total_ctas, st);
}
}  // namespace smc
