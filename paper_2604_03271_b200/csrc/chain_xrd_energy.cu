// chain_xrd_energy.cu -- instantiates k_chain<FAM_XRD, *, *, true, NZ_DYN> (see chain.cuh).
#include "chain.cuh"

namespace smc {
cudaError_t launch_chain_xrd_energy(const Shape& s, int dmax, const GroupDesc* gds, const int* list,
                                    const int* prefix, int n_list, int total_ctas, cudaStream_t st) {
  return launch_chain_fam<FAM_XRD, true, NZ_DYN>(s, dmax, gds, list, prefix, n_list, total_ctas, st);
}
}  // namespace smc
