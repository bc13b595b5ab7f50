// run_variants.cu -- instantiates two of the eight k_run / k_run_cluster variants
// (VAR = 2*DILU_VGROUP and 2*DILU_VGROUP + 1); see variants.h.  Compiled twice per group:
// DILU_HOT_SMEM=1 for the shared-memory kernels (hot pointers asserted shared, see
// hot_view in sim_kernel.cuh), DILU_HOT_SMEM=0 for the global-memory and cluster kernels.
#define DILU_VARIANT_TU
#include "sim_kernel.cuh"
#include "variants.h"

#ifndef DILU_VGROUP
#error "compile with -DDILU_VGROUP=0..3"
#endif
#define DILU_CAT2(a, b) a##b
#define DILU_CAT(a, b) DILU_CAT2(a, b)

namespace dilu {

#if DILU_HOT_SMEM   // hot region in shared memory: k_run<true, *> only
RunFn DILU_CAT(run_fn_smem_group, DILU_VGROUP)(int var) {
  constexpr int V0 = 2 * DILU_VGROUP, V1 = V0 + 1;
  return (var & 1) ? k_run<true, V1> : k_run<true, V0>;
}
#else               // hot region in global memory: k_run<false, *> and the cluster engine
RunFn DILU_CAT(run_fn_gmem_group, DILU_VGROUP)(int var) {
  constexpr int V0 = 2 * DILU_VGROUP, V1 = V0 + 1;
  return (var & 1) ? k_run<false, V1> : k_run<false, V0>;
}

ClusterFn DILU_CAT(cluster_fn_group, DILU_VGROUP)(int var) {
  constexpr int V0 = 2 * DILU_VGROUP, V1 = V0 + 1;
  return (var & 1) ? k_run_cluster<V1> : k_run_cluster<V0>;
}
#endif

}  // namespace dilu
