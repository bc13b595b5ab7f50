// variants.h -- host-side handles of the k_run / k_run_cluster instantiations.
//
// The eight kernel variants (VAR bit0 fused sub-second batches, bit1 literal Alg.2
// periods, bit2 request-level latency) are instantiated in four translation units
// (run_variants.cu compiled with DILU_VGROUP = 0..3, two variants each) so they compile
// in parallel; dilu_api.cu launches them through these function pointers.
#pragma once
#include <stdint.h>

namespace dilu {
struct Params;
typedef void (*RunFn)(Params, int32_t*, int32_t, int32_t, int32_t, const int32_t*, const int32_t*,
                      int32_t*, int32_t*);
typedef void (*ClusterFn)(Params, int32_t, int32_t, int32_t, const int32_t*, const int32_t*,
                          int32_t*, int32_t*);
// group g holds VAR 2g and 2g + 1
RunFn run_fn_smem_group0(int var);   // DILU_HOT_SMEM=1 units
RunFn run_fn_smem_group1(int var);
RunFn run_fn_smem_group2(int var);
RunFn run_fn_smem_group3(int var);
RunFn run_fn_gmem_group0(int var);   // DILU_HOT_SMEM=0 units
RunFn run_fn_gmem_group1(int var);
RunFn run_fn_gmem_group2(int var);
RunFn run_fn_gmem_group3(int var);
ClusterFn cluster_fn_group0(int var);
ClusterFn cluster_fn_group1(int var);
ClusterFn cluster_fn_group2(int var);
ClusterFn cluster_fn_group3(int var);
}  // namespace dilu
