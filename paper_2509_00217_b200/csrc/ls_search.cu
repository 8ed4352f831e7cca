// ls_search.cu — standalone launch of the search-loop environment step
// (ls_envstep.cuh); the fused PPO round (ls_policy.cu) calls the same code.
#include <cuda_runtime.h>

#include "ls_envstep.cuh"
#include "ls_kernels.h"

namespace ls {

namespace {

template <bool NEU>
__global__ void env_step_kernel(const uint64_t* __restrict__ tab, const TabLayout L, const EvalMeta M,
                                const ls_search_state S, const int64_t* __restrict__ action, double* reward_out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) env_step<NEU>(tab, L, M, S, action, reward_out);
}

}  // namespace

cudaError_t launch_env_step(bool neumaier, const uint64_t* tab, const TabLayout& L, const EvalMeta& M,
                            const ls_search_state& S, const int64_t* action, double* reward_out, cudaStream_t s) {
  if (neumaier) env_step_kernel<true><<<1, 32, 0, s>>>(tab, L, M, S, action, reward_out);
  else env_step_kernel<false><<<1, 32, 0, s>>>(tab, L, M, S, action, reward_out);
  return cudaGetLastError();
}

}  // namespace ls
