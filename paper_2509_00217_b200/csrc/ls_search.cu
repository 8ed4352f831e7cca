// ls_search.cu — standalone launch of the search-loop environment step
// (ls_envstep.cuh); the fused PPO round (ls_policy.cu) calls the same code.
#include <cuda_runtime.h>

#include "ls_envstep.cuh"
#include "ls_kernels.h"

namespace ls {

namespace {

template <bool NEU>
__global__ void env_step_kernel(const uint64_t* __restrict__ tab, const __grid_constant__ TabLayout L,
                                const __grid_constant__ EvalMeta M, const __grid_constant__ ls_search_state S,
                                const int64_t* __restrict__ action, double* reward_out) {
  extern __shared__ int64_t dyn[];
  __shared__ int act[LS_MAX_HEADS];
  for (int h = threadIdx.x; h < M.A; h += blockDim.x) act[h] = (int)action[h];
  int64_t* ev = dyn;
  double* er = reinterpret_cast<double*>(dyn + S.elite_capacity * M.A);
  env_step_block<NEU, true>(tab, L, M, S, act, reward_out, ev, er);
}

}  // namespace

cudaError_t launch_env_step(bool neumaier, const uint64_t* tab, const TabLayout& L, const EvalMeta& M,
                            const ls_search_state& S, const int64_t* action, double* reward_out, cudaStream_t s) {
  const size_t smem = sizeof(int64_t) * (size_t)S.elite_capacity * (M.A + 1);
  if (neumaier) env_step_kernel<true><<<1, 128, smem, s>>>(tab, L, M, S, action, reward_out);
  else env_step_kernel<false><<<1, 128, smem, s>>>(tab, L, M, S, action, reward_out);
  return cudaGetLastError();
}

}  // namespace ls
