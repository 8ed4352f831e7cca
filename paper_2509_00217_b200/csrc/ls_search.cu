// ls_search.cu — the sequential callers of the cost model:
//   * env_step_kernel: one SearchEnv.step + EliteBuffer.offer on device state
//     (ls_envstep.cuh; the fused PPO round in ls_policy.cu calls the same code);
//   * eval_one_kernel: the scalar simulate() seam with host-mapped results
//     (no copies, no stream sync: the host spins on a sequence word);
//   * sa_chain_kernel: a whole simulated-annealing chain (baselines.py:112-145)
//     in one launch — mutate, env step, Metropolis accept, step after step.
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

// One strategy (vector passed by value in the launch parameters), verdict
// written straight into host-mapped memory, then the sequence word.
template <bool NEU>
__global__ void eval_one_kernel(const uint64_t* __restrict__ tab, const __grid_constant__ TabLayout L,
                                const __grid_constant__ EvalMeta M, const __grid_constant__ OneArgs a) {
  if (threadIdx.x != 0) return;
  Verdict v;
  double mem;
  score_vector<NEU, true>(tab, L, M, a.vec, v, mem);
  volatile OneOut* o = a.out;
  o->f[0] = v.thr;
  o->f[1] = v.tpot;
  o->f[2] = mem;
  o->f[3] = v.comp;
  o->f[4] = v.comm;
  o->f[5] = v.pipe;
  o->reason = v.reason;
  __threadfence_system();  // the verdict lands before the sequence word
  o->seq = a.seq;
}

// The simulated-annealing chain of baselines.py:112-145 on device state. The
// host pre-draws the chain's randomness in the reference's order (the draws
// do not depend on the chain's decisions): the first vector, per proposal
// the mutated heads and their integers(k - 1) draws, and the acceptance
// uniform; temperatures are the reference's cosine_decay values. Every
// evaluation is SearchEnv.step (reward against the best raw seen strictly
// before, best updated after, log append); acceptance is the Metropolis rule
// u < (delta >= 0 ? 1 : T <= 0 ? 0 : exp(delta / T)).
template <bool NEU>
__global__ void sa_chain_kernel(const uint64_t* __restrict__ tab, const __grid_constant__ TabLayout L,
                                const __grid_constant__ EvalMeta M, const __grid_constant__ ls_sa_plan P) {
  if (threadIdx.x != 0) return;
  const int A = M.A;
  const ls_search_state& S = P.env;
  int cur[LS_MAX_HEADS], cand[LS_MAX_HEADS];
  for (int h = 0; h < A; ++h) cur[h] = P.init[h];
  double best = *S.best_raw, cur_reward = 0.0;
  int64_t pos = *S.log_pos;
  for (int s = 0; s < P.steps && pos < S.log_capacity; ++s) {
    if (s > 0) {
      for (int h = 0; h < A; ++h) cand[h] = cur[h];
      for (int j = 0; j < P.moves; ++j) {  // distinct heads: cand[c] still equals cur[c]
        const int c = P.coords[(s - 1) * P.moves + j], d = P.drawn[(s - 1) * P.moves + j];
        cand[c] = d < cur[c] ? d : d + 1;
      }
    } else {
      for (int h = 0; h < A; ++h) cand[h] = cur[h];
    }
    Verdict v;
    double mem;
    score_vector<NEU, true>(tab, L, M, cand, v, mem);
    const bool valid = v.reason == LS_REASON_NONE;
    const double raw = valid ? v.thr : 0.0;
    const double reward = valid ? S.alpha * raw + S.beta * (raw - best) : S.penalty;
    if (valid && raw > best) best = raw;
    for (int h = 0; h < A; ++h) S.log_vec[pos * A + h] = (uint8_t)cand[h];
    S.log_raw[pos] = raw;
    S.log_reward[pos] = reward;
    S.log_reason[pos] = (uint8_t)v.reason;
    ++pos;
    if (s == 0) {
      cur_reward = reward;
      continue;
    }
    const double delta = reward - cur_reward, T = P.temperature[s - 1];
    const double p = delta >= 0.0 ? 1.0 : (T <= 0.0 ? 0.0 : exp(delta / T));
    if (P.u[s - 1] < p) {
      for (int h = 0; h < A; ++h) cur[h] = cand[h];
      cur_reward = reward;
    }
  }
  *S.best_raw = best;
  *S.log_pos = pos;
}

// A stream waits for another stream's completion signal: one thread polls
// the word (acquire loads, backing off with __nanosleep) until it reaches seq.
// The fallback of ls_stream_wait_signal when cuStreamWaitValue32 is missing
// (LS_WAIT_MEMOP=0 selects it). Gives up after ~10 s (no hang if the signal
// never comes).
__global__ void wait_signal_kernel(const uint32_t* __restrict__ sig, uint32_t seq) {
  unsigned ns = 128;
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(sig) : "memory");
    if ((int32_t)(v - seq) >= 0) return;
    __nanosleep(ns);
    if (ns < 4096) ns *= 2;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 10000000000ull) return;
  }
}

}  // namespace

cudaError_t launch_wait_signal(const uint32_t* sig, uint32_t seq, cudaStream_t s) {
  // the SM this thread spins on keeps the shared-memory carve-out the
  // evaluate kernels need, so their CTAs can still land beside it
  static const bool attr = [] {
    cudaFuncSetAttribute(wait_signal_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                         (int)cudaSharedmemCarveoutMaxShared);
    return true;
  }();
  (void)attr;
  wait_signal_kernel<<<1, 1, 0, s>>>(sig, seq);
  return cudaGetLastError();
}

cudaError_t launch_eval_one(bool neumaier, const uint64_t* tab, const TabLayout& L, const EvalMeta& M,
                            const OneArgs& a, cudaStream_t s) {
  if (neumaier) eval_one_kernel<true><<<1, 32, 0, s>>>(tab, L, M, a);
  else eval_one_kernel<false><<<1, 32, 0, s>>>(tab, L, M, a);
  return cudaGetLastError();
}

cudaError_t launch_sa_chain(bool neumaier, const uint64_t* tab, const TabLayout& L, const EvalMeta& M,
                            const ls_sa_plan& p, cudaStream_t s) {
  if (neumaier) sa_chain_kernel<true><<<1, 32, 0, s>>>(tab, L, M, p);
  else sa_chain_kernel<false><<<1, 32, 0, s>>>(tab, L, M, p);
  return cudaGetLastError();
}

cudaError_t launch_env_step(bool neumaier, const uint64_t* tab, const TabLayout& L, const EvalMeta& M,
                            const ls_search_state& S, const int64_t* action, double* reward_out, cudaStream_t s) {
  const size_t smem = sizeof(int64_t) * (size_t)S.elite_capacity * (M.A + 1);
  if (neumaier) env_step_kernel<true><<<1, 128, smem, s>>>(tab, L, M, S, action, reward_out);
  else env_step_kernel<false><<<1, 128, smem, s>>>(tab, L, M, S, action, reward_out);
  return cudaGetLastError();
}

}  // namespace ls
