// ls_envstep.cuh — one environment step of a learning search (device code).
//
// Fuses what the reference does in Python per sampled action:
//   SearchEnv.step (env.py:152-180): score the strategy, Eq.-1 reward
//     alpha*raw + beta*(raw - best) against the best raw seen strictly
//     before, flat penalty when invalid, best update after the reward,
//     eval-log append;
//   EliteBuffer.offer (policy.py:86-102), valid strategies only: reject a
//     duplicate vector, reject reward <= min when full, else insert after
//     every entry with reward >= the newcomer's (the reference's stable sort).
// Called by ONE thread: the step is strictly sequential (the next action's
// observation depends on this step's elite update).
#pragma once
#include <math.h>

#include "ls_evaluate.cuh"

namespace ls {

// Score one index vector (A indices, each checked against its head size like
// decode_strategy, strategy.py:245-263): gate() then full_path() — the same
// code as the batched kernels. mem: memory_bytes as SimResult carries it.
template <bool NEU, bool LDG, typename V>
__device__ __forceinline__ void score_vector(const uint64_t* __restrict__ tab, const TabLayout& L,
                                             const EvalMeta& M, const V* vec, Verdict& v, double& mem) {
  uint32_t bad = 0, Y = 0;
  int idx[4] = {0, 0, 0, 0};
  for (int h = 0; h < M.A; ++h) {
    const int x = (int)vec[h];
    bad |= (x < 0 || x >= (int)M.head_size[h]) ? 1u : 0u;
    const uint32_t byte = (uint32_t)(x & 0xff);
    if (h < 4) {
      idx[h] = (int)byte;
    } else {
      const int slot = M.head_slot[h];
      if (slot >= 0) Y |= (byte & 3u) << (2 * slot);
    }
  }
  v.thr = v.tpot = v.comp = v.comm = v.pipe = 0.0;
  mem = 0.0;
  if (bad) {
    v.reason = LS_REASON_DECODE_ERROR;
    return;
  }
  Decoded c;
  c.t = idx[0];
  c.e = idx[1];
  c.p = idx[2];
  c.b = idx[3];
  c.Y = Y;
  v.reason = gate(tab, L, M, c, mem);
  if (v.reason == LS_REASON_NONE) full_path<NEU, LDG>(tab, L, M, c, v);
}

// Thread-0 core. ev/er: the elite buffer (shared-memory copy); returns true
// when the buffer changed. tab is global (LDG) or a shared-memory copy.
template <bool NEU, bool LDG>
__device__ __noinline__ bool env_step_core(const uint64_t* __restrict__ tab, const TabLayout& L, const EvalMeta& M,
                                           const ls_search_state& S, const int* action, double* reward_out,
                                           int64_t* ev, double* er) {
  const int A = M.A;
  const int64_t pos = *S.log_pos;
  const double best = *S.best_raw;
  if (pos < 0 || pos >= S.log_capacity) {  // budget guard: nothing scored
    *reward_out = __longlong_as_double(0x7ff8000000000000LL);
    return false;
  }
  Verdict v;
  double mem;
  score_vector<NEU, LDG>(tab, L, M, action, v, mem);
  const bool bad = v.reason == LS_REASON_DECODE_ERROR;
  const bool valid = v.reason == LS_REASON_NONE;
  double raw = 0.0, reward;
  if (valid) {
    raw = v.thr;
    reward = S.alpha * raw + S.beta * (raw - best);
  } else {
    reward = bad ? __longlong_as_double(0x7ff8000000000000LL) : S.penalty;
  }
  if (valid && raw > best) *S.best_raw = raw;
  // eval-log append
  for (int h = 0; h < A; ++h) S.log_vec[pos * A + h] = (uint8_t)(action[h] & 0xff);
  S.log_raw[pos] = raw;
  S.log_reward[pos] = reward;
  S.log_reason[pos] = (uint8_t)v.reason;
  *S.log_pos = pos + 1;
  *reward_out = reward;
  if (!valid) return false;

  // EliteBuffer.offer: entries are contiguous from slot 0, best first
  const int T = S.elite_capacity;
  int cnt = 0;
  while (cnt < T && !isinf(er[cnt])) ++cnt;
  for (int i = 0; i < cnt; ++i) {
    bool same = true;
    for (int h = 0; h < A; ++h) same &= ev[i * A + h] == (int64_t)action[h];
    if (same) return false;  // duplicate vector
  }
  if (cnt >= T) {
    if (reward <= er[T - 1]) return false;
    cnt = T - 1;  // the last entry is evicted
  }
  int at = cnt;  // stable: after every entry with reward >= the newcomer's
  while (at > 0 && er[at - 1] < reward) {
    er[at] = er[at - 1];
    for (int h = 0; h < A; ++h) ev[at * A + h] = ev[(at - 1) * A + h];
    --at;
  }
  er[at] = reward;
  for (int h = 0; h < A; ++h) ev[at * A + h] = action[h];
  return true;
}

// Block-cooperative step: every thread of the block must call it. The elite
// buffer is staged through shared memory (ev: >= T*A, er: >= T) so the
// sequential part runs on on-chip data; action: A indices visible to thread 0.
template <bool NEU, bool LDG>
__device__ __forceinline__ void env_step_block(const uint64_t* __restrict__ tab, const TabLayout& L,
                                               const EvalMeta& M, const ls_search_state& S, const int* action,
                                               double* reward_out, int64_t* ev, double* er) {
  __shared__ int changed;
  const int T = S.elite_capacity, TA = T * M.A;
  for (int i = threadIdx.x; i < TA; i += blockDim.x) ev[i] = S.elite_vec[i];
  for (int i = threadIdx.x; i < T; i += blockDim.x) er[i] = S.elite_reward[i];
  __syncthreads();
  if (threadIdx.x == 0) changed = env_step_core<NEU, LDG>(tab, L, M, S, action, reward_out, ev, er) ? 1 : 0;
  __syncthreads();
  if (changed) {
    for (int i = threadIdx.x; i < TA; i += blockDim.x) S.elite_vec[i] = ev[i];
    for (int i = threadIdx.x; i < T; i += blockDim.x) S.elite_reward[i] = er[i];
  }
}

}  // namespace ls
