// ls_kernels.h — internal launch interface between the C ABI (ls_capi.cu)
// and the kernels. Not part of the public ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "ls_tables.cuh"

namespace ls {

struct EvalArgs {
  const uint8_t* planes;
  const uint64_t* words;  // packed candidate words (GEN_WORDS) instead of planes
  int64_t n;
  int64_t stride;
  uint8_t* reason;
  double *thr, *tpot, *mem, *comp, *comm, *pipe;
  bool sparse_thr;  // throughput written for gate survivors only (compact results read it where reason == 0)
};

struct LaunchPlan {
  bool tma;        // TMA-ring two-pass kernel (aligned planes, A <= 16)
  bool smem_gate;  // gate tables staged into shared memory
  int64_t max_blocks;
  bool sweep_fits = false;  // ls_sweep: sweep_kernel's tables fit in shared memory (else eval_ws_kernel)
  bool pdl = false;         // fused evaluate + elite: programmatic dependent launch
  const float* tabf = nullptr;  // ls_sweep fp32 fast mode: the fp32 copy of the tables
};

cudaError_t build_tables(const ls_workload_desc& d, const TabLayout& L, uint64_t* out, cudaStream_t stream);
// Layer-sum memo (ls_memo.cu): entries and builder.
int64_t memo_entries(const TabLayout& L);
cudaError_t build_memo(bool neumaier, const uint64_t* tab, const TabLayout& L, const EvalMeta& M, double2* memo,
                       cudaStream_t s);

// Fused evaluate + top-k by raw (eval_ws_kernel<..., TOPK>): every CTA emits
// its elite list to part[blockIdx.x * k ..] / part_counts[blockIdx.x]; the
// last CTA to finish merges them into out / count_out.
struct TopkArgs {
  int k;
  int64_t index_base;
  ls_elite_rec* part;
  int32_t* part_counts;
  unsigned long long* floor;  // device word, zeroed before launch
  unsigned int* done;         // CTAs finished (zeroed before launch): the last one merges every CTA list
  unsigned int* tile_ctr;     // dynamic tile claims after each CTA's first (zero before launch), or null
  uint32_t* signal;           // optional: the last CTA stores seq here (release) once out / count_out are written
  uint32_t seq;
  uint8_t* const* sinks;      // optional (device array): the last CTA copies the elite block (k records + a
  int nsinks;                 // count | seq << 32 word at row k) to each sink, peers' memory included
  ls_elite_rec* out;          // final top-k and its count
  int32_t* count_out;
};

// Candidate sources of eval_ws_kernel.
enum : int { GEN_PLANES = 0, GEN_UNIFORM = 1, GEN_ENUM = 2, GEN_ENUM_ADMISSIBLE = 3, GEN_WORDS = 4 };

// Packed candidate word (A <= 16): axis head h in bits [2(h-4), 2(h-4)+2)
// (= the Y word), and from bit 24 the coarse rank ((t*ne + e)*np + p)*nb + b.
struct PackMeta {
  uint32_t axis_mask;  // low 2(A-4) bits
  uint32_t ncoarse;    // nt * ne * np * nb
  uint32_t nt, ne, np, nb;
  uint64_t m_e, m_p, m_b;  // ceil(2^64 / d) (exact floor division of ranks < 2^24)
};
PackMeta pack_meta(const ls_workload_desc& d);

// On-device candidate stream: index -> (coarse rank, axis rank) -> decoded
// candidate. Axis ranks split into a high and a low group of axis heads whose
// packed Y fields come from two small tables.
struct GenMeta {
  int64_t start;  // stream index of the launch's first candidate
  uint64_t seed;
  uint64_t coarse_size, axis_size, lo_size;
  uint64_t m_axis, m_lo, m_b, m_p, m_e;  // ceil(2^64 / d) for the divisors above
  uint64_t nb, np, ne;
  const uint32_t* hi_tab;  // [axis_size / lo_size] packed Y of the high group
  const uint32_t* lo_tab;  // [lo_size] packed Y of the low group
  PackMeta pk;             // GEN_WORDS field layout
};

bool tma_eligible(const EvalArgs& a, int A);
cudaError_t launch_sweep(const LaunchPlan& lp, bool neumaier, int mode, const uint64_t* tab, const TabLayout& L,
                         const EvalMeta& M, int64_t n, const TopkArgs& tk, const GenMeta& gm, cudaStream_t s);
cudaError_t launch_generate(int mode, const GenMeta& gm, int64_t n, int A, uint8_t* planes, int64_t stride,
                            cudaStream_t s);
cudaError_t launch_pack(const PackMeta& pk, int A, const uint8_t* planes, int64_t stride, int64_t n, uint64_t* words,
                        cudaStream_t s);
int64_t ws_grid(const LaunchPlan& lp, int64_t n, int mode);  // CTAs of one eval_ws_kernel launch
int64_t sweep_grid(const LaunchPlan& lp, int64_t n, int mode);         // CTAs of one sweep_kernel launch (ls_sweep)
int sweep_ctas_per_sm();
size_t sweep_smem_bytes(const TabLayout& L, uint64_t hi_size, uint64_t lo_size, int mode, bool f32);
cudaError_t build_tables_f32(const uint64_t* tab, int words, float* out, cudaStream_t s);
size_t prepare_sweep_kernels(size_t optin);  // -> dynamic shared memory budget of sweep_kernel
int fused_k_max();
cudaError_t launch_evaluate_topk(const LaunchPlan& lp, bool neumaier, const uint64_t* tab, const TabLayout& L,
                                 const EvalMeta& M, const EvalArgs& a, const TopkArgs& tk, cudaStream_t s,
                                 const PackMeta* pk = nullptr);
cudaError_t prepare_eval_kernels(const TabLayout& L, int A, bool smem_gate);
int tma_blocks_per_sm(const TabLayout& L, int A, bool smem_gate);
int generic_blocks_per_sm();
size_t tma_smem_bytes(const TabLayout& L, int A, bool smem_gate);
size_t tma_smem_budget(const cudaDeviceProp& prop);  // dynamic smem one eval_ws_kernel CTA may use
cudaError_t launch_evaluate(const LaunchPlan& lp, bool neumaier, const uint64_t* tab, const TabLayout& L,
                            const EvalMeta& M, const EvalArgs& a, cudaStream_t s, const PackMeta* pk = nullptr);

// Reward scan (ls_select.cu)
size_t scan_scratch_bytes(int64_t n);
cudaError_t launch_reward_scan(const uint8_t* reason, const double* thr, int64_t n, double b0, double alpha,
                               double beta, double penalty, double* reward, double* best_out, void* scratch,
                               int num_sms, cudaStream_t s);

// Valid-raw compaction (ls_select.cu): raws of the reason == 0 candidates in
// index order -> out[0..count), *count_out = count (device int64).
size_t compact_scratch_bytes(int64_t n);
cudaError_t launch_valid_compact(const uint8_t* reason, const double* thr, int64_t n, double* out, int64_t* count_out,
                                 void* scratch, cudaStream_t s);

// Top-k (ls_select.cu)
struct TopkMeta {
  int A;
  int64_t code_stride[LS_MAX_HEADS];
};
size_t topk_scratch_bytes(int64_t n, int k, int num_sms);
cudaError_t launch_topk(const TopkMeta& tm, const uint8_t* planes, int64_t stride, const uint8_t* reason,
                        const double* thr, const double* key, int64_t n, int k, int64_t index_base,
                        ls_elite_rec* out, int32_t* count_out, void* scratch, int num_sms, cudaStream_t s);
cudaError_t launch_topk_merge_steps(const ls_elite_rec* blocks, int world, int steps, int k, ls_elite_rec* out,
                                    int32_t* counts_out, cudaStream_t s, int rank_stride = 0, uint32_t seq0 = 0,
                                    int32_t* err = nullptr);
cudaError_t launch_topk_merge(const ls_elite_rec* recs, const int32_t* counts, int m, int k_in, int k,
                              const unsigned long long* floor,
                              ls_elite_rec* out, int32_t* count_out, cudaStream_t s);

// Scalar seam (ls_search.cu): one vector in the launch parameters, the
// verdict in host-mapped memory followed by the sequence word.
struct OneOut {
  double f[6];  // throughput, tpot, memory, compute, comm, pipeline
  uint32_t reason;
  uint32_t seq;
};
struct OneArgs {
  uint8_t vec[LS_MAX_HEADS];
  OneOut* out;
  uint32_t seq;
};
cudaError_t launch_eval_one(bool neumaier, const uint64_t* tab, const TabLayout& L, const EvalMeta& M,
                            const OneArgs& a, cudaStream_t s);
cudaError_t launch_wait_signal(const uint32_t* sig, uint32_t seq, cudaStream_t s);
cudaError_t launch_sa_chain(bool neumaier, const uint64_t* tab, const TabLayout& L, const EvalMeta& M,
                            const ls_sa_plan& p, cudaStream_t s);

// Search-loop environment step (ls_search.cu)
cudaError_t launch_env_step(bool neumaier, const uint64_t* tab, const TabLayout& L, const EvalMeta& M,
                            const ls_search_state& S, const int64_t* action, double* reward_out, cudaStream_t s);

// Fused PPO rounds (ls_policy.cu)
struct PpoCtx {
  const uint64_t* tab;
  TabLayout L;
  EvalMeta M;
  bool neumaier;
};
bool ppo_layout(const ls_policy_dims& D, ls_policy_layout* out);
size_t ppo_workspace_bytes(const ls_policy_dims& D);
cudaError_t ppo_prime(const ls_ppo_plan& p, const PpoCtx& c, cudaStream_t s);
cudaError_t ppo_round(const ls_ppo_plan& p, const PpoCtx& c, int n, cudaStream_t s);
cudaError_t ppo_forward(const ls_ppo_plan& p, const PpoCtx& c, int n, double* logp, double* value, cudaStream_t s);
cudaError_t ppo_update(const ls_ppo_plan& p, const PpoCtx& c, int n, cudaStream_t s);

}  // namespace ls
