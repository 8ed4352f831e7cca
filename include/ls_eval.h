/*
 * ls_eval.h — C ABI of the B200 batched strategy evaluator (libls_eval.so).
 *
 * Drop-in boundary for the Learn-to-Shard cost model. The reference has no
 * native code and no batched API: every caller scores one candidate at a
 * time through
 *
 *     SearchEnv.evaluate_raw(strategy) -> SimResult
 *         pkg/src/shardsearch/env.py:140-150   (the seam, called from step :152-180)
 *     simulate(SimRequest) -> SimResult
 *         pkg/src/shardsearch/simulator.py:239-341
 *
 * This header is what a binding for that seam links against (ctypes stub in
 * INTEGRATION.md). Everything is POD: plain pointers, sizes and status codes;
 * no C++ exceptions or torch types cross it. Device buffers are owned by the
 * caller; a context owns only its per-workload tables. All device entry points
 * are stream-ordered and asynchronous; a context is immutable after creation,
 * so concurrent calls on distinct streams are safe.
 *
 * Candidate wire format: the reference's flat index vector
 * (strategy.py:220-263, encode_strategy / decode_strategy), stored
 * struct-of-arrays: head h of candidate i is planes[h * plane_stride + i]
 * (one uint8 per head). Heads 0..3 index the tp/ep/pp/batch domains, heads
 * 4.. are per-operator axis choices (AxisChoice, strategy.py:17-28).
 */
#ifndef LS_EVAL_H
#define LS_EVAL_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LS_ABI_VERSION 1u
#define LS_MAX_DOMAIN 64 /* entries per tp/ep/pp/batch domain */
#define LS_MAX_HEADS 64  /* max vector length A */
#define LS_NUM_OPS 12    /* canonical fused operators, strategy.py:65-78 */

/* Status codes returned by every entry point. */
enum {
  LS_OK = 0,
  LS_ERR_INVALID_ARGUMENT = 1,
  LS_ERR_CUDA = 2,
  LS_ERR_OUT_OF_MEMORY = 3,
  LS_ERR_UNSUPPORTED = 4
};

/* Verdict codes, in InvalidReason declaration order (simulator.py:48-53).
 * LS_REASON_DECODE_ERROR marks a vector decode_strategy would reject with
 * DecodingError (strategy.py:245-254); the Python facade raises it. */
enum {
  LS_REASON_NONE = 0,
  LS_REASON_OVER_DEVICE_BUDGET = 1,
  LS_REASON_LAYOUT_ERROR = 2,
  LS_REASON_OOM = 3,
  LS_REASON_SLO_VIOLATION = 4,
  LS_REASON_DECODE_ERROR = 255
};

/* Canonical fused operators, in _CANONICAL_OPS order (strategy.py:65-78). */
enum {
  LS_OP_EMBEDDING = 0,
  LS_OP_QKV_PROJ = 1,
  LS_OP_KV_CACHE_IO = 2,
  LS_OP_ATTN_CORE = 3,
  LS_OP_ATTN_OUT_PROJ = 4,
  LS_OP_ROUTER_GATE = 5,
  LS_OP_EXPERT_FFN1 = 6,
  LS_OP_EXPERT_FFN2 = 7,
  LS_OP_SHARED_FFN1 = 8,
  LS_OP_SHARED_FFN2 = 9,
  LS_OP_FINAL_NORM = 10,
  LS_OP_LM_HEAD = 11
};

/* Float summation order of _plan_times (simulator.py:232-235): Python's
 * builtin sum() is a naive left fold up to 3.11 and Neumaier-compensated
 * from 3.12 on. The evaluator reproduces whichever the caller names. */
enum { LS_SUM_NAIVE = 0, LS_SUM_NEUMAIER = 1 };

/* Top-k keys. */
enum {
  LS_KEY_RAW = 0,   /* raw throughput of valid candidates (build_report by_raw, ppo.py:441-447) */
  LS_KEY_REWARD = 1 /* shaped reward of valid candidates (EliteBuffer.offer, policy.py:86-102) */
};

/* One workload: ModelSpec + HardwareSpec + SimRequest knobs + ActionSpaceSpec. */
typedef struct ls_workload_desc {
  uint32_t abi_version; /* = LS_ABI_VERSION */
  uint32_t sum_mode;    /* LS_SUM_NAIVE / LS_SUM_NEUMAIER */
  /* ModelSpec, model.py:13-36 */
  int64_t num_layers, hidden_dim, num_heads, head_dim, num_kv_heads, ffn_dim;
  int64_t num_experts, experts_per_token, vocab_size, dtype_bytes;
  int32_t has_shared_expert;
  int32_t reserved0;
  /* HardwareSpec, model.py:74-93 */
  double peak_flops, hbm_bandwidth, hbm_capacity, intra_node_bw, inter_node_bw;
  int64_t node_size, device_budget;
  double kernel_overhead, per_collective_latency;
  /* SimRequest, simulator.py:56-73 */
  int64_t context_len;
  double slo_tpot;
  /* ActionSpaceSpec, strategy.py:106-175: domains in head order tp, ep, pp, batch */
  int32_t domain_len[4];
  int64_t domain[4][LS_MAX_DOMAIN];
  int32_t vector_length; /* A = 4 + len(op_names) */
  /* Axis source per canonical op (Strategy.axis_of, strategy.py:209-214):
   * op_head[k] >= 4 is the head index that controls op k; -1 means the op
   * is not controlled and takes op_pinned[k] (pins, default UNSHARDED). */
  int8_t op_head[LS_NUM_OPS];
  int8_t op_pinned[LS_NUM_OPS];
} ls_workload_desc;

/* Per-candidate results, struct-of-arrays. reason is required; any other
 * pointer may be NULL to skip that field. Field conventions follow SimResult
 * (simulator.py:89-97, :246-255): over-budget / layout-error / decode-error
 * leave every number 0; OOM sets only memory_bytes; SLO sets tpot, memory and
 * the breakdown with throughput 0. */
typedef struct ls_result_soa {
  uint8_t* reason;
  double* throughput; /* tokens/s/chip, the raw objective */
  double* tpot_s;
  double* memory_bytes;
  double* compute_s;
  double* comm_s;
  double* pipeline_s;
} ls_result_soa;

/* One elite / top-k record. code is the candidate's mixed-radix rank over the
 * head sizes (head 0 most significant), i.e. its index in
 * itertools.product(*map(range, head_sizes)) order; index is the candidate's
 * global position in the evaluated stream. */
typedef struct ls_elite_rec {
  double key;    /* raw or reward, per key kind */
  double raw;    /* raw throughput */
  int64_t index; /* global candidate index (ties: smaller wins) */
  uint64_t code; /* mixed-radix vector code (dedupe + decode) */
} ls_elite_rec;

typedef struct ls_ctx ls_ctx;

/* Last error message of the calling thread ("" when none). */
const char* ls_last_error(void);
uint32_t ls_abi_version(void);

/* Validate the workload, build its per-workload tables on `device`. */
int ls_ctx_create(const ls_workload_desc* desc, int device, ls_ctx** out);
int ls_ctx_destroy(ls_ctx* ctx);
/* Size of the encodable space (product of head sizes); 0 if it overflows. */
uint64_t ls_space_size(const ls_ctx* ctx);

/* Arithmetic of the on-device sweeps (ls_sweep): LS_PREC_FP64 (default) is
 * bit-exact; LS_PREC_FP32 is the fp32 fast mode — the plan walk on an fp32
 * copy of the time tables with plain fp32 sums and division, raw throughput
 * within 1e-5 relative of the reference's (measured ~2e-6 worst), every verdict
 * reason exact (integer and memory gates in fp64; the SLO gate re-decided in
 * fp64 within 1e-5 of the boundary). Elite order may differ from fp64 mode
 * only among candidates whose raws agree to ~1e-5. Other entry points are
 * always fp64. */
enum { LS_PREC_FP64 = 0, LS_PREC_FP32 = 1 };
int ls_set_precision(ls_ctx* ctx, int precision);

/* Leave `sms` SMs free of the persistent evaluate kernels (default 0), so a
 * concurrent stream (e.g. the cross-rank elite all-gather + merge of the
 * previous step) runs beside them instead of delaying one of their CTAs. */
int ls_reserve_sms(ls_ctx* ctx, int sms);

/* Score n candidates already resident on the device (SoA planes). */
int ls_evaluate(ls_ctx* ctx, const uint8_t* planes, int64_t n, int64_t plane_stride,
                const ls_result_soa* out, void* stream);

/* Same, from and to HOST memory: chunked H2D copy -> evaluate -> D2H copy,
 * double-buffered across two internal streams; returns when results are in
 * host memory. Host buffers should be pinned (ls_host_alloc) for full speed. */
int ls_evaluate_host(ls_ctx* ctx, const uint8_t* host_planes, int64_t n, int64_t plane_stride,
                     const ls_result_soa* host_out);

/* Packed candidates (vectors of <= 16 heads): one uint64 word per candidate,
 *   word = Y | crank << 24
 * Y: axis head h (4 <= h < A) in bits [2(h-4), 2(h-4)+2); crank: the coarse
 * rank ((t*ne + e)*np + p)*nb + b over the tp/ep/pp/batch domain indices.
 * 8 B per candidate instead of A bytes of planes, and the coarse rank
 * indexes the gate table directly. Malformed words (bits above 24 + 24, an
 * axis field of 3, a rank past the coarse space, bits above head A) evaluate
 * to LS_REASON_DECODE_ERROR, like out-of-range plane bytes.
 * ls_packed_layout reports the rank's shift (24) and the coarse space size. */
int ls_packed_layout(ls_ctx* ctx, int32_t* coarse_shift, int64_t* coarse_size);
int ls_pack(ls_ctx* ctx, const uint8_t* planes, int64_t plane_stride, int64_t n, uint64_t* words, void* stream);
int ls_evaluate_packed(ls_ctx* ctx, const uint64_t* words, int64_t n, const ls_result_soa* out, void* stream);
int ls_evaluate_host_packed(ls_ctx* ctx, const uint64_t* host_words, int64_t n, const ls_result_soa* host_out);

/* Compact host results: the reason byte of every candidate plus the raw
 * throughput of the VALID ones (reason 0) only, in index order — all that
 * SearchEnv.step consumes (env.py:165-172; raw is 0 for every invalid
 * candidate, and the valid positions are the zero reason bytes). About 1 B
 * per candidate comes back instead of 9. Input `format`:
 *   LS_HOST_PLANES  A uint8 planes plane_stride apart (the reference's index
 *                   vectors, SoA), copied as they are (A B/candidate over
 *                   PCIe); with LS_HOST_PACK=1 in the environment at context
 *                   creation they are instead packed into 8-byte candidate
 *                   words on host worker threads inside the call (chunk by
 *                   chunk, beside the copies and kernels of earlier chunks),
 *                   which wins only when the host has cores to spare;
 *   LS_HOST_WORDS   packed candidate words, as ls_evaluate_packed takes them.
 * valid_raw holds up to `capacity` doubles; *valid_count receives the number
 * of valid candidates (LS_ERR_INVALID_ARGUMENT when it exceeds capacity).
 * Blocking; pinned host buffers (ls_host_alloc) copy fastest. */
enum { LS_HOST_PLANES = 0, LS_HOST_WORDS = 1 };
int ls_evaluate_host_compact(ls_ctx* ctx, int format, const void* host_in, int64_t n, int64_t plane_stride,
                             uint8_t* reason_out, double* valid_raw, int64_t capacity, int64_t* valid_count);

/* Pinned host memory helpers for ls_evaluate_host callers. */
int ls_host_alloc(size_t bytes, void** out);
int ls_host_free(void* ptr);

/* Reward shaping of SearchEnv.step (env.py:159-164, :178-179) over a batch:
 *   b_i = max(b0, max{raw_j : j < i, valid_j})     (exclusive running best)
 *   reward_i = alpha*raw_i + beta*(raw_i - b_i)  if valid_i else penalty
 * raw_i is throughput for valid candidates and 0 otherwise. best_out (device,
 * optional) receives max(b0, all valid raw), the env's best_raw afterwards.
 * scratch must hold ls_scan_scratch_bytes(n) bytes of device memory. */
size_t ls_scan_scratch_bytes(int64_t n);
int ls_reward_scan(ls_ctx* ctx, const uint8_t* reason, const double* throughput, int64_t n,
                   double b0, double alpha, double beta, double penalty, double* reward_out,
                   double* best_out, void* scratch, void* stream);

/* Top-k of valid candidates by (key desc, index asc) over DISTINCT vectors
 * (first occurrence kept), written best first to out[0..k) on the device;
 * count_out (device int32) receives the number of records filled (<= k).
 * key is `throughput` for LS_KEY_RAW or the reward array for LS_KEY_REWARD.
 * index_base is added to local positions (global stream offset). planes are
 * the candidate vectors (for the dedupe code). scratch must hold
 * ls_topk_scratch_bytes(n, k) bytes. k <= 64. */
size_t ls_topk_scratch_bytes(int64_t n, int k);
int ls_topk(ls_ctx* ctx, const uint8_t* planes, int64_t plane_stride, const uint8_t* reason,
            const double* throughput, const double* key, int64_t n, int k, int64_t index_base,
            ls_elite_rec* out, int32_t* count_out, void* scratch, void* stream);

/* Fused evaluate + elite (the sweep path): score n device-resident
 * candidates and reduce the valid ones to the top-k by RAW throughput over
 * distinct vectors (LS_KEY_RAW semantics of ls_topk) in the same pass.
 * `out` may be NULL (or out->reason NULL): then no per-candidate verdicts
 * are written at all (16 B/candidate of HBM traffic). k <= 32. scratch must
 * hold ls_evaluate_topk_scratch_bytes(ctx, n, k) bytes of device memory,
 * zero-filled before its first use (every call leaves its sync words zero,
 * so one call is one kernel launch); calls that may run concurrently (other
 * streams) need distinct scratch buffers.
 * Unaligned planes or vectors longer than 16 heads need `out` with reason and
 * throughput (evaluated first, then reduced by ls_topk). */
size_t ls_evaluate_topk_scratch_bytes(const ls_ctx* ctx, int64_t n, int k);
int ls_evaluate_topk(ls_ctx* ctx, const uint8_t* planes, int64_t n, int64_t plane_stride,
                     const ls_result_soa* out, int k, int64_t index_base, ls_elite_rec* topk_out,
                     int32_t* count_out, void* scratch, void* stream);

/* On-device candidate streams: the candidates are generated in registers,
 * never read from memory (0 B/candidate of input traffic).
 *   LS_GEN_UNIFORM          i.i.d. uniform over every head (the random-walk
 *                           proposal, baselines.py:50-54), a counter-based
 *                           function of (seed, stream index);
 *   LS_GEN_ENUM             stream index i -> the i-th vector of
 *                           itertools.product over all head domains (the
 *                           order of the reference's exhaustive sweeps);
 *   LS_GEN_ENUM_ADMISSIBLE  the same over admissible axes only
 *                           (FusedOpDescriptor.admits, strategy.py:57-59).
 * Vectors of up to 16 heads. */
enum { LS_GEN_UNIFORM = 1, LS_GEN_ENUM = 2, LS_GEN_ENUM_ADMISSIBLE = 3 };

/* Length of an enumeration stream (0 for LS_GEN_UNIFORM or on error). */
uint64_t ls_stream_size(ls_ctx* ctx, int mode);
/* Materialise stream positions [start, start + n) as SoA planes. */
int ls_generate(ls_ctx* ctx, int mode, uint64_t seed, int64_t start, int64_t n, uint8_t* planes,
                int64_t plane_stride, void* stream);
/* Evaluate stream positions [start, start + n) and reduce them to the top-k
 * by raw throughput over distinct vectors (index = stream position). k <= 32,
 * n <= 2^40 per call (split larger enumerations, e.g. baselines._sweep);
 * scratch as for ls_evaluate_topk_scratch_bytes(ctx, n, k). */
int ls_sweep(ls_ctx* ctx, int mode, uint64_t seed, int64_t start, int64_t n, int k, ls_elite_rec* topk_out,
             int32_t* count_out, void* scratch, void* stream);

/* Merge m device-resident record lists (e.g. the all-gathered per-rank top-k)
 * into the global top-k with the same ordering and dedupe rule. List l starts
 * at recs[l * k_in] (k_in: the list stride in records, >= its count). */
int ls_topk_merge(const ls_elite_rec* recs, const int32_t* counts, int m, int k_in, int k,
                  ls_elite_rec* out, int32_t* count_out, void* stream);
/* The cross-rank merge of a group of exchanged steps in one launch: `blocks`
 * holds, for rank r and step j, the (k + 1) x 32 B exchange block (k records,
 * then a row starting with the int32 count) at record (r * steps + j) * (k + 1)
 * — the layout of one all-gather of each rank's consecutive blocks. Step j's
 * merged top-k goes to out[j * k ..], its count to counts_out[j]. k <= 32. */
int ls_topk_merge_steps(const void* blocks, int world, int steps, int k, ls_elite_rec* out, int32_t* counts_out,
                        void* stream);

/* ls_evaluate_topk over packed words (fused path only: k <= 32). */
int ls_evaluate_packed_topk(ls_ctx* ctx, const uint64_t* words, int64_t n, const ls_result_soa* out, int k,
                            int64_t index_base, ls_elite_rec* topk_out, int32_t* count_out, void* scratch,
                            void* stream);

/* ---- Search-loop step (device-resident environment state) ---------------
 * One sequential environment step of a learning search, entirely on the
 * device so a whole search round can be captured in a CUDA graph:
 *   SearchEnv.step (env.py:134-180: score, Eq.-1 reward against the best raw
 *   seen strictly before, flat penalty when invalid, best update, eval-log
 *   append) and the valid-only EliteBuffer.offer (policy.py:86-102: reject
 *   duplicates, reject reward <= min when full, stable insert by reward desc).
 * The action is `A` int64 indices on the device. All state pointers are
 * device memory owned by the caller. Writes the step's reward to
 * *reward_out. If *log_pos >= log_capacity nothing is scored and the
 * step's reason is LS_REASON_DECODE_ERROR with reward NaN (budget guard). */
typedef struct ls_search_state {
  double* best_raw;      /* [1] env.best_raw */
  int64_t* elite_vec;    /* [elite_capacity * A], best first */
  double* elite_reward;  /* [elite_capacity]; -inf marks an empty slot */
  int32_t elite_capacity;
  int64_t* log_pos;      /* [1] next eval-log slot (= evaluations done) */
  int64_t log_capacity;
  uint8_t* log_vec;      /* [log_capacity * A] */
  double* log_raw;       /* [log_capacity] raw (0 when invalid) */
  double* log_reward;    /* [log_capacity] */
  uint8_t* log_reason;   /* [log_capacity] LS_REASON_* */
  double alpha, beta, penalty;
} ls_search_state;

int ls_env_step(ls_ctx* ctx, const ls_search_state* state, const int64_t* action, double* reward_out, void* stream);

/* ---- Scalar seam ----------------------------------------------------------
 * simulate() for ONE strategy (simulator.py:239-341) with host memory on both
 * sides: `vector` holds A index bytes; reason_out receives the verdict and
 * fields_out (optional) the six SimResult numbers in ls_result_soa order
 * (throughput, tpot_s, memory_bytes, compute_s, comm_s, pipeline_s). Blocking
 * and low-latency: the vector travels in the launch parameters and the
 * verdict comes back through host-mapped memory (no copies, no stream
 * synchronisation). Thread-safe (calls on one context serialise). */
int ls_evaluate_one(ls_ctx* ctx, const uint8_t* vector, uint8_t* reason_out, double* fields_out);

/* ---- Simulated annealing chain on the device ------------------------------
 * baselines.simulated_annealing (baselines.py:112-145) as one launch: `steps`
 * SearchEnv.step evaluations on the env state (best_raw, log_*, alpha, beta,
 * penalty of `env`; its elite fields are unused), the first of `init`, each
 * later one of a mutation of the current vector (coords/drawn: the heads
 * mutate_vector picks and its integers(k - 1) draws, `moves` per proposal),
 * accepted when u < Metropolis(delta, temperature). The randomness is drawn
 * on the host in the reference's order; all pointers are device memory. */
typedef struct ls_sa_plan {
  int32_t steps;
  int32_t moves;
  const int32_t* init;        /* [A] */
  const int32_t* coords;      /* [(steps - 1) * moves] */
  const int32_t* drawn;       /* [(steps - 1) * moves] */
  const double* u;            /* [steps - 1] */
  const double* temperature;  /* [steps - 1] */
  ls_search_state env;
} ls_sa_plan;

int ls_sa_chain(ls_ctx* ctx, const ls_sa_plan* plan, void* stream);

/* ---- Fused PPO search rounds ---------------------------------------------
 * The reference's elite-conditioned policy (policy.py:213-499: embedding,
 * one post-norm single-head attention block, mean pool, masked categorical
 * heads, value head) and its chunked PPO loop (ppo.py:170-359) as float64
 * device kernels: sampling (inverse CDF on caller-supplied uniforms,
 * policy.py:205-210), the env step above, the clipped-surrogate loss with
 * its exact gradient (ppo.py:203-294), backward, and Adam (ppo.py:130-161).
 *
 * Parameters live in ONE float64 arena in the layout ls_policy_layout_of
 * returns (reference names in LS_PSEG_* order; q/k/v packed as [d, 3d],
 * heads packed as [d, heads*kmax] with zero padding columns). Every pointer
 * below is device memory owned by the caller. */
enum {
  LS_PSEG_EMBED_W = 0, LS_PSEG_EMBED_B, LS_PSEG_WQKV, LS_PSEG_BQKV, LS_PSEG_WO, LS_PSEG_BO,
  LS_PSEG_LN1_G, LS_PSEG_LN1_B, LS_PSEG_FFN_W1, LS_PSEG_FFN_B1, LS_PSEG_FFN_W2, LS_PSEG_FFN_B2,
  LS_PSEG_LN2_G, LS_PSEG_LN2_B, LS_PSEG_HEAD_W, LS_PSEG_HEAD_B, LS_PSEG_VALUE_W1, LS_PSEG_VALUE_B1,
  LS_PSEG_VALUE_W2, LS_PSEG_VALUE_B2, LS_PSEG_COUNT
};

typedef struct ls_policy_dims {
  int32_t obs_dim;     /* vector_length (= number of heads) */
  int32_t width;       /* d */
  int32_t ffn_width;   /* f */
  int32_t history_len; /* T, observation rows */
  int32_t num_heads;
  int32_t kmax;        /* largest head size */
  int32_t n_steps;     /* rollout samples per update */
} ls_policy_dims;

typedef struct ls_policy_layout {
  int64_t off[LS_PSEG_COUNT]; /* element offsets into the arena */
  int64_t total;              /* arena length in doubles */
} ls_policy_layout;

int ls_policy_layout_of(const ls_policy_dims* dims, ls_policy_layout* out);
/* Scratch for activations and their gradients; 0 if dims are unsupported
 * (n_steps * history_len > 16, or a stage's shared-memory staging > 160 KB). */
size_t ls_ppo_workspace_bytes(const ls_policy_dims* dims);

typedef struct ls_ppo_plan {
  ls_policy_dims dims;
  double* params;          /* arena */
  double* adam_m;          /* arena-shaped first moments */
  double* adam_v;          /* arena-shaped second moments */
  double* grad_out;        /* optional arena-shaped gradient of the last epoch (tests) */
  void* workspace;         /* ls_ppo_workspace_bytes */
  const uint8_t* blocked;  /* [num_heads * kmax] 1 = inadmissible or padding */
  const int32_t* head_size;/* [num_heads] */
  const double* obs_denom; /* [obs_dim] max(k - 1, 1) */
  ls_search_state env;
  const double* uniforms;  /* chunk's draws, num_heads per sample, indexed by *spent */
  const double* lr_table;  /* chunk's learning rate, indexed by samples spent before the update */
  int64_t* spent;          /* [1] samples taken in this chunk */
  int64_t* adam_step;      /* [1] Adam step count of this chunk's optimizer */
  int32_t* status;         /* [1] bit 0 every head confident, bit 1 non-finite loss/params */
  double* batch_obs;       /* [n_steps * history_len * obs_dim] */
  int64_t* batch_action;   /* [n_steps * num_heads] */
  double* batch_logp;      /* [n_steps] */
  double* batch_value;     /* [n_steps] */
  double* batch_reward;    /* [n_steps] */
  double tau, clip_eps, value_coef, entropy_coef, beta1, beta2, adam_eps;
  int32_t epochs;
} ls_ppo_plan;

/* Forward of the current observation into sample slot 0 (after a parameter
 * reset: the next round's first sample reads it). */
int ls_ppo_prime(ls_ctx* ctx, const ls_ppo_plan* plan, void* stream);
/* One round (run_chunk loop body, ppo.py:350-358): n samples (each: sample,
 * env step, elite offer), `epochs` PPO updates, then the confidence check of
 * the new parameters on the current observation, which also primes the next
 * round's first sample. Capturable in a CUDA graph. */
int ls_ppo_round(ls_ctx* ctx, const ls_ppo_plan* plan, int n, void* stream);
/* Tests: forward of batch_obs slots [0, n) -> log-probs [n, heads*kmax] and values [n]. */
int ls_ppo_forward(ls_ctx* ctx, const ls_ppo_plan* plan, int n, double* logp_out, double* value_out, void* stream);
/* Tests: `epochs` updates on the batch_* arrays as given (no sampling). */
int ls_ppo_update(ls_ctx* ctx, const ls_ppo_plan* plan, int n, void* stream);

/* ---- Completion signal of a fused launch ----------------------------------
 * ls_evaluate_packed_topk, plus: once the launch's last CTA has written
 * topk_out / count_out it stores `seq` to *signal (device memory or pinned,
 * mapped host memory; system-scope release, so a host thread polling the
 * word sees the records complete). Another stream waits for that elite with ls_stream_wait_signal
 * (cuStreamWaitValue32 until *signal >= seq; LS_WAIT_MEMOP=0 or a driver
 * without it: a one-thread polling kernel, giving up after ~10 s) rather than
 * an event recorded between two fused launches — a stream operation there
 * would serialise launches that otherwise overlap (programmatic dependent
 * launch). Used for the cross-rank elite exchange beside the next batch. */
int ls_evaluate_packed_topk_signal(ls_ctx* ctx, const uint64_t* words, int64_t n, const ls_result_soa* out, int k,
                                   int64_t index_base, ls_elite_rec* topk_out, int32_t* count_out, void* scratch,
                                   uint32_t* signal, uint32_t seq, void* stream);
int ls_stream_wait_signal(void* stream, const uint32_t* signal, uint32_t seq);

/* Multi-GPU elite exchange over peer memory (replaces the NCCL all-gather of
 * the per-rank top-k blocks, reference: the driver loop that compares every
 * worker's best). Each rank owns a ring of exchange blocks
 * [world][slots][k + 1][32 B] in its own HBM and maps its peers' rings with
 * CUDA IPC; for step t the fused launch's last CTA writes its elite block
 * (k records, then a count | seq << 32 word at row k, release-stored after a
 * system-scope fence) into slot t of every rank's ring — sinks is a DEVICE
 * array of nsinks destination pointers, seq != 0 the step's sequence number.
 * ls_topk_merge_steps_wait merges `steps` consecutive slots of the local ring
 * (rank r's block of step j at blocks + (r * rank_stride + j) * (k + 1)
 * records) after waiting, on the device, until each block carries seq0 + j;
 * a block that does not arrive within ~10 s sets *err (device int) to 1. */
#define LS_IPC_HANDLE_BYTES 64
int ls_evaluate_packed_topk_sinks(ls_ctx* ctx, const uint64_t* words, int64_t n, const ls_result_soa* out, int k,
                                  int64_t index_base, ls_elite_rec* topk_out, int32_t* count_out, void* scratch,
                                  void* const* sinks, int nsinks, uint32_t seq, void* stream);
int ls_topk_merge_steps_wait(const void* blocks, int world, int steps, int rank_stride, int k, uint32_t seq0,
                             ls_elite_rec* out, int32_t* counts_out, int32_t* err, void* stream);
int ls_ipc_alloc(size_t bytes, void** dptr_out); /* zeroed device memory of its own allocation (the ring) */
int ls_ipc_free(void* dptr);
int ls_ipc_handle(const void* dptr, void* handle_out); /* dptr: a base returned by ls_ipc_alloc */
int ls_ipc_open(const void* handle, void** dptr_out);
int ls_ipc_close(void* dptr);

#ifdef __cplusplus
}
#endif
#endif /* LS_EVAL_H */
