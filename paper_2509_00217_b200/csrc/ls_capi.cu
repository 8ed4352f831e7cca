// ls_capi.cu — the C ABI of libls_eval.so (declared in include/ls_eval.h).
//
// Owns per-workload contexts (validated descriptor, device tables, launch
// plan) and the host<->device pipeline of ls_evaluate_host. No exception
// crosses the ABI; every entry returns a status and records a message
// retrievable with ls_last_error().
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "../../include/ls_eval.h"
#include "ls_formulas.cuh"
#include "ls_kernels.h"

using namespace ls;

// ABI layouts the Python ctypes mirrors (_native.py) and tests rely on
static_assert(sizeof(ls_workload_desc) == 2280, "ls_workload_desc layout");
static_assert(sizeof(ls_elite_rec) == 32, "ls_elite_rec layout");
static_assert(sizeof(ls_search_state) == 104, "ls_search_state layout");
static_assert(sizeof(ls_policy_layout) == 168, "ls_policy_layout layout");
static_assert(sizeof(ls_ppo_plan) == 344, "ls_ppo_plan layout");
static_assert(sizeof(ls_sa_plan) == 152, "ls_sa_plan layout");

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  return fail(LS_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

struct DeviceGuard {
  int prev = -1;
  bool ok = true;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) ok = cudaSetDevice(dev) == cudaSuccess;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// Host pipeline: chunks of 2^kHostChunkLog2 candidates, up to kPipe in flight on
// their own streams, so the H2D of later chunks overlaps the D2H of earlier
// ones (two copy engines). LS_HOST_CHUNK_LOG2 / LS_HOST_PIPE override the
// defaults (tuning knobs, read at context creation).
constexpr int kHostChunkLog2 = 22;
constexpr int kPipe = 8;  // capacity; the depth in use is ls_ctx::pipe
constexpr int kPipeDefault = 2;

// Persistent host worker pool: run(fn, parts) calls fn(part) for part in
// [0, parts) across the workers and the calling thread, and returns when all
// are done. Used to pack host planes into candidate words inside the host
// pipeline, in parallel with the copies and kernels of earlier chunks.
class HostPool {
 public:
  explicit HostPool(int workers) {
    for (int i = 0; i < workers; ++i) threads_.emplace_back([this] { loop(); });
  }
  ~HostPool() {
    {
      std::lock_guard<std::mutex> l(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : threads_) t.join();
  }
  int size() const { return (int)threads_.size() + 1; }
  void run(const std::function<void(int)>& fn, int parts) {
    {
      std::lock_guard<std::mutex> l(mu_);
      fn_ = &fn;
      parts_ = parts;
      next_ = 0;
      left_ = parts;
      ++gen_;
    }
    cv_.notify_all();
    work();
    std::unique_lock<std::mutex> l(mu_);
    done_.wait(l, [this] { return left_ == 0; });
    fn_ = nullptr;
  }

 private:
  void work() {
    for (;;) {
      int part;
      const std::function<void(int)>* fn;
      {
        std::lock_guard<std::mutex> l(mu_);
        if (!fn_ || next_ >= parts_) return;
        part = next_++;
        fn = fn_;
      }
      (*fn)(part);
      std::lock_guard<std::mutex> l(mu_);
      if (--left_ == 0) done_.notify_all();
    }
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> l(mu_);
        cv_.wait(l, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
      }
      work();
    }
  }
  std::vector<std::thread> threads_;
  std::mutex mu_;
  std::condition_variable cv_, done_;
  const std::function<void(int)>* fn_ = nullptr;
  int parts_ = 0, next_ = 0, left_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

}  // namespace

struct ls_ctx {
  ls_workload_desc desc;
  TabLayout L;
  EvalMeta M;
  TopkMeta TM;
  int device = 0;
  int num_sms = 148;
  uint64_t* d_tab = nullptr;
  float* d_tabf = nullptr;   // fp32 copy of the tables (ls_set_precision LS_PREC_FP32)
  double2* d_memo = nullptr;  // layer-sum memo (ls_memo.cu), or null
  std::atomic<int> precision{0};
  bool smem_gate = false;
  int64_t blocks_tma = 0, blocks_generic = 0;
  int tma_per_sm = 1;
  size_t sweep_smem = 0;  // dynamic shared memory sweep_kernel may use
  std::atomic<int> reserved_sms{0};  // SMs the persistent kernels leave free (ls_reserve_sms)
  uint64_t space_size = 0;
  // on-device candidate streams, built lazily per mode
  std::mutex gen_mu;
  GenMeta gen[4] = {};
  bool gen_ready[4] = {};
  uint32_t* gen_tabs[4] = {};
  // scalar seam: host-mapped verdict block, own stream
  std::mutex one_mu;
  OneOut* one = nullptr;  // pinned + mapped (UVA: the same pointer on the device)
  cudaStream_t one_stream = nullptr;
  uint32_t one_seq = 0;
  // host pipeline
  std::mutex host_mu;
  int64_t host_chunk = int64_t(1) << kHostChunkLog2;
  int pipe = kPipeDefault;
  cudaStream_t hs[kPipe] = {};
  uint8_t* h_planes[kPipe] = {};
  uint8_t* h_reason[kPipe] = {};
  double* h_f[kPipe][6] = {};
  // compact host results: valid raws per slot, their count, pinned staging
  double* d_vraw[kPipe] = {};
  int64_t* d_vcnt[kPipe] = {};
  void* d_cscr[kPipe] = {};
  uint64_t* hp_words[kPipe] = {};  // pinned: host-packed candidate words of the slot's chunk
  int64_t* hp_cnt = nullptr;       // pinned [kPipe]
  cudaEvent_t ev_in[kPipe] = {}, ev_cnt[kPipe] = {};
  HostPool* pool = nullptr;
  // fused evaluate + elite: PDL between consecutive launches, scratch half per buffer
  bool pdl = true;
  bool host_pack = false;  // LS_HOST_PLANES: pack on host threads (8 B/candidate over PCIe) instead of raw planes
  std::mutex parity_mu;
  std::unordered_map<uintptr_t, uint8_t> parity;
};

namespace {

bool finite_pos(double x) { return std::isfinite(x) && x > 0; }

int validate(const ls_workload_desc& d) {
  if (d.abi_version != LS_ABI_VERSION) return fail(LS_ERR_INVALID_ARGUMENT, "abi_version mismatch");
  if (d.sum_mode > 1) return fail(LS_ERR_INVALID_ARGUMENT, "sum_mode must be 0 (naive) or 1 (neumaier)");
  const int64_t ints[] = {d.num_layers,  d.hidden_dim,        d.num_heads,  d.head_dim,   d.num_kv_heads,
                          d.ffn_dim,     d.num_experts,       d.experts_per_token, d.vocab_size, d.dtype_bytes,
                          d.node_size,   d.device_budget,     d.context_len};
  for (int64_t v : ints)
    if (v < 1 || v > (int64_t(1) << 40)) return fail(LS_ERR_INVALID_ARGUMENT, "model/hardware integers must be in [1, 2^40]");
  if (d.num_heads * d.head_dim != d.hidden_dim)
    return fail(LS_ERR_INVALID_ARGUMENT, "model.num_heads * model.head_dim must equal model.hidden_dim");
  if (d.num_heads % d.num_kv_heads) return fail(LS_ERR_INVALID_ARGUMENT, "model.num_kv_heads must divide model.num_heads");
  if (d.experts_per_token > d.num_experts)
    return fail(LS_ERR_INVALID_ARGUMENT, "model.experts_per_token must not exceed model.num_experts");
  if (!finite_pos(d.peak_flops) || !finite_pos(d.hbm_bandwidth) || !finite_pos(d.hbm_capacity) ||
      !finite_pos(d.intra_node_bw) || !finite_pos(d.inter_node_bw))
    return fail(LS_ERR_INVALID_ARGUMENT, "hardware rates must be positive and finite");
  if (!(std::isfinite(d.kernel_overhead) && d.kernel_overhead >= 0) ||
      !(std::isfinite(d.per_collective_latency) && d.per_collective_latency >= 0))
    return fail(LS_ERR_INVALID_ARGUMENT, "hardware overheads must be non-negative and finite");
  if (!finite_pos(d.slo_tpot)) return fail(LS_ERR_INVALID_ARGUMENT, "slo_tpot must be positive");
  for (int h = 0; h < 4; ++h) {
    if (d.domain_len[h] < 1 || d.domain_len[h] > LS_MAX_DOMAIN)
      return fail(LS_ERR_INVALID_ARGUMENT, "domain lengths must be in [1, 64]");
    for (int j = 0; j < d.domain_len[h]; ++j)
      if (d.domain[h][j] < 1 || d.domain[h][j] > (1 << 20))
        return fail(LS_ERR_INVALID_ARGUMENT, "domain values must be in [1, 2^20]");
  }
  if (d.vector_length < 4 || d.vector_length > LS_MAX_HEADS)
    return fail(LS_ERR_INVALID_ARGUMENT, "vector_length must be in [4, 64]");
  bool used[LS_MAX_HEADS] = {};
  for (int k = 0; k < LS_NUM_OPS; ++k) {
    const int h = d.op_head[k];
    if (h == -1) {
      if (d.op_pinned[k] < 0 || d.op_pinned[k] > 2) return fail(LS_ERR_INVALID_ARGUMENT, "op_pinned must be 0..2");
      continue;
    }
    if (h < 4 || h >= d.vector_length || used[h])
      return fail(LS_ERR_INVALID_ARGUMENT, "op_head entries must be distinct heads in [4, vector_length)");
    used[h] = true;
  }
  // exact int->double conversions (< 2^53) for every product the model forms
  const double lim = 9007199254740992.0;
  const double h = (double)d.hidden_dim;
  const double qkv = (double)((d.num_heads + 2 * d.num_kv_heads) * d.head_dim);
  const double dense = 2.0 * d.vocab_size * h + d.num_layers * (h * qkv + h * h + h * d.num_experts + 4 * h) +
                       (d.has_shared_expert ? d.num_layers * 2.0 * h * d.ffn_dim : 0.0) + h;
  const double routed = (double)d.num_layers * d.num_experts * 2.0 * h * d.ffn_dim;
  int64_t bmax = 0;
  for (int j = 0; j < d.domain_len[3]; ++j) bmax = std::max<int64_t>(bmax, d.domain[3][j]);
  const double widest = std::max({h, qkv, (double)d.ffn_dim, (double)d.vocab_size});
  if (dense * d.dtype_bytes >= lim || routed * d.dtype_bytes >= lim ||
      (double)bmax * d.experts_per_token * widest * d.dtype_bytes >= lim)
    return fail(LS_ERR_UNSUPPORTED, "workload integers exceed 2^53: exact float64 parity is not guaranteed");
  return LS_OK;
}

void build_meta(ls_ctx* c) {
  const ls_workload_desc& d = c->desc;
  EvalMeta& M = c->M;
  std::memset(&M, 0, sizeof(M));
  M.A = d.vector_length;
  int slot[LS_MAX_HEADS];
  head_slots(d, slot);
  for (int h = 0; h < LS_MAX_HEADS; ++h) {
    M.head_size[h] = h < 4 ? (uint8_t)d.domain_len[h] : 3;
    M.head_slot[h] = (int8_t)slot[h];
  }
  for (int k = 0; k < LS_NUM_OPS; ++k) {
    const int h = d.op_head[k];
    M.op_src[k] = (int8_t)(h >= 0 ? 2 * slot[h] : -1);
    M.op_pin[k] = (int8_t)(h >= 0 ? 0 : d.op_pinned[k]);
  }
  M.canon_runs = 0;
  M.canon_or = 0;
  for (int k = 0; k < LS_NUM_OPS; ++k) {
    if (M.op_src[k] < 0) {
      M.canon_or |= (uint32_t)M.op_pin[k] << (2 * k);
      continue;
    }
    const int r = M.canon_runs - 1;
    if (r >= 0 && M.canon_shl[r] + M.canon_len[r] == 2 * k && M.canon_shr[r] + M.canon_len[r] == M.op_src[k]) {
      M.canon_len[r] += 2;  // extends the run
    } else {
      M.canon_shr[M.canon_runs] = (uint8_t)M.op_src[k];
      M.canon_len[M.canon_runs] = 2;
      M.canon_shl[M.canon_runs] = (uint8_t)(2 * k);
      ++M.canon_runs;
    }
  }
  M.canon_ident = M.canon_or == 0 && M.canon_runs == 1 && M.canon_shr[0] == 0 && M.canon_shl[0] == 0 &&
                  M.canon_len[0] == 2 * LS_NUM_OPS;
  M.attn_src = M.op_src[LS_OP_ATTN_CORE];
  M.attn_pin = M.op_pin[LS_OP_ATTN_CORE];
  M.attn_shift = M.attn_src >= 0 ? M.attn_src + 1 : 31;
  M.attn_or = M.attn_src >= 0 ? 0u : (M.attn_pin == 2 ? 0x80000000u : 0u);
  M.node_size = d.node_size;
  M.num_layers_d = (double)d.num_layers;
  M.slo_tpot = d.slo_tpot;
  M.hbm_capacity = d.hbm_capacity;
  // mixed-radix place values, head 0 most significant
  unsigned __int128 stride = 1;
  bool overflow = false;
  for (int h = d.vector_length - 1; h >= 0; --h) {
    M.code_stride[h] = (int64_t)stride;
    stride *= M.head_size[h];
    if (stride >= ((unsigned __int128)1 << 63)) overflow = true;
  }
  c->space_size = overflow ? 0 : (uint64_t)stride;
  c->TM.A = M.A;
  for (int h = 0; h < LS_MAX_HEADS; ++h) c->TM.code_stride[h] = M.code_stride[h];
}

uint64_t ceil_recip(uint64_t d) {  // ceil(2^64 / d), d >= 2
  const unsigned __int128 one = (unsigned __int128)1 << 64;
  return (uint64_t)((one + d - 1) / d);
}

// Mixed-radix tables of one candidate stream mode (see GenMeta). Axis heads
// take radix 3 (GEN_UNIFORM, GEN_ENUM) or the number of axes the op they
// control admits (GEN_ENUM_ADMISSIBLE, FusedOpDescriptor.admits,
// strategy.py:57-59); the last min(6, #axis heads) heads form the low group.
int build_gen(ls_ctx* c, int mode) {
  if (c->gen_ready[mode]) return LS_OK;
  const ls_workload_desc& d = c->desc;
  const int A = d.vector_length;
  if (A > 16) return fail(LS_ERR_UNSUPPORTED, "on-device candidate streams support vectors of up to 16 heads");
  int radix[16], axes[16][3];
  for (int h = 4; h < A; ++h) {
    radix[h] = 3;
    for (int v = 0; v < 3; ++v) axes[h][v] = v;
    if (mode == GEN_ENUM_ADMISSIBLE) {
      for (int k = 0; k < LS_NUM_OPS; ++k) {
        if (d.op_head[k] != h) continue;
        if ((k == LS_OP_SHARED_FFN1 || k == LS_OP_SHARED_FFN2) && !d.has_shared_expert) break;
        const int mask = admits_mask(k);
        int r = 0;
        for (int v = 0; v < 3; ++v)
          if ((mask >> v) & 1) axes[h][r++] = v;
        radix[h] = r;
      }
    }
  }
  const int naxis = A - 4, nlo = naxis < 6 ? naxis : 6, lo0 = A - nlo;
  uint64_t lo_size = 1, hi_size = 1;
  for (int h = lo0; h < A; ++h) lo_size *= radix[h];
  for (int h = 4; h < lo0; ++h) hi_size *= radix[h];
  std::vector<uint32_t> tab(hi_size + lo_size);
  auto fill = [&](uint32_t* out, uint64_t size, int h0, int h1) {
    for (uint64_t r = 0; r < size; ++r) {
      uint64_t x = r;
      uint32_t y = 0;
      for (int h = h1 - 1; h >= h0; --h) {
        y |= (uint32_t)axes[h][x % radix[h]] << (2 * (h - 4));
        x /= radix[h];
      }
      out[r] = y;
    }
  };
  fill(tab.data(), hi_size, 4, lo0);
  fill(tab.data() + hi_size, lo_size, lo0, A);
  cudaError_t e;
  if ((e = cudaMalloc(&c->gen_tabs[mode], tab.size() * 4)) != cudaSuccess) return cuda_fail(e, "gen tables");
  if ((e = cudaMemcpy(c->gen_tabs[mode], tab.data(), tab.size() * 4, cudaMemcpyHostToDevice)) != cudaSuccess)
    return cuda_fail(e, "gen tables copy");
  GenMeta& g = c->gen[mode];
  g.coarse_size = (uint64_t)d.domain_len[0] * d.domain_len[1] * d.domain_len[2] * d.domain_len[3];
  g.lo_size = lo_size;
  g.axis_size = lo_size * hi_size;
  g.nb = (uint64_t)d.domain_len[3];
  g.np = (uint64_t)d.domain_len[2];
  g.ne = (uint64_t)d.domain_len[1];
  g.m_axis = g.axis_size > 1 ? ceil_recip(g.axis_size) : 0;
  g.m_lo = lo_size > 1 ? ceil_recip(lo_size) : 0;
  g.m_b = g.nb > 1 ? ceil_recip(g.nb) : 0;
  g.m_p = g.np > 1 ? ceil_recip(g.np) : 0;
  g.m_e = g.ne > 1 ? ceil_recip(g.ne) : 0;
  g.hi_tab = c->gen_tabs[mode];
  g.lo_tab = c->gen_tabs[mode] + hi_size;
  c->gen_ready[mode] = true;
  return LS_OK;
}

uint64_t stream_size(const GenMeta& g) {
  const unsigned __int128 t = (unsigned __int128)g.coarse_size * g.axis_size;
  return t >> 62 ? 0 : (uint64_t)t;
}

}  // namespace

namespace ls {
PackMeta pack_meta(const ls_workload_desc& d) {
  PackMeta pk{};
  const int A = d.vector_length;
  pk.axis_mask = A > 4 ? (uint32_t)((1ull << (2 * (A - 4))) - 1ull) : 0u;
  pk.nt = (uint32_t)d.domain_len[0];
  pk.ne = (uint32_t)d.domain_len[1];
  pk.np = (uint32_t)d.domain_len[2];
  pk.nb = (uint32_t)d.domain_len[3];
  pk.ncoarse = (uint32_t)d.domain_len[0] * pk.ne * pk.np * pk.nb;
  auto magic = [](uint64_t v) {
    return v <= 1 ? 0ull : (uint64_t)((((unsigned __int128)1 << 64) + v - 1) / v);
  };
  pk.m_e = magic(pk.ne);
  pk.m_p = magic(pk.np);
  pk.m_b = magic(pk.nb);
  return pk;
}
}  // namespace ls

extern "C" {

const char* ls_last_error(void) { return g_err.c_str(); }
uint32_t ls_abi_version(void) { return LS_ABI_VERSION; }

int ls_ctx_create(const ls_workload_desc* desc, int device, ls_ctx** out) {
  g_err.clear();
  if (!desc || !out) return fail(LS_ERR_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  int rc = validate(*desc);
  if (rc) return rc;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0) return fail(LS_ERR_CUDA, "no CUDA device available");
  if (device < 0 || device >= ndev) return fail(LS_ERR_INVALID_ARGUMENT, "device ordinal out of range");
  DeviceGuard g(device);
  if (!g.ok) return fail(LS_ERR_CUDA, "cudaSetDevice failed");
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, device);
  if (prop.major < 10) return fail(LS_ERR_UNSUPPORTED, "libls_eval.so is built for sm_100a (B200)");
  ls_ctx* c = new ls_ctx();
  c->desc = *desc;
  c->device = device;
  c->num_sms = prop.multiProcessorCount;
  c->L = make_layout(c->desc);
  build_meta(c);
  const size_t tab_bytes = (size_t)c->L.words * 8;
  if ((e = cudaMalloc(&c->d_tab, tab_bytes)) != cudaSuccess) {
    delete c;
    return cuda_fail(e, "cudaMalloc(tables)");
  }
  if ((e = build_tables(c->desc, c->L, c->d_tab, 0)) != cudaSuccess || (e = cudaDeviceSynchronize()) != cudaSuccess) {
    cudaFree(c->d_tab);
    delete c;
    return cuda_fail(e, "build_tables");
  }
  // the layer-sum memo when it stays small (12.6 MB for the default domains);
  // LS_MEMO=0 disables it (the walk then sums per candidate)
  {
    const int64_t entries = memo_entries(c->L);
    const char* v = getenv("LS_MEMO");
    if ((!v || atoi(v) != 0) && entries * (int64_t)sizeof(double2) <= (int64_t(64) << 20)) {
      if ((e = cudaMalloc(&c->d_memo, sizeof(double2) * (size_t)entries)) != cudaSuccess ||
          (e = build_memo(c->desc.sum_mode == LS_SUM_NEUMAIER, c->d_tab, c->L, c->M, c->d_memo, 0)) != cudaSuccess ||
          (e = cudaDeviceSynchronize()) != cudaSuccess) {
        cudaFree(c->d_memo);
        cudaFree(c->d_tab);
        delete c;
        return cuda_fail(e, "layer-sum memo");
      }
      c->M.memo = c->d_memo;
    }
  }
  // the workload's tables go to shared memory when they fit beside the ring
  // at the kernel's CTAs-per-SM; otherwise both passes read them through L1
  c->smem_gate = tma_smem_bytes(c->L, c->desc.vector_length, true) <= tma_smem_budget(prop);
  c->sweep_smem = prepare_sweep_kernels((size_t)prop.sharedMemPerBlockOptin);
  if (c->desc.vector_length <= 16) {
    prepare_eval_kernels(c->L, c->desc.vector_length, c->smem_gate);
    c->tma_per_sm = std::max(1, tma_blocks_per_sm(c->L, c->desc.vector_length, c->smem_gate));
    c->blocks_tma = (int64_t)c->num_sms * c->tma_per_sm;
  }
  c->blocks_generic = (int64_t)c->num_sms * std::max(1, generic_blocks_per_sm());
  if ((e = cudaGetLastError()) != cudaSuccess) {
    cudaFree(c->d_tab);
    delete c;
    return cuda_fail(e, "kernel setup");
  }
  if (const char* v = getenv("LS_HOST_CHUNK_LOG2")) {
    const int l = atoi(v);
    if (l >= 16 && l <= 26) c->host_chunk = int64_t(1) << l;
  }
  if (const char* v = getenv("LS_PDL")) c->pdl = atoi(v) != 0;
  if (const char* v = getenv("LS_HOST_PACK")) c->host_pack = atoi(v) != 0;
  if (const char* v = getenv("LS_HOST_PIPE")) {
    const int p = atoi(v);
    if (p >= 2 && p <= kPipe) c->pipe = p;
  }
  *out = c;
  return LS_OK;
}

int ls_ctx_destroy(ls_ctx* c) {
  if (!c) return LS_OK;
  DeviceGuard g(c->device);
  for (int s = 0; s < kPipe; ++s) {
    if (c->hs[s]) cudaStreamDestroy(c->hs[s]);
    cudaFree(c->h_planes[s]);
    cudaFree(c->h_reason[s]);
    for (int f = 0; f < 6; ++f) cudaFree(c->h_f[s][f]);
  }
  for (int s = 0; s < kPipe; ++s) {
    cudaFree(c->d_vraw[s]);
    cudaFree(c->d_vcnt[s]);
    cudaFree(c->d_cscr[s]);
    if (c->hp_words[s]) cudaFreeHost(c->hp_words[s]);
    if (c->ev_in[s]) cudaEventDestroy(c->ev_in[s]);
    if (c->ev_cnt[s]) cudaEventDestroy(c->ev_cnt[s]);
  }
  if (c->hp_cnt) cudaFreeHost(c->hp_cnt);
  delete c->pool;
  for (int m = 0; m < 4; ++m) cudaFree(c->gen_tabs[m]);
  if (c->one_stream) cudaStreamDestroy(c->one_stream);
  if (c->one) cudaFreeHost(c->one);
  cudaFree(c->d_tab);
  cudaFree(c->d_tabf);
  cudaFree(c->d_memo);
  delete c;
  return LS_OK;
}

uint64_t ls_space_size(const ls_ctx* c) { return c ? c->space_size : 0; }

int ls_set_precision(ls_ctx* c, int precision) {
  g_err.clear();
  if (!c || (precision != LS_PREC_FP64 && precision != LS_PREC_FP32))
    return fail(LS_ERR_INVALID_ARGUMENT, "precision must be LS_PREC_FP64 or LS_PREC_FP32");
  std::lock_guard<std::mutex> lock(c->gen_mu);
  if (precision == LS_PREC_FP32 && !c->d_tabf) {
    DeviceGuard g(c->device);
    const size_t bytes = ((size_t)c->L.words * 4 + 15) & ~size_t(15);
    cudaError_t e;
    if ((e = cudaMalloc(&c->d_tabf, bytes)) != cudaSuccess) return cuda_fail(e, "cudaMalloc(fp32 tables)");
    if ((e = cudaMemset(c->d_tabf, 0, bytes)) != cudaSuccess ||
        (e = build_tables_f32(c->d_tab, c->L.words, c->d_tabf, 0)) != cudaSuccess ||
        (e = cudaDeviceSynchronize()) != cudaSuccess)
      return cuda_fail(e, "fp32 tables");
  }
  c->precision.store(precision);
  return LS_OK;
}

int ls_reserve_sms(ls_ctx* c, int sms) {
  g_err.clear();
  if (!c || sms < 0 || sms >= c->num_sms) return fail(LS_ERR_INVALID_ARGUMENT, "reserved SMs must be in [0, num_sms)");
  c->reserved_sms.store(sms);
  return LS_OK;
}

// CTAs of the persistent evaluate kernels: every SM not reserved, times CTAs per SM
static int64_t tma_grid_cap(const ls_ctx* c) {
  return c->blocks_tma > 0 ? (int64_t)(c->num_sms - c->reserved_sms.load()) * c->tma_per_sm : 0;
}


static int do_evaluate(ls_ctx* c, const uint8_t* planes, int64_t n, int64_t stride, const ls_result_soa* out,
                       cudaStream_t s, const uint64_t* words = nullptr) {
  if (n < 0 || !out) return fail(LS_ERR_INVALID_ARGUMENT, "bad evaluate arguments");
  if (n == 0) return LS_OK;
  if (!out->reason || (!planes && !words)) return fail(LS_ERR_INVALID_ARGUMENT, "null candidates or reason buffer");
  if (!words && stride < n) return fail(LS_ERR_INVALID_ARGUMENT, "plane_stride must be >= n");
  EvalArgs a{};
  a.planes = planes;
  a.words = words;
  a.n = n;
  a.stride = stride;
  a.reason = out->reason;
  a.thr = out->throughput;
  a.tpot = out->tpot_s;
  a.mem = out->memory_bytes;
  a.comp = out->compute_s;
  a.comm = out->comm_s;
  a.pipe = out->pipeline_s;
  LaunchPlan lp;
  lp.tma = tma_eligible(a, c->M.A) && c->blocks_tma > 0;
  lp.smem_gate = c->smem_gate;
  lp.max_blocks = lp.tma ? tma_grid_cap(c) : c->blocks_generic;
  PackMeta pk;
  if (words) {
    if (!lp.tma)
      return fail(LS_ERR_UNSUPPORTED, "packed candidates need vectors of <= 16 heads and 16-byte aligned buffers");
    pk = pack_meta(c->desc);
  }
  cudaError_t e = launch_evaluate(lp, c->desc.sum_mode == LS_SUM_NEUMAIER, c->d_tab, c->L, c->M, a, s,
                                  words ? &pk : nullptr);
  if (e != cudaSuccess) return cuda_fail(e, "evaluate launch");
  return LS_OK;
}

int ls_evaluate(ls_ctx* c, const uint8_t* planes, int64_t n, int64_t plane_stride, const ls_result_soa* out,
                void* stream) {
  g_err.clear();
  if (!c) return fail(LS_ERR_INVALID_ARGUMENT, "null context");
  DeviceGuard g(c->device);
  return do_evaluate(c, planes, n, plane_stride, out, static_cast<cudaStream_t>(stream));
}


int ls_packed_layout(ls_ctx* c, int32_t* coarse_shift, int64_t* coarse_size) {
  g_err.clear();
  if (!c || !coarse_shift || !coarse_size) return fail(LS_ERR_INVALID_ARGUMENT, "null argument");
  if (c->desc.vector_length > 16) return fail(LS_ERR_UNSUPPORTED, "packed candidates need vectors of <= 16 heads");
  *coarse_shift = 24;
  *coarse_size = (int64_t)pack_meta(c->desc).ncoarse;
  return LS_OK;
}

int ls_pack(ls_ctx* c, const uint8_t* planes, int64_t plane_stride, int64_t n, uint64_t* words, void* stream) {
  g_err.clear();
  if (!c || n < 0 || (n > 0 && (!planes || !words)) || plane_stride < n)
    return fail(LS_ERR_INVALID_ARGUMENT, "bad pack arguments");
  if (c->desc.vector_length > 16) return fail(LS_ERR_UNSUPPORTED, "packed candidates need vectors of <= 16 heads");
  DeviceGuard g(c->device);
  cudaError_t e = launch_pack(pack_meta(c->desc), c->desc.vector_length, planes, plane_stride, n, words,
                              static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? LS_OK : cuda_fail(e, "pack launch");
}

int ls_evaluate_packed(ls_ctx* c, const uint64_t* words, int64_t n, const ls_result_soa* out, void* stream) {
  g_err.clear();
  if (!c) return fail(LS_ERR_INVALID_ARGUMENT, "null context");
  if (n > 0 && !words) return fail(LS_ERR_INVALID_ARGUMENT, "null words");
  DeviceGuard g(c->device);
  return do_evaluate(c, nullptr, n, n, out, static_cast<cudaStream_t>(stream), words);
}

static int host_pipeline(ls_ctx* c, const uint8_t* host_planes, int64_t plane_stride, const uint64_t* host_words,
                         int64_t n, const ls_result_soa* host_out);

int ls_evaluate_host_packed(ls_ctx* c, const uint64_t* host_words, int64_t n, const ls_result_soa* host_out) {
  g_err.clear();
  if (!c || !host_out || n < 0) return fail(LS_ERR_INVALID_ARGUMENT, "bad evaluate_host_packed arguments");
  if (n == 0) return LS_OK;
  if (!host_out->reason || !host_words) return fail(LS_ERR_INVALID_ARGUMENT, "bad evaluate_host_packed arguments");
  if (c->desc.vector_length > 16) return fail(LS_ERR_UNSUPPORTED, "packed candidates need vectors of <= 16 heads");
  return host_pipeline(c, nullptr, 0, host_words, n, host_out);
}

int ls_evaluate_host(ls_ctx* c, const uint8_t* host_planes, int64_t n, int64_t plane_stride,
                     const ls_result_soa* host_out) {
  g_err.clear();
  if (!c || !host_out || n < 0) return fail(LS_ERR_INVALID_ARGUMENT, "bad evaluate_host arguments");
  if (n == 0) return LS_OK;
  if (!host_out->reason || !host_planes || plane_stride < n)
    return fail(LS_ERR_INVALID_ARGUMENT, "bad evaluate_host arguments");
  return host_pipeline(c, host_planes, plane_stride, nullptr, n, host_out);
}

// Chunked H2D -> evaluate -> D2H, kPipe chunks in flight on kPipe streams.
static int host_pipeline(ls_ctx* c, const uint8_t* host_planes, int64_t plane_stride, const uint64_t* host_words,
                         int64_t n, const ls_result_soa* host_out) {
  std::lock_guard<std::mutex> lock(c->host_mu);
  DeviceGuard g(c->device);
  const int A = c->desc.vector_length;
  double* hf[6] = {host_out->throughput, host_out->tpot_s, host_out->memory_bytes,
                   host_out->compute_s,  host_out->comm_s, host_out->pipeline_s};
  cudaError_t e;
  const int64_t chunk_n = c->host_chunk;
  for (int s = 0; s < c->pipe; ++s) {
    if (!c->hs[s] && (e = cudaStreamCreateWithFlags(&c->hs[s], cudaStreamNonBlocking)) != cudaSuccess)
      return cuda_fail(e, "stream create");
    if (!c->h_planes[s]) {
      if ((e = cudaMalloc(&c->h_planes[s], (size_t)LS_MAX_HEADS * chunk_n)) != cudaSuccess ||
          (e = cudaMalloc(&c->h_reason[s], chunk_n)) != cudaSuccess)
        return cuda_fail(e, "pipeline buffers");
    }
    for (int f = 0; f < 6; ++f)
      if (hf[f] && !c->h_f[s][f] && (e = cudaMalloc(&c->h_f[s][f], sizeof(double) * chunk_n)) != cudaSuccess)
        return cuda_fail(e, "pipeline buffers");
  }
  int64_t chunk = 0;
  for (int64_t off = 0; off < n; off += chunk_n, ++chunk) {
    const int s = (int)(chunk % c->pipe);
    const int64_t cnt = std::min<int64_t>(chunk_n, n - off);
    cudaStream_t st = c->hs[s];
    if (host_words) {
      if ((e = cudaMemcpyAsync(c->h_planes[s], host_words + off, sizeof(uint64_t) * (size_t)cnt,
                               cudaMemcpyHostToDevice, st)) != cudaSuccess)
        return cuda_fail(e, "H2D words");
    } else if ((e = cudaMemcpy2DAsync(c->h_planes[s], (size_t)cnt, host_planes + off, (size_t)plane_stride,
                                      (size_t)cnt, A, cudaMemcpyHostToDevice, st)) != cudaSuccess) {
      return cuda_fail(e, "H2D planes");
    }
    ls_result_soa dev;
    dev.reason = c->h_reason[s];
    double** dv[6] = {&dev.throughput, &dev.tpot_s, &dev.memory_bytes, &dev.compute_s, &dev.comm_s, &dev.pipeline_s};
    for (int f = 0; f < 6; ++f) *dv[f] = hf[f] ? c->h_f[s][f] : nullptr;
    int rc = host_words ? do_evaluate(c, nullptr, cnt, cnt, &dev, st, reinterpret_cast<const uint64_t*>(c->h_planes[s]))
                        : do_evaluate(c, c->h_planes[s], cnt, cnt, &dev, st);
    if (rc) return rc;
    if ((e = cudaMemcpyAsync(host_out->reason + off, dev.reason, (size_t)cnt, cudaMemcpyDeviceToHost, st)) !=
        cudaSuccess)
      return cuda_fail(e, "D2H reason");
    for (int f = 0; f < 6; ++f)
      if (hf[f] && (e = cudaMemcpyAsync(hf[f] + off, *dv[f], sizeof(double) * cnt, cudaMemcpyDeviceToHost, st)) !=
                       cudaSuccess)
        return cuda_fail(e, "D2H field");
  }
  for (int s = 0; s < c->pipe; ++s)
    if ((e = cudaStreamSynchronize(c->hs[s])) != cudaSuccess) return cuda_fail(e, "pipeline sync");
  return LS_OK;
}

// Host planes -> packed candidate words (the ls_pack / pack4_kernel rule:
// a head out of range gives an all-ones word, which decodes as an error).
// SWAR over 8 candidates per step: one 8-byte load per plane, per-byte range
// checks, the axis heads folded four per byte (2-bit fields), then per
// candidate the coarse rank and the Y word from byte extracts.
static inline uint64_t ld64(const uint8_t* p) {
  uint64_t v;
  std::memcpy(&v, p, 8);
  return v;
}
static void pack_host_range(const uint8_t* planes, int64_t stride, int A, const PackMeta& pk, int64_t lo, int64_t hi,
                            uint64_t* out) {
  constexpr uint64_t kOnes = 0x0101010101010101ull, kHigh = 0x8080808080808080ull, kM3 = 0x0303030303030303ull;
  const uint64_t sz[4] = {pk.nt * kOnes, pk.ne * kOnes, pk.np * kOnes, pk.nb * kOnes};
  auto word = [&](uint32_t t, uint32_t e, uint32_t p, uint32_t b, uint64_t y, bool bad) {
    const uint64_t rank = ((uint64_t)(t * pk.ne + e) * pk.np + p) * pk.nb + b;
    return bad ? ~0ull : (y | rank << 24);
  };
  int64_t i = lo;
  for (; i + 8 <= hi; i += 8) {
    uint64_t w[16];
    for (int h = 0; h < 16; ++h) w[h] = h < A ? ld64(planes + (int64_t)h * stride + i) : 0;
    uint64_t bad = 0;  // per byte: bit 7 set when that candidate has a head out of range
    for (int h = 0; h < 4; ++h) bad |= (((w[h] | kHigh) - sz[h]) | w[h]) & kHigh;
    uint64_t q[3];
    for (int g = 0; g < 3; ++g) {
      const uint64_t a = w[4 + 4 * g], b = w[5 + 4 * g], c = w[6 + 4 * g], d = w[7 + 4 * g];
      bad |= ((((a | kHigh) - 3 * kOnes) | a) | (((b | kHigh) - 3 * kOnes) | b) | (((c | kHigh) - 3 * kOnes) | c) |
              (((d | kHigh) - 3 * kOnes) | d)) & kHigh;
      q[g] = (a & kM3) | (b & kM3) << 2 | (c & kM3) << 4 | (d & kM3) << 6;
    }
    for (int j = 0; j < 8; ++j) {
      const int sh = 8 * j;
      const uint64_t y = ((q[0] >> sh) & 255) | ((q[1] >> sh) & 255) << 8 | ((q[2] >> sh) & 255) << 16;
      out[i - lo + j] = word((uint32_t)(w[0] >> sh) & 255, (uint32_t)(w[1] >> sh) & 255, (uint32_t)(w[2] >> sh) & 255,
                             (uint32_t)(w[3] >> sh) & 255, y, (bad >> sh) & 0x80);
    }
  }
  for (; i < hi; ++i) {  // the < 8 tail
    uint32_t v[16] = {};
    for (int h = 0; h < A; ++h) v[h] = planes[(int64_t)h * stride + i];
    bool bad = v[0] >= pk.nt || v[1] >= pk.ne || v[2] >= pk.np || v[3] >= pk.nb;
    uint64_t y = 0;
    for (int h = 4; h < 16; ++h) {
      bad |= v[h] > 2;
      y |= (uint64_t)(v[h] & 3u) << (2 * (h - 4));
    }
    out[i - lo] = word(v[0], v[1], v[2], v[3], y, bad);
  }
}

// Chunked host -> device -> compact host results (see ls_evaluate_host_compact).
static int host_pipeline_compact(ls_ctx* c, int format, const void* host_in, int64_t stride, int64_t n,
                                 uint8_t* reason_out, double* valid_raw, int64_t capacity, int64_t* valid_count) {
  std::lock_guard<std::mutex> lock(c->host_mu);
  DeviceGuard g(c->device);
  const int A = c->desc.vector_length;
  const PackMeta pk = pack_meta(c->desc);
  const int64_t chunk_n = c->host_chunk;
  cudaError_t e;
  for (int s = 0; s < c->pipe; ++s) {
    if (!c->hs[s] && (e = cudaStreamCreateWithFlags(&c->hs[s], cudaStreamNonBlocking)) != cudaSuccess)
      return cuda_fail(e, "stream create");
    if (!c->h_planes[s]) {
      if ((e = cudaMalloc(&c->h_planes[s], (size_t)LS_MAX_HEADS * chunk_n)) != cudaSuccess ||
          (e = cudaMalloc(&c->h_reason[s], chunk_n)) != cudaSuccess)
        return cuda_fail(e, "pipeline buffers");
    }
    if (!c->h_f[s][0] && (e = cudaMalloc(&c->h_f[s][0], sizeof(double) * chunk_n)) != cudaSuccess)
      return cuda_fail(e, "pipeline buffers");
    if (!c->d_vraw[s]) {
      if ((e = cudaMalloc(&c->d_vraw[s], sizeof(double) * chunk_n)) != cudaSuccess ||
          (e = cudaMalloc(&c->d_vcnt[s], sizeof(int64_t))) != cudaSuccess ||
          (e = cudaMalloc(&c->d_cscr[s], compact_scratch_bytes(chunk_n))) != cudaSuccess ||
          (e = cudaEventCreateWithFlags(&c->ev_in[s], cudaEventDisableTiming)) != cudaSuccess ||
          (e = cudaEventCreateWithFlags(&c->ev_cnt[s], cudaEventDisableTiming)) != cudaSuccess)
        return cuda_fail(e, "compact buffers");
    }
    if (format == LS_HOST_PLANES && c->host_pack && !c->hp_words[s] &&
        (e = cudaHostAlloc(reinterpret_cast<void**>(&c->hp_words[s]), sizeof(uint64_t) * chunk_n,
                           cudaHostAllocPortable)) != cudaSuccess)
      return cuda_fail(e, "pinned staging");
  }
  if (!c->hp_cnt && (e = cudaHostAlloc(reinterpret_cast<void**>(&c->hp_cnt), sizeof(int64_t) * kPipe,
                                       cudaHostAllocPortable)) != cudaSuccess)
    return cuda_fail(e, "pinned counts");
  if (format == LS_HOST_PLANES && c->host_pack && !c->pool) {
    int w = (int)std::thread::hardware_concurrency() - 1;
    if (const char* v = getenv("LS_HOST_THREADS")) w = atoi(v) - 1;
    c->pool = new HostPool(std::max(0, std::min(w, 255)));
  }
  const int64_t nchunks = (n + chunk_n - 1) / chunk_n;
  int64_t total = 0;
  int rc = LS_OK;
  // second half of chunk j: its valid count is known -> copy exactly that many raws
  auto finish = [&](int64_t j) -> int {
    const int s = (int)(j % c->pipe);
    cudaError_t err = cudaEventSynchronize(c->ev_cnt[s]);
    if (err != cudaSuccess) return cuda_fail(err, "compact count");
    const int64_t cnt = c->hp_cnt[s];
    if (total + cnt > capacity) {
      total += cnt;
      return fail(LS_ERR_INVALID_ARGUMENT, "valid_raw capacity is smaller than the number of valid candidates");
    }
    if (cnt > 0 && (err = cudaMemcpyAsync(valid_raw + total, c->d_vraw[s], sizeof(double) * cnt,
                                          cudaMemcpyDeviceToHost, c->hs[s])) != cudaSuccess)
      return cuda_fail(err, "D2H valid raws");
    total += cnt;
    return LS_OK;
  };
  for (int64_t j = 0; j < nchunks && rc == LS_OK; ++j) {
    const int s = (int)(j % c->pipe);
    const int64_t off = j * chunk_n, cnt = std::min<int64_t>(chunk_n, n - off);
    cudaStream_t st = c->hs[s];
    const uint64_t* src;
    const bool raw_planes = format == LS_HOST_PLANES && !c->host_pack;
    const int64_t dstride = (cnt + 15) & ~int64_t(15);  // device plane stride: TMA-aligned
    if (raw_planes) {  // the planes themselves cross PCIe (A B/candidate); the device reads them directly
      if ((e = cudaMemcpy2DAsync(c->h_planes[s], (size_t)dstride, static_cast<const uint8_t*>(host_in) + off,
                                 (size_t)stride, (size_t)cnt, A, cudaMemcpyHostToDevice, st)) != cudaSuccess ||
          (e = cudaEventRecord(c->ev_in[s], st)) != cudaSuccess) {
        rc = cuda_fail(e, "H2D planes");
        break;
      }
      src = nullptr;
    } else if (format == LS_HOST_PLANES) {
      // the slot's staging buffer is free once its previous H2D finished
      if (j >= c->pipe && (e = cudaEventSynchronize(c->ev_in[s])) != cudaSuccess) {
        rc = cuda_fail(e, "staging reuse");
        break;
      }
      const uint8_t* planes = static_cast<const uint8_t*>(host_in) + off;
      uint64_t* dst = c->hp_words[s];
      const int parts = std::max(1, std::min<int>(c->pool->size() * 2, (int)(cnt / 8192)));
      c->pool->run([&](int q) {
        const int64_t lo = cnt * q / parts, hi = cnt * (q + 1) / parts;
        pack_host_range(planes, stride, A, pk, lo, hi, dst + lo);
      }, parts);
      src = dst;
    } else {
      src = static_cast<const uint64_t*>(host_in) + off;
    }
    uint64_t* dwords = reinterpret_cast<uint64_t*>(c->h_planes[s]);
    if (!raw_planes && ((e = cudaMemcpyAsync(dwords, src, sizeof(uint64_t) * (size_t)cnt, cudaMemcpyHostToDevice,
                                             st)) != cudaSuccess ||
                        (e = cudaEventRecord(c->ev_in[s], st)) != cudaSuccess)) {
      rc = cuda_fail(e, "H2D words");
      break;
    }
    EvalArgs a{};
    if (raw_planes) {
      a.planes = c->h_planes[s];
      a.stride = dstride;
    } else {
      a.words = dwords;
      a.stride = cnt;
    }
    a.n = cnt;
    a.reason = c->h_reason[s];
    a.thr = c->h_f[s][0];
    a.sparse_thr = true;
    LaunchPlan lp{tma_eligible(a, A), c->smem_gate, tma_grid_cap(c)};
    if (!lp.tma) lp.max_blocks = c->blocks_generic;
    if ((e = launch_evaluate(lp, c->desc.sum_mode == LS_SUM_NEUMAIER, c->d_tab, c->L, c->M, a, st,
                             raw_planes ? nullptr : &pk)) !=
            cudaSuccess ||
        (e = launch_valid_compact(a.reason, a.thr, cnt, c->d_vraw[s], c->d_vcnt[s], c->d_cscr[s], st)) !=
            cudaSuccess ||
        (e = cudaMemcpyAsync(reason_out + off, a.reason, (size_t)cnt, cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
        (e = cudaMemcpyAsync(c->hp_cnt + s, c->d_vcnt[s], sizeof(int64_t), cudaMemcpyDeviceToHost, st)) !=
            cudaSuccess ||
        (e = cudaEventRecord(c->ev_cnt[s], st)) != cudaSuccess) {
      rc = cuda_fail(e, "compact chunk");
      break;
    }
    if (j >= 1) rc = finish(j - 1);
  }
  if (rc == LS_OK && nchunks > 0) rc = finish(nchunks - 1);
  for (int s = 0; s < c->pipe; ++s) {
    e = cudaStreamSynchronize(c->hs[s]);
    if (rc == LS_OK && e != cudaSuccess) rc = cuda_fail(e, "pipeline sync");
  }
  if (valid_count) *valid_count = total;
  return rc;
}

int ls_evaluate_host_compact(ls_ctx* c, int format, const void* host_in, int64_t n, int64_t plane_stride,
                             uint8_t* reason_out, double* valid_raw, int64_t capacity, int64_t* valid_count) {
  g_err.clear();
  if (!c || n < 0 || capacity < 0 || (format != LS_HOST_PLANES && format != LS_HOST_WORDS))
    return fail(LS_ERR_INVALID_ARGUMENT, "bad evaluate_host_compact arguments");
  if (valid_count) *valid_count = 0;
  if (n == 0) return LS_OK;
  if (!host_in || !reason_out || (capacity > 0 && !valid_raw) || (format == LS_HOST_PLANES && plane_stride < n))
    return fail(LS_ERR_INVALID_ARGUMENT, "bad evaluate_host_compact arguments");
  if (c->desc.vector_length > 16 || c->blocks_tma == 0)
    return fail(LS_ERR_UNSUPPORTED, "compact host results need vectors of <= 16 heads");
  if (format == LS_HOST_WORDS && ((uintptr_t)host_in % 8) != 0)
    return fail(LS_ERR_INVALID_ARGUMENT, "packed words must be 8-byte aligned");
  return host_pipeline_compact(c, format, host_in, plane_stride, n, reason_out, valid_raw, capacity, valid_count);
}

int ls_host_alloc(size_t bytes, void** out) {
  g_err.clear();
  if (!out) return fail(LS_ERR_INVALID_ARGUMENT, "null out");
  cudaError_t e = cudaHostAlloc(out, bytes ? bytes : 1, cudaHostAllocPortable);
  return e == cudaSuccess ? LS_OK : cuda_fail(e, "cudaHostAlloc");
}

int ls_host_free(void* p) {
  cudaError_t e = cudaFreeHost(p);
  return e == cudaSuccess ? LS_OK : cuda_fail(e, "cudaFreeHost");
}

size_t ls_scan_scratch_bytes(int64_t n) { return scan_scratch_bytes(n); }

int ls_reward_scan(ls_ctx* c, const uint8_t* reason, const double* throughput, int64_t n, double b0, double alpha,
                   double beta, double penalty, double* reward_out, double* best_out, void* scratch, void* stream) {
  g_err.clear();
  if (!c || n < 0 || (n > 0 && (!reason || !throughput || !reward_out || !scratch)))
    return fail(LS_ERR_INVALID_ARGUMENT, "bad reward_scan arguments");
  DeviceGuard g(c->device);
  cudaError_t e = launch_reward_scan(reason, throughput, n, b0, alpha, beta, penalty, reward_out, best_out, scratch,
                                     c->num_sms, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? LS_OK : cuda_fail(e, "reward_scan launch");
}

size_t ls_topk_scratch_bytes(int64_t n, int k) { return topk_scratch_bytes(n, k < 1 ? 1 : k, 0); }

int ls_topk(ls_ctx* c, const uint8_t* planes, int64_t plane_stride, const uint8_t* reason, const double* throughput,
            const double* key, int64_t n, int k, int64_t index_base, ls_elite_rec* out, int32_t* count_out,
            void* scratch, void* stream) {
  g_err.clear();
  if (!c || n < 0 || k < 1 || k > 64 || !out || !count_out || !scratch ||
      (n > 0 && (!planes || !reason || !throughput || !key)) || plane_stride < n)
    return fail(LS_ERR_INVALID_ARGUMENT, "bad topk arguments (k must be in [1, 64])");
  if (c->space_size == 0) return fail(LS_ERR_UNSUPPORTED, "vector codes overflow 63 bits for this action space");
  DeviceGuard g(c->device);
  cudaError_t e = launch_topk(c->TM, planes, plane_stride, reason, throughput, key, n, k, index_base, out, count_out,
                              scratch, c->num_sms, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? LS_OK : cuda_fail(e, "topk launch");
}

// Scratch of the fused evaluate + top-k: two halves, used by alternate calls
// on the same buffer (consecutive fused launches overlap under PDL, so one
// launch's last CTA still merges in its half while the next fills the
// other). A half: 32 bytes of sync words at a fixed offset (the global pruning
// floor, the finished-CTA counter, the tile claim counter), then the per-CTA
// lists and counts. The sync words must be zero before the first call on a
// buffer; each launch's last CTA leaves its half's words zero again, so a call
// is one launch (no per-call memset).
// The half size does not depend on k: the second half's sync words sit at the
// same offset for every call on a buffer, whatever k earlier calls used.
// Sync words at the head of each fused scratch half: the floor and the done
// counter share a line; the tile-claim counter has its own 128-byte line (the
// floor's atomics, frequent while the elite lists fill, would queue the
// claims behind them); the CTA lists start after them.
constexpr size_t kSyncBytes = 256;
constexpr size_t kClaimOffset = 128;

static size_t fused_half_bytes(const ls_ctx* c, int /*k*/) {
  const size_t lists = std::max<size_t>((size_t)c->blocks_tma, (size_t)c->num_sms * sweep_ctas_per_sm());
  return (kSyncBytes + lists * (size_t)fused_k_max() * sizeof(ls_elite_rec) + lists * 4 + 255) & ~size_t(255);
}

static uint8_t* fused_half(ls_ctx* c, void* scratch, int k) {
  std::lock_guard<std::mutex> l(c->parity_mu);
  uint8_t& p = c->parity[reinterpret_cast<uintptr_t>(scratch)];
  uint8_t* h = static_cast<uint8_t*>(scratch) + (p ? fused_half_bytes(c, k) : 0);
  p ^= 1;
  return h;
}

static TopkArgs fused_topk_args(void* half, int64_t grid, int k, int64_t index_base, ls_elite_rec* out,
                                int32_t* count_out) {
  TopkArgs tk{};
  tk.k = k;
  tk.index_base = index_base;
  tk.floor = static_cast<unsigned long long*>(half);
  tk.done = reinterpret_cast<unsigned int*>(tk.floor + 1);
  tk.tile_ctr = reinterpret_cast<unsigned int*>(static_cast<uint8_t*>(half) + kClaimOffset);
  tk.part = reinterpret_cast<ls_elite_rec*>(static_cast<uint8_t*>(half) + kSyncBytes);
  tk.part_counts = reinterpret_cast<int32_t*>(tk.part + grid * k);
  tk.out = out;
  tk.count_out = count_out;
  return tk;
}

size_t ls_evaluate_topk_scratch_bytes(const ls_ctx* c, int64_t n, int k) {
  if (!c || k < 1) return 0;
  return std::max(2 * fused_half_bytes(c, k), topk_scratch_bytes(n, k, 0));
}

static int evaluate_topk_impl(ls_ctx* c, const uint8_t* planes, const uint64_t* words, int64_t n,
                              int64_t plane_stride, const ls_result_soa* out, int k, int64_t index_base,
                              ls_elite_rec* topk_out, int32_t* count_out, void* scratch, void* stream,
                              uint32_t* signal = nullptr, uint32_t seq = 0, uint8_t* const* sinks = nullptr,
                              int nsinks = 0);

int ls_evaluate_topk(ls_ctx* c, const uint8_t* planes, int64_t n, int64_t plane_stride, const ls_result_soa* out,
                     int k, int64_t index_base, ls_elite_rec* topk_out, int32_t* count_out, void* scratch,
                     void* stream) {
  g_err.clear();
  if (!c || n < 0 || k < 1 || !topk_out || !count_out || !scratch || (n > 0 && !planes) || plane_stride < n)
    return fail(LS_ERR_INVALID_ARGUMENT, "bad evaluate_topk arguments");
  return evaluate_topk_impl(c, planes, nullptr, n, plane_stride, out, k, index_base, topk_out, count_out, scratch,
                            stream);
}

int ls_evaluate_packed_topk_signal(ls_ctx* c, const uint64_t* words, int64_t n, const ls_result_soa* out, int k,
                                   int64_t index_base, ls_elite_rec* topk_out, int32_t* count_out, void* scratch,
                                   uint32_t* signal, uint32_t seq, void* stream) {
  g_err.clear();
  if (!c || n < 0 || k < 1 || k > fused_k_max() || !topk_out || !count_out || !scratch || (n > 0 && !words) ||
      !signal)
    return fail(LS_ERR_INVALID_ARGUMENT, "bad evaluate_packed_topk_signal arguments");
  return evaluate_topk_impl(c, nullptr, words, n, n, out, k, index_base, topk_out, count_out, scratch, stream, signal,
                            seq);
}

int ls_evaluate_packed_topk_sinks(ls_ctx* c, const uint64_t* words, int64_t n, const ls_result_soa* out, int k,
                                  int64_t index_base, ls_elite_rec* topk_out, int32_t* count_out, void* scratch,
                                  void* const* sinks, int nsinks, uint32_t seq, void* stream) {
  g_err.clear();
  if (!c || n < 1 || k < 1 || k > fused_k_max() || !topk_out || !count_out || !scratch || !words || !sinks ||
      nsinks < 1 || nsinks > 32 || seq == 0)
    return fail(LS_ERR_INVALID_ARGUMENT, "bad evaluate_packed_topk_sinks arguments");
  return evaluate_topk_impl(c, nullptr, words, n, n, out, k, index_base, topk_out, count_out, scratch, stream,
                            nullptr, seq, reinterpret_cast<uint8_t* const*>(sinks), nsinks);
}

int ls_topk_merge_steps_wait(const void* blocks, int world, int steps, int rank_stride, int k, uint32_t seq0,
                             ls_elite_rec* out, int32_t* counts_out, int32_t* err, void* stream) {
  g_err.clear();
  if (!blocks || world < 1 || world > 1024 || steps < 1 || rank_stride < steps || k < 1 || k > 32 || !out ||
      !counts_out || seq0 == 0)
    return fail(LS_ERR_INVALID_ARGUMENT, "bad topk_merge_steps_wait arguments");
  cudaError_t e = launch_topk_merge_steps(static_cast<const ls_elite_rec*>(blocks), world, steps, k, out, counts_out,
                                          static_cast<cudaStream_t>(stream), rank_stride, seq0, err);
  return e == cudaSuccess ? LS_OK : cuda_fail(e, "topk_merge_steps_wait launch");
}

int ls_ipc_alloc(size_t bytes, void** dptr_out) {
  g_err.clear();
  if (!bytes || !dptr_out) return fail(LS_ERR_INVALID_ARGUMENT, "bad ipc_alloc arguments");
  cudaError_t e = cudaMalloc(dptr_out, bytes);  // its own allocation: an IPC handle maps exactly this base
  if (e == cudaSuccess) e = cudaMemset(*dptr_out, 0, bytes);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  return e == cudaSuccess ? LS_OK : cuda_fail(e, "ipc_alloc");
}

int ls_ipc_free(void* dptr) {
  g_err.clear();
  if (!dptr) return fail(LS_ERR_INVALID_ARGUMENT, "null ipc_free argument");
  cudaError_t e = cudaFree(dptr);
  return e == cudaSuccess ? LS_OK : cuda_fail(e, "ipc_free");
}

int ls_ipc_handle(const void* dptr, void* handle_out) {
  g_err.clear();
  if (!dptr || !handle_out) return fail(LS_ERR_INVALID_ARGUMENT, "null ipc_handle argument");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, const_cast<void*>(dptr));
  if (e != cudaSuccess) return cuda_fail(e, "cudaIpcGetMemHandle");
  static_assert(sizeof(h) == LS_IPC_HANDLE_BYTES, "IPC handle size");
  memcpy(handle_out, &h, sizeof(h));
  return LS_OK;
}

int ls_ipc_open(const void* handle, void** dptr_out) {
  g_err.clear();
  if (!handle || !dptr_out) return fail(LS_ERR_INVALID_ARGUMENT, "null ipc_open argument");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  cudaError_t e = cudaIpcOpenMemHandle(dptr_out, h, cudaIpcMemLazyEnablePeerAccess);
  return e == cudaSuccess ? LS_OK : cuda_fail(e, "cudaIpcOpenMemHandle");
}

int ls_ipc_close(void* dptr) {
  g_err.clear();
  if (!dptr) return fail(LS_ERR_INVALID_ARGUMENT, "null ipc_close argument");
  cudaError_t e = cudaIpcCloseMemHandle(dptr);
  return e == cudaSuccess ? LS_OK : cuda_fail(e, "cudaIpcCloseMemHandle");
}

// cuStreamWaitValue32 from the driver (resolved once through the runtime: no -lcuda)
typedef int (*StreamWaitValue32Fn)(void* stream, unsigned long long addr, uint32_t value, unsigned int flags);

int ls_stream_wait_signal(void* stream, const uint32_t* signal, uint32_t seq) {
  g_err.clear();
  static StreamWaitValue32Fn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<StreamWaitValue32Fn>(p);
  });
  if (!signal) return fail(LS_ERR_INVALID_ARGUMENT, "null signal");
  static const bool mem_op = [] {
    const char* v = getenv("LS_WAIT_MEMOP");
    return !v || atoi(v) != 0;
  }();
  if (!mem_op || !fn) {  // a one-thread polling kernel on the waiting stream instead
    cudaError_t e = launch_wait_signal(signal, seq, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? LS_OK : cuda_fail(e, "wait_signal launch");
  }
  constexpr unsigned kGeq = 0x0;  // CU_STREAM_WAIT_VALUE_GEQ
  const int r = fn(stream, reinterpret_cast<unsigned long long>(signal), seq, kGeq);
  return r == 0 ? LS_OK : fail(LS_ERR_CUDA, "cuStreamWaitValue32 failed (" + std::to_string(r) + ")");
}

int ls_evaluate_packed_topk(ls_ctx* c, const uint64_t* words, int64_t n, const ls_result_soa* out, int k,
                            int64_t index_base, ls_elite_rec* topk_out, int32_t* count_out, void* scratch,
                            void* stream) {
  g_err.clear();
  if (!c || n < 0 || k < 1 || !topk_out || !count_out || !scratch || (n > 0 && !words))
    return fail(LS_ERR_INVALID_ARGUMENT, "bad evaluate_packed_topk arguments");
  return evaluate_topk_impl(c, nullptr, words, n, n, out, k, index_base, topk_out, count_out, scratch, stream);
}

static int evaluate_topk_impl(ls_ctx* c, const uint8_t* planes, const uint64_t* words, int64_t n,
                              int64_t plane_stride, const ls_result_soa* out, int k, int64_t index_base,
                              ls_elite_rec* topk_out, int32_t* count_out, void* scratch, void* stream,
                              uint32_t* signal, uint32_t seq, uint8_t* const* sinks, int nsinks) {
  DeviceGuard g(c->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  EvalArgs a{};
  a.planes = planes;
  a.words = words;
  a.n = n;
  a.stride = plane_stride;
  if (out) {
    a.reason = out->reason;
    a.thr = out->throughput;
    a.tpot = out->tpot_s;
    a.mem = out->memory_bytes;
    a.comp = out->compute_s;
    a.comm = out->comm_s;
    a.pipe = out->pipeline_s;
  }
  if (!a.reason) a.thr = a.tpot = a.mem = a.comp = a.comm = a.pipe = nullptr;
  cudaError_t e;
  if (k <= fused_k_max() && c->blocks_tma > 0 && tma_eligible(a, c->M.A)) {
    LaunchPlan lp{true, c->smem_gate, tma_grid_cap(c)};
    lp.pdl = c->pdl;
    const int64_t grid = ws_grid(lp, n, words ? GEN_WORDS : GEN_PLANES);
    TopkArgs tk = fused_topk_args(fused_half(c, scratch, k), grid, k, index_base, topk_out, count_out);
    tk.signal = signal;
    tk.seq = seq;
    tk.sinks = sinks;
    tk.nsinks = nsinks;
    if (n == 0) {
      if (nsinks > 0) return fail(LS_ERR_INVALID_ARGUMENT, "an empty batch has no elite to send to sinks");
      cudaMemsetAsync(count_out, 0, sizeof(int32_t), s);
      if (signal) cudaMemcpyAsync(signal, &seq, sizeof(seq), cudaMemcpyHostToDevice, s);
      return LS_OK;
    }
    const PackMeta pk = pack_meta(c->desc);
    if ((e = launch_evaluate_topk(lp, c->desc.sum_mode == LS_SUM_NEUMAIER, c->d_tab, c->L, c->M, a, tk, s,
                                  words ? &pk : nullptr)) != cudaSuccess)
      return cuda_fail(e, "evaluate_topk launch");
    return LS_OK;
  }
  if (words) return fail(LS_ERR_UNSUPPORTED, "packed candidates need k <= 32 and 16-byte aligned buffers");
  if (!a.reason || !a.thr)
    return fail(LS_ERR_UNSUPPORTED,
                "unaligned planes, k > 32 or vectors longer than 16 heads need per-candidate reason + throughput "
                "outputs");
  int rc = do_evaluate(c, planes, n, plane_stride, out, s);
  if (rc) return rc;
  if (c->space_size == 0) return fail(LS_ERR_UNSUPPORTED, "vector codes overflow 63 bits for this action space");
  if (k > 64) return fail(LS_ERR_INVALID_ARGUMENT, "k must be <= 64");
  e = launch_topk(c->TM, planes, plane_stride, a.reason, a.thr, a.thr, n, k, index_base, topk_out, count_out, scratch,
                  c->num_sms, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(scratch, 0, kSyncBytes, s);  // the fused path's sync words, zero again
  if (e == cudaSuccess)
    e = cudaMemsetAsync(static_cast<uint8_t*>(scratch) + fused_half_bytes(c, k), 0, kSyncBytes, s);
  return e == cudaSuccess ? LS_OK : cuda_fail(e, "topk launch");
}

int ls_topk_merge_steps(const void* blocks, int world, int steps, int k, ls_elite_rec* out, int32_t* counts_out,
                        void* stream) {
  g_err.clear();
  if (!blocks || world < 1 || world > 1024 || steps < 1 || k < 1 || k > 32 || !out || !counts_out)
    return fail(LS_ERR_INVALID_ARGUMENT, "bad topk_merge_steps arguments");
  cudaError_t e = launch_topk_merge_steps(static_cast<const ls_elite_rec*>(blocks), world, steps, k, out, counts_out,
                                          static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? LS_OK : cuda_fail(e, "topk_merge_steps launch");
}

int ls_topk_merge(const ls_elite_rec* recs, const int32_t* counts, int m, int k_in, int k, ls_elite_rec* out,
                  int32_t* count_out, void* stream) {
  g_err.clear();
  if (!recs || !counts || m < 1 || k_in < 1 || k_in > (1 << 20) || k < 1 || k > 64 || !out || !count_out)
    return fail(LS_ERR_INVALID_ARGUMENT, "bad topk_merge arguments");
  cudaError_t e =
      launch_topk_merge(recs, counts, m, k_in, k, nullptr, out, count_out, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? LS_OK : cuda_fail(e, "topk_merge launch");
}

int ls_env_step(ls_ctx* c, const ls_search_state* st, const int64_t* action, double* reward_out, void* stream) {
  g_err.clear();
  if (!c || !st || !action || !reward_out) return fail(LS_ERR_INVALID_ARGUMENT, "null env_step argument");
  if (!st->best_raw || !st->log_pos || !st->log_vec || !st->log_raw || !st->log_reward || !st->log_reason ||
      st->log_capacity < 0 || st->elite_capacity < 1 || !st->elite_vec || !st->elite_reward)
    return fail(LS_ERR_INVALID_ARGUMENT, "incomplete search state");
  DeviceGuard g(c->device);
  cudaError_t e = launch_env_step(c->desc.sum_mode == LS_SUM_NEUMAIER, c->d_tab, c->L, c->M, *st, action, reward_out,
                                  static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? LS_OK : cuda_fail(e, "env_step launch");
}

int ls_evaluate_one(ls_ctx* c, const uint8_t* vector, uint8_t* reason_out, double* fields_out) {
  g_err.clear();
  if (!c || !vector || !reason_out) return fail(LS_ERR_INVALID_ARGUMENT, "null evaluate_one argument");
  std::lock_guard<std::mutex> lock(c->one_mu);
  DeviceGuard g(c->device);
  cudaError_t e;
  if (!c->one) {
    if ((e = cudaStreamCreateWithFlags(&c->one_stream, cudaStreamNonBlocking)) != cudaSuccess)
      return cuda_fail(e, "stream create");
    if ((e = cudaHostAlloc(reinterpret_cast<void**>(&c->one), sizeof(OneOut), cudaHostAllocMapped)) != cudaSuccess)
      return cuda_fail(e, "mapped verdict block");
    std::memset(c->one, 0, sizeof(OneOut));
  }
  OneArgs a{};
  std::memcpy(a.vec, vector, (size_t)c->desc.vector_length);
  a.out = c->one;
  a.seq = ++c->one_seq;
  if (a.seq == 0) a.seq = c->one_seq = 1;
  if ((e = launch_eval_one(c->desc.sum_mode == LS_SUM_NEUMAIER, c->d_tab, c->L, c->M, a, c->one_stream)) !=
      cudaSuccess)
    return cuda_fail(e, "evaluate_one launch");
  volatile OneOut* o = c->one;
  for (uint64_t spins = 0; o->seq != a.seq; ++spins) {
    if ((spins & 0xfff) == 0xfff) {  // a failed kernel never writes the word
      e = cudaStreamQuery(c->one_stream);
      if (e != cudaSuccess && e != cudaErrorNotReady) return cuda_fail(e, "evaluate_one");
      if (e == cudaSuccess && o->seq != a.seq) return fail(LS_ERR_CUDA, "evaluate_one: verdict never arrived");
    }
  }
  std::atomic_thread_fence(std::memory_order_acquire);
  *reason_out = (uint8_t)o->reason;
  if (fields_out)
    for (int f = 0; f < 6; ++f) fields_out[f] = o->f[f];
  return LS_OK;
}

int ls_sa_chain(ls_ctx* c, const ls_sa_plan* p, void* stream) {
  g_err.clear();
  if (!c || !p || p->steps < 1 || p->moves < 0 || !p->init || (p->steps > 1 && (!p->u || !p->temperature)) ||
      (p->moves > 0 && p->steps > 1 && (!p->coords || !p->drawn)))
    return fail(LS_ERR_INVALID_ARGUMENT, "bad sa plan");
  const ls_search_state& s = p->env;
  if (!s.best_raw || !s.log_pos || !s.log_vec || !s.log_raw || !s.log_reward || !s.log_reason)
    return fail(LS_ERR_INVALID_ARGUMENT, "incomplete search state");
  DeviceGuard g(c->device);
  cudaError_t e = launch_sa_chain(c->desc.sum_mode == LS_SUM_NEUMAIER, c->d_tab, c->L, c->M, *p,
                                  static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? LS_OK : cuda_fail(e, "sa_chain launch");
}

int ls_policy_layout_of(const ls_policy_dims* dims, ls_policy_layout* out) {
  g_err.clear();
  if (!dims || !out || !ppo_layout(*dims, out)) return fail(LS_ERR_INVALID_ARGUMENT, "bad policy dims");
  return LS_OK;
}

size_t ls_ppo_workspace_bytes(const ls_policy_dims* dims) { return dims ? ppo_workspace_bytes(*dims) : 0; }

static int ppo_check(ls_ctx* c, const ls_ppo_plan* p, int n) {
  if (!c || !p) return fail(LS_ERR_INVALID_ARGUMENT, "null context or plan");
  if (ppo_workspace_bytes(p->dims) == 0)
    return fail(LS_ERR_UNSUPPORTED, "policy dims unsupported by the fused kernels (n_steps*history_len > 16, "
                                    "heads != obs_dim, or shared-memory staging too large)");
  if (p->dims.obs_dim != c->desc.vector_length) return fail(LS_ERR_INVALID_ARGUMENT, "obs_dim != vector_length");
  if (n < 1 || n > p->dims.n_steps) return fail(LS_ERR_INVALID_ARGUMENT, "n must be in [1, n_steps]");
  if (!p->params || !p->adam_m || !p->adam_v || !p->workspace || !p->blocked || !p->head_size || !p->obs_denom ||
      !p->spent || !p->adam_step || !p->status || !p->batch_obs || !p->batch_action || !p->batch_logp ||
      !p->batch_value || !p->batch_reward || !p->lr_table || p->epochs < 1)
    return fail(LS_ERR_INVALID_ARGUMENT, "incomplete ppo plan");
  return LS_OK;
}

static PpoCtx ppo_ctx(const ls_ctx* c) {
  PpoCtx x;
  x.tab = c->d_tab;
  x.L = c->L;
  x.M = c->M;
  x.neumaier = c->desc.sum_mode == LS_SUM_NEUMAIER;
  return x;
}

int ls_ppo_prime(ls_ctx* c, const ls_ppo_plan* p, void* stream) {
  g_err.clear();
  int rc = ppo_check(c, p, 1);
  if (rc) return rc;
  DeviceGuard g(c->device);
  cudaError_t e = ppo_prime(*p, ppo_ctx(c), static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? LS_OK : cuda_fail(e, "ppo_prime");
}

int ls_ppo_round(ls_ctx* c, const ls_ppo_plan* p, int n, void* stream) {
  g_err.clear();
  int rc = ppo_check(c, p, n);
  if (rc) return rc;
  if (!p->uniforms || !p->env.best_raw || !p->env.log_pos || !p->env.elite_vec || !p->env.elite_reward)
    return fail(LS_ERR_INVALID_ARGUMENT, "incomplete search state");
  DeviceGuard g(c->device);
  cudaError_t e = ppo_round(*p, ppo_ctx(c), n, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? LS_OK : cuda_fail(e, "ppo_round");
}

int ls_ppo_forward(ls_ctx* c, const ls_ppo_plan* p, int n, double* logp_out, double* value_out, void* stream) {
  g_err.clear();
  int rc = ppo_check(c, p, n);
  if (rc) return rc;
  if (!logp_out || !value_out) return fail(LS_ERR_INVALID_ARGUMENT, "null output");
  DeviceGuard g(c->device);
  cudaError_t e = ppo_forward(*p, ppo_ctx(c), n, logp_out, value_out, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? LS_OK : cuda_fail(e, "ppo_forward");
}

int ls_ppo_update(ls_ctx* c, const ls_ppo_plan* p, int n, void* stream) {
  g_err.clear();
  int rc = ppo_check(c, p, n);
  if (rc) return rc;
  DeviceGuard g(c->device);
  cudaError_t e = ppo_update(*p, ppo_ctx(c), n, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? LS_OK : cuda_fail(e, "ppo_update");
}

uint64_t ls_stream_size(ls_ctx* c, int mode) {
  if (!c || mode < LS_GEN_UNIFORM || mode > LS_GEN_ENUM_ADMISSIBLE) return 0;
  std::lock_guard<std::mutex> lock(c->gen_mu);
  DeviceGuard g(c->device);
  if (build_gen(c, mode)) return 0;
  return mode == LS_GEN_UNIFORM ? 0 : stream_size(c->gen[mode]);
}

static int gen_meta(ls_ctx* c, int mode, uint64_t seed, int64_t start, int64_t n, GenMeta* out) {
  if (mode < LS_GEN_UNIFORM || mode > LS_GEN_ENUM_ADMISSIBLE) return fail(LS_ERR_INVALID_ARGUMENT, "bad stream mode");
  if (start < 0 || n < 0) return fail(LS_ERR_INVALID_ARGUMENT, "negative start or n");
  std::lock_guard<std::mutex> lock(c->gen_mu);
  int rc = build_gen(c, mode);
  if (rc) return rc;
  *out = c->gen[mode];
  out->start = start;
  out->seed = seed;
  if (mode != LS_GEN_UNIFORM) {
    const uint64_t total = stream_size(*out);
    if (total == 0) return fail(LS_ERR_UNSUPPORTED, "enumeration space too large for exact 64-bit indexing");
    if ((uint64_t)start + (uint64_t)n > total) return fail(LS_ERR_INVALID_ARGUMENT, "start + n exceeds the stream size");
  } else if ((uint64_t)start + (uint64_t)n >= (1ull << 40)) {
    return fail(LS_ERR_INVALID_ARGUMENT, "uniform stream indices must stay below 2^40");
  }
  return LS_OK;
}

int ls_generate(ls_ctx* c, int mode, uint64_t seed, int64_t start, int64_t n, uint8_t* planes, int64_t plane_stride,
                void* stream) {
  g_err.clear();
  if (!c || (n > 0 && !planes) || plane_stride < n) return fail(LS_ERR_INVALID_ARGUMENT, "bad generate arguments");
  DeviceGuard g(c->device);
  GenMeta gm;
  int rc = gen_meta(c, mode, seed, start, n, &gm);
  if (rc) return rc;
  cudaError_t e =
      launch_generate(mode, gm, n, c->desc.vector_length, planes, plane_stride, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? LS_OK : cuda_fail(e, "generate launch");
}

int ls_sweep(ls_ctx* c, int mode, uint64_t seed, int64_t start, int64_t n, int k, ls_elite_rec* topk_out,
             int32_t* count_out, void* scratch, void* stream) {
  g_err.clear();
  if (!c || n < 0 || k < 1 || k > fused_k_max() || !topk_out || !count_out || !scratch)
    return fail(LS_ERR_INVALID_ARGUMENT, "bad sweep arguments (k must be in [1, 32])");
  if (n > (int64_t(1) << 40))  // the launch's 32-bit chunk / tile claim counters
    return fail(LS_ERR_INVALID_ARGUMENT, "a sweep launch covers at most 2^40 stream positions: split it");
  if (c->blocks_tma == 0) return fail(LS_ERR_UNSUPPORTED, "sweeps need vectors of up to 16 heads");
  DeviceGuard g(c->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  GenMeta gm;
  int rc = gen_meta(c, mode, seed, start, n, &gm);
  if (rc) return rc;
  if (n == 0) {
    cudaMemsetAsync(count_out, 0, sizeof(int32_t), s);
    return LS_OK;
  }
  LaunchPlan lp{true, c->smem_gate, tma_grid_cap(c)};
  const GenMeta& gen = c->gen[mode];
  const bool f32 = c->precision.load() == LS_PREC_FP32;
  lp.sweep_fits = sweep_smem_bytes(c->L, gen.axis_size / gen.lo_size, gen.lo_size, mode, f32) <= c->sweep_smem;
  if (f32) {
    if (!lp.sweep_fits) return fail(LS_ERR_UNSUPPORTED, "fp32 sweep: tables do not fit in shared memory");
    lp.tabf = c->d_tabf;
  }
  if (lp.sweep_fits) lp.max_blocks = tma_grid_cap(c) / c->tma_per_sm * sweep_ctas_per_sm();
  const int64_t grid = lp.sweep_fits ? sweep_grid(lp, n, mode) : ws_grid(lp, n, mode);
  TopkArgs tk = fused_topk_args(fused_half(c, scratch, k), grid, k, start, topk_out, count_out);
  cudaError_t e;
  if ((e = launch_sweep(lp, c->desc.sum_mode == LS_SUM_NEUMAIER, mode, c->d_tab, c->L, c->M, n, tk, gm, s)) !=
      cudaSuccess)
    return cuda_fail(e, "sweep launch");
  return LS_OK;
}

}  // extern "C"
