// ls_formulas.cuh — the reference's cost formulas, one table entry at a time.
//
// Every expression keeps Python's left-to-right evaluation order and the
// exact point where an int operand meets a float.
// This translation unit family is compiled with --fmad=false, so no
// multiply-add is contracted into an FMA: each * and + rounds separately,
// exactly like CPython's float ops. Integer true division a/b (Python)
// equals IEEE double(a)/double(b) because every operand is < 2^53
// (checked when the context is created).
#pragma once
#include <stdint.h>

#include "../../include/ls_eval.h"

namespace ls {

__host__ __device__ inline double py_max(double a, double b) { return b > a ? b : a; }
__host__ __device__ inline float py_max(float a, float b) { return b > a ? b : a; }
__host__ __device__ inline double py_min(double a, double b) { return b < a ? b : a; }

// op_time, simulator.py:100-104
__host__ __device__ inline double op_time(const ls_workload_desc& d, double flops, double bytes) {
  return py_max(flops / d.peak_flops, bytes / d.hbm_bandwidth) + d.kernel_overhead;
}

// ceil(log2 n) as an integer bit length, simulator.py:115
__host__ __device__ inline int64_t ceil_log2(int64_t n) {
  int64_t h = 0;
  for (int64_t v = n - 1; v > 0; v >>= 1) ++h;
  return h;
}

// collective_time, simulator.py:107-120, for fam AR (2(n-1)/n) or ONCE ((n-1)/n)
__host__ __device__ inline double coll_time(const ls_workload_desc& d, bool all_reduce, int64_t n,
                                            double payload, bool intra) {
  if (n <= 1) return 0.0;
  const double bw = intra ? d.intra_node_bw : d.inter_node_bw;
  double volume;
  if (all_reduce)
    volume = ((2.0 * (double)(n - 1)) / (double)n) * payload;
  else
    volume = ((double)(n - 1) / (double)n) * payload;
  return volume / bw + d.per_collective_latency * (double)ceil_log2(n);
}

// point-to-point stage handoff, simulator.py:113-114 / :294-301
__host__ __device__ inline double p2p_time(const ls_workload_desc& d, double payload, bool intra) {
  const double bw = intra ? d.intra_node_bw : d.inter_node_bw;
  return payload / bw + d.per_collective_latency;
}

__host__ __device__ inline int64_t qkv_out_dim(const ls_workload_desc& d) {
  return (d.num_heads + 2 * d.num_kv_heads) * d.head_dim;
}

// _kv_share, simulator.py:123-132
__host__ __device__ inline int64_t kv_share(const ls_workload_desc& d, int64_t tp, bool attn_dim1) {
  if (attn_dim1) return tp < d.num_kv_heads ? tp : d.num_kv_heads;
  return 1;
}

// matmul() inside _op_cost, simulator.py:178-185
__host__ __device__ inline double matmul_time(const ls_workload_desc& d, double t, int64_t in, int64_t out,
                                              double wc, int64_t s) {
  const double flops = (((2.0 * t) * (double)in) * (double)out) / (double)s;
  const double weight = (((wc * (double)in) * (double)out) * (double)d.dtype_bytes) / (double)s;
  const double act = (t * (double)(in + out)) * (double)d.dtype_bytes;
  return op_time(d, flops, weight + act);
}

// op_time(_op_cost(step)) for one planned op instance, simulator.py:163-221.
// axis: the op's AxisChoice; t: the step's token count; attn_dim1 selects
// the KV share for kv_cache_io / attn_core.
__host__ __device__ inline double op_cost_time(const ls_workload_desc& d, int op, int axis, double t, int64_t tp,
                                               int64_t ep, bool attn_dim1) {
  const int64_t h = d.hidden_dim, dt = d.dtype_bytes;
  const int64_t s = axis != 0 ? tp : 1;
  switch (op) {
    case LS_OP_EMBEDDING:
      return op_time(d, 0.0, (((2.0 * t) * (double)h) * (double)dt) / (double)s);
    case LS_OP_QKV_PROJ:
      return matmul_time(d, t, h, qkv_out_dim(d), 1.0, s);
    case LS_OP_KV_CACHE_IO: {
      const int64_t share = kv_share(d, tp, attn_dim1);
      return op_time(d, 0.0,
                     ((((t * 2.0) * (double)d.num_kv_heads) * (double)d.head_dim) * (double)dt) / (double)share);
    }
    case LS_OP_ATTN_CORE: {
      const double hl = (double)d.num_heads / (double)s;
      const int64_t share = kv_share(d, tp, attn_dim1);
      const double kv_read = ((((t * (double)d.context_len) * 2.0) * ((double)d.num_kv_heads / (double)share)) *
                              (double)d.head_dim) *
                             (double)dt;
      const double q_io = (((2.0 * t) * hl) * (double)d.head_dim) * (double)dt;
      const double flops = (((4.0 * t) * hl) * (double)d.head_dim) * (double)d.context_len;
      return op_time(d, flops, kv_read + q_io);
    }
    case LS_OP_ATTN_OUT_PROJ:
      return matmul_time(d, t, d.num_heads * d.head_dim, h, 1.0, s);
    case LS_OP_ROUTER_GATE:
      return matmul_time(d, t, h, d.num_experts, 1.0, s);
    case LS_OP_EXPERT_FFN1:
    case LS_OP_EXPERT_FFN2: {
      const double local = (double)d.num_experts / (double)ep;
      const double active = t > 0 ? py_min(local, t) : 0.0;
      if (op == LS_OP_EXPERT_FFN1) return matmul_time(d, t, h, d.ffn_dim, active, s);
      return matmul_time(d, t, d.ffn_dim, h, active, s);
    }
    case LS_OP_SHARED_FFN1:
      return matmul_time(d, t, h, d.ffn_dim, 1.0, s);
    case LS_OP_SHARED_FFN2:
      return matmul_time(d, t, d.ffn_dim, h, 1.0, s);
    case LS_OP_FINAL_NORM:
      return op_time(d, (8.0 * t) * (double)h, ((2.0 * t) * (double)h) * (double)dt);
    default:  // LS_OP_LM_HEAD
      return matmul_time(d, t, h, d.vocab_size, 1.0, s);
  }
}

// routed_tokens = batch * experts_per_token / ep, layout.py:397
__host__ __device__ inline double routed_tokens(const ls_workload_desc& d, int64_t batch, int64_t ep) {
  return (double)(batch * d.experts_per_token) / (double)ep;
}

// count_parameters (model.py:149-170): dense and routed-expert parameters.
__host__ __device__ inline void param_counts(const ls_workload_desc& d, int64_t* dense, int64_t* routed) {
  const int64_t h = d.hidden_dim;
  const int64_t per_expert = 2 * h * d.ffn_dim;
  const int64_t attention = d.num_layers * (h * qkv_out_dim(d) + d.num_heads * d.head_dim * h);
  const int64_t router = d.num_layers * (h * d.num_experts);
  const int64_t shared = d.has_shared_expert ? d.num_layers * per_expert : 0;
  const int64_t norms = d.num_layers * (4 * h) + h;
  *dense = d.vocab_size * h + d.vocab_size * h + attention + router + shared + norms;
  *routed = d.num_layers * d.num_experts * per_expert;
}

// _shard_extent, layout.py:158-179 (-1: no extent on that axis)
__host__ __device__ inline int64_t shard_extent(const ls_workload_desc& d, int op, int axis) {
  const int64_t h = d.hidden_dim;
  switch (op) {
    case LS_OP_EMBEDDING: return axis == 1 ? d.vocab_size : h;
    case LS_OP_QKV_PROJ: return axis == 1 ? h : d.num_heads;
    case LS_OP_ATTN_CORE: return axis == 2 ? d.num_heads : -1;
    case LS_OP_ATTN_OUT_PROJ: return axis == 1 ? d.num_heads : h;
    case LS_OP_EXPERT_FFN1:
    case LS_OP_SHARED_FFN1: return axis == 1 ? h : d.ffn_dim;
    case LS_OP_EXPERT_FFN2:
    case LS_OP_SHARED_FFN2: return axis == 1 ? d.ffn_dim : h;
    case LS_OP_LM_HEAD: return axis == 1 ? h : d.vocab_size;
    default: return -1;
  }
}

// FusedOpDescriptor.admits over _CANONICAL_OPS (strategy.py:65-78):
// bit a set when axis a is admitted.
__host__ __device__ inline int admits_mask(int op) {
  switch (op) {
    case LS_OP_KV_CACHE_IO:
    case LS_OP_ROUTER_GATE:
    case LS_OP_FINAL_NORM: return 1;
    case LS_OP_ATTN_CORE: return 1 | 4;
    default: return 7;
  }
}

}  // namespace ls
