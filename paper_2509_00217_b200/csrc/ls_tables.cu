// ls_tables.cu — device-side construction of the per-workload tables.
//
// One thread per table word. Each word is the reference's own expression for
// that (op, axis, tp, batch[, ep][, attn axis]) tuple (ls_formulas.cuh), so
// the evaluate kernel only has to gather and sum. Runs once per context.
#include "ls_formulas.cuh"
#include "ls_tables.cuh"

namespace ls {

namespace {

__device__ inline uint64_t dbits(double x) { return (uint64_t)__double_as_longlong(x); }


// Decompose a flat row-major index over dims (d0..d3) into 4 coordinates.
__device__ inline void unflat(int i, int d1, int d2, int d3, int* c0, int* c1, int* c2, int* c3) {
  *c3 = i % d3;
  i /= d3;
  *c2 = i % d2;
  i /= d2;
  *c1 = i % d1;
  *c0 = i / d1;
}

// Gate bits of one (tp, ep, pp) (see GATE_* in ls_tables.cuh): device budget
// (simulator.py:257), pp | num_layers and ep vs num_experts (simulator.py:268,
// layout.py:371-374), and per axis field whether the op it controls is
// inadmissible under DIM0 / DIM1 or its sharded extent does not divide tp
// (layout.py:214-221); UNSHARDED is always admitted and never sharded.
__device__ uint32_t gate_bits(const ls_workload_desc& d, int64_t tp, int64_t ep, int64_t pp) {
  int slot[LS_MAX_HEADS];
  head_slots(d, slot);
  uint32_t g = 0;
  if (tp * ep * pp > d.device_budget) g |= GATE_BUDGET;
  if (ep > d.num_experts || d.num_experts % ep != 0 || d.num_layers % pp != 0) g |= GATE_LAYOUT;
  for (int op = 0; op < LS_NUM_OPS; ++op) {
    if ((op == LS_OP_SHARED_FFN1 || op == LS_OP_SHARED_FFN2) && !d.has_shared_expert) continue;
    for (int a = 1; a < 3; ++a) {
      bool bad = !((admits_mask(op) >> a) & 1);
      if (!bad && tp > 1) {
        const int64_t ext = shard_extent(d, op, a);
        bad = ext < 0 || ext % tp != 0;
      }
      if (!bad) continue;
      const int h = d.op_head[op];
      if (h >= 0) g |= 1u << (2 * slot[h] + (a - 1));
      else if (d.op_pinned[op] == a) g |= GATE_PINNED;
    }
  }
  return g;
}

// memory_per_device terms (simulator.py:135-160), each in the reference's order
__device__ double weights_mem(const ls_workload_desc& d, int64_t tp, int64_t ep, int64_t pp) {
  int64_t dense, routed;
  param_counts(d, &dense, &routed);
  return ((double)(dense * d.dtype_bytes) / (double)tp) / (double)pp +
         ((double)(routed * d.dtype_bytes) / (double)(ep * tp)) / (double)pp;
}
__device__ double kv_mem(const ls_workload_desc& d, int64_t tp, int64_t pp, int64_t b, bool attn_dim1) {
  const int64_t share = kv_share(d, tp, attn_dim1);
  return ((((2.0 * ((double)d.num_layers / (double)pp)) * ((double)(d.num_kv_heads * d.head_dim) / (double)share)) *
           (double)d.context_len) *
          (double)b) *
         (double)d.dtype_bytes;
}
__device__ double ws_mem(const ls_workload_desc& d, int64_t b) {
  return ((2.0 * (double)b) * (double)(d.hidden_dim + d.ffn_dim)) * (double)d.dtype_bytes;
}

// Coarse gate word of one (t, e, p, b) (COARSE_RS_SHIFT): the axis-field bits
// and, per attention layout, the static reason in gate order; the OOM test is
// gate()'s expression (w + kv) + ws > capacity.
__device__ uint32_t coarse_word(const ls_workload_desc& d, const TabLayout& L, int c) {
  const int b = c % L.nb, p = (c / L.nb) % L.np, e = (c / (L.nb * L.np)) % L.ne, t = c / (L.nb * L.np * L.ne);
  const int64_t TP = d.domain[0][t], EP = d.domain[1][e], PP = d.domain[2][p], B = d.domain[3][b];
  const uint32_t g = gate_bits(d, TP, EP, PP);
  const double w = weights_mem(d, TP, EP, PP), ws = ws_mem(d, B);
  const bool oom0 = (w + kv_mem(d, TP, PP, B, false)) + ws > d.hbm_capacity;
  const bool oom1 = (w + kv_mem(d, TP, PP, B, true)) + ws > d.hbm_capacity;
  auto rs = [&](bool oom) -> uint32_t {
    if (g & GATE_BUDGET) return LS_REASON_OVER_DEVICE_BUDGET;
    if (g & (GATE_PINNED | GATE_LAYOUT)) return LS_REASON_LAYOUT_ERROR;
    return oom ? LS_REASON_OOM : LS_REASON_NONE;
  };
  return (g & GATE_FIELDS) | rs(oom0) << COARSE_RS_SHIFT | rs(oom1) << (COARSE_RS_SHIFT + 2);
}

__device__ uint64_t table_word(const ls_workload_desc& d, const TabLayout& L, int w) {
  const int nt = L.nt, ne = L.ne, np = L.np, nb = L.nb;
  const int64_t* TP = d.domain[0];
  const int64_t* EP = d.domain[1];
  const int64_t* PP = d.domain[2];
  const int64_t* B = d.domain[3];
  int c0, c1, c2, c3;
  // [axis][t][b] op-time segments of the batch-token walkers
  const struct {
    int off, op;
  } dense3[] = {{L.opt_emb, LS_OP_EMBEDDING}, {L.opt_qkv, LS_OP_QKV_PROJ}, {L.opt_out, LS_OP_ATTN_OUT_PROJ},
                {L.opt_sh1, LS_OP_SHARED_FFN1}, {L.opt_sh2, LS_OP_SHARED_FFN2}, {L.opt_lmh, LS_OP_LM_HEAD}};
  for (int k = 0; k < 6; ++k) {
    const int off = dense3[k].off, op = dense3[k].op;
    if ((op == LS_OP_SHARED_FFN1 || op == LS_OP_SHARED_FFN2) && !L.has_shared) continue;
    if (w >= off && w < off + 3 * nt * nb) {
      const int i = w - off, b = i % nb, t = (i / nb) % nt, a = i / (nb * nt);
      return dbits(op_cost_time(d, op, a, (double)B[b], TP[t], 1, false));
    }
  }
  // kv_cache_io / attn_core: [attn_dim1][t][b]
  if (w >= L.opt_kv && w < L.opt_kv + 2 * nt * nb) {
    const int i = w - L.opt_kv, b = i % nb, t = (i / nb) % nt, a2 = i / (nb * nt);
    return dbits(op_cost_time(d, LS_OP_KV_CACHE_IO, 0, (double)B[b], TP[t], 1, a2 != 0));
  }
  if (w >= L.opt_attn && w < L.opt_attn + 2 * nt * nb) {
    const int i = w - L.opt_attn, b = i % nb, t = (i / nb) % nt, a2 = i / (nb * nt);
    return dbits(op_cost_time(d, LS_OP_ATTN_CORE, a2 ? 2 : 0, (double)B[b], TP[t], 1, a2 != 0));
  }
  if (w >= L.opt_router && w < L.opt_router + nb)
    return dbits(op_cost_time(d, LS_OP_ROUTER_GATE, 0, (double)B[w - L.opt_router], 1, 1, false));
  if (w >= L.opt_norm && w < L.opt_norm + nb)
    return dbits(op_cost_time(d, LS_OP_FINAL_NORM, 0, (double)B[w - L.opt_norm], 1, 1, false));
  // expert ops: [axis][t][e][b], tokens = routed tokens
  for (int k = 0; k < 2; ++k) {
    const int off = k ? L.opt_ffn2 : L.opt_ffn1;
    if (w >= off && w < off + 3 * nt * ne * nb) {
      unflat(w - off, nt, ne, nb, &c0, &c1, &c2, &c3);
      const double rt = routed_tokens(d, B[c3], EP[c2]);
      return dbits(op_cost_time(d, k ? LS_OP_EXPERT_FFN2 : LS_OP_EXPERT_FFN1, c0, rt, TP[c1], EP[c2], false));
    }
  }
  // TP-group collectives: [cls][fam][t][b], tokens = batch
  if (w >= L.coll && w < L.coll + 8 * nt * nb) {
    unflat(w - L.coll, 2, nt, nb, &c0, &c1, &c2, &c3);
    const int64_t feats[4] = {qkv_out_dim(d), d.hidden_dim, d.ffn_dim, d.vocab_size};
    const double payload = ((double)B[c3] * (double)feats[c0]) * (double)d.dtype_bytes;
    return dbits(coll_time(d, c1 == 0, TP[c2], payload, TP[c2] <= d.node_size));
  }
  // routed ffn1->ffn2 reconcile: [fam][t][e][b], tokens = routed tokens
  if (w >= L.rtf && w < L.rtf + 2 * nt * ne * nb) {
    unflat(w - L.rtf, nt, ne, nb, &c0, &c1, &c2, &c3);
    const double payload = (routed_tokens(d, B[c3], EP[c2]) * (double)d.ffn_dim) * (double)d.dtype_bytes;
    return dbits(coll_time(d, c0 == 0, TP[c1], payload, TP[c1] <= d.node_size));
  }
  // expert dispatch / combine all_to_all: [t][e][b] over the EP group
  if (w >= L.a2a && w < L.a2a + nt * ne * nb) {
    unflat(w - L.a2a, 1, nt, ne * nb, &c0, &c1, &c2, &c3);
    const int t = c2, e = c3 / nb, b = c3 % nb;
    const double payload = (routed_tokens(d, B[b], EP[e]) * (double)d.hidden_dim) * (double)d.dtype_bytes;
    return dbits(coll_time(d, false, EP[e], payload, TP[t] * EP[e] <= d.node_size));
  }
  // gate entry per (t, e, p): word 0 = weights per device (memory_per_device,
  // simulator.py:147-150); word 1 = gate bits | kv row base << 32
  if (w >= L.tep && w < L.tep + 2 * nt * ne * np) {
    const int i = (w - L.tep) / 2, t = i / (ne * np), e = (i / np) % ne, p = i % np;
    if ((w - L.tep) % 2 == 0) return dbits(weights_mem(d, TP[t], EP[e], PP[p]));
    return (uint64_t)gate_bits(d, TP[t], EP[e], PP[p]) | ((uint64_t)((t * np + p) * nb) << 32);
  }
  // KV cache per device: [attn_dim1][t][p][b]
  if (w >= L.mem_kv && w < L.mem_kv + 2 * nt * np * nb) {
    unflat(w - L.mem_kv, nt, np, nb, &c0, &c1, &c2, &c3);
    return dbits(kv_mem(d, TP[c1], PP[c2], B[c3], c0 != 0));
  }
  if (w >= L.mem_ws && w < L.mem_ws + nb) return dbits(ws_mem(d, B[w - L.mem_ws]));
  if (L.coarse_words && w >= L.coarse && w < L.coarse + L.coarse_words) {
    const int c0i = 2 * (w - L.coarse), nc = nt * ne * np * nb;
    const uint64_t lo = c0i < nc ? coarse_word(d, L, c0i) : 0u, hi = c0i + 1 < nc ? coarse_word(d, L, c0i + 1) : 0u;
    return lo | (hi << 32);
  }
  // stage handoff hop: [intra][b]
  if (w >= L.hop && w < L.hop + 2 * nb) {
    const int i = w - L.hop, b = i % nb;
    return dbits(p2p_time(d, (double)(B[b] * d.hidden_dim * d.dtype_bytes), i / nb != 0));
  }
  if (w >= L.batch_d && w < L.batch_d + nb) return dbits((double)B[w - L.batch_d]);
  if (w >= L.lps_d && w < L.lps_d + np) return dbits((double)(d.num_layers / PP[w - L.lps_d]));
  if (w >= L.ppm1_d && w < L.ppm1_d + np) return dbits((double)(PP[w - L.ppm1_d] - 1));
  if (w >= L.tpv && w < L.tpv + nt) return (uint64_t)TP[w - L.tpv];
  if (w >= L.epv && w < L.epv + ne) return (uint64_t)EP[w - L.epv];
  if (w >= L.ppv && w < L.ppv + np) return (uint64_t)PP[w - L.ppv];
  return 0;  // padding
}

__global__ void build_tables_kernel(const ls_workload_desc d, const TabLayout L, uint64_t* out) {
  for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < L.words; w += gridDim.x * blockDim.x)
    out[w] = table_word(d, L, w);
}

}  // namespace

cudaError_t build_tables(const ls_workload_desc& d, const TabLayout& L, uint64_t* out, cudaStream_t stream) {
  const int threads = 256;
  int blocks = (L.words + threads - 1) / threads;
  if (blocks < 1) blocks = 1;
  build_tables_kernel<<<blocks, threads, 0, stream>>>(d, L, out);
  return cudaGetLastError();
}

namespace {
__global__ void tables_f32_kernel(const uint64_t* __restrict__ tab, int words, float* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < words) out[i] = (float)__longlong_as_double((long long)tab[i]);  // round to nearest
}
}  // namespace

// fp32 copy of every table word read as a double (only the time segments are
// read from it, by the fp32 fast mode of ls_sweep).
cudaError_t build_tables_f32(const uint64_t* tab, int words, float* out, cudaStream_t s) {
  tables_f32_kernel<<<(words + 255) / 256, 256, 0, s>>>(tab, words, out);
  return cudaGetLastError();
}

}  // namespace ls
