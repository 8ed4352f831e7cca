/*
 * shardsim_oracle.c — CPU restatement of the reference cost model.
 *
 * TEST INFRASTRUCTURE ONLY. This file is the parity checker for the CUDA
 * evaluator and the CPU baseline arm of bench.py. Nothing in the product path
 * (paper_2509_00217_b200/) links, loads or calls it.
 *
 * It restates, operation for operation, the reference's per-candidate path
 *     decode_strategy   pkg/src/shardsearch/strategy.py:245-263
 *     plan_layer        pkg/src/shardsearch/layout.py:347-456 (walker :301-344)
 *     simulate          pkg/src/shardsearch/simulator.py:239-341
 * as a direct state-machine walk (no precomputed tables) so it shares no
 * structure with the GPU kernel it checks. Every float expression keeps
 * Python's left-to-right evaluation order and int->double promotion point;
 * build with -ffp-contract=off so no FMA contraction changes a rounding.
 *
 * Pinned: tests/test_oracle_golden.py checks it bit-for-bit against golden
 * vectors produced by the reference itself (tests/golden/make_golden.py).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/ls_eval.h"

enum { AX_UNSHARDED = 0, AX_DIM0 = 1, AX_DIM1 = 2 };
/* Layout kinds (layout.py:34-37). A sharded layout carries its axis. */
enum { LK_REPLICATED = 0, LK_SHARDED = 1, LK_PARTIAL = 2 };
/* CollectiveKind (layout.py:40-46) */
enum { CK_NOOP = 0, CK_ALL_REDUCE, CK_ALL_GATHER, CK_REDUCE_SCATTER, CK_ALL_TO_ALL, CK_P2P };
/* OpClass (strategy.py:31-38) */
enum { OC_DENSE = 0, OC_MOE, OC_ATTN, OC_ROUTER, OC_ELEM };

typedef struct { int kind, axis; int64_t group; } layout_t;
typedef struct { int kind; int64_t group; double payload; int intra; } coll_t;
typedef struct { int op, axis; double tokens; int ncoll; coll_t coll[4]; } step_t;
typedef struct { int nsteps; step_t steps[12]; int nexit; coll_t exit[8]; } plan_t;

typedef struct {
  int64_t tp, ep, pp, batch;
  int axis[LS_NUM_OPS]; /* Strategy.axis_of per canonical op */
} strat_t;

/* _CANONICAL_OPS class and admissible shard axes (strategy.py:65-78). */
static const int k_op_class[LS_NUM_OPS] = {OC_DENSE, OC_DENSE, OC_ELEM,  OC_ATTN,
                                           OC_DENSE, OC_ROUTER, OC_MOE,  OC_MOE,
                                           OC_DENSE, OC_DENSE, OC_ELEM,  OC_DENSE};
/* bit a set: axis a admitted (UNSHARDED always). */
static const int k_admits[LS_NUM_OPS] = {7, 7, 1, 5, 7, 1, 7, 7, 7, 7, 1, 7};

/* TensorLayout constructors collapse to replicated on a one-device group
 * (layout.py:77-93). */
static layout_t mk(int kind, int axis, int64_t g) {
  layout_t l;
  if (g == 1) kind = LK_REPLICATED;
  l.kind = kind;
  l.axis = kind == LK_SHARDED ? axis : 0;
  l.group = g;
  return l;
}
static int leq(layout_t a, layout_t b) {
  return a.kind == b.kind && a.axis == b.axis && a.group == b.group;
}

/* transition, layout.py:119-155. Returns the collective kind, -1 on error. */
static int transition_kind(layout_t src, layout_t dst) {
  if (leq(src, dst)) return CK_NOOP;
  if (src.kind == LK_REPLICATED) return dst.kind == LK_SHARDED ? CK_NOOP : -1;
  if (src.kind == LK_SHARDED) {
    if (dst.kind == LK_REPLICATED) return CK_ALL_GATHER;
    if (dst.kind == LK_SHARDED) return CK_ALL_TO_ALL;
    return -1;
  }
  if (dst.kind == LK_REPLICATED) return CK_ALL_REDUCE;
  if (dst.kind == LK_SHARDED) return CK_REDUCE_SCATTER;
  return -1;
}

/* _shard_extent, layout.py:158-179; -1 when the op has no extent on axis. */
static int64_t shard_extent(const ls_workload_desc* m, int op, int axis) {
  int64_t h = m->hidden_dim;
  switch (op) {
    case LS_OP_EMBEDDING: return axis == AX_DIM0 ? m->vocab_size : h;
    case LS_OP_QKV_PROJ: return axis == AX_DIM0 ? h : m->num_heads;
    case LS_OP_ATTN_CORE: return axis == AX_DIM1 ? m->num_heads : -1;
    case LS_OP_ATTN_OUT_PROJ: return axis == AX_DIM0 ? m->num_heads : h;
    case LS_OP_EXPERT_FFN1:
    case LS_OP_SHARED_FFN1: return axis == AX_DIM0 ? h : m->ffn_dim;
    case LS_OP_EXPERT_FFN2:
    case LS_OP_SHARED_FFN2: return axis == AX_DIM0 ? m->ffn_dim : h;
    case LS_OP_LM_HEAD: return axis == AX_DIM0 ? h : m->vocab_size;
    default: return -1;
  }
}

/* _out_features, layout.py:284-298 */
static int64_t out_features(const ls_workload_desc* m, int op) {
  switch (op) {
    case LS_OP_EMBEDDING: return m->hidden_dim;
    case LS_OP_QKV_PROJ:
    case LS_OP_KV_CACHE_IO: return (m->num_heads + 2 * m->num_kv_heads) * m->head_dim;
    case LS_OP_ATTN_CORE: return m->num_heads * m->head_dim;
    case LS_OP_ATTN_OUT_PROJ: return m->hidden_dim;
    case LS_OP_ROUTER_GATE: return m->num_experts;
    case LS_OP_EXPERT_FFN1:
    case LS_OP_SHARED_FFN1: return m->ffn_dim;
    case LS_OP_EXPERT_FFN2:
    case LS_OP_SHARED_FFN2: return m->hidden_dim;
    case LS_OP_FINAL_NORM: return m->hidden_dim;
    default: return m->vocab_size;
  }
}

/* _required_input, layout.py:182-197. has_req=0 for elementwise ops. */
static layout_t required_input(int op, int axis, int64_t tp, int* has_req) {
  int cls = k_op_class[op];
  *has_req = 1;
  if (cls == OC_ELEM) {
    *has_req = 0;
    return mk(LK_REPLICATED, 0, tp);
  }
  if (cls == OC_ROUTER) return mk(LK_REPLICATED, 0, tp);
  if (cls == OC_ATTN) return axis == AX_DIM1 ? mk(LK_SHARDED, AX_DIM1, tp) : mk(LK_REPLICATED, 0, tp);
  return axis == AX_DIM0 ? mk(LK_SHARDED, AX_DIM1, tp) : mk(LK_REPLICATED, 0, tp);
}

/* infer_output_layout, layout.py:200-240. Returns 0, or -1 for LayoutError. */
static int infer_output(const ls_workload_desc* m, int op, layout_t in, int axis, layout_t* out) {
  int64_t tp = in.group;
  int has_req;
  layout_t req;
  int cls = k_op_class[op];
  if (!((k_admits[op] >> axis) & 1)) return -1;
  if (axis != AX_UNSHARDED && tp > 1) {
    int64_t ext = shard_extent(m, op, axis);
    if (ext < 0 || ext % tp != 0) return -1;
  }
  req = required_input(op, axis, tp, &has_req);
  if (has_req && !leq(in, req)) return -1;
  if (cls == OC_ELEM) *out = in;
  else if (cls == OC_ROUTER) *out = mk(LK_REPLICATED, 0, tp);
  else if (cls == OC_ATTN) *out = axis == AX_DIM1 ? mk(LK_SHARDED, AX_DIM1, tp) : mk(LK_REPLICATED, 0, tp);
  else if (axis == AX_UNSHARDED) *out = mk(LK_REPLICATED, 0, tp);
  else if (axis == AX_DIM1) *out = mk(LK_SHARDED, AX_DIM1, tp);
  else *out = mk(LK_PARTIAL, 0, tp);
  return 0;
}

/* _Walker, layout.py:301-344 */
typedef struct {
  const ls_workload_desc* m;
  const strat_t* s;
  double tokens;
  int tp_intra;
  layout_t state;
  int64_t features;
  int npending;
  coll_t pending[8];
  int nsteps;
  step_t steps[12];
} walker_t;

static void walker_init(walker_t* w, const ls_workload_desc* m, const strat_t* s, double tokens, int tp_intra) {
  w->m = m;
  w->s = s;
  w->tokens = tokens;
  w->tp_intra = tp_intra;
  w->state = mk(LK_REPLICATED, 0, s->tp);
  w->features = m->hidden_dim;
  w->npending = 0;
  w->nsteps = 0;
}

/* _Walker.tensor_bytes: tokens * features * dtype, left to right. */
static double walker_bytes(const walker_t* w) {
  return w->tokens * (double)w->features * (double)w->m->dtype_bytes;
}

static int walker_reconcile(walker_t* w, layout_t target) {
  int kind;
  if (leq(w->state, target)) return 0;
  kind = transition_kind(w->state, target);
  if (kind < 0) return -1;
  if (kind != CK_NOOP) {
    coll_t c;
    c.kind = kind;
    c.group = w->state.group;
    c.payload = walker_bytes(w);
    c.intra = w->tp_intra;
    w->pending[w->npending++] = c;
  }
  w->state = target;
  return 0;
}

static int walker_run_op(walker_t* w, int op) {
  int axis = w->s->axis[op], has_req, i;
  layout_t req = required_input(op, axis, w->s->tp, &has_req), out;
  step_t* st;
  if (has_req && walker_reconcile(w, req)) return -1;
  if (infer_output(w->m, op, w->state, axis, &out)) return -1;
  st = &w->steps[w->nsteps++];
  st->op = op;
  st->axis = axis;
  st->tokens = w->tokens;
  st->ncoll = w->npending;
  for (i = 0; i < w->npending; ++i) st->coll[i] = w->pending[i];
  w->npending = 0;
  w->state = out;
  w->features = out_features(w->m, op);
  return 0;
}

/* plan_layer, layout.py:347-456. ops: canonical indices in walk order.
 * Returns 0, or -1 on LayoutError. */
static int plan_layer(const ls_workload_desc* m, const int* ops, int nops, const strat_t* s, plan_t* plan) {
  int64_t tp = s->tp, ep = s->ep;
  int tp_intra = tp <= m->node_size;
  int ep_intra = tp * ep <= m->node_size;
  int i, has_expert = 0, branch = nops, has_shared = 0;
  walker_t w;
  for (i = 0; i < nops; ++i) {
    if (ops[i] == LS_OP_EXPERT_FFN1 || ops[i] == LS_OP_EXPERT_FFN2) has_expert = 1;
    if (ops[i] == LS_OP_SHARED_FFN1) has_shared = 1;
    if (ops[i] == LS_OP_ROUTER_GATE && branch == nops) branch = i;
  }
  if (has_expert) {
    if (ep > m->num_experts) return -1;
    if (m->num_experts % ep != 0) return -1;
  }
  walker_init(&w, m, s, (double)s->batch, tp_intra);
  for (i = 0; i < branch; ++i) {
    if (walker_run_op(&w, ops[i])) return -1;
    if (ops[i] == LS_OP_ATTN_OUT_PROJ && walker_reconcile(&w, mk(LK_REPLICATED, 0, tp))) return -1;
  }
  if (branch < nops) {
    walker_t ew, sw;
    double routed, dispatch_bytes;
    layout_t expert_state, shared_state;
    int64_t hidden_bytes;
    coll_t a2a;
    if (walker_run_op(&w, LS_OP_ROUTER_GATE)) return -1;
    w.state = mk(LK_REPLICATED, 0, tp);
    w.features = m->hidden_dim;

    /* routed_tokens = batch * top_k / ep (int product, true division) */
    routed = (double)(s->batch * m->experts_per_token) / (double)ep;
    dispatch_bytes = routed * (double)m->hidden_dim * (double)m->dtype_bytes;
    walker_init(&ew, m, s, routed, tp_intra);
    a2a.kind = CK_ALL_TO_ALL;
    a2a.group = ep;
    a2a.payload = dispatch_bytes;
    a2a.intra = ep_intra;
    if (ep > 1) ew.pending[ew.npending++] = a2a;
    if (walker_run_op(&ew, LS_OP_EXPERT_FFN1)) return -1;
    if (walker_run_op(&ew, LS_OP_EXPERT_FFN2)) return -1;
    /* expert_exit = leftover pending + combine */
    expert_state = ew.state;

    if (has_shared) {
      walker_init(&sw, m, s, (double)s->batch, tp_intra);
      if (walker_run_op(&sw, LS_OP_SHARED_FFN1)) return -1;
      if (walker_run_op(&sw, LS_OP_SHARED_FFN2)) return -1;
      shared_state = sw.state;
    }
    for (i = 0; i < ew.nsteps; ++i) w.steps[w.nsteps++] = ew.steps[i];
    for (i = 0; i < ew.npending; ++i) w.pending[w.npending++] = ew.pending[i];
    if (ep > 1) w.pending[w.npending++] = a2a;
    if (has_shared) {
      for (i = 0; i < sw.nsteps; ++i) w.steps[w.nsteps++] = sw.steps[i];
      for (i = 0; i < sw.npending; ++i) w.pending[w.npending++] = sw.pending[i];
    }
    hidden_bytes = s->batch * m->hidden_dim * m->dtype_bytes;
    if (has_shared && !leq(shared_state, expert_state)) {
      layout_t sides[2];
      int k;
      sides[0] = expert_state;
      sides[1] = shared_state;
      for (k = 0; k < 2; ++k) {
        int kind = transition_kind(sides[k], mk(LK_REPLICATED, 0, tp));
        if (kind < 0) return -1;
        if (kind != CK_NOOP) {
          coll_t c;
          c.kind = kind;
          c.group = sides[k].group;
          c.payload = (double)hidden_bytes;
          c.intra = tp_intra;
          w.pending[w.npending++] = c;
        }
      }
      w.state = mk(LK_REPLICATED, 0, tp);
    } else {
      w.state = expert_state;
    }
    w.features = m->hidden_dim;
  }
  if (walker_reconcile(&w, mk(LK_REPLICATED, 0, tp))) return -1;
  plan->nsteps = w.nsteps;
  for (i = 0; i < w.nsteps; ++i) plan->steps[i] = w.steps[i];
  plan->nexit = w.npending;
  for (i = 0; i < w.npending; ++i) plan->exit[i] = w.pending[i];
  return 0;
}

/* ---- roofline cost model, simulator.py ---- */

/* Python max(a, b) / min(a, b): the first argument wins ties. */
static double py_max(double a, double b) { return b > a ? b : a; }
static double py_min(double a, double b) { return b < a ? b : a; }

/* op_time, simulator.py:100-104 */
static double op_time(double flops, double bytes, const ls_workload_desc* m) {
  return py_max(flops / m->peak_flops, bytes / m->hbm_bandwidth) + m->kernel_overhead;
}

/* ceil(log2 n) for n >= 1 as an integer bit length (simulator.py:115). */
static int64_t ceil_log2(int64_t n) {
  int64_t h = 0, v = n - 1;
  while (v > 0) {
    ++h;
    v >>= 1;
  }
  return h;
}

/* collective_time, simulator.py:107-120 */
static double collective_time(const coll_t* c, const ls_workload_desc* m) {
  int64_t n = c->group;
  double bw, volume;
  if (c->kind == CK_NOOP || n <= 1) return 0.0;
  bw = c->intra ? m->intra_node_bw : m->inter_node_bw;
  if (c->kind == CK_P2P) return c->payload / bw + m->per_collective_latency;
  if (c->kind == CK_ALL_REDUCE)
    volume = ((2.0 * (double)(n - 1)) / (double)n) * c->payload;
  else
    volume = ((double)(n - 1) / (double)n) * c->payload;
  return volume / bw + m->per_collective_latency * (double)ceil_log2(n);
}

/* _kv_share, simulator.py:123-132 */
static int64_t kv_share(const ls_workload_desc* m, const strat_t* s) {
  if (s->axis[LS_OP_ATTN_CORE] == AX_DIM1) return s->tp < m->num_kv_heads ? s->tp : m->num_kv_heads;
  return 1;
}

/* memory_per_device, simulator.py:135-160 (count_parameters, model.py:149-170) */
static double memory_per_device(const ls_workload_desc* m, const strat_t* s) {
  int64_t h = m->hidden_dim, d = m->dtype_bytes;
  int64_t qkv_out = (m->num_heads + 2 * m->num_kv_heads) * m->head_dim;
  int64_t per_layer_attn = h * qkv_out + m->num_heads * m->head_dim * h;
  int64_t per_layer_router = h * m->num_experts;
  int64_t per_expert = 2 * h * m->ffn_dim;
  int64_t per_layer_norms = 4 * h;
  int64_t shared = m->has_shared_expert ? per_expert : 0;
  int64_t embedding = m->vocab_size * h, lm_head = m->vocab_size * h;
  int64_t attention = m->num_layers * per_layer_attn;
  int64_t router = m->num_layers * per_layer_router;
  int64_t routed = m->num_layers * m->num_experts * per_expert;
  int64_t shared_total = m->num_layers * shared;
  int64_t norms = m->num_layers * per_layer_norms + h;
  int64_t dense = embedding + lm_head + attention + router + shared_total + norms;
  double weight = ((double)(dense * d) / (double)s->tp) / (double)s->pp +
                  ((double)(routed * d) / (double)(s->ep * s->tp)) / (double)s->pp;
  double kv = ((((2.0 * ((double)m->num_layers / (double)s->pp)) *
                 ((double)(m->num_kv_heads * m->head_dim) / (double)kv_share(m, s))) *
                (double)m->context_len) *
               (double)s->batch) *
              (double)d;
  double workspace = ((2.0 * (double)s->batch) * (double)(h + m->ffn_dim)) * (double)d;
  return (weight + kv) + workspace;
}

/* matmul helper inside _op_cost, simulator.py:178-185 */
static void matmul(double t, int64_t in, int64_t outd, double wc, int64_t s, int64_t d, double* flops, double* bytes) {
  double weight, act;
  *flops = (((2.0 * t) * (double)in) * (double)outd) / (double)s;
  weight = (((wc * (double)in) * (double)outd) * (double)d) / (double)s;
  act = (t * (double)(in + outd)) * (double)d;
  *bytes = weight + act;
}

/* _op_cost, simulator.py:163-221 */
static void op_cost(const step_t* st, const ls_workload_desc* m, const strat_t* s, double* flops, double* bytes) {
  double t = st->tokens;
  int64_t h = m->hidden_dim, d = m->dtype_bytes;
  int64_t sdiv = st->axis != AX_UNSHARDED ? s->tp : 1;
  int64_t qkv_out = (m->num_heads + 2 * m->num_kv_heads) * m->head_dim;
  switch (st->op) {
    case LS_OP_EMBEDDING:
      *flops = 0.0;
      *bytes = (((2.0 * t) * (double)h) * (double)d) / (double)sdiv;
      return;
    case LS_OP_QKV_PROJ: matmul(t, h, qkv_out, 1.0, sdiv, d, flops, bytes); return;
    case LS_OP_KV_CACHE_IO: {
      int64_t share = kv_share(m, s);
      *flops = 0.0;
      *bytes = ((((t * 2.0) * (double)m->num_kv_heads) * (double)m->head_dim) * (double)d) / (double)share;
      return;
    }
    case LS_OP_ATTN_CORE: {
      double hl = (double)m->num_heads / (double)sdiv;
      int64_t share = kv_share(m, s);
      double kv_read = ((((t * (double)m->context_len) * 2.0) * ((double)m->num_kv_heads / (double)share)) *
                        (double)m->head_dim) *
                       (double)d;
      double q_io = (((2.0 * t) * hl) * (double)m->head_dim) * (double)d;
      *flops = (((4.0 * t) * hl) * (double)m->head_dim) * (double)m->context_len;
      *bytes = kv_read + q_io;
      return;
    }
    case LS_OP_ATTN_OUT_PROJ: matmul(t, m->num_heads * m->head_dim, h, 1.0, sdiv, d, flops, bytes); return;
    case LS_OP_ROUTER_GATE: matmul(t, h, m->num_experts, 1.0, sdiv, d, flops, bytes); return;
    case LS_OP_EXPERT_FFN1:
    case LS_OP_EXPERT_FFN2: {
      double local = (double)m->num_experts / (double)s->ep;
      double active = t > 0 ? py_min(local, t) : 0.0;
      if (st->op == LS_OP_EXPERT_FFN1) matmul(t, h, m->ffn_dim, active, sdiv, d, flops, bytes);
      else matmul(t, m->ffn_dim, h, active, sdiv, d, flops, bytes);
      return;
    }
    case LS_OP_SHARED_FFN1: matmul(t, h, m->ffn_dim, 1.0, sdiv, d, flops, bytes); return;
    case LS_OP_SHARED_FFN2: matmul(t, m->ffn_dim, h, 1.0, sdiv, d, flops, bytes); return;
    case LS_OP_FINAL_NORM:
      *flops = (8.0 * t) * (double)h;
      *bytes = ((2.0 * t) * (double)h) * (double)d;
      return;
    default: matmul(t, h, m->vocab_size, 1.0, sdiv, d, flops, bytes); return;
  }
}

/* builtin sum() over floats with int start 0 (CPython bltinmodule.c):
 * naive left fold (<= 3.11) or Neumaier compensation (>= 3.12). */
typedef struct { double f, c; int n, mode; } pysum_t;
static void pysum_init(pysum_t* a, int mode) {
  a->f = 0.0;
  a->c = 0.0;
  a->n = 0;
  a->mode = mode;
}
static void pysum_add(pysum_t* a, double x) {
  if (a->n++ == 0) {
    a->f = 0.0 + x;
    return;
  }
  if (a->mode == LS_SUM_NEUMAIER) {
    double t = a->f + x;
    if (fabs(a->f) >= fabs(x)) a->c += (a->f - t) + x;
    else a->c += (x - t) + a->f;
    a->f = t;
  } else {
    a->f = a->f + x;
  }
}
static double pysum_result(const pysum_t* a) {
  if (a->mode == LS_SUM_NEUMAIER && a->c != 0.0 && isfinite(a->c)) return a->f + a->c;
  return a->f;
}

/* _plan_times, simulator.py:224-236 */
static void plan_times(const plan_t* p, const ls_workload_desc* m, const strat_t* s, double* comp, double* comm) {
  pysum_t a, b;
  int i, j;
  pysum_init(&a, (int)m->sum_mode);
  pysum_init(&b, (int)m->sum_mode);
  for (i = 0; i < p->nsteps; ++i) {
    double fl, by;
    op_cost(&p->steps[i], m, s, &fl, &by);
    pysum_add(&a, op_time(fl, by, m));
  }
  /* LayerPlan.all_collectives order, layout.py:270-275 */
  for (i = 0; i < p->nsteps; ++i)
    for (j = 0; j < p->steps[i].ncoll; ++j) pysum_add(&b, collective_time(&p->steps[i].coll[j], m));
  for (i = 0; i < p->nexit; ++i) pysum_add(&b, collective_time(&p->exit[i], m));
  *comp = pysum_result(&a);
  *comm = pysum_result(&b);
}

typedef struct {
  uint8_t reason;
  double throughput, tpot, memory, compute, comm, pipeline;
} or_result;

/* simulate, simulator.py:239-341, on an already decoded strategy. */
static void simulate(const ls_workload_desc* m, const strat_t* s, or_result* r) {
  int layer_ops[9], n_layer = 0, pre_ops[1] = {LS_OP_EMBEDDING}, post_ops[2] = {LS_OP_FINAL_NORM, LS_OP_LM_HEAD};
  plan_t lp, pp_, po;
  int64_t world = s->tp * s->ep * s->pp;
  double memory, lc, lm, prc, prm, poc, pom, hop_s, compute, comm, pipe, tpot, body, c0, cmax, thr;
  int k;
  memset(r, 0, sizeof(*r));
  if (world > m->device_budget) {
    r->reason = LS_REASON_OVER_DEVICE_BUDGET;
    return;
  }
  for (k = LS_OP_QKV_PROJ; k <= LS_OP_SHARED_FFN2; ++k) {
    if ((k == LS_OP_SHARED_FFN1 || k == LS_OP_SHARED_FFN2) && !m->has_shared_expert) continue;
    layer_ops[n_layer++] = k;
  }
  if (m->num_layers % s->pp != 0 || plan_layer(m, layer_ops, n_layer, s, &lp) || plan_layer(m, pre_ops, 1, s, &pp_) ||
      plan_layer(m, post_ops, 2, s, &po)) {
    r->reason = LS_REASON_LAYOUT_ERROR;
    return;
  }
  memory = memory_per_device(m, s);
  if (memory > m->hbm_capacity) {
    r->reason = LS_REASON_OOM;
    r->memory = memory;
    return;
  }
  plan_times(&lp, m, s, &lc, &lm);
  plan_times(&pp_, m, s, &prc, &prm);
  plan_times(&po, m, s, &poc, &pom);
  {
    coll_t hop;
    hop.kind = CK_P2P;
    hop.group = 2;
    hop.payload = (double)(s->batch * m->hidden_dim * m->dtype_bytes);
    hop.intra = world <= m->node_size;
    hop_s = s->pp > 1 ? collective_time(&hop, m) : 0.0;
  }
  compute = ((double)m->num_layers * lc + prc) + poc;
  comm = ((double)m->num_layers * lm + prm) + pom;
  pipe = (double)(s->pp - 1) * hop_s;
  tpot = (compute + comm) + pipe;
  body = (double)(m->num_layers / s->pp) * (lc + lm);
  /* stage cycles, simulator.py:311-322 (max keeps the first of equals) */
  c0 = body + (prc + prm);
  if (s->pp == 1) {
    cmax = c0 + (poc + pom);
  } else {
    int64_t st;
    cmax = c0 + hop_s;
    for (st = 1; st < s->pp; ++st) {
      double cyc = st == s->pp - 1 ? body + (poc + pom) : body + hop_s;
      cmax = py_max(cmax, cyc);
    }
  }
  thr = ((double)s->batch / cmax) / (double)world;
  r->tpot = tpot;
  r->memory = memory;
  r->compute = compute;
  r->comm = comm;
  r->pipeline = pipe;
  if (tpot > m->slo_tpot) {
    r->reason = LS_REASON_SLO_VIOLATION;
    return;
  }
  r->reason = LS_REASON_NONE;
  r->throughput = thr;
}

/* decode_strategy, strategy.py:245-263, from one SoA column. */
static int decode(const ls_workload_desc* m, const uint8_t* planes, int64_t stride, int64_t i, strat_t* s) {
  int h, k;
  int v[LS_MAX_HEADS];
  for (h = 0; h < m->vector_length; ++h) {
    int size = h < 4 ? m->domain_len[h] : 3;
    v[h] = planes[(int64_t)h * stride + i];
    if (v[h] >= size) return -1;
  }
  s->tp = m->domain[0][v[0]];
  s->ep = m->domain[1][v[1]];
  s->pp = m->domain[2][v[2]];
  s->batch = m->domain[3][v[3]];
  for (k = 0; k < LS_NUM_OPS; ++k) s->axis[k] = m->op_head[k] >= 0 ? v[(int)m->op_head[k]] : m->op_pinned[k];
  return 0;
}

/* ---- exported entry points (ctypes from tests/ and bench.py) ---- */

int or_simulate_batch_range(const ls_workload_desc* m, const uint8_t* planes, int64_t stride, int64_t lo, int64_t hi,
                            uint8_t* reason, double* thr, double* tpot, double* mem, double* comp, double* comm,
                            double* pipe) {
  int64_t i;
  for (i = lo; i < hi; ++i) {
    strat_t s;
    or_result r;
    if (decode(m, planes, stride, i, &s)) {
      memset(&r, 0, sizeof(r));
      r.reason = LS_REASON_DECODE_ERROR;
    } else {
      simulate(m, &s, &r);
    }
    reason[i] = r.reason;
    if (thr) thr[i] = r.throughput;
    if (tpot) tpot[i] = r.tpot;
    if (mem) mem[i] = r.memory;
    if (comp) comp[i] = r.compute;
    if (comm) comm[i] = r.comm;
    if (pipe) pipe[i] = r.pipeline;
  }
  return 0;
}

typedef struct {
  const ls_workload_desc* m;
  const uint8_t* planes;
  int64_t stride, lo, hi;
  uint8_t* reason;
  double *thr, *tpot, *mem, *comp, *comm, *pipe;
} job_t;

static void* run_job(void* arg) {
  job_t* j = (job_t*)arg;
  or_simulate_batch_range(j->m, j->planes, j->stride, j->lo, j->hi, j->reason, j->thr, j->tpot, j->mem, j->comp,
                          j->comm, j->pipe);
  return NULL;
}

/* Multi-threaded batch: contiguous slices over `threads` pthreads. */
int or_simulate_batch(const ls_workload_desc* m, const uint8_t* planes, int64_t stride, int64_t n, uint8_t* reason,
                      double* thr, double* tpot, double* mem, double* comp, double* comm, double* pipe, int threads) {
  pthread_t tid[256];
  job_t jobs[256];
  int t;
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  for (t = 0; t < threads; ++t) {
    jobs[t].m = m;
    jobs[t].planes = planes;
    jobs[t].stride = stride;
    jobs[t].lo = n * t / threads;
    jobs[t].hi = n * (t + 1) / threads;
    jobs[t].reason = reason;
    jobs[t].thr = thr;
    jobs[t].tpot = tpot;
    jobs[t].mem = mem;
    jobs[t].comp = comp;
    jobs[t].comm = comm;
    jobs[t].pipe = pipe;
    if (threads == 1) run_job(&jobs[t]);
    else pthread_create(&tid[t], NULL, run_job, &jobs[t]);
  }
  if (threads > 1)
    for (t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
  return 0;
}

/* Plan introspection for tests: kinds/groups/payloads of the layer plan's
 * all_collectives() in order. Returns count, or -1 on layout error. */
int or_layer_plan(const ls_workload_desc* m, const uint8_t* vec, int* kinds, int64_t* groups, double* payloads,
                  int* intra, int cap) {
  strat_t s;
  plan_t p;
  int layer_ops[9], n = 0, k, i, j, c = 0;
  if (decode(m, vec, 1, 0, &s)) return -2;
  for (k = LS_OP_QKV_PROJ; k <= LS_OP_SHARED_FFN2; ++k) {
    if ((k == LS_OP_SHARED_FFN1 || k == LS_OP_SHARED_FFN2) && !m->has_shared_expert) continue;
    layer_ops[n++] = k;
  }
  if (plan_layer(m, layer_ops, n, &s, &p)) return -1;
  for (i = 0; i < p.nsteps; ++i)
    for (j = 0; j < p.steps[i].ncoll; ++j, ++c)
      if (c < cap) {
        kinds[c] = p.steps[i].coll[j].kind;
        groups[c] = p.steps[i].coll[j].group;
        payloads[c] = p.steps[i].coll[j].payload;
        intra[c] = p.steps[i].coll[j].intra;
      }
  for (i = 0; i < p.nexit; ++i, ++c)
    if (c < cap) {
      kinds[c] = p.exit[i].kind;
      groups[c] = p.exit[i].group;
      payloads[c] = p.exit[i].payload;
      intra[c] = p.exit[i].intra;
    }
  return c;
}
