// ls_evaluate.cuh — per-candidate scoring on the device (table-driven).
//
// score() restates simulate() (simulator.py:239-341) for one decoded
// candidate: gate order budget -> layout -> memory -> SLO, the layer/pre/post
// plan walk of plan_layer (layout.py:347-456) reduced to the layout-state
// algebra on axis codes, Python-sum() accumulation (simulator.py:232-235) of
// table-gathered op and collective times, then the pipeline totals.
#pragma once
#include <stdint.h>

#include "ls_formulas.cuh"
#include "ls_tables.cuh"

namespace ls {

struct Verdict {
  uint32_t reason;
  double thr, tpot, mem, comp, comm, pipe;
};

// CPython builtin sum() over floats with int start 0: Neumaier compensation
// from 3.12 (NEU) or the naive left fold before it.
template <bool NEU>
struct PySum {
  double f, c;
  __device__ __forceinline__ void first(double x) {
    f = 0.0 + x;
    c = 0.0;
  }
  __device__ __forceinline__ void add(double x) {
    const double t = f + x;
    if (NEU) c += fabs(f) >= fabs(x) ? (f - t) + x : (x - t) + f;
    f = t;
  }
  __device__ __forceinline__ double result() const {
    if (NEU && c != 0.0 && isfinite(c)) return f + c;
    return f;
  }
};

// Collective family of reconciling producer state `from` to demand `to`
// (transition, layout.py:119-155; states are axis codes, see ST_*):
// R->* none, S->S none, S->R all_gather, P->S reduce_scatter, P->R all_reduce.
__device__ __forceinline__ int fam(int from, int to) {
  if (from == ST_R) return FAM_NONE;
  if (from == ST_S) return to == ST_S ? FAM_NONE : FAM_ONCE;
  return to == ST_S ? FAM_ONCE : FAM_AR;
}
// Input demanded by a matmul under `axis` (_required_input, layout.py:194-197).
__device__ __forceinline__ int req(int axis) { return axis == 1 ? ST_S : ST_R; }

__device__ __forceinline__ double dget(const uint64_t* T, int i) {
  return __longlong_as_double((long long)T[i]);
}

template <bool NEU>
struct Accum {
  PySum<NEU> s;
  int n;
  __device__ __forceinline__ void init() { n = 0; }
  __device__ __forceinline__ void push(double x) {
    if (n++ == 0) s.first(x);
    else s.add(x);
  }
  __device__ __forceinline__ double result() const { return n ? s.result() : 0.0; }
};

// Score one decoded candidate. t,e,p,b: domain indices; X: 2-bit axis per
// canonical op. Returns reason; fills v per SimResult field conventions.
template <bool NEU>
__device__ __forceinline__ void score(const uint64_t* __restrict__ T, const TabLayout& L, const EvalMeta& M, int t,
                                      int e, int p, int b, uint32_t X, Verdict& v) {
  v.thr = v.tpot = v.mem = v.comp = v.comm = v.pipe = 0.0;
  // gate 1: world_size > device_budget (simulator.py:257)
  if ((T[L.ovb + t * L.ne + e] >> p) & 1) {
    v.reason = LS_REASON_OVER_DEVICE_BUDGET;
    return;
  }
  // gate 2: pp | num_layers, ep vs num_experts, per-op admissibility and
  // extent divisibility (simulator.py:268, layout.py:371-374, :214-221)
  {
    const uint32_t lo = X & 0x555555u, hi = (X >> 1) & 0x555555u;
    const uint64_t bad = ((~(lo | hi) & 0x555555u) & T[L.bad + t]) | ((lo & ~hi) & T[L.bad + L.nt + t]) |
                         ((hi & ~lo) & T[L.bad + 2 * L.nt + t]);
    if (bad | ((M.pp_bad >> p) & 1) | ((M.ep_bad >> e) & 1)) {
      v.reason = LS_REASON_LAYOUT_ERROR;
      return;
    }
  }
  const int ax_emb = X & 3, ax_qkv = (X >> 2) & 3, ax_attn = (X >> 6) & 3, ax_out = (X >> 8) & 3;
  const int ax_f1 = (X >> 12) & 3, ax_f2 = (X >> 14) & 3, ax_s1 = (X >> 16) & 3, ax_s2 = (X >> 18) & 3;
  const int ax_lmh = (X >> 22) & 3;
  const int a2 = ax_attn == 2;
  const int nt = L.nt, ne = L.ne, np = L.np, nb = L.nb;

  // gate 3: memory_per_device > hbm_capacity (simulator.py:135-160, :279)
  const double mem = (dget(T, L.mem_w + (t * ne + e) * np + p) + dget(T, L.mem_kv + ((a2 * nt + t) * np + p) * nb + b)) +
                     dget(T, L.mem_ws + b);
  v.mem = mem;
  if (mem > M.hbm_capacity) {
    v.reason = LS_REASON_OOM;
    return;
  }

  const int tb = t * nb + b, teb = (t * ne + e) * nb + b;
  const bool tp_gt1 = (int64_t)T[L.tpv + t] > 1;
  const bool ep_gt1 = (int64_t)T[L.epv + e] > 1;

  // layer plan compute: qkv, kv, attn, out, router, ffn1, ffn2[, sh1, sh2]
  Accum<NEU> lc;
  lc.init();
  lc.push(dget(T, L.opt_qkv + ax_qkv * nt * nb + tb));
  lc.push(dget(T, L.opt_kv + a2 * nt * nb + tb));
  lc.push(dget(T, L.opt_attn + a2 * nt * nb + tb));
  lc.push(dget(T, L.opt_out + ax_out * nt * nb + tb));
  lc.push(dget(T, L.opt_router + b));
  lc.push(dget(T, L.opt_ffn1 + ax_f1 * nt * ne * nb + teb));
  lc.push(dget(T, L.opt_ffn2 + ax_f2 * nt * ne * nb + teb));
  if (L.has_shared) {
    lc.push(dget(T, L.opt_sh1 + ax_s1 * nt * nb + tb));
    lc.push(dget(T, L.opt_sh2 + ax_s2 * nt * nb + tb));
  }
  // layer plan collectives in all_collectives() order (layout.py:270-275)
  Accum<NEU> lm;
  lm.init();
  const int coll_cls = L.coll;  // [cls][fam-1][t][b]
#define LS_TP_COLL(cls, f) dget(T, coll_cls + ((cls) * 2 + ((f) - 1)) * nt * nb + tb)
  const int st_attn = a2 ? ST_S : ST_R;
  if (tp_gt1) {
    int f;
    if ((f = fam(ax_qkv, st_attn))) lm.push(LS_TP_COLL(CLS_QKV, f));  // feed attn_core
    if ((f = fam(st_attn, req(ax_out)))) lm.push(LS_TP_COLL(CLS_H, f));  // feed attn_out_proj
    if ((f = fam(ax_out, ST_R))) lm.push(LS_TP_COLL(CLS_H, f));          // attention residual
  }
  const double a2a = ep_gt1 ? dget(T, L.a2a + teb) : 0.0;
  if (ep_gt1) lm.push(a2a);  // expert dispatch
  if (tp_gt1) {
    int f;
    if ((f = fam(ax_f1, req(ax_f2)))) lm.push(dget(T, L.rtf + (f - 1) * nt * ne * nb + teb));  // feed ffn2
    if (L.has_shared && (f = fam(ax_s1, req(ax_s2)))) lm.push(LS_TP_COLL(CLS_F, f));        // feed sh2
  }
  if (ep_gt1) lm.push(a2a);  // expert combine
  if (tp_gt1) {
    int f;
    if (L.has_shared && ax_s2 != ax_f2) {  // branch outputs disagree: align both
      if ((f = fam(ax_f2, ST_R))) lm.push(LS_TP_COLL(CLS_H, f));
      if ((f = fam(ax_s2, ST_R))) lm.push(LS_TP_COLL(CLS_H, f));
    } else if ((f = fam(ax_f2, ST_R))) {  // layer exit
      lm.push(LS_TP_COLL(CLS_H, f));
    }
  }
  const double layer_c = lc.result(), layer_m = lm.result();

  // pre plan (embedding) and post plan (final_norm, lm_head)
  const double pre_c = 0.0 + dget(T, L.opt_emb + ax_emb * nt * nb + tb);
  double pre_m = 0.0, post_m = 0.0;
  if (tp_gt1) {
    int f;
    if ((f = fam(ax_emb, ST_R))) pre_m = 0.0 + LS_TP_COLL(CLS_H, f);
    if ((f = fam(ax_lmh, ST_R))) post_m = 0.0 + LS_TP_COLL(CLS_V, f);
  }
#undef LS_TP_COLL
  PySum<NEU> po;
  po.first(dget(T, L.opt_norm + b));
  po.add(dget(T, L.opt_lmh + ax_lmh * nt * nb + tb));
  const double post_c = po.result();

  // totals and pipeline stages (simulator.py:286-323)
  const int64_t tpv = (int64_t)T[L.tpv + t], epv = (int64_t)T[L.epv + e], ppv = (int64_t)T[L.ppv + p];
  const int64_t world = tpv * epv * ppv;
  const double hop = ppv > 1 ? dget(T, L.hop + (world <= M.node_size ? nb : 0) + b) : 0.0;
  const double compute = (M.num_layers_d * layer_c + pre_c) + post_c;
  const double comm = (M.num_layers_d * layer_m + pre_m) + post_m;
  const double pipe = dget(T, L.ppm1_d + p) * hop;
  const double tpot = (compute + comm) + pipe;
  const double body = dget(T, L.lps_d + p) * (layer_c + layer_m);
  const double c0 = body + (pre_c + pre_m);
  double cmax;
  if (ppv == 1) {
    cmax = c0 + (post_c + post_m);
  } else {
    cmax = c0 + hop;
    if (ppv > 2) cmax = py_max(cmax, body + hop);
    cmax = py_max(cmax, body + (post_c + post_m));
  }
  v.tpot = tpot;
  v.comp = compute;
  v.comm = comm;
  v.pipe = pipe;
  // gate 4: tpot > slo_tpot (simulator.py:325)
  if (tpot > M.slo_tpot) {
    v.reason = LS_REASON_SLO_VIOLATION;
    return;
  }
  v.reason = LS_REASON_NONE;
  v.thr = (dget(T, L.batch_d + b) / cmax) / (double)world;
}

}  // namespace ls
