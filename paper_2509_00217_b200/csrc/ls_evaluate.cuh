// ls_evaluate.cuh — per-candidate scoring on the device (table-driven).
//
// simulate() (simulator.py:239-341) split in two passes:
//   gate()      integer/bitmask gates in the reference's order — device
//               budget (:257), layout (:268, layout.py:371-374, :214-221) —
//               then the memory model (:135-160, :279). Every candidate.
//   full_path() only for candidates that fit in memory: the plan walk of
//               plan_layer (layout.py:347-456) reduced to the layout-state
//               algebra on axis codes, Python-sum() accumulation
//               (simulator.py:232-235) of table-gathered op and collective
//               times, pipeline totals (:286-323) and the SLO gate (:325).
#pragma once
#include <stdint.h>

#include <type_traits>

#include "ls_formulas.cuh"
#include "ls_tables.cuh"

namespace ls {

struct Verdict {
  uint32_t reason;
  double thr, tpot, comp, comm, pipe;
};

// CPython builtin sum() over floats with int start 0: Neumaier compensation
// from 3.12 (NEU) or the naive left fold before it. CPython adds the first
// float to the int 0 exactly (0 + x == x) and compensates from the second
// on; starting from f = c = 0 and compensating every add gives the same bits
// (the first add's error is exactly 0), so there is no first-element case.
// The compensation term is the exact rounding error of f + x. CPython gets it
// with Fast2Sum after ordering the operands by magnitude
// (fabs(f) >= fabs(x) ? (f - t) + x : (x - t) + f); Knuth's branch-free
// TwoSum computes the same exact error (both are exact for finite sums under
// round-to-nearest), without the compare and selects. Adding 0.0 leaves both
// f and c unchanged, so an absent term can be added as 0.0 (branch-free).
template <bool NEU, typename R = double>
struct PySum {
  R f = R(0), c = R(0);
  __device__ __forceinline__ void add(R x) {
    const R t = f + x;
    if (NEU) {
      const R xp = t - f, fp = t - xp;
      c += (f - fp) + (x - xp);
    }
    f = t;
  }
  __device__ __forceinline__ R result() const {
    if (NEU && c != R(0) && isfinite(c)) return f + c;
    return f;
  }
};

// Collective family of reconciling producer state `from` to demand `to`
// (transition, layout.py:119-155; states are axis codes, see ST_*):
// R->* none, S->S none, S->R all_gather, P->S reduce_scatter, P->R all_reduce.
// As a 2-bit table indexed by 3*from + to: (P,R) -> AR, (P,S) -> ONCE, (S,R) -> ONCE.
__device__ __forceinline__ int fam(int from, int to) {
  constexpr uint32_t kFam = (FAM_AR << 6) | (FAM_ONCE << 10) | (FAM_ONCE << 12);
  return (int)((kFam >> (2 * (3 * from + to))) & 3u);
}
// Input demanded by a matmul under `axis` (_required_input, layout.py:194-197).
__device__ __forceinline__ int req(int axis) { return axis == 1 ? ST_S : ST_R; }

__device__ __forceinline__ double dget(const uint64_t* T, int i) { return __longlong_as_double((long long)T[i]); }
// read-only global path (L1) for the fp64 time tables
__device__ __forceinline__ double gget(const uint64_t* __restrict__ T, int i) {
  return __longlong_as_double((long long)__ldg(reinterpret_cast<const unsigned long long*>(T) + i));
}
__device__ __forceinline__ uint64_t gword(const uint64_t* __restrict__ T, int i) {
  return __ldg(reinterpret_cast<const unsigned long long*>(T) + i);
}
// LDG: table in global memory (read-only path) or any address space (smem copy)
template <bool LDG>
__device__ __forceinline__ double tget(const uint64_t* __restrict__ T, int i) {
  return LDG ? gget(T, i) : dget(T, i);
}
template <bool LDG>
__device__ __forceinline__ uint64_t tword(const uint64_t* __restrict__ T, int i) {
  return LDG ? gword(T, i) : T[i];
}

// A decoded candidate: domain indices and Y, the 2-bit axis of every axis
// head in its field slot (ls_tables.cuh head_slots).
struct Decoded {
  int t, e, p, b;
  uint32_t Y;
};

// The 12 canonical ops' axes as 2-bit fields in canonical op order (op k at
// bits 2k): the head fields of Y moved by the workload's runs of consecutive
// controlled ops, pinned ops' axes OR-ed in (EvalMeta canon_*). For the
// default 12-op spaces this is one run, Y itself.
__device__ __forceinline__ uint32_t canon_y(const EvalMeta& M, uint32_t Y) {
  if (M.canon_ident) return Y;  // one run from bit 0, nothing pinned
  uint32_t yc = M.canon_or;
  for (int r = 0; r < M.canon_runs; ++r)
    yc |= ((Y >> M.canon_shr[r]) & ((1u << M.canon_len[r]) - 1u)) << M.canon_shl[r];
  return yc;
}
__device__ __forceinline__ int cax(uint32_t yc, int k) { return (int)((yc >> (2 * k)) & 3u); }

// attn_core sharded on DIM1 (the high bit of its 2-bit field), or its pin.
__device__ __forceinline__ uint32_t attn_dim1(const EvalMeta& M, uint32_t Y) {
  return ((Y | M.attn_or) >> M.attn_shift) & 1u;
}

// Gate pass (every candidate), branch-free: one 128-bit lookup of the
// (t, e, p) entry gives the weights term, the gate bits and the kv row; the
// reason is then selected in the reference's gate order — device budget
// (simulator.py:257), layout (:268, layout.py:371-374, :214-221), memory
// (:135-160, :279). Returns LS_REASON_NONE for survivors (which still need
// full_path). mem is set only when the memory gate ran, as in SimResult.
// Indices must be in range (callers clamp decode-failed candidates).
__device__ __forceinline__ uint32_t gate(const uint64_t* G, const TabLayout& L, const EvalMeta& M, const Decoded& c,
                                         double& mem) {
  const int tep = (c.t * L.ne + c.e) * L.np + c.p;
  const uint4 ent = *reinterpret_cast<const uint4*>(G + L.tep + 2 * tep);
  const double w = __hiloint2double((int)ent.y, (int)ent.x);
  const uint32_t bits = ent.z, kv_row = ent.w;
  const uint32_t a2 = attn_dim1(M, c.Y);
  const double m = (w + dget(G, L.mem_kv + (int)(a2 * (uint32_t)(L.nt * L.np * L.nb) + kv_row) + c.b)) +
                   dget(G, L.mem_ws + c.b);
  const bool over = (bits & GATE_BUDGET) != 0;
  const bool bad = ((c.Y & bits & GATE_FIELDS) | (bits & (GATE_PINNED | GATE_LAYOUT))) != 0;
  const uint32_t reason = over ? LS_REASON_OVER_DEVICE_BUDGET
                               : (bad ? LS_REASON_LAYOUT_ERROR : (m > M.hbm_capacity ? LS_REASON_OOM : LS_REASON_NONE));
  mem = (over || bad) ? 0.0 : m;
  return reason;
}

// Raw-mode gate (no memory_bytes output) from a coarse word: the static
// reason of the candidate's attention layout, unless the budget passed and an
// axis field is inadmissible (a layout error, gate order of simulator.py:257-284).
__device__ __forceinline__ uint32_t coarse_reason(uint32_t cw, uint32_t Y, uint32_t a2) {
  const uint32_t rs = (cw >> (COARSE_RS_SHIFT + 2 * a2)) & 3u;
  return ((Y & cw & GATE_FIELDS) != 0 && rs != LS_REASON_OVER_DEVICE_BUDGET) ? (uint32_t)LS_REASON_LAYOUT_ERROR : rs;
}
__device__ __forceinline__ uint32_t gate_coarse(const uint32_t* C, const TabLayout& L, const EvalMeta& M,
                                                const Decoded& c) {
  return coarse_reason(C[((c.t * L.ne + c.e) * L.np + c.p) * L.nb + c.b], c.Y, attn_dim1(M, c.Y));
}

// Same, from the coarse rank ((t*ne + e)*np + p)*nb + b directly.
__device__ __forceinline__ uint32_t gate_rank(const uint32_t* C, const EvalMeta& M, uint32_t rank, uint32_t Y) {
  return coarse_reason(C[rank], Y, attn_dim1(M, Y));
}

// fp64 pass for a candidate that passed gate(). T: the full table (global).
// The layer plan's two Python sums (simulator.py:224-236): compute over
// qkv, kv, attn, out, router, ffn1, ffn2[, sh1, sh2] and the collectives in
// all_collectives() order (layout.py:270-275) — functions of (t, e, b) and the
// axes of qkv, attn (DIM1 or not), out, ffn1, ffn2, sh1, sh2 only.
template <bool NEU, bool LDG, bool F32, typename R>
__device__ __forceinline__ void layer_sums(const uint64_t* __restrict__ T, const float* __restrict__ Tf,
                                           const TabLayout& L, int t, int e, int b, bool tp_gt1, bool ep_gt1,
                                           int ax_qkv, int a2, int ax_out, int ax_f1, int ax_f2, int ax_s1,
                                           int ax_s2, R& layer_c, R& layer_m) {
  auto get = [&](int i) -> R {
    if constexpr (F32) return Tf[i];
    else return tget<LDG>(T, i);
  };
  const int nt = L.nt, ne = L.ne, nb = L.nb;
  const int tb = t * nb + b, teb = (t * ne + e) * nb + b;
  // layer plan compute: qkv, kv, attn, out, router, ffn1, ffn2[, sh1, sh2]
  PySum<NEU && !F32, R> lc;
  lc.add(get(L.opt_qkv + ax_qkv * nt * nb + tb));
  lc.add(get(L.opt_kv + a2 * nt * nb + tb));
  lc.add(get(L.opt_attn + a2 * nt * nb + tb));
  lc.add(get(L.opt_out + ax_out * nt * nb + tb));
  lc.add(get(L.opt_router + b));
  lc.add(get(L.opt_ffn1 + ax_f1 * nt * ne * nb + teb));
  lc.add(get(L.opt_ffn2 + ax_f2 * nt * ne * nb + teb));
  if (L.has_shared) {
    lc.add(get(L.opt_sh1 + ax_s1 * nt * nb + tb));
    lc.add(get(L.opt_sh2 + ax_s2 * nt * nb + tb));
  }
  // layer plan collectives in all_collectives() order (layout.py:270-275);
  // a collective that is not emitted is added as 0.0 (an exact no-op of the
  // sum), so the walk is branch-free: (f) ? time : 0.0 from an in-range slot
  PySum<NEU && !F32, R> lm;
#define LS_TP_COLL(cls, f) get(L.coll + ((cls) * 2 + ((f) - 1 + ((f) == 0))) * nt * nb + tb)
#define LS_OPT(f, x) ((f) ? (x) : R(0))
  const int st_attn = a2 ? ST_S : ST_R;
  const int tpm = tp_gt1 ? 3 : 0;  // with tp == 1 no TP collective is emitted (fam & 0)
  int f;
  f = fam(ax_qkv, st_attn) & tpm;
  lm.add(LS_OPT(f, LS_TP_COLL(CLS_QKV, f)));  // feed attn_core
  f = fam(st_attn, req(ax_out)) & tpm;
  lm.add(LS_OPT(f, LS_TP_COLL(CLS_H, f)));  // feed attn_out_proj
  f = fam(ax_out, ST_R) & tpm;
  lm.add(LS_OPT(f, LS_TP_COLL(CLS_H, f)));  // attention residual
  const R a2a = ep_gt1 ? get(L.a2a + teb) : R(0);
  lm.add(a2a);  // expert dispatch (0.0 when ep == 1)
  f = fam(ax_f1, req(ax_f2)) & tpm;
  lm.add(LS_OPT(f, get(L.rtf + (f - 1 + (f == 0)) * nt * ne * nb + teb)));  // feed ffn2
  if (L.has_shared) {
    f = fam(ax_s1, req(ax_s2)) & tpm;
    lm.add(LS_OPT(f, LS_TP_COLL(CLS_F, f)));  // feed sh2
  }
  lm.add(a2a);  // expert combine
  if (L.has_shared && ax_s2 != ax_f2) {  // branch outputs disagree: align both
    f = fam(ax_f2, ST_R) & tpm;
    lm.add(LS_OPT(f, LS_TP_COLL(CLS_H, f)));
    f = fam(ax_s2, ST_R) & tpm;
    lm.add(LS_OPT(f, LS_TP_COLL(CLS_H, f)));
  } else {  // layer exit
    f = fam(ax_f2, ST_R) & tpm;
    lm.add(LS_OPT(f, LS_TP_COLL(CLS_H, f)));
  }
  layer_c = lc.result();
  layer_m = lm.result();
#undef LS_TP_COLL
#undef LS_OPT
}

// Index of a layer-sum memo entry (EvalMeta::memo): (t, e, b) then the axes,
// mixed radix; the shared-expert axes only when the model has one.
// (32-bit: the memo is built only below 2^22 entries)
__device__ __forceinline__ int memo_key(const TabLayout& L, int t, int e, int b, int ax_qkv, int a2, int ax_out,
                                        int ax_f1, int ax_f2, int ax_s1, int ax_s2) {
  int k = (((((t * L.ne + e) * L.nb + b) * 3 + ax_qkv) * 2 + a2) * 3 + ax_out) * 3 + ax_f1;
  k = k * 3 + ax_f2;
  if (L.has_shared) k = (k * 3 + ax_s1) * 3 + ax_s2;
  return k;
}

//
// F32 (the fp32 fast mode of ls_sweep, ls_set_precision): the same walk on the
// fp32 copy of the time tables Tf (each entry the double correctly rounded),
// plain fp32 sums (no compensation), fp32 division — raw within ~2e-6
// relative of the fp64 value. The SLO gate is re-decided exactly in fp64 when
// tpot lies within 1e-5 relative of slo_tpot, so every verdict reason is the
// reference's; the integer gates and the memory gate run before, in fp64.
template <bool NEU, bool LDG = true, bool F32 = false>
__device__ __forceinline__ void full_path(const uint64_t* __restrict__ T, const TabLayout& L, const EvalMeta& M,
                                          const Decoded& c, Verdict& v, const float* __restrict__ Tf = nullptr) {
  using R = typename std::conditional<F32, float, double>::type;
  auto get = [&](int i) -> R {
    if constexpr (F32) return Tf[i];
    else return tget<LDG>(T, i);
  };
  const int t = c.t, e = c.e, p = c.p, b = c.b;
  const uint32_t yc = canon_y(M, c.Y);
  const int ax_emb = cax(yc, LS_OP_EMBEDDING), ax_qkv = cax(yc, LS_OP_QKV_PROJ);
  const int ax_attn = cax(yc, LS_OP_ATTN_CORE), ax_out = cax(yc, LS_OP_ATTN_OUT_PROJ);
  const int ax_f1 = cax(yc, LS_OP_EXPERT_FFN1), ax_f2 = cax(yc, LS_OP_EXPERT_FFN2);
  const int ax_s1 = cax(yc, LS_OP_SHARED_FFN1), ax_s2 = cax(yc, LS_OP_SHARED_FFN2);
  const int ax_lmh = cax(yc, LS_OP_LM_HEAD);
  const int a2 = ax_attn == 2;
  const int nt = L.nt, nb = L.nb;
  const int tb = t * nb + b;
  const int64_t tpv = (int64_t)tword<LDG>(T, L.tpv + t), epv = (int64_t)tword<LDG>(T, L.epv + e);
  const int64_t ppv = (int64_t)tword<LDG>(T, L.ppv + p);
  const bool tp_gt1 = tpv > 1, ep_gt1 = epv > 1;

  // layer sums: from the workload's memo table (exact values computed once
  // by the same code, layer_sums) or walked here
  R layer_c, layer_m;
  if (M.memo) {  // (the fp32 fast mode rounds the exact sums to fp32)
    const double2 lv = __ldg(M.memo + memo_key(L, t, e, b, ax_qkv, a2, ax_out, ax_f1, ax_f2, ax_s1, ax_s2));
    layer_c = (R)lv.x;
    layer_m = (R)lv.y;
  } else {
    layer_sums<NEU, LDG, F32, R>(T, Tf, L, t, e, b, tp_gt1, ep_gt1, ax_qkv, a2, ax_out, ax_f1, ax_f2, ax_s1, ax_s2,
                                 layer_c, layer_m);
  }
#define LS_TP_COLL(cls, f) get(L.coll + ((cls) * 2 + ((f) - 1 + ((f) == 0))) * nt * nb + tb)
#define LS_OPT(f, x) ((f) ? (x) : R(0))
  const int tpm = tp_gt1 ? 3 : 0;  // with tp == 1 no TP collective is emitted (fam & 0)
  int f;

  // pre plan (embedding) and post plan (final_norm, lm_head)
  const R pre_c = R(0) + get(L.opt_emb + ax_emb * nt * nb + tb);
  f = fam(ax_emb, ST_R) & tpm;
  const R pre_m = R(0) + LS_OPT(f, LS_TP_COLL(CLS_H, f));
  f = fam(ax_lmh, ST_R) & tpm;
  const R post_m = R(0) + LS_OPT(f, LS_TP_COLL(CLS_V, f));
#undef LS_TP_COLL
#undef LS_OPT
  PySum<NEU && !F32, R> po;
  po.add(get(L.opt_norm + b));
  po.add(get(L.opt_lmh + ax_lmh * nt * nb + tb));
  const R post_c = po.result();

  // totals and pipeline stages (simulator.py:286-323)
  const int64_t world = tpv * epv * ppv;
  const R hop = ppv > 1 ? get(L.hop + (world <= M.node_size ? nb : 0) + b) : R(0);
  const R nl = (R)M.num_layers_d;
  const R compute = (nl * layer_c + pre_c) + post_c;
  const R comm = (nl * layer_m + pre_m) + post_m;
  const R pipe = get(L.ppm1_d + p) * hop;
  const R tpot = (compute + comm) + pipe;
  const R body = get(L.lps_d + p) * (layer_c + layer_m);
  const R c0 = body + (pre_c + pre_m);
  R cmax;
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
  if (F32) {  // near the SLO boundary the fp32 tpot cannot decide gate 4: redo it in fp64
    const R slo = (R)M.slo_tpot;
    if (fabs(tpot - slo) <= (R)1e-5 * slo) {
      full_path<NEU, LDG, false>(T, L, M, c, v);
      return;
    }
  }
  // gate 4: tpot > slo_tpot (simulator.py:325)
  if ((double)tpot > M.slo_tpot) {
    v.reason = LS_REASON_SLO_VIOLATION;
    v.thr = 0.0;
    return;
  }
  v.reason = LS_REASON_NONE;
  v.thr = (double)((get(L.batch_d + b) / cmax) / (R)world);
}

}  // namespace ls
