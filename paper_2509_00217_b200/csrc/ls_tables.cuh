// ls_tables.cuh — per-workload lookup tables of the B200 evaluator.
//
// The reference recomputes every operator cost and collective cost from
// scratch for every candidate (simulator.py:163-236, layout.py:347-456).
// Each of those quantities is a pure function of a few domain indices —
// (op, axis, tp, batch[, ep][, attention axis]) — so a workload compiles
// into a few thousand float64 words computed ONCE per context by
// build_tables (ls_tables.cu) with exactly the reference's expression order.
// Kernels then only gather and sum per candidate, which removes ~66 IEEE
// divisions per full-path candidate while staying bit-identical (each entry
// IS the value the reference computes).
//
// The buffer starts with the GATE segment — everything the first pass needs
// (budget / layout bitmasks and the three memory terms) — which the evaluate
// kernel bulk-copies into shared memory. The op / collective time segments
// behind it are read through L1 by the compacted fp64 pass.
//
// Axis words. Candidates are decoded into Y: 2 bits per AXIS HEAD (heads
// 4.., in head order), the order the SoA planes arrive in. Layout masks are
// therefore built per head; the fp64 pass maps heads back to canonical ops
// through EvalMeta::op_src.
//
// All words are 8 bytes: doubles, or int64/uint64 bit patterns.
#pragma once
#include <stdint.h>

#include <vector_types.h>

#include "../../include/ls_eval.h"

namespace ls {

// Layout states of an activation over the TP group (layout.py:34-37). The
// code equals the producing matmul's axis: UNSHARDED->R, DIM0->P, DIM1->S.
enum : int { ST_R = 0, ST_P = 1, ST_S = 2 };
// Collective families: AR pays 2(n-1)/n, the rest (AG, RS, A2A) (n-1)/n
// (simulator.py:116-119).
enum : int { FAM_NONE = 0, FAM_AR = 1, FAM_ONCE = 2 };
// Payload classes of TP-group collectives: tokens x features x dtype.
enum : int { CLS_QKV = 0, CLS_H = 1, CLS_F = 2, CLS_V = 3 };

// Gate bits of a [t][e][p] entry. An axis field of Y holds 0 (UNSHARDED,
// never a layout error), 1 (DIM0: only its low bit set) or 2 (DIM1: only its
// high bit set), so "some op's axis is inadmissible or its extent does not
// divide tp" (layout.py:214-221) is the single test  Y & GATE_FIELDS-mask:
// bit 2f flags DIM0 bad for field f, bit 2f+1 flags DIM1 bad.
enum : uint32_t {
  GATE_FIELDS = 0x00ffffffu,  // 12 axis fields x {DIM0, DIM1}
  GATE_PINNED = 1u << 24,     // a pinned (uncontrolled) op is a layout error at this tp
  GATE_LAYOUT = 1u << 25,     // pp does not divide num_layers, or ep vs num_experts
  GATE_BUDGET = 1u << 26      // tp * ep * pp > device_budget
};

// Coarse gate words: one uint32 per (t, e, p, b) = the 24 axis-field bits of
// the (t, e, p) entry plus, for each attention layout (attn_core on DIM1 or
// not), the reason the candidate-independent gates give in the reference's
// order — over budget (1), pinned-op / pp / ep layout error (2), OOM (3) or
// none (0) — so a raw-mode gate is one shared-memory load, one field test and
// one select. Built only when the coarse space is small enough to stage.
enum : uint32_t { COARSE_RS_SHIFT = 24 };  // 2-bit static reason at 24 (attn not DIM1) and 26 (DIM1)
constexpr int kCoarseMax = 6144;

// Offsets (in 8-byte words) of every table segment inside one buffer.
struct TabLayout {
  int nt, ne, np, nb;  // tp / ep / pp / batch domain sizes
  int has_shared;
  // gate segment (staged to shared memory)
  // [t][e][p] x 2 words: {weights per device (f64),
  //   lo32 = gate bits (GATE_*), hi32 = kv row base ((t*np + p)*nb)}
  int tep;
  int mem_kv, mem_ws;
  int gate_words;  // words of the gate segment, even
  // op-time segments
  int opt_emb, opt_qkv, opt_kv, opt_attn, opt_out, opt_router, opt_ffn1, opt_ffn2;
  int opt_sh1, opt_sh2, opt_norm, opt_lmh;
  // collective-time segments
  int coll, rtf, a2a;
  // pipeline hop, per-index doubles
  int hop, batch_d, lps_d, ppm1_d;
  // integer segments
  int tpv, epv, ppv;
  // coarse gate words (uint32 [t][e][p][b], two per table word), 0 if too large
  int coarse, coarse_words;
  int words;  // total, even (16-byte multiple)
};

// Warp-uniform per-workload scalars, passed by value as a kernel parameter.
struct EvalMeta {
  int A;                              // vector length
  int attn_src;                       // 2*(h-4) of the head controlling attn_core, or -1
  int attn_pin;                       // attn_core axis when not controlled
  int attn_shift;                     // attn_core is DIM1: ((Y | attn_or) >> attn_shift) & 1
  uint32_t attn_or;                   //   (shift 31 and a constant bit 31 when pinned; Y < 2^24)
  int pad0_;
  uint8_t head_size[LS_MAX_HEADS];    // domain size per head
  int8_t head_slot[LS_MAX_HEADS];     // Y field of each head (head_slots), -1 none
  int8_t op_src[LS_NUM_OPS];          // per canonical op: bit shift of its field in Y, or -1 (pinned)
  int8_t op_pin[LS_NUM_OPS];          // pinned axis of uncontrolled ops (default UNSHARDED)
  int64_t node_size;
  double num_layers_d;
  double slo_tpot;
  double hbm_capacity;
  int64_t code_stride[LS_MAX_HEADS];  // mixed-radix place value per head
  // canonical axis word (canon_y): runs of consecutive controlled ops whose
  // head fields are consecutive too: bits [shr, shr + len) of Y -> bit shl
  int canon_runs;
  uint8_t canon_shr[LS_NUM_OPS], canon_len[LS_NUM_OPS], canon_shl[LS_NUM_OPS];
  uint32_t canon_or;  // pinned ops' axes at their canonical fields
  int canon_ident;    // canon_y(Y) == Y (12 controlled ops, heads in canonical order)
  int pad1_;
  // layer-sum memo (ls_memo.cu): (layer compute, layer collectives) per
  // memo_key(t, e, b, layer axes), or null (then walked per candidate)
  const double2* memo;
};

__host__ __device__ inline int round2(int w) { return (w + 1) & ~1; }

// 2-bit field slot of each axis head in the Y word. For A <= 16 (the TMA
// kernel's domain) slot = h - 4, so planes map to fields positionally; for
// longer vectors only the heads that control a canonical op get a slot
// (0..11, in head order) and the rest are range-checked only (-1).
__host__ __device__ inline void head_slots(const ls_workload_desc& d, int* slot) {
  for (int h = 0; h < LS_MAX_HEADS; ++h) slot[h] = -1;
  if (d.vector_length <= 16) {
    for (int h = 4; h < d.vector_length; ++h) slot[h] = h - 4;
    return;
  }
  int next = 0;
  for (int h = 4; h < d.vector_length; ++h)
    for (int k = 0; k < LS_NUM_OPS; ++k)
      if (d.op_head[k] == h) slot[h] = next++;
}

inline TabLayout make_layout(const ls_workload_desc& d) {
  TabLayout L{};
  L.nt = d.domain_len[0];
  L.ne = d.domain_len[1];
  L.np = d.domain_len[2];
  L.nb = d.domain_len[3];
  L.has_shared = d.has_shared_expert ? 1 : 0;
  const int nt = L.nt, ne = L.ne, np = L.np, nb = L.nb;
  int w = 0;
  auto seg = [&](int words) {
    int at = w;
    w += round2(words);
    return at;
  };
  L.tep = seg(2 * nt * ne * np);
  L.mem_kv = seg(2 * nt * np * nb);
  L.mem_ws = seg(nb);
  L.gate_words = w;
  L.opt_emb = seg(3 * nt * nb);
  L.opt_qkv = seg(3 * nt * nb);
  L.opt_kv = seg(2 * nt * nb);
  L.opt_attn = seg(2 * nt * nb);
  L.opt_out = seg(3 * nt * nb);
  L.opt_router = seg(nb);
  L.opt_ffn1 = seg(3 * nt * ne * nb);
  L.opt_ffn2 = seg(3 * nt * ne * nb);
  L.opt_sh1 = seg(L.has_shared ? 3 * nt * nb : 0);
  L.opt_sh2 = seg(L.has_shared ? 3 * nt * nb : 0);
  L.opt_norm = seg(nb);
  L.opt_lmh = seg(3 * nt * nb);
  L.coll = seg(4 * 2 * nt * nb);
  L.rtf = seg(2 * nt * ne * nb);
  L.a2a = seg(nt * ne * nb);
  L.hop = seg(2 * nb);
  L.batch_d = seg(nb);
  L.lps_d = seg(np);
  L.ppm1_d = seg(np);
  L.tpv = seg(nt);
  L.epv = seg(ne);
  L.ppv = seg(np);
  const int nc = nt * ne * np * nb;
  L.coarse_words = nc <= kCoarseMax ? round2((nc + 1) / 2) : 0;
  L.coarse = seg(L.coarse_words);
  L.words = round2(w);
  return L;
}

}  // namespace ls
