"""Batched GPU evaluator: the drop-in for the reference's per-candidate path.

``Evaluator`` owns one libls_eval context (one workload on one device) and
exposes the batched API of SURVEY.md §8(b):

* ``evaluate(planes)``      — score [A, N] uint8 SoA candidates resident on the
  GPU; every element equals ``simulate(SimRequest(decode_strategy(v)))``
  (reference simulator.py:239-341) bit for bit.
* ``evaluate_host(planes)`` — the same from/to host memory (pipelined copies).
* ``reward_scan(...)``      — Eq.-1 rewards with the exclusive running best
  of ``SearchEnv.step`` (env.py:159-164, :178-179).
* ``topk(...)``             — elite top-k over distinct vectors
  (EliteBuffer.offer, policy.py:86-102; build_report(by_raw), ppo.py:441-447).

Tensors are torch CUDA tensors; calls are enqueued on torch's current stream
of the evaluator's device, so they order naturally with surrounding torch work.
"""

from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from ._native import EliteRec, NativeUnavailable, ResultSoA, check
from .strategy import codes_to_vectors
from .workload import Workload

__all__ = ["Evaluator", "BatchResult", "Elite", "FIELDS", "REASON_NAMES", "NativeUnavailable"]

FIELDS = ("throughput", "tpot_s", "memory_bytes", "compute_s", "comm_s", "pipeline_s")
REASON_NAMES = {0: "none", 1: "over_device_budget", 2: "layout_error", 3: "oom", 4: "slo_violation",
                255: "decode_error"}
_REC_BYTES = ctypes.sizeof(EliteRec)


@dataclass
class BatchResult:
    """Per-candidate verdicts (struct of arrays); absent fields are None."""

    reason: torch.Tensor
    throughput: torch.Tensor | None = None
    tpot_s: torch.Tensor | None = None
    memory_bytes: torch.Tensor | None = None
    compute_s: torch.Tensor | None = None
    comm_s: torch.Tensor | None = None
    pipeline_s: torch.Tensor | None = None

    @property
    def valid(self) -> torch.Tensor:
        return self.reason == 0

    def numpy(self) -> dict:
        out = {"reason": self.reason.cpu().numpy()}
        for f in FIELDS:
            t = getattr(self, f)
            if t is not None:
                out[f] = t.cpu().numpy()
        return out


@dataclass(frozen=True)
class Elite:
    """One top-k record: the vector, its key (raw or reward), raw, global index."""

    vector: tuple[int, ...]
    key: float
    raw: float
    index: int


def _cuda_device(device) -> torch.device:
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    if isinstance(device, int):
        return torch.device("cuda", device)
    dev = torch.device(device)
    if dev.type != "cuda":
        raise ValueError(f"the evaluator runs on CUDA devices only, got {dev}")
    return torch.device("cuda", dev.index if dev.index is not None else torch.cuda.current_device())


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


class Evaluator:
    """One workload compiled onto one CUDA device."""

    def __init__(self, workload: Workload, device=None):
        self._lib = _native.lib(require_gpu=True)
        self.workload = workload
        self.space = workload.space
        self.device = _cuda_device(device)
        self.desc = workload.desc()
        handle = ctypes.c_void_p()
        check(self._lib.ls_ctx_create(ctypes.byref(self.desc), self.device.index, ctypes.byref(handle)))
        self._ctx = handle
        self.vector_length = self.desc.vector_length
        self.head_sizes = tuple(int(self.desc.domain_len[h]) if h < 4 else 3 for h in range(self.vector_length))
        self.space_size = int(self._lib.ls_space_size(self._ctx))
        self._scratch: dict[int, torch.Tensor] = {}  # fused-call scratch per CUDA stream
        self._one_bufs = threading.local()

    # -- lifecycle ----------------------------------------------------------

    def close(self) -> None:
        if getattr(self, "_ctx", None):
            self._lib.ls_ctx_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def _stream(self):
        return ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def _check_planes(self, planes: torch.Tensor):
        if planes.dtype != torch.uint8 or planes.dim() != 2:
            raise TypeError("planes must be a 2-D uint8 tensor [A, N]")
        if planes.shape[0] != self.vector_length:
            raise ValueError(f"planes have {planes.shape[0]} heads, the action space has {self.vector_length}")
        if planes.shape[1] > 1 and planes.stride(1) != 1:
            raise ValueError("planes must be contiguous along candidates (stride(1) == 1)")
        n = planes.shape[1]
        stride = planes.stride(0) if planes.shape[0] > 1 else max(n, 1)
        return n, max(stride, n)

    def wait_signal(self, signal: torch.Tensor, seq: int, stream=None) -> None:
        """Make ``stream`` (default: the current one) wait until ``signal`` >= seq."""
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        check(self._lib.ls_stream_wait_signal(ctypes.c_void_p(st.cuda_stream), _ptr(signal), int(seq)))

    def set_precision(self, precision: str) -> None:
        """"fp64" (default, bit-exact) or "fp32": the fp32 fast mode of the on-device
        sweeps (``sweep`` / ``exhaustive_search`` / ``random_sweep``), raw within 1e-5
        relative, reasons exact (ls_set_precision)."""
        modes = {"fp64": 0, "fp32": 1}
        if precision not in modes:
            raise ValueError(f"precision must be 'fp64' or 'fp32', got {precision!r}")
        check(self._lib.ls_set_precision(self._ctx, modes[precision]))

    def reserve_sms(self, sms: int) -> None:
        """Leave ``sms`` SMs free of the persistent evaluate kernels (ls_reserve_sms)."""
        check(self._lib.ls_reserve_sms(self._ctx, int(sms)))

    # -- evaluation ---------------------------------------------------------

    def evaluate_one(self, vector) -> tuple[int, tuple[float, ...]]:
        """One strategy, host in / host out, lowest latency (ls_evaluate_one):
        (reason code, (throughput, tpot_s, memory_bytes, compute_s, comm_s, pipeline_s))."""
        a = self.vector_length
        if len(vector) != a:
            raise ValueError(f"vector has {len(vector)} heads, the action space has {a}")
        try:
            raw = bytes(vector) if isinstance(vector, (tuple, list)) else np.asarray(vector).astype(np.uint8).tobytes()
            if not isinstance(vector, (tuple, list)) and np.any(np.asarray(vector) > 255):
                raise ValueError
        except (ValueError, TypeError):
            if any(not 0 <= int(x) <= 255 for x in vector):
                return 255, (0.0,) * 6  # decode error, like an out-of-range plane byte
            raw = bytes(int(x) for x in vector)
        buf = self._one_bufs
        if not hasattr(buf, "reason"):  # per-thread verdict buffers
            buf.reason, buf.fields = ctypes.c_uint8(), (ctypes.c_double * 6)()
        check(self._lib.ls_evaluate_one(self._ctx, raw, ctypes.byref(buf.reason), buf.fields))
        return buf.reason.value, tuple(buf.fields)

    def evaluate(self, planes: torch.Tensor, fields=("throughput",), out: BatchResult | None = None) -> BatchResult:
        """Score candidates resident on the device. ``fields``: subset of FIELDS or "all"."""
        if planes.device != self.device:
            raise ValueError(f"planes live on {planes.device}, evaluator on {self.device}")
        n, stride = self._check_planes(planes)
        if fields == "all":
            fields = FIELDS
        if out is None:
            out = BatchResult(reason=torch.empty(n, dtype=torch.uint8, device=self.device))
            for f in fields:
                setattr(out, f, torch.empty(n, dtype=torch.float64, device=self.device))
        soa = ResultSoA(_ptr(out.reason), *(_ptr(getattr(out, f)) for f in FIELDS))
        check(self._lib.ls_evaluate(self._ctx, ctypes.c_void_p(planes.data_ptr()), n, stride, ctypes.byref(soa),
                                    self._stream()))
        return out

    def evaluate_host(self, planes: np.ndarray | torch.Tensor, fields=("throughput",), out: dict | None = None) -> dict:
        """Score host-resident [A, N] planes; results come back as numpy arrays.

        Copies are pipelined with the kernels inside the library; pass pinned
        memory (``pinned_planes``) for full PCIe bandwidth.
        """
        if isinstance(planes, torch.Tensor):
            if planes.is_cuda:
                raise ValueError("evaluate_host takes host memory; use evaluate() for device tensors")
            arr = planes.numpy()
        else:
            arr = np.asarray(planes)
        if arr.dtype != np.uint8 or arr.ndim != 2 or arr.shape[0] != self.vector_length:
            raise ValueError(f"expected uint8 planes of shape [{self.vector_length}, N]")
        if arr.shape[1] and arr.strides[1] != 1:
            arr = np.ascontiguousarray(arr)
        n = arr.shape[1]
        stride = arr.strides[0] if arr.shape[0] > 1 else max(n, 1)
        if fields == "all":
            fields = FIELDS
        if out is None:
            out = {"reason": np.empty(n, dtype=np.uint8)}
            for f in fields:
                out[f] = np.empty(n, dtype=np.float64)
        elif any(len(v) < n for v in out.values()):
            raise ValueError("out arrays are shorter than the batch")
        soa = ResultSoA(ctypes.c_void_p(out["reason"].ctypes.data),
                        *(ctypes.c_void_p(out[f].ctypes.data) if f in out else None for f in FIELDS))
        check(self._lib.ls_evaluate_host(self._ctx, ctypes.c_void_p(arr.ctypes.data), n, max(stride, n),
                                         ctypes.byref(soa)))
        return out

    def sa_chain(self, init, coords, drawn, u, temperature, moves: int, best_raw: float, alpha: float, beta: float,
                 penalty: float):
        """One simulated-annealing chain of len(u) + 1 evaluations in ONE kernel
        (ls_sa_chain). Returns numpy (vectors [n, A] u8, raws, rewards, reasons u8)
        and the best raw afterwards."""
        steps = len(u) + 1
        dev = self.device
        a = self.vector_length
        t_i32 = lambda x: torch.as_tensor(np.asarray(x, dtype=np.int32).reshape(-1)).to(dev)  # noqa: E731
        t_f64 = lambda x: torch.as_tensor(np.asarray(x, dtype=np.float64).reshape(-1)).to(dev)  # noqa: E731
        init_d, coords_d, drawn_d = t_i32(init), t_i32(coords), t_i32(drawn)
        u_d, temp_d = t_f64(u), t_f64(temperature)
        best = torch.tensor([best_raw], dtype=torch.float64, device=dev)
        pos = torch.zeros(1, dtype=torch.int64, device=dev)
        log_vec = torch.zeros(steps * a, dtype=torch.uint8, device=dev)
        log_raw = torch.zeros(steps, dtype=torch.float64, device=dev)
        log_reward = torch.zeros(steps, dtype=torch.float64, device=dev)
        log_reason = torch.zeros(steps, dtype=torch.uint8, device=dev)
        env = _native.SearchState(_ptr(best), None, None, 0, _ptr(pos), steps, _ptr(log_vec), _ptr(log_raw),
                                  _ptr(log_reward), _ptr(log_reason), float(alpha), float(beta), float(penalty))
        plan = _native.SaPlan(steps, int(moves), _ptr(init_d), _ptr(coords_d) if coords_d.numel() else None,
                              _ptr(drawn_d) if drawn_d.numel() else None, _ptr(u_d) if steps > 1 else None,
                              _ptr(temp_d) if steps > 1 else None, env)
        check(self._lib.ls_sa_chain(self._ctx, ctypes.byref(plan), self._stream()))
        return (log_vec.view(steps, a).cpu().numpy(), log_raw.cpu().numpy(), log_reward.cpu().numpy(),
                log_reason.cpu().numpy(), float(best.item()))

    # -- reward shaping + elites -------------------------------------------

    def reward_scan(self, reason: torch.Tensor, throughput: torch.Tensor, b0: float = 0.0, alpha: float = 1.0,
                    beta: float = 1.0, penalty: float = -10.0):
        """Per-candidate Eq.-1 rewards and the running best after the batch."""
        n = reason.shape[0]
        reward = torch.empty(n, dtype=torch.float64, device=self.device)
        best = torch.empty(1, dtype=torch.float64, device=self.device)
        scratch = torch.empty(int(self._lib.ls_scan_scratch_bytes(n)), dtype=torch.uint8, device=self.device)
        check(self._lib.ls_reward_scan(self._ctx, _ptr(reason), _ptr(throughput), n, float(b0), float(alpha),
                                       float(beta), float(penalty), _ptr(reward), _ptr(best), _ptr(scratch),
                                       self._stream()))
        return reward, best

    def topk_records(self, planes: torch.Tensor, reason: torch.Tensor, throughput: torch.Tensor,
                     key: torch.Tensor | None = None, k: int = 3, index_base: int = 0):
        """Device top-k: returns (records uint8 tensor [k, 32], count int32 tensor [1])."""
        n, stride = self._check_planes(planes)
        if key is None:
            key = throughput
        recs = torch.empty((k, _REC_BYTES), dtype=torch.uint8, device=self.device)
        count = torch.empty(1, dtype=torch.int32, device=self.device)
        scratch = torch.empty(int(self._lib.ls_topk_scratch_bytes(n, k)), dtype=torch.uint8, device=self.device)
        check(self._lib.ls_topk(self._ctx, _ptr(planes), stride, _ptr(reason), _ptr(throughput), _ptr(key), n, int(k),
                                int(index_base), _ptr(recs), _ptr(count), _ptr(scratch), self._stream()))
        return recs, count

    def topk(self, planes, reason, throughput, key=None, k: int = 3, index_base: int = 0) -> list[Elite]:
        """Top-k valid candidates over distinct vectors, best first."""
        recs, count = self.topk_records(planes, reason, throughput, key, k, index_base)
        return self.decode_records(recs, count)

    def decode_records(self, recs: torch.Tensor, count: torch.Tensor) -> list[Elite]:
        n = int(count.item())
        if n < 0:
            raise RuntimeError("elite exchange timed out: a peer rank never published its block")
        raw = recs[:n].cpu().numpy().view(np.dtype([("key", "<f8"), ("raw", "<f8"), ("index", "<i8"), ("code", "<u8")]))
        raw = raw.reshape(-1)
        vecs = codes_to_vectors(raw["code"], self.space) if n else np.zeros((0, self.vector_length), np.int64)
        return [Elite(tuple(int(x) for x in vecs[i]), float(raw["key"][i]), float(raw["raw"][i]), int(raw["index"][i]))
                for i in range(n)]

    def evaluate_topk(self, planes: torch.Tensor, k: int = 3, index_base: int = 0, out: BatchResult | None = None,
                      fields=("throughput",), verdicts: bool = True, into: torch.Tensor | None = None):
        """Fused sweep: score the batch and reduce it to the top-k by raw in one pass.

        With ``verdicts=False`` nothing per-candidate is written (16 B of HBM
        traffic per candidate); otherwise ``out`` (allocated if None) receives
        the same verdicts ``evaluate`` produces. Returns (out, records, count).
        """
        if planes.device != self.device:
            raise ValueError(f"planes live on {planes.device}, evaluator on {self.device}")
        n, stride = self._check_planes(planes)
        fused_ok = (planes.data_ptr() % 16 == 0 and stride % 16 == 0 and self.vector_length <= 16 and k <= 32)
        if not verdicts and not fused_ok:
            # the fused sweep needs TMA-aligned planes; otherwise evaluate, then reduce
            out, recs, count = self.evaluate_topk(planes, k, index_base, None, ("throughput",), True)
            return None, recs, count
        if verdicts and out is None:
            out = BatchResult(reason=torch.empty(n, dtype=torch.uint8, device=self.device))
            for f in (FIELDS if fields == "all" else fields):
                setattr(out, f, torch.empty(n, dtype=torch.float64, device=self.device))
        soa = ResultSoA(_ptr(out.reason), *(_ptr(getattr(out, f)) for f in FIELDS)) if verdicts else None
        recs, count = self._elite_out(k, into)
        scratch = self._fused_scratch(n, k)
        check(self._lib.ls_evaluate_topk(self._ctx, ctypes.c_void_p(planes.data_ptr()), n, stride,
                                         ctypes.byref(soa) if soa is not None else None, int(k), int(index_base),
                                         _ptr(recs), _ptr(count), _ptr(scratch), self._stream()))
        return (out if verdicts else None), recs, count

    # -- packed candidate words (8 B per candidate) ---------------------------

    def packed_layout(self) -> tuple[int, int]:
        """(bit shift of the coarse rank, coarse space size) of packed words."""
        sh, size = ctypes.c_int32(), ctypes.c_int64()
        check(self._lib.ls_packed_layout(self._ctx, ctypes.byref(sh), ctypes.byref(size)))
        return sh.value, size.value

    def pack(self, planes: torch.Tensor) -> torch.Tensor:
        """Device SoA planes -> packed uint64 words (as int64 storage)."""
        n, stride = self._check_planes(planes)
        words = torch.empty(n, dtype=torch.int64, device=self.device)
        check(self._lib.ls_pack(self._ctx, ctypes.c_void_p(planes.data_ptr()), stride, n, _ptr(words),
                                self._stream()))
        return words

    def _check_words(self, words: torch.Tensor) -> int:
        if words.device != self.device:
            raise ValueError(f"words live on {words.device}, evaluator on {self.device}")
        if words.dtype not in (torch.int64, torch.uint64) or words.dim() != 1 or not words.is_contiguous():
            raise ValueError("packed candidates must be a contiguous 1-D 64-bit tensor")
        return words.shape[0]

    def _alloc(self, n: int, fields) -> BatchResult:
        out = BatchResult(reason=torch.empty(n, dtype=torch.uint8, device=self.device))
        for f in (FIELDS if fields == "all" else fields):
            setattr(out, f, torch.empty(n, dtype=torch.float64, device=self.device))
        return out

    def evaluate_packed(self, words: torch.Tensor, fields=("throughput",), out: BatchResult | None = None) -> BatchResult:
        """Score packed candidate words resident on the device."""
        n = self._check_words(words)
        if out is None:
            out = self._alloc(n, fields)
        soa = ResultSoA(_ptr(out.reason), *(_ptr(getattr(out, f)) for f in FIELDS))
        check(self._lib.ls_evaluate_packed(self._ctx, ctypes.c_void_p(words.data_ptr()), n, ctypes.byref(soa),
                                           self._stream()))
        return out

    def _fused_scratch(self, n: int, k: int, stream=None) -> torch.Tensor:
        """Scratch of the fused evaluate + elite kernels, one buffer per CUDA stream
        (calls on different streams may overlap and must not share the CTA lists
        and sync words). Zero-filled once: every call leaves its sync words zero.
        A buffer is only ever used on the stream it was allocated on."""
        nbytes = int(self._lib.ls_evaluate_topk_scratch_bytes(self._ctx, int(n), int(k)))
        key = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        buf = self._scratch.get(key)
        if buf is None or buf.numel() < nbytes:
            buf = torch.zeros(max(nbytes, 4096), dtype=torch.uint8, device=self.device)
            self._scratch[key] = buf
        return buf

    def _elite_out(self, k: int, into: torch.Tensor | None):
        """(records, count) outputs: fresh tensors, or views of a caller's [(k + 1), 32]
        uint8 buffer (records in rows 0..k-1, the int32 count at the start of row k) —
        one contiguous message for the cross-rank all-gather."""
        if into is None:  # one allocation for both
            into = torch.empty((k + 1, _REC_BYTES), dtype=torch.uint8, device=self.device)
            return into[:k], into[k, :4].view(torch.int32)
        if into.shape != (k + 1, _REC_BYTES) or into.dtype != torch.uint8 or not into.is_contiguous():
            raise ValueError("into must be a contiguous [(k + 1), 32] uint8 tensor")
        return into[:k], into[k, :4].view(torch.int32)

    def evaluate_packed_topk(self, words: torch.Tensor, k: int = 3, index_base: int = 0,
                             out: BatchResult | None = None, fields=("throughput",), verdicts: bool = True,
                             into: torch.Tensor | None = None, signal: torch.Tensor | None = None, seq: int = 0):
        """Fused evaluate + top-k by raw over packed words. Returns (out, records, count).

        ``signal`` (a device uint32/int32 tensor of one element): the launch stores ``seq``
        there once the records are written, for ``wait_signal`` on another stream."""
        n = self._check_words(words)
        if verdicts and out is None:
            out = self._alloc(n, fields)
        soa = ResultSoA(_ptr(out.reason), *(_ptr(getattr(out, f)) for f in FIELDS)) if verdicts else None
        recs, count = self._elite_out(k, into)
        st = torch.cuda.current_stream(self.device)
        scratch = self._fused_scratch(n, k, st)
        sp = ctypes.c_void_p(st.cuda_stream)
        if signal is not None:
            check(self._lib.ls_evaluate_packed_topk_signal(
                self._ctx, ctypes.c_void_p(words.data_ptr()), n, ctypes.byref(soa) if soa is not None else None,
                int(k), int(index_base), _ptr(recs), _ptr(count), _ptr(scratch), _ptr(signal), int(seq), sp))
        else:
            check(self._lib.ls_evaluate_packed_topk(self._ctx, ctypes.c_void_p(words.data_ptr()), n,
                                                    ctypes.byref(soa) if soa is not None else None, int(k),
                                                    int(index_base), _ptr(recs), _ptr(count), _ptr(scratch), sp))
        return (out if verdicts else None), recs, count

    def fused_plan(self, words: torch.Tensor, k: int = 3, out: BatchResult | None = None,
                   into: torch.Tensor | None = None, index_base: int = 0,
                   signal: torch.Tensor | None = None, sinks: torch.Tensor | None = None) -> "FusedPlan":
        """A prepared ``evaluate_packed_topk`` over fixed buffers on the current stream:
        each call of the plan enqueues the fused launch with arguments marshalled
        once (the per-call host cost of the small-batch regime). With ``signal``,
        ``plan(seq)`` is ``evaluate_packed_topk(..., signal=signal, seq=seq)``."""
        return FusedPlan(self, words, k, out, into, index_base, signal, sinks)

    def evaluate_host_packed(self, words: np.ndarray, fields=("throughput",), out: dict | None = None) -> dict:
        """Score host-resident packed words (pinned for full PCIe speed); numpy results."""
        arr = np.ascontiguousarray(words)
        if arr.dtype not in (np.uint64, np.int64) or arr.ndim != 1:
            raise ValueError("packed candidates must be a 1-D 64-bit array")
        n = arr.shape[0]
        if fields == "all":
            fields = FIELDS
        if out is None:
            out = {"reason": np.empty(n, dtype=np.uint8)}
            for f in fields:
                out[f] = np.empty(n, dtype=np.float64)
        elif any(len(v) < n for v in out.values()):
            raise ValueError("out arrays are shorter than the batch")
        soa = ResultSoA(ctypes.c_void_p(out["reason"].ctypes.data),
                        *(ctypes.c_void_p(out[f].ctypes.data) if f in out else None for f in FIELDS))
        check(self._lib.ls_evaluate_host_packed(self._ctx, ctypes.c_void_p(arr.ctypes.data), n, ctypes.byref(soa)))
        return out

    # -- compact host results -------------------------------------------------

    def evaluate_host_compact(self, candidates: np.ndarray, reason: np.ndarray | None = None,
                              valid_raw: np.ndarray | None = None) -> tuple[np.ndarray, np.ndarray]:
        """Score HOST candidates — [A, N] uint8 planes (the reference's index
        vectors; packed on host threads inside the call) or N packed 64-bit words —
        and return (reason [N] uint8, raws of the valid candidates in index order).
        ~1 B per candidate crosses PCIe back (ls_evaluate_host_compact);
        ``scatter_raw`` rebuilds the dense raw array. Pinned buffers copy fastest."""
        arr = np.asarray(candidates)
        if arr.ndim == 2:
            if arr.dtype != np.uint8 or arr.shape[0] != self.vector_length:
                raise ValueError(f"expected uint8 planes of shape [{self.vector_length}, N]")
            if arr.shape[1] and arr.strides[1] != 1:
                arr = np.ascontiguousarray(arr)
            fmt, n = 0, arr.shape[1]
            stride = arr.strides[0] if arr.shape[0] > 1 else max(n, 1)
        elif arr.ndim == 1 and arr.dtype in (np.uint64, np.int64):
            arr = np.ascontiguousarray(arr)
            fmt, n, stride = 1, arr.shape[0], arr.shape[0]
        else:
            raise ValueError("candidates must be [A, N] uint8 planes or N packed 64-bit words")
        if reason is None:
            reason = np.empty(n, dtype=np.uint8)
        if valid_raw is None:
            valid_raw = np.empty(max(n, 1), dtype=np.float64)
        if len(reason) < n:
            raise ValueError("reason buffer is shorter than the batch")
        count = ctypes.c_int64()
        check(self._lib.ls_evaluate_host_compact(self._ctx, fmt, ctypes.c_void_p(arr.ctypes.data), n,
                                                 max(int(stride), n), ctypes.c_void_p(reason.ctypes.data),
                                                 ctypes.c_void_p(valid_raw.ctypes.data), len(valid_raw),
                                                 ctypes.byref(count)))
        return reason[:n], valid_raw[: count.value]

    @staticmethod
    def scatter_raw(reason: np.ndarray, valid_raw: np.ndarray) -> np.ndarray:
        """Dense raw array (0 for invalid candidates) from compact host results."""
        out = np.zeros(len(reason), dtype=np.float64)
        out[np.flatnonzero(reason == 0)] = valid_raw
        return out

    # -- on-device candidate streams ----------------------------------------

    def stream_size(self, mode: int) -> int:
        """Length of an enumeration stream (GEN_ENUM / GEN_ENUM_ADMISSIBLE). Raises
        NativeError when the library cannot enumerate it (a space beyond exact 64-bit
        indexing, vectors of more than 16 heads) — 0 is never a valid size."""
        size = int(self._lib.ls_stream_size(self._ctx, int(mode)))
        if size == 0:
            msg = self._lib.ls_last_error().decode("utf-8", "replace")
            raise _native.NativeError(_native.LS_ERR_UNSUPPORTED,
                                      msg or "stream size unavailable (uniform streams are unbounded)")
        return size

    def generate(self, mode: int, n: int, start: int = 0, seed: int = 0) -> torch.Tensor:
        """Stream positions [start, start + n) as [A, N] uint8 planes on the device."""
        planes = torch.empty((self.vector_length, max(int(n), 0)), dtype=torch.uint8, device=self.device)
        check(self._lib.ls_generate(self._ctx, int(mode), int(seed) & (2**64 - 1), int(start), int(n),
                                    _ptr(planes), max(int(n), 1), self._stream()))
        return planes

    def sweep(self, mode: int, n: int, start: int = 0, seed: int = 0, k: int = 8):
        """Evaluate stream positions [start, start + n) generated on the device
        and return the top-k by raw over distinct vectors (records, count)."""
        recs = torch.empty((k, _REC_BYTES), dtype=torch.uint8, device=self.device)
        count = torch.empty(1, dtype=torch.int32, device=self.device)
        scratch = self._fused_scratch(n, k)
        check(self._lib.ls_sweep(self._ctx, int(mode), int(seed) & (2**64 - 1), int(start), int(n), int(k),
                                 _ptr(recs), _ptr(count), _ptr(scratch), self._stream()))
        return recs, count

    def merge_records(self, recs: torch.Tensor, counts: torch.Tensor, k_in: int, k: int, into=None):
        """Merge m stacked record lists ([m*k_in, 32] bytes, counts [m]) into one top-k
        (into: optional preallocated ([k, 32] uint8, [1] int32) outputs)."""
        m = counts.shape[0]
        if into is not None:
            out, count = into
        else:
            out = torch.empty((k, _REC_BYTES), dtype=torch.uint8, device=self.device)
            count = torch.empty(1, dtype=torch.int32, device=self.device)
        check(self._lib.ls_topk_merge(_ptr(recs), _ptr(counts), m, int(k_in), int(k), _ptr(out), _ptr(count),
                                      self._stream()))
        return out, count


def pinned_planes(a: int, n: int) -> torch.Tensor:
    """Page-locked [A, N] uint8 host buffer for evaluate_host."""
    return torch.empty((a, n), dtype=torch.uint8).pin_memory()


def pinned_results(n: int, fields=("throughput",)) -> dict:
    """Page-locked numpy result arrays for evaluate_host(out=...)."""
    if fields == "all":
        fields = FIELDS
    out = {"reason": torch.empty(n, dtype=torch.uint8).pin_memory().numpy()}
    for f in fields:
        out[f] = torch.empty(n, dtype=torch.float64).pin_memory().numpy()
    return out


class FusedPlan:
    """``Evaluator.fused_plan``: one fused evaluate + elite launch over fixed device
    buffers (candidate words, verdicts, elite records) on the stream current at
    creation. Calling it enqueues the launch and returns (records, count)."""

    def __init__(self, ev: Evaluator, words: torch.Tensor, k: int, out: BatchResult | None, into, index_base: int,
                 signal: torch.Tensor | None = None, sinks: torch.Tensor | None = None):
        n = ev._check_words(words)
        self.ev, self.words, self.out = ev, words, out
        self.recs, self.count = ev._elite_out(k, into)
        st = torch.cuda.current_stream(ev.device)
        self.scratch = ev._fused_scratch(n, k, st)
        self._soa = ResultSoA(_ptr(out.reason), *(_ptr(getattr(out, f)) for f in FIELDS)) if out is not None else None
        self.key = (words.data_ptr(), n, k, index_base, self.recs.data_ptr(),
                    None if out is None else (out.reason.data_ptr(), out.throughput.data_ptr() if out.throughput
                                              is not None else 0), st.cuda_stream,
                    None if signal is None else signal.data_ptr())
        self.signal = signal
        head = (ev._ctx, ctypes.c_void_p(words.data_ptr()), ctypes.c_int64(n),
                ctypes.byref(self._soa) if self._soa is not None else None, ctypes.c_int(k),
                ctypes.c_int64(index_base), _ptr(self.recs), _ptr(self.count), _ptr(self.scratch))
        self._stream = ctypes.c_void_p(st.cuda_stream)
        self.sinks = sinks
        if sinks is not None:  # the elite block also goes to these device pointers (peer-memory exchange)
            self._fn = ev._lib.ls_evaluate_packed_topk_sinks
            self._head = head + (_ptr(sinks), int(sinks.numel()))
        elif signal is None:
            self._fn = ev._lib.ls_evaluate_packed_topk
            self._args = head + (self._stream,)
        else:
            self._fn = ev._lib.ls_evaluate_packed_topk_signal
            self._head = head + (_ptr(signal),)

    def __call__(self, seq: int | None = None):
        if self.signal is None and self.sinks is None:
            rc = self._fn(*self._args)
        else:
            rc = self._fn(*self._head, seq, self._stream)
        if rc:
            check(rc)
        return self.recs, self.count
