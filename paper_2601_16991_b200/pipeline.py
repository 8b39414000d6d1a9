"""The SALR linear forward on the B200 behind the reference engine's API
(``pkg/src/salr/pipeline.py``).

The reference's two-stage engine -- a decoder thread filling a bounded SPSC
ring with dense tiles and a compute thread multiplying them
(``pipeline.py:110-331``) -- is one persistent CUDA kernel here
(``csrc/salr_linear.cu``): a TMA warp streams compressed tiles into a
shared-memory ring, decoder warps expand them into TMEM, a single thread
issues tcgen05 MMAs, and mbarriers play the ring's Empty -> Filled ->
Consumed -> Empty slot protocol.

``PipelineConfig`` keeps the reference fields and validation
(``pipeline.py:63-86``).  Mapping onto the kernel:

* ``ring_capacity`` -> shared-memory ring slots (clamped to what fits);
* ``overlap=False`` -> a one-slot ring: decode of tile k+1 waits for the MMA
  of tile k (the serial schedule);
* ``tile_rows`` / ``tile_col_bytes`` -> accepted and validated; the device
  tile is fixed at 64 rows x 16 bitmap bytes (the TB format).

As in the reference, the result does not depend on the schedule: the
per-column accumulation order is fixed, so serial and overlapped runs (and
all ring capacities) are bit-identical for a given CTA count.
"""

from __future__ import annotations

import ctypes
import math
import statistics
from dataclasses import dataclass, field
from enum import Enum

import torch

from . import _lib
from .bitmap import BitmapSparseMatrix
from .errors import ConfigError, DomainError, SalrError, ShapeError, VerificationError
from .fusion import FusedAdapters
from .linalg import as_matrix

__all__ = ["SlotState", "PipelineConfig", "PipelineProbe", "BenchResult", "pipelined_matmul",
           "pipelined_forward", "validate_transitions", "bench", "salr_linear"]


class SlotState(Enum):
    EMPTY = "empty"
    FILLED = "filled"
    CONSUMED = "consumed"


_LEGAL = {
    (SlotState.EMPTY, SlotState.FILLED),
    (SlotState.FILLED, SlotState.CONSUMED),
    (SlotState.CONSUMED, SlotState.EMPTY),
}


@dataclass(frozen=True)
class PipelineConfig:
    """Tile and ring dimensions (reference ``pipeline.py:63-86``)."""

    tile_rows: int = 64
    tile_col_bytes: int = 8
    ring_capacity: int = 4
    overlap: bool = True

    def __post_init__(self):
        if self.tile_rows < 1 or self.tile_col_bytes < 1:
            raise ConfigError(f"tile dims must be positive, got ({self.tile_rows}, {self.tile_col_bytes})")
        if self.ring_capacity < 1:
            raise ConfigError(f"ring_capacity must be >= 1, got {self.ring_capacity}")
        if self.overlap and self.ring_capacity < 2:
            raise ConfigError("overlap requires ring_capacity >= 2")

    @property
    def device_stages(self) -> int:
        """Shared-memory ring slots requested from the kernel: 1 for the
        serial schedule (``overlap=False``); otherwise at least the 8 slots
        the kernel is tuned for (the reference's ``ring_capacity`` counts
        decoded tiles in flight; the device ring holds records *and* decoded
        tiles, and results are bit-identical for every depth).  ``salr_linear``
        takes an explicit ``stages=`` for schedule experiments."""
        return 1 if not self.overlap else max(self.ring_capacity, 8)


@dataclass
class PipelineProbe:
    """Fault-injection and audit hooks (reference ``pipeline.py:89-103``),
    run on the device ring of the fused kernel.

    ``decode_delay`` / ``compute_delay``: host callables cannot run inside a
    CUDA kernel (ConfigError); a number is the maximum jitter in
    nanoseconds slept before every tile decode / MMA issue (a per-tile hash
    of ``seed``).  ``record`` fills ``transitions`` with ``(slot, old,
    new)`` for every ring-slot transition of every CTA (slot = cta * stages
    + stage; audit with ``validate_transitions(probe, probe.capacity)``) and
    sets ``produced`` / ``consumed``.
    """

    decode_delay: object = None
    compute_delay: object = None
    record: bool = False
    transitions: list = field(default_factory=list)
    produced: int = 0
    consumed: int = 0
    seed: int = 0
    capacity: int = 0  # slots of the last recorded launch (ctas * stages)


def validate_transitions(probe: PipelineProbe, capacity: int) -> None:
    """Audit a transition log against the slot protocol (``pipeline.py:334-370``)."""
    if probe.produced != probe.consumed:
        raise VerificationError(f"produced {probe.produced} != consumed {probe.consumed}")
    states = [SlotState.EMPTY] * capacity
    for step, (idx, old, new) in enumerate(probe.transitions):
        if not 0 <= idx < capacity:
            raise VerificationError(f"step {step}: slot index {idx} out of range")
        if states[idx] is not old:
            raise VerificationError(f"step {step}: slot {idx} was {states[idx]}, transition claims {old}")
        if (old, new) not in _LEGAL:
            raise VerificationError(f"step {step}: illegal transition {old} -> {new} on slot {idx}")
        states[idx] = new
    for idx, st in enumerate(states):
        if st is not SlotState.EMPTY:
            raise VerificationError(f"slot {idx} left in state {st} at shutdown")
    fills = sum(1 for _, old, _ in probe.transitions if old is SlotState.EMPTY)
    if fills != probe.produced:
        raise VerificationError(f"recorded fills {fills} != produced count {probe.produced}")


# ---------------------------------------------------------------------------
# kernel launch

_WS: dict = {}
_WS_TURN: dict = {}


def _workspace(M: int, N: int, K: int, r_pad: int, num_ctas: int, device) -> torch.Tensor:
    """Per-device scratch (grown on demand, zeroed at allocation; the kernels
    leave its counters in a reusable state).  Two workspaces alternate from
    call to call, so a launch that overlaps the tail of the previous one
    (programmatic dependent launch) never shares scratch with it.  Calls on
    one device must be stream-ordered: pass ``workspace=`` for concurrent
    streams."""
    need = int(_lib.load().salr_linear_workspace_bytes(M, N, K, r_pad, num_ctas))
    turn = _WS_TURN.get(device.index, 0)
    _WS_TURN[device.index] = turn ^ 1
    ws = _WS.get((device.index, turn))
    if ws is None or ws.numel() < need:
        # grow both buffers together (the caching allocator keeps the old ones
        # alive until the work queued on them is done)
        size = max(need, 1 << 21)
        for t in (0, 1):
            _WS[(device.index, t)] = torch.zeros(size, dtype=torch.uint8, device=device)
        ws = _WS[(device.index, turn)]
    return ws


def _prep_x(x, K: int, check_finite: bool):
    """(X, max|X| or None, leading dimension): bf16, K padded to a multiple of
    8; with ``check_finite`` also max|X| (one reduction: a non-finite entry
    makes it non-finite) -> DomainError.  A bf16 device matrix whose rows are
    16-byte aligned -- e.g. the leading columns of the previous linear's
    output -- is passed as it is with its row stride (no copy kernel between
    two chained launches)."""
    if (isinstance(x, torch.Tensor) and x.is_cuda and x.dtype == torch.bfloat16 and x.dim() == 2
            and x.shape[0] >= 1 and x.shape[1] == K and K % 8 == 0 and x.stride(1) == 1
            and x.stride(0) >= K and x.stride(0) % 8 == 0 and x.data_ptr() % 16 == 0
            and x.device.index == torch.cuda.current_device()):
        xmax = None
        if check_finite:
            xmax = float(x.abs().amax())
            if not math.isfinite(xmax):
                raise DomainError("x contains non-finite entries")
        return x, xmax, int(x.stride(0))
    xm = as_matrix(x, "x", require_finite=False)
    if xm.shape[1] != K:
        raise ShapeError(f"x cols {xm.shape[1]} != sparse rows {K}")
    xmax = None
    if check_finite:
        xmax = float(xm.abs().amax())
        if not math.isfinite(xmax):
            raise DomainError("x contains non-finite entries")
    if xm.dtype != torch.bfloat16:
        xm = xm.to(torch.bfloat16)
    if K % 8:
        xm = torch.nn.functional.pad(xm, (0, 8 - K % 8))
    xm = xm.contiguous()
    if xm.data_ptr() % 16:  # e.g. a single-row slice at an odd column offset
        xm = xm.clone()
    return xm, xmax, int(xm.shape[1])


# the in-kernel U accumulator (int64 fixed point, 2^-26) is exact enough for
# |U| bounds inside this window; outside it U comes from the fp32 pre-kernel
_U_FIXED_MIN, _U_FIXED_MAX = 2.0 ** -6, 2.0 ** 34
_FLAG_PDL, _FLAG_U_FP32, _FLAG_NM24 = 1, 2, 4

_launches = 0


def launch_count() -> int:
    """Kernel launches issued by :func:`salr_linear` since the last reset (one
    fused launch per forward for M <= 256; two when U comes from the fp32
    pre-kernel) -- the device analog of the reference's product counter."""
    return _launches


def reset_launch_count() -> None:
    global _launches
    _launches = 0


def salr_linear(x, s: BitmapSparseMatrix, fused: FusedAdapters | None = None, *, out: torch.Tensor | None = None,
                out_dtype: torch.dtype = torch.float32, stages: int = 0, num_ctas: int = 0,
                check_finite: bool = True, workspace: torch.Tensor | None = None, pdl: bool = False,
                dense_prefill: bool | None = None) -> torch.Tensor:
    """Launch the fused B200 kernel: ``x @ decode(s) [+ (x @ a_cat) @ b_cat]``.

    ``x`` is rounded to bf16 (the compute format); ``s`` is used with bf16
    values (converted once and cached if it holds float32 values).
    ``pdl=True`` launches as a programmatic dependent of the preceding kernel
    (weight streaming overlaps its tail); only valid when that kernel does not
    read ``out`` and the default alternating workspaces are used.
    ``dense_prefill``: None (default) takes the decode-to-dense + tensor-core
    GEMM path from ``DENSE_PREFILL_MIN_M`` tokens on with the default
    schedule; True / False force it / the fused kernels.
    """
    _lib.require_cuda()
    if not isinstance(s, BitmapSparseMatrix):
        raise SalrError("s must be a BitmapSparseMatrix")
    rec2, off2, max_rec2, nm24 = s.kernel_operand()
    xb, xmax, ldx = _prep_x(x, s.rows, check_finite)
    M = int(xb.shape[0])
    N = s.cols
    if fused is not None and (fused.d_in != s.rows or fused.d_out != s.cols):
        raise ShapeError(f"fused adapter dims {(fused.d_in, fused.d_out)} != weight dims {(s.rows, s.cols)}")
    if out_dtype not in (torch.float32, torch.bfloat16):
        raise DomainError(f"out_dtype must be float32 or bfloat16, got {out_dtype}")
    if out is None:
        out = torch.empty((M, N), dtype=out_dtype, device=xb.device)
    elif out.shape != (M, N) or out.dtype not in (torch.float32, torch.bfloat16) or not out.is_contiguous():
        raise ShapeError("out must be a contiguous (M, N) float32/bfloat16 tensor")
    tail = None
    if fused is not None and fused.total_rank > 128:
        # the kernel's adapter operand holds 128 ranks: the rest is added by
        # two fp32 device GEMMs after the launch (rare; the fused path covers
        # the paper's configurations, R = 32..128)
        fused, tail = fused.split(128)
    flags = (_FLAG_PDL if pdl else 0) | (_FLAG_NM24 if nm24 else 0)
    if fused is not None:
        acat, bct = fused.device_operands()
        r_pad = fused.r_pad
        if xmax is not None:
            bound = s.rows * xmax * fused.amax_a
            if bound > _U_FIXED_MAX or (0.0 < bound < _U_FIXED_MIN):
                flags |= _FLAG_U_FP32
    else:
        acat = bct = None
        r_pad = 0
    global _launches
    if dense_prefill is None:
        dense_prefill = stages == 0 and num_ctas == 0 and (
            M >= DENSE_PREFILL_MIN_M or (M > 128 and s.rows * s.cols <= DENSE_SMALL_W_MAX))
    if dense_prefill:
        _launches += 1
        _dense_prefill(xb, s, fused, out, rec2, off2, nm24)
    else:
        ws = _workspace(M, N, s.rows, r_pad, num_ctas, xb.device) if workspace is None else workspace
        _launches += 1 if (fused is None or (M <= 256 and not flags & _FLAG_U_FP32)) else 2
        _lib.check(_lib.load().salr_linear_forward(
            _lib.ptr(xb), M, s.rows, ldx, _lib.ptr(rec2), _lib.ptr(off2), max_rec2, N,
            _lib.ptr(acat), _lib.ptr(bct), r_pad, _lib.ptr(out), _lib.dtype_code(out.dtype), N,
            _lib.ptr(ws), int(ws.numel()), int(stages), int(num_ctas), flags, _lib.stream_ptr()))
    if tail is not None:
        xf = xb[:, : s.rows].float()
        out += ((xf @ tail.a_cat.float()) @ tail.b_cat.float()).to(out.dtype)
    return out


# Prefill-size products (M > 256 tokens, default schedule):
# the weight is decoded once per call into a dense bf16 scratch
# (salr_tb2_decode / salr_nm24_decode, HBM-bound, ~30 us for 4096x14336) and
# multiplied on the tensor cores by cuBLAS, the adapters folded into the same
# GEMM along K: [X | U_hi | U_lo] @ [W; B_cat; B_cat], U = X A_cat split into
# two bf16 halves as in the fused kernel.  With 512+ tokens the decode is
# amortised and the GEMM is tensor-bound; the fused prefill kernel re-reads
# X per column tile.  Measured: faster than the fused
# prefill kernel at every M > 256 (the decode-size kernel wins up to 256).
DENSE_PREFILL_MIN_M = 257
# Between 129 and 256 tokens the fused decode-size kernel streams the weight
# twice (two 128-token chunks): there the dense path wins for weights up to
# ~32 M entries (q, k, v, o, q|k|v) and loses for the MLP ones
# (profiles/r02_prefill_compare_midM.jsonl).
DENSE_SMALL_W_MAX = 32 * 1024 * 1024
_DENSE_SCRATCH: dict = {}


def _dense_scratch(rows: int, cols: int, device) -> torch.Tensor:
    """bf16 scratch per (device, stream) -- calls on one stream are ordered,
    calls on different streams get their own -- grown on demand, viewed as
    rows x cols."""
    key = (device.index, torch.cuda.current_stream(device).cuda_stream)
    buf = _DENSE_SCRATCH.get(key)
    if buf is None or buf.numel() < rows * cols:
        buf = torch.empty(rows * cols, dtype=torch.bfloat16, device=device)
        _DENSE_SCRATCH[key] = buf
    return buf[: rows * cols].view(rows, cols)


_SIDE_STREAMS: dict = {}


def _side_stream(device) -> torch.cuda.Stream:
    st = _SIDE_STREAMS.get(device.index)
    if st is None:
        st = _SIDE_STREAMS[device.index] = torch.cuda.Stream(device)
    return st


def _dense_prefill(xb, s, fused, out, rec, off, nm24):
    K, N = s.rows, s.cols
    rp = fused.r_pad if fused is not None else 0
    w = _dense_scratch(K + 2 * rp, N, xb.device)
    lib = _lib.load()
    main = torch.cuda.current_stream(xb.device)
    xk = xb[:, :K]
    side = None
    if fused is not None:
        # U = X A_cat and the [X | U_hi | U_lo] operand on a side stream,
        # concurrently with the (HBM-bound) weight decode
        side = _side_stream(xb.device)
        side.wait_stream(main)
        with torch.cuda.stream(side):
            acat, bct = fused.device_operands()
            u = torch.mm(xk, acat, out_dtype=torch.float32)
            hi = u.to(torch.bfloat16)
            lo = (u - hi.float()).to(torch.bfloat16)
            xk = torch.cat([xk, hi, lo], dim=1)
    st = _lib.stream_ptr()
    if nm24:
        _lib.check(lib.salr_nm24_decode(_lib.ptr(rec), K, N, _lib.ptr(w), N, st))
    else:
        _lib.check(lib.salr_tb2_decode(_lib.ptr(rec), _lib.ptr(off), K, N, _lib.ptr(w), N, st))
    if side is not None:
        bt = bct[:N].t()
        w[K:K + rp].copy_(bt)
        w[K + rp:].copy_(bt)
        main.wait_stream(side)
        xk.record_stream(main)
    if out.dtype == torch.float32:
        torch.mm(xk, w, out_dtype=torch.float32, out=out)
    else:
        torch.mm(xk, w, out=out)


_CHAIN_WS: dict = {}
_CHAIN_TURN: dict = {}


def _chain_workspace(M: int, L: int, device) -> torch.Tensor:
    """Per-device chain scratch, two alternating buffers (as ``_workspace``)."""
    need = int(_lib.load().salr_chain_workspace_bytes(M, L))
    turn = _CHAIN_TURN.get(device.index, 0)
    _CHAIN_TURN[device.index] = turn ^ 1
    ws = _CHAIN_WS.get((device.index, turn))
    if ws is None or ws.numel() < need:
        for t in (0, 1):
            _CHAIN_WS[(device.index, t)] = torch.zeros(need, dtype=torch.uint8, device=device)
        ws = _CHAIN_WS[(device.index, turn)]
    return ws


def salr_chain(x, linears, outs, *, pdl: bool = False, workspace: torch.Tensor | None = None):
    """A chain of SALR linears in ONE persistent launch: ``outs[0] = x @ W_0
    [+ adapters]``, ``outs[l] = outs[l-1][:, :K_l] @ W_l [+ adapters]``
    (bf16 outputs).  ``linears`` is a list of ``(BitmapSparseMatrix,
    FusedAdapters | None)``, at most 4, M <= 256.  The weight stream runs
    through the linear boundaries; only the next linear's X tiles wait for the
    previous output (see csrc/salr_chain.cuh).  Results equal running
    :func:`salr_linear` per linear on the same grid."""
    _lib.require_cuda()
    L = len(linears)
    if not 1 <= L <= 4 or len(outs) != L:
        raise ConfigError("a chain holds 1..4 linears and one output per linear")
    xb, _, ldx0 = _prep_x(x, linears[0][0].rows, False)
    M = int(xb.shape[0])
    if M > 256:
        raise ConfigError("chained linears are decode-size (M <= 256)")
    arr = (_lib.ChainLinear * L)()
    keep = []
    prev_n = None
    for l, ((s, fused), y) in enumerate(zip(linears, outs)):
        if not isinstance(s, BitmapSparseMatrix):
            raise SalrError("chain entries must be BitmapSparseMatrix")
        if y.shape != (M, s.cols) or y.dtype != torch.bfloat16 or not y.is_contiguous():
            raise ShapeError(f"outs[{l}] must be a contiguous ({M}, {s.cols}) bfloat16 tensor")
        if l and s.rows > prev_n:
            raise ShapeError(f"linear {l} reads {s.rows} columns of a {prev_n}-column output")
        if s.rows % 8:
            raise ShapeError("chained linears need K a multiple of 8")
        if fused is not None and fused.total_rank > 128:
            raise ConfigError("chained linears take fused rank <= 128")
        if s.is_nm24():
            raise ConfigError("chained linears read TB2 records; NM24 matrices run through salr_linear")
        rec2, off2, mx = s.compute_format()
        acat = bct = None
        r_pad = 0
        if fused is not None:
            acat, bct = fused.device_operands()
            r_pad = fused.r_pad
        keep += [rec2, off2, acat, bct]
        arr[l] = _lib.ChainLinear(_lib.ptr(rec2), _lib.ptr(off2), mx, s.rows, s.cols, _lib.ptr(acat),
                                  _lib.ptr(bct), r_pad, _lib.ptr(y), s.cols)
        prev_n = s.cols
    ws = workspace if workspace is not None else _chain_workspace(M, L, xb.device)
    global _launches
    _launches += 1
    _lib.check(_lib.load().salr_chain_forward(ctypes.addressof(arr), L, _lib.ptr(xb), M, ldx0,
                                              _lib.ptr(ws), int(ws.numel()), _FLAG_PDL if pdl else 0,
                                              _lib.stream_ptr()))
    return outs


def _check_probe(probe):
    if probe is None:
        return
    for d in (probe.decode_delay, probe.compute_delay):
        if d is not None and not isinstance(d, (int, float)):
            raise ConfigError("host delay callables cannot be injected into the device pipeline; pass the "
                              "maximum device jitter in nanoseconds instead")


def _run_probed(probe, fn):
    """Run one launch with the device probe armed; decode the log into the
    reference's (slot, old, new) transition list."""
    if probe is None:
        return fn()
    delay = int(max(probe.decode_delay or 0, probe.compute_delay or 0))
    lib = _lib.load()
    words = 1 << 20
    log = torch.zeros(words, dtype=torch.int32, device="cuda")
    _lib.check(lib.salr_debug_set_probe(_lib.ptr(log), words, delay, int(probe.seed) & 0xFFFFFFFF))
    try:
        out = fn()
        torch.cuda.synchronize()
    finally:
        lib.salr_debug_set_probe(None, 0, 0, 0)
    head = log[:4].cpu().tolist()
    n = head[0]
    if n > words - 4:
        raise VerificationError(f"probe log overflow ({n} transitions)")
    info = (ctypes.c_int32 * 12)()
    lib.salr_debug_last_launch(ctypes.addressof(info))
    probe.capacity = int(info[0]) * int(info[1])
    probe.produced += head[1]
    probe.consumed += head[2]
    if probe.record:
        ent = log[4:4 + n].cpu().tolist()
        st = (SlotState.EMPTY, SlotState.FILLED, SlotState.CONSUMED)
        probe.transitions.extend(((e >> 8) & 0xFFFFFF, st[(e >> 4) & 15], st[e & 15]) for e in ent)
    return out


def pipelined_matmul(x, s: BitmapSparseMatrix, cfg: PipelineConfig, probe: PipelineProbe | None = None,
                     out_dtype: torch.dtype = torch.float32) -> torch.Tensor:
    """``x @ decode(s)`` through the fused kernel (``pipeline.py:258-272``)."""
    _check_probe(probe)
    return _run_probed(probe, lambda: salr_linear(x, s, None, out_dtype=out_dtype, stages=cfg.device_stages))


def pipelined_forward(x, s: BitmapSparseMatrix, fused: FusedAdapters, cfg: PipelineConfig,
                      probe: PipelineProbe | None = None, out_dtype: torch.dtype = torch.float32) -> torch.Tensor:
    """The SALR linear ``x @ decode(s) + (x @ a_cat) @ b_cat`` (``pipeline.py:275-331``)."""
    _check_probe(probe)
    if fused.d_in != s.rows or fused.d_out != s.cols:
        raise ShapeError(f"fused adapter dims {(fused.d_in, fused.d_out)} != weight dims {(s.rows, s.cols)}")
    return _run_probed(probe, lambda: salr_linear(x, s, fused, out_dtype=out_dtype, stages=cfg.device_stages))


@dataclass(frozen=True)
class BenchResult:
    serial_s: float
    overlapped_s: float
    speedup: float


def bench(x_shape, s: BitmapSparseMatrix, cfg: PipelineConfig, repeats: int = 5, seed: int = 0) -> BenchResult:
    """Median device times of the serial (1-slot ring) and overlapped
    schedules with a bit-identity gate (``pipeline.py:380-436``).  Timed with
    CUDA events; absolute numbers come from ``bench.py``."""
    if repeats < 3:
        raise DomainError("repeats must be >= 3")
    g = torch.Generator().manual_seed(seed)
    x = torch.randn(tuple(x_shape), generator=g).to(torch.bfloat16)
    serial = PipelineConfig(cfg.tile_rows, cfg.tile_col_bytes, cfg.ring_capacity, overlap=False)
    over = PipelineConfig(cfg.tile_rows, cfg.tile_col_bytes, max(cfg.ring_capacity, 2), overlap=True)
    a = pipelined_matmul(x, s, serial)
    b = pipelined_matmul(x, s, over)
    if not torch.equal(a, b):
        raise VerificationError("serial and overlapped outputs differ")
    xd, _, _ = _prep_x(x, s.rows, True)

    def timed(c):
        pipelined_matmul(xd, s, c)
        ts = []
        for _ in range(repeats):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            pipelined_matmul(xd, s, c)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) / 1e3)
        return float(statistics.median(ts))

    ts, to = timed(serial), timed(over)
    return BenchResult(serial_s=ts, overlapped_s=to, speedup=ts / to)
