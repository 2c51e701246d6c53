"""Direct sparse convolution engine (/root/reference/pkg/src/unsparse/engine.py).

Same public surface -- ExecConfig, VirtualBlock, plan_blocks,
sparse_conv_forward, sparse_conv_1d, time_median, autotune_sb -- but the work
runs on the B200: the host plans a tile (usc_plan_make), packs the CsrFilter
into the kernel's entry stream once per plan (usc_pack, cached on the filter),
and launches the sm_100a kernel (usc_conv_forward) on the current CUDA stream.
There is no CPU fallback: without the native library or a CUDA device these
functions raise.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from .csr import CsrFilter
from .tensor import ConvGeometry, DenseTensor4, PrecisionMode

SB_CANDIDATES = (2, 4, 8)


@dataclass(frozen=True)
class ExecConfig:
    """engine.py:25-41 plus the B200 tile knobs (0 = planner's choice).

    sub_batch keeps the reference's meaning (samples per virtual block, must
    divide the batch); worker_count is accepted for API parity.  On the GPU a
    virtual block is a CTA: ``samples_per_cta`` samples x ``ch_per_cta`` output
    channels, ``pix_per_thread`` output pixels per thread, ``chunk_channels``
    input channels per shared-memory stage.
    """

    sub_batch: int = 1
    worker_count: int = 1
    pix_per_thread: int = 0
    ch_per_cta: int = 0
    samples_per_cta: int = 0
    chunk_channels: int = 0
    kernel: int = 0
    threads: int = 0
    pixel_warps: int = 0
    stages: int = 0
    rows_per_thread: int = 0
    ent_reserve: int = 0
    pixel_classes: int = 0
    window: int = 0

    def __post_init__(self):
        if self.sub_batch < 1:
            raise ValueError("sub_batch must be >= 1")
        if self.worker_count < 1:
            raise ValueError("worker_count must be >= 1")

    def block_count(self, batch: int, out_channels: int) -> int:
        if batch % self.sub_batch:
            raise ValueError(f"sub_batch {self.sub_batch} does not divide batch {batch}")
        return (batch * out_channels) // self.sub_batch

    def to_c(self) -> _lib.ExecCfg:
        return _lib.ExecCfg(self.sub_batch, self.worker_count, self.pix_per_thread, self.ch_per_cta,
                            self.samples_per_cta, self.chunk_channels, self.threads, self.kernel,
                            self.pixel_warps, self.stages, self.rows_per_thread, self.ent_reserve,
                            self.pixel_classes, self.window)


@dataclass(frozen=True)
class VirtualBlock:
    """engine.py:44-50."""

    out_channel: int
    sample_start: int
    sample_count: int


def plan_blocks(geometry: ConvGeometry, batch: int, sub_batch: int) -> list[VirtualBlock]:
    """engine.py:53-61: batch*D/sb_S blocks, d-major then sample groups."""
    if batch % sub_batch:
        raise ValueError(f"sub_batch {sub_batch} does not divide batch {batch}")
    return [VirtualBlock(d, g0, sub_batch)
            for d in range(geometry.out_channels)
            for g0 in range(0, batch, sub_batch)]


# ---------------------------------------------------------------------------
# plans and device packs

def dtype_of(precision: PrecisionMode) -> int:
    return _lib.USC_F16 if precision is PrecisionMode.BINARY16 else _lib.USC_F32


def make_plan(geometry: ConvGeometry, n: int, dtype: int, config: ExecConfig | None) -> _lib.Plan:
    cfg = (config or ExecConfig()).to_c()
    plan = _lib.Plan()
    g = _lib.make_geometry(geometry)
    _lib.check(_lib.lib().usc_plan_make(_lib.ref(g), n, dtype, _lib.ref(cfg), _lib.ref(plan)), "plan")
    return plan


def plan_for(filt: CsrFilter, n: int, dtype: int, config: ExecConfig | None, payload, table=None,
             device=None):
    """make_plan + device_pack.  For kernel-3 plans the shared-memory entry reserve is
    sized from the filter itself: a plan at chunk length CC is packed dry to measure
    its densest (group, chunk) block, then re-planned with exactly that reserve; when
    input tile + entries no longer fit, CC shrinks until they do."""
    config = config or ExecConfig()
    # fitted plans are cached on the (immutable) filter, so a repeated call costs a
    # dict lookup instead of two make_plan calls and a dry pack of the whole filter
    key = (n, dtype, config, id(payload), None if table is None else np.asarray(table, np.float32).tobytes())
    cache = filt._extra.setdefault("plans", {})
    hit = cache.get(key)
    if hit is None or hit[1] is not payload:
        hit = cache[key] = (fit_plan(filt, n, dtype, config, payload, table), payload)
    plan = hit[0]
    blob, _ = device_pack(filt, plan, payload, table, device)
    return plan, blob


def fit_plan(filt: CsrFilter, n: int, dtype: int, config: ExecConfig | None, payload, table=None) -> _lib.Plan:
    """The planning half of plan_for (host only)."""
    config = config or ExecConfig()
    plan = make_plan(filt.geometry, n, dtype, config)
    if plan.kernel in (3, 4) and not config.ent_reserve:
        fields = {f: getattr(config, f) for f in config.__dataclass_fields__}
        cc, best = plan.CC, None
        while cc >= 1 and best is None:
            fields.update(chunk_channels=cc, ent_reserve=256)
            try:
                probe = make_plan(filt.geometry, n, dtype, ExecConfig(**fields))
                fields.update(chunk_channels=probe.CC,
                              ent_reserve=max(256, _max_block(filt, probe, payload, table)))
                best = make_plan(filt.geometry, n, dtype, ExecConfig(**fields))
            except ValueError:
                if config.chunk_channels:
                    raise
                cc = cc * 3 // 4 if cc > 1 else 0
        if best is None:
            raise ValueError("no chunk length fits this filter's entry blocks in shared memory")
        plan = best
    return plan


def _max_block(filt, plan, payload, table=None) -> int:
    worst = ctypes.c_int64(0)
    tbl = None if table is None else np.ascontiguousarray(table, np.float32)
    _lib.check(_lib.lib().usc_pack(_lib.ref(plan), _lib.np_ptr(filt.row_ptr), _lib.np_ptr(filt.col_offsets),
                                   _lib.np_ptr(np.ascontiguousarray(payload)), filt.n_nz,
                                   None if tbl is None else _lib.np_ptr(tbl), None, 0,
                                   _lib.ref(worst)), "pack")
    return int(worst.value)


def _pack_key(plan: _lib.Plan, device) -> tuple:
    return (plan.dtype, plan.kernel, plan.DT, plan.CC, plan.HS, plan.TWs, plan.in_.ws, plan.in_.hp,
            plan.transposed, plan.groups, plan.n_chunks, plan.ent_stage_bytes, plan.WC, plan.DW,
            plan.ncls_r, plan.ncls_c, plan.in_.interleave, plan.window, str(device))


def device_pack(filt: CsrFilter, plan: _lib.Plan, payload: np.ndarray, table=None, device=None):
    """Kernel entry stream of `filt` for `plan`, cached on the filter (uint8 CUDA tensor)."""
    import torch
    device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    key = _pack_key(plan, device)
    hit = filt._packs.get(key)
    if hit is not None:
        return hit
    L = _lib.lib()
    size = ctypes.c_int64(0)
    _lib.check(L.usc_pack_size(_lib.ref(plan), filt.n_nz, _lib.ref(size)), "pack")
    blob = np.zeros(size.value, np.uint8)
    n_ent = ctypes.c_int64(0)
    tbl = None if table is None else np.ascontiguousarray(table, np.float32)
    _lib.check(L.usc_pack(_lib.ref(plan), _lib.np_ptr(filt.row_ptr), _lib.np_ptr(filt.col_offsets),
                          _lib.np_ptr(payload), filt.n_nz,
                          None if tbl is None else _lib.np_ptr(tbl), _lib.np_ptr(blob), blob.size,
                          _lib.ref(n_ent)), "pack")
    dev = torch.from_numpy(blob).to(device)
    filt._packs[key] = (dev, int(n_ent.value))
    return filt._packs[key]


def padded_input(x_dev, plan: _lib.Plan, stream=None):
    """Plain NCHW storage tensor -> the plan's padded layout (zero_pad, tensor.py:225-235)."""
    import torch
    lay = plan.in_
    # the batch-interleaved kernel stages int8 codes as binary16 (exact)
    dt = torch.float16 if (plan.kernel in (3, 4) and plan.dtype == _lib.USC_I8) else x_dev.dtype
    out = torch.empty(lay.elems(plan.n), dtype=dt, device=x_dev.device)
    _lib.check(_lib.lib().usc_pad_input(_lib.ref(lay), plan.dtype, plan.n, _lib.t_ptr(x_dev),
                                        _lib.t_ptr(out), _lib.stream_ptr(stream)), "pad")
    return out


def launch(plan: _lib.Plan, blob, x_pad, y, epi: _lib.Epilogue | None = None, stream=None):
    """One kernel launch: usc_conv_forward on the current (or given) stream."""
    _lib.check(_lib.lib().usc_conv_forward(_lib.ref(plan), _lib.t_ptr(blob), _lib.t_ptr(x_pad),
                                           _lib.t_ptr(y), None if epi is None else _lib.ref(epi),
                                           _lib.stream_ptr(stream)), "conv")


def _storage_dtype(dtype: int):
    import torch
    return {_lib.USC_F32: torch.float32, _lib.USC_F16: torch.float16, _lib.USC_I8: torch.int8,
            _lib.USC_CB4: torch.float16}[dtype]


def _check_call(input: DenseTensor4, filt: CsrFilter, config: ExecConfig):
    g = filt.geometry
    g.check_input(input)
    if input.precision is not filt.precision:
        raise ValueError("input and filter precisions differ")
    if input.n % config.sub_batch:
        raise ValueError(f"sub_batch {config.sub_batch} does not divide batch {input.n}")


def sparse_conv_forward(input: DenseTensor4, filt: CsrFilter,
                        config: ExecConfig | None = None) -> DenseTensor4:
    """engine.py:64-111 on the B200.

    Validation as the reference (77-82); the padded input is materialised on the
    device (83); the output (84) is written once per element by the kernel
    (the virtual-block plan of 85-108 is the CTA grid); BINARY16 outputs are
    rounded with saturation inside the kernel epilogue (109-110).  The result
    is bit-identical to the reference and device-resident (``.data`` copies it
    to the host on first access).
    """
    import torch
    config = config or ExecConfig()
    _check_call(input, filt, config)
    g = filt.geometry
    if input.n == 0:  # no virtual blocks (engine.py:85-88): the empty output, nothing launched
        return DenseTensor4(np.zeros((0, g.out_channels, g.out_h, g.out_w), np.float32), input.precision)
    dtype = dtype_of(input.precision)
    plan, blob = plan_for(filt, input.n, dtype, config, filt.weights)
    x = input.device()
    x_pad = padded_input(x, plan)
    y = torch.empty((input.n, g.out_channels, g.out_h, g.out_w), dtype=_storage_dtype(dtype),
                    device=x.device)
    launch(plan, blob, x_pad, y)
    return DenseTensor4._adopt(y, input.precision)


def sparse_conv_1d(input: DenseTensor4, filt: CsrFilter,
                   config: ExecConfig | None = None) -> DenseTensor4:
    """engine.py:114-124 (one-dimensional layers run as their H/W transpose)."""
    if input.h != 1 and input.w != 1:
        raise ValueError(f"input {input.shape} is not one-dimensional")
    return sparse_conv_forward(input, filt, config)


def sparse_conv_blocks(xflat, row_ptr, col_offsets, theta, out, blocks, sb, x_size, s_h, s_w,
                       padded_w, stream=None):
    """The numba FFI kernels.sparse_conv_blocks (kernels.py:57-100) with device tensors:
    xflat f32[n*x_size] (materialised padded input), row_ptr/col_offsets int64,
    theta f32, out f32[n,D,Yh,Yw], blocks int64[nb,2].  Writes only the blocks'
    output slices, every stored entry in stored order."""
    _, D, Yh, Yw = out.shape
    blocks = blocks.reshape(-1, 2)
    _lib.check(_lib.lib().usc_sparse_conv_blocks(
        _lib.t_ptr(xflat), _lib.t_ptr(row_ptr), _lib.t_ptr(col_offsets), _lib.t_ptr(theta),
        _lib.t_ptr(out), _lib.t_ptr(blocks), blocks.shape[0], sb, x_size, s_h, s_w, padded_w, D, Yh,
        Yw, _lib.stream_ptr(stream)), "sparse_conv_blocks")


# ---------------------------------------------------------------------------
# timing and autotuning

def _sync():
    import torch
    if torch.cuda.is_available():
        torch.cuda.synchronize()


def time_median(fn, repeats: int = 9, warmup: int = 2) -> float:
    """engine.py:127-136: median wall time of fn() in ms; the device is
    synchronised after every call so asynchronous launches are fully timed."""
    for _ in range(warmup):
        fn()
    _sync()
    times = []
    for _ in range(repeats):
        t0 = time.perf_counter()
        fn()
        _sync()
        times.append(time.perf_counter() - t0)
    return float(np.median(times) * 1e3)


def time_median_cuda(fn, repeats: int = 9, warmup: int = 2, inner: int = 2) -> float:
    """Median device time of fn() in ms, CUDA events on the current stream.  A
    device-side spin is queued ahead of the start event so the timed launches are
    already enqueued when the GPU reaches it: the host's per-launch cost (ctypes,
    tensor-map encoding) never shows up as idle time between the events."""
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    times = []
    for _ in range(repeats):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(300_000)  # ~150 us of device time to enqueue behind
        a.record()
        for _ in range(inner):
            fn()
        b.record()
        b.synchronize()
        times.append(a.elapsed_time(b) / inner)
    return float(np.median(times))


def tile_candidates(geometry: ConvGeometry, n: int, sb_values, precision=PrecisionMode.BINARY32,
                    kernels=None) -> list[ExecConfig]:
    """The autotuner's search space (the paper's hand-chosen block count,
    PAPER.md:739-749, becomes a searched tile).  Kernel 3 (batch-interleaved,
    fp32): pixels per thread x output channels per CTA.  Kernel 1 (padded NCHW):
    samples per CTA (the sb_S analogue) x pixels per thread x channels per CTA."""
    out = []
    yw = geometry.out_w if geometry.input_w != 1 else geometry.out_h
    if kernels is None:
        kernels = (3, 1)
    if 3 in kernels:
        # every compiled k_bi instance x every split of its warps into pixel warps (WS)
        # and channel warps; skip pixel blocks wider/taller than the map and splits
        # that leave pixel warps idle
        yh = geometry.out_h if geometry.input_w != 1 else geometry.out_w
        sw = geometry.stride[1] if geometry.input_w != 1 else geometry.stride[0]
        h16 = precision is PrecisionMode.BINARY16
        for nw, pc, pr, dw, isw, spl in _lib.bi_instances(h16):
            if isw != sw or pc > max(1, yw) and pc > 1 or pr > yh or (spl == 2 and n <= 32 and not h16):
                continue
            strips = -(-yh // pr) * -(-yw // pc)
            for ws in (w for w in range(1, nw + 1) if nw % w == 0):
                if ws > strips:
                    break
                # per-pixel-class runs (halo taps dropped) for 1x1 blocks on small maps
                classes = (0, 1) if (pc == 1 or pr == 1) and yh * yw <= 64 else (0,)
                for st in (2, 3):
                    for pcl in classes:
                        out.append(ExecConfig(sub_batch=min(sb_values), pix_per_thread=pc, rows_per_thread=pr,
                                              ch_per_cta=dw * (nw // ws), kernel=3, threads=nw * 32,
                                              pixel_warps=ws, stages=st, samples_per_cta=32 * spl,
                                              pixel_classes=pcl))
    if 5 in kernels and geometry.stride == (1, 1) and geometry.filter_w in (1, 3) and geometry.input_w != 1:
        # register-window variant of kernel 3 (k_bw, opt-in "kernel 5" of the search): one row
        # of PC pixels per thread, the warp's DW slots sharing one entry stream and each
        # (c, kh) input-row window loaded into registers once.  Measured 2-2.6x slower than
        # k_bi on the VGG layers: the per-entry jump-table dispatch (LDC + BRX)
        # is a latency chain 8-12 warps per SM cannot hide, so it is not in the default search.
        yh, fam = geometry.out_h, 1 if precision is PrecisionMode.BINARY16 else 0
        for f, nw, pc, dw, kw in _lib.bw_instances():
            if f != fam or kw != geometry.filter_w or pc > max(1, yw) and pc > 1:
                continue
            strips = yh * -(-yw // pc)
            for ws in (w for w in range(1, nw + 1) if nw % w == 0):
                if ws > strips:
                    break
                for st in (2, 3):
                    out.append(ExecConfig(sub_batch=min(sb_values), pix_per_thread=pc, rows_per_thread=1,
                                          ch_per_cta=dw * (nw // ws), kernel=3, threads=nw * 32, pixel_warps=ws,
                                          stages=st, samples_per_cta=64, window=1))
    if 4 in kernels and precision is PrecisionMode.BINARY32 and geometry.stride == (1, 1):
        # tensor-memory-fed fp32 BI64 (kernel 4, opt-in: measured slower than kernel 3 on the
        # VGG layers -- short TMEM-bounded chunks, fill and per-load R2UR cost more issue
        # slots than the shared-memory port saves)
        yh = geometry.out_h if geometry.input_w != 1 else geometry.out_w
        for nw, pc, pr, dw, _, _ in _lib.bi_instances(tmem=True):
            if pc > max(1, yw) and pc > 1 or pr > yh:
                continue
            strips = -(-yh // pr) * -(-yw // pc)
            for ws in (w for w in range(1, nw + 1) if nw % w == 0):
                if ws > strips:
                    break
                for st in (3, 4):
                    out.append(ExecConfig(sub_batch=min(sb_values), pix_per_thread=pc, rows_per_thread=pr,
                                          ch_per_cta=dw * (nw // ws), kernel=4, threads=nw * 32,
                                          pixel_warps=ws, stages=st, samples_per_cta=64))
    if 1 in kernels:
        ps = [p for p in (2, 4, 8) if p <= max(2, yw)]
        for sb in sb_values:
            for p in ps:
                for dt in (8, 16):
                    out.append(ExecConfig(sub_batch=sb, samples_per_cta=sb if sb > 1 else 0,
                                          pix_per_thread=p, ch_per_cta=dt, kernel=1))
    feasible, seen = [], set()
    for cfg in out:  # drop tiles that do not fit and duplicates of the same resolved plan
        try:
            plan = make_plan(geometry, n, dtype_of(precision), cfg)
        except ValueError:
            continue
        key = (plan.kernel, plan.P, plan.PR, plan.PC, plan.DT, plan.DW, plan.WS, plan.NS, plan.CC,
               plan.threads, plan.stages, plan.ncls_r, plan.ncls_c, plan.window)
        if key not in seen:
            seen.add(key)
            feasible.append(cfg)
    return feasible


def autotune_sb(input: DenseTensor4, filt: CsrFilter, candidates=SB_CANDIDATES, worker_count: int = 1,
                repeats: int = 9, warmup: int = 2, noise_floor: float = 0.02) -> ExecConfig:
    """engine.py:139-170 on the GPU: time every (sb, tile) candidate with CUDA
    events and return the fastest; medians within `noise_floor` of the best are
    ties resolved toward the smaller sub-batch (then the earlier candidate).
    Candidates that do not divide the batch are skipped; with none usable the
    search runs with sb = 1."""
    import torch
    n = input.n
    usable = sorted(c for c in set(candidates) if n % c == 0) or [1]
    if n == 0:  # nothing to time: every candidate divides an empty batch
        return ExecConfig(usable[0], worker_count)
    g = filt.geometry
    dtype = dtype_of(input.precision)
    x = input.device()
    results = []
    pads = {}
    for cfg in tile_candidates(g, n, usable, input.precision):
        try:
            plan, blob = plan_for(filt, n, dtype, cfg, filt.weights)
        except ValueError:
            continue
        lk = plan.in_.key()
        if lk not in pads:
            pads[lk] = padded_input(x, plan)
        y = torch.empty((n, g.out_channels, g.out_h, g.out_w), dtype=_storage_dtype(dtype),
                        device=x.device)
        ms = time_median_cuda(lambda: launch(plan, blob, pads[lk], y), repeats, warmup)
        results.append((ms, cfg))
    best = min(ms for ms, _ in results)
    filt._packs.clear()  # the candidates' device packs (the caller re-packs its pick)
    for sb in usable:  # ascending, so the smallest near-tie wins
        for ms, cfg in results:
            if cfg.sub_batch == sb and ms <= best * (1.0 + noise_floor):
                return ExecConfig(cfg.sub_batch, worker_count, cfg.pix_per_thread, cfg.ch_per_cta,
                                  cfg.samples_per_cta, cfg.chunk_channels, cfg.kernel, cfg.threads,
                                  cfg.pixel_warps, cfg.stages, cfg.rows_per_thread, cfg.ent_reserve,
                                  cfg.pixel_classes, cfg.window)
    return ExecConfig(usable[0], worker_count)


def autotune_native(input: DenseTensor4, filt: CsrFilter, repeats: int = 9, warmup: int = 2,
                    noise_floor: float = 0.02, payload=None, table=None, dtype: int | None = None) -> ExecConfig:
    """The tile search through the C ABI (usc_autotune): what a non-Python caller of
    libunsparse_b200.so runs.  Same candidates and rule as autotune_sb
    on the fp32 / binary16 path."""
    dtype = dtype_of(input.precision) if dtype is None else dtype
    x = input.device()
    payload = filt.weights if payload is None else np.ascontiguousarray(payload)
    tbl = None if table is None else np.ascontiguousarray(table, np.float32)
    g = _lib.make_geometry(filt.geometry)
    best = _lib.ExecCfg()
    ms = ctypes.c_float(0.0)
    _lib.check(_lib.lib().usc_autotune(_lib.ref(g), input.n, dtype, _lib.np_ptr(filt.row_ptr),
                                       _lib.np_ptr(filt.col_offsets), _lib.np_ptr(payload), filt.n_nz,
                                       None if tbl is None else _lib.np_ptr(tbl), _lib.t_ptr(x), repeats, warmup,
                                       noise_floor, _lib.ref(best), _lib.ref(ms), _lib.stream_ptr()), "autotune")
    return ExecConfig(best.sub_batch, best.worker_count, best.pix_per_thread, best.ch_per_cta,
                      best.samples_per_cta, best.chunk_channels, best.kernel, best.threads, best.pixel_warps,
                      best.stages, best.rows_per_thread, best.ent_reserve, best.pixel_classes, best.window)
