"""Pruned ResNet-50 for CIFAR-scale inputs on the sparse engine (BASELINE configs[2]).

The reference has no ResNet; SURVEY.md §8d (cfg3) defines the network from its
pieces: a 3x3 stem (stride 1, no max-pool), bottleneck stages at 32/16/8/4 with
widths 64/128/256/512 (3/4/6/3 blocks, expansion 4, stride on the 3x3 and the
projection), 53 sparse convs.  Two precisions, as the reference's modes:
  fp32 -- every conv bit-identical to sparse_conv_forward; block output
          relu(conv3 + shortcut);
  fp16 -- 16b/16b (quantization.py:257-301): binary16 weights and activations,
          every layer output rounded to binary16 (the conv hook), the residual add
          rounded again, then ReLU.
Stride-2 layers use the reference's exact geometries (ConvGeometry rejects 32 -> 16
with pad 1, tensor.py:186-190): the 3x3 reads the top/left 33x33 window of its
34x34 zero-haloed input (pad 0), the 1x1 projection the top/left 31x31 window --
through usc_conv_forward_view, no copies; the 1x1 projection runs as a stride-1 plan over
every 2nd pixel (usc_conv_forward_strided).  Every activation stays resident in the
BI64 layout; the residual add and ReLU are fused into conv3's epilogue.
"""

from __future__ import annotations

import ctypes
import zlib

import numpy as np

from . import _lib
from .csr import build_csr
from .engine import ExecConfig, launch, plan_for, tile_candidates, time_median_cuda
from .pruning import synthesize_masked_weights
from .tensor import ConvGeometry, PrecisionMode

STAGES = ((64, 3, 1), (128, 4, 2), (256, 6, 2), (512, 3, 2))  # (width, blocks, stride)


def resnet50_layers(hw: int = 32):
    """[(name, ConvGeometry, role, stride)] in execution order; role in {stem, c1, c2,
    c3, proj}."""
    out = [("stem", ConvGeometry(3, 64, 3, 3, hw, hw, padding=(1, 1)), "stem", 1)]
    c_in = 64
    for si, (width, blocks, stride) in enumerate(STAGES):
        for b in range(blocks):
            s = stride if b == 0 else 1
            tag = f"s{si}b{b}"
            out.append((f"{tag}.c1", ConvGeometry(c_in, width, 1, 1, hw, hw), "c1", 1))
            if s == 2:
                out.append((f"{tag}.c2", ConvGeometry(width, width, 3, 3, hw + 1, hw + 1, stride=(2, 2)), "c2", 2))
            else:
                out.append((f"{tag}.c2", ConvGeometry(width, width, 3, 3, hw, hw, padding=(1, 1)), "c2", 1))
            hw_out = hw // s
            if b == 0:
                if s == 2:
                    g = ConvGeometry(c_in, 4 * width, 1, 1, hw - 1, hw - 1, stride=(2, 2))
                else:
                    g = ConvGeometry(c_in, 4 * width, 1, 1, hw, hw)
                out.append((f"{tag}.proj", g, "proj", s))
            out.append((f"{tag}.c3", ConvGeometry(width, 4 * width, 1, 1, hw_out, hw_out), "c3", 1))
            c_in, hw = 4 * width, hw_out
    return out


def resnet50_weights(sparsity: float, seed: int = 0, precision=PrecisionMode.BINARY32):
    rng = np.random.default_rng([seed, zlib.crc32(b"resnet50-cifar"), int(round(sparsity * 1000))])
    return [synthesize_masked_weights(g, sparsity, rng, precision) for _, g, _, _ in resnet50_layers()]


class SparseResNet50:
    """ResNet-50 CIFAR conv trunk (53 sparse convs) on one GPU for a fixed batch.
    forward(x): plain NCHW (n,3,32,32) -> (n,2048,4,4) features."""

    def __init__(self, weights, batch: int, precision=PrecisionMode.BINARY32, device=None, backends=None):
        import torch
        self.precision = precision
        self.dtype = _lib.USC_F16 if precision is PrecisionMode.BINARY16 else _lib.USC_F32
        self.tdtype = torch.float16 if self.dtype == _lib.USC_F16 else torch.float32
        self.eb = 2 if self.dtype == _lib.USC_F16 else 4
        self.batch = batch
        self.device = torch.device(device or "cuda")
        self.layers = resnet50_layers()
        # (plan geometry, pixel step): a stride-2 1x1 projection runs as a stride-1 1x1
        # plan over every 2nd pixel (usc_conv_forward_strided: the TMA map skips the
        # pixels the projection never reads); same entries, same order, same bits
        self.eff = []
        for _, g, role, s in self.layers:
            if role == "proj" and s > 1:
                self.eff.append((ConvGeometry(g.in_channels, g.out_channels, 1, 1, g.out_h, g.out_w), s))
            else:
                self.eff.append((g, 1))
        self.filters = [build_csr(w, eg) for w, (eg, _) in zip(weights, self.eff)]
        self.weights = weights
        self.configs = [ExecConfig(samples_per_cta=64) for _ in self.layers]
        self.backends = list(backends) if backends is not None else ["sparse"] * len(self.layers)
        self.tc_cfg = {}  # per tensor-core conv: (pixels per tile, K splits), 0 = automatic (autotune_tc)
        self._check_backends()
        self.graph = None
        self._build()

    # -- per-layer backend (the reference's backend_config, bench.py:212-227) ----------
    def dense_eligible(self, li: int) -> bool:
        """cuDNN may run conv `li`: binary16 network (the 1e-2 tolerance path; fp32 stays
        all-sparse and bitwise) and channel counts the BI64<->NHWC transposes take."""
        g = self.layers[li][1]
        return (self.dtype == _lib.USC_F16 and g.in_channels % 16 == 0 and g.out_channels % 16 == 0)

    def tc_eligible(self, li: int) -> bool:
        """The tensor-core backend (dense.py) may run conv li: binary16 network, channels
        in % 64 and out % 128, 1x1 / 3x3, stride 1 / 2."""
        from .dense import tc_eligible
        _, g, role, s = self.layers[li]
        return self.dtype == _lib.USC_F16 and tc_eligible(g.in_channels, g.out_channels, g.filter_h, s)

    def _check_backends(self):
        if len(self.backends) != len(self.layers):
            raise ValueError(f"{len(self.backends)} backends for {len(self.layers)} convs")
        for li, b in enumerate(self.backends):
            if b not in ("sparse", "dense", "tc"):
                raise ValueError(f"unknown backend {b!r}")
            if b == "dense" and not self.dense_eligible(li):
                raise ValueError(f"conv {self.layers[li][0]} cannot run dense (binary16 networks with "
                                 f"channels % 16 == 0 only)")
            if b == "tc" and not self.tc_eligible(li):
                raise ValueError(f"conv {self.layers[li][0]} cannot run on the tensor-core backend")

    def _dense_weight(self, li):
        import torch
        if not hasattr(self, "_dense_w"):
            self._dense_w = {}
        if li not in self._dense_w:
            w = torch.from_numpy(np.array(self.weights[li].data)).to(self.device, torch.float16)
            self._dense_w[li] = w.contiguous(memory_format=torch.channels_last)
        return self._dense_w[li]

    def _dense_fn(self, li, x_act, relu, res_act, out_act):
        """cuDNN (torch conv2d: binary16 on tensor cores, channels_last) for conv li on the
        NHWC form of its input; the epilogue in binary16 as the hooks define it:
        sat16(conv) (+ shortcut, sat16 again), ReLU; the NHWC result becomes out_act's."""
        import torch
        _, g, role, s = self.layers[li]
        w = self._dense_weight(li)
        k = g.filter_h

        L = _lib.lib()

        def fn(stream=None):
            y = torch.nn.functional.conv2d(x_act.nhwc_now(), w, stride=s, padding=k // 2)
            if not y.is_contiguous(memory_format=torch.channels_last):
                y = y.contiguous(memory_format=torch.channels_last)
            # one in-place pass: sat16 (binary16 hook, tensor.py:55-60), + shortcut, sat16, ReLU
            r = None if res_act is None else res_act.nhwc_now()
            _lib.check(L.usc_f16_epilogue(_lib.t_ptr(y), None if r is None else _lib.t_ptr(r), y.numel(),
                                          int(relu), _lib.stream_ptr(stream)), "f16 epilogue")
            out_act.held[0] = y
        return fn

    # -- buffers -------------------------------------------------------------------
    def _lay(self, c, hw, halo):
        return _lib.act_layout(c, hw, hw, halo, halo, self.eb, 64)

    def _buf(self, lay):
        import torch
        return torch.zeros(lay.elems(self.batch), dtype=self.tdtype, device=self.device)

    def _build(self):
        """Steps in execution order.  Every activation has a canonical BI64 layout (the halo
        its sparse consumers read) and, when a dense (cuDNN) conv touches it, an NHWC form;
        a form is materialised by a transpose step the first time a consumer needs it, so a
        chain of dense convs stays in NHWC and transposes only run at sparse/dense borders."""
        import torch
        n = self.batch
        net = self
        self.steps = []  # (li, plan, blob, x, x_view_layout | None, y, epilogue) | (li, None, .., fn)
        self._tc_launch = {}  # tensor-core conv -> (launch(twp, splits, ws), input layout, shortcut)
        self.in_layout = self._lay(3, 32, 1)
        self.x_buf = self._buf(self.in_layout)
        L = _lib.lib()

        class Act:
            def __init__(self, c, hw, lay, buf=None):
                self.c, self.hw, self.lay, self.buf = c, hw, lay, buf
                self.held = [None]  # NHWC tensor (written at run time by its producer)
                self.has_nhwc = False

            def bi(self):  # the BI64 buffer, adding an NHWC -> BI transpose the first time
                if self.buf is None:
                    self.buf = net._buf(self.lay)
                    act = self

                    def fn(stream=None):
                        _lib.check(L.usc_nhwc_to_bi(_lib.ref(act.lay), n, _lib.t_ptr(act.held[0]),
                                                    _lib.t_ptr(act.buf), None, None, 0,
                                                    _lib.stream_ptr(stream)), "nhwc_to_bi")
                    net.steps.append((-1, None, None, None, None, None, fn))
                return self.buf

            def nhwc(self):  # request the NHWC form, adding a BI -> NHWC transpose the first time
                if not self.has_nhwc:
                    self.has_nhwc = True
                    t = torch.empty((n, self.c, self.hw, self.hw), dtype=torch.float16, device=net.device,
                                    memory_format=torch.channels_last)
                    self.held[0] = t
                    act = self

                    def fn(stream=None):
                        _lib.check(L.usc_bi_to_nhwc(_lib.ref(act.lay), n, _lib.t_ptr(act.buf), _lib.t_ptr(t),
                                                    _lib.stream_ptr(stream)), "bi_to_nhwc")
                        act.held[0] = t
                    net.steps.append((-1, None, None, None, None, None, fn))
                return self

            def nhwc_now(self):
                return self.held[0]

        def conv(li, xa, c_out, hw_out, halo, relu=True, residual=None):
            name, g, role, s = self.layers[li]
            ya = Act(c_out, hw_out, self._lay(c_out, hw_out, halo))
            if self.backends[li] == "tc":  # tensor cores straight on the BI64 buffers
                from .dense import dense_conv, dense_workspace, pack_weights
                if not hasattr(self, "_tc_w"):
                    self._tc_w = {}
                if li not in self._tc_w:
                    self._tc_w[li] = pack_weights(self.weights[li], self.device)
                w, x, x_lay = self._tc_w[li], xa.bi(), xa.lay
                y = ya.buf = self._buf(ya.lay)
                r, r_lay = (None, None) if residual is None else (residual.bi(), residual.lay)
                twp, sp = self.tc_cfg.get(li, (0, 0))
                ws = dense_workspace(g.in_channels, g.out_channels, g.filter_h, s, n, x_lay, residual is not None,
                                     self.device, twp, sp)

                def launch(twp, sp, ws, stream=None, w=w, x=x, x_lay=x_lay, y=y, y_lay=ya.lay, r=r, r_lay=r_lay,
                           relu=relu, g=g, s=s):
                    dense_conv(w, g.in_channels, g.out_channels, g.filter_h, s, n, x, x_lay, y, y_lay, r, r_lay,
                               relu, stream, ws, twp, sp)
                self._tc_launch[li] = (launch, x_lay, residual is not None)

                def fn(stream=None, launch=launch, twp=twp, sp=sp, ws=ws):
                    launch(twp, sp, ws, stream)
                self.steps.append((li, None, None, None, None, None, fn))
                return ya
            if self.backends[li] == "dense":
                xa.nhwc()
                if residual is not None:
                    residual.nhwc()
                ya.has_nhwc = True
                self.steps.append((li, None, None, None, None, None, self._dense_fn(li, xa, relu, residual, ya)))
                return ya
            x, x_lay = xa.bi(), xa.lay
            plan, blob = plan_for(self.filters[li], n, self.dtype, self.configs[li], self.filters[li].weights,
                                  device=self.device)
            if plan.in_.interleave != 64:
                raise RuntimeError(f"{name}: the network needs BI64 plans")
            e = _lib.Epilogue()
            e.relu, e.scale, e.out_padded, e.out = int(relu), 1.0, 1, ya.lay
            if residual is not None:
                e.residual, e.res_layout, e.res = 1, residual.lay, residual.bi().data_ptr()
            y = ya.buf = self._buf(ya.lay)
            # a window of a larger buffer (the stride-2 exact geometries) goes through the view
            # entry; a stride-2 projection through the strided view
            step = self.eff[li][1]
            view = None
            if step > 1:
                if x_lay.pad_h or x_lay.pad_w:
                    raise RuntimeError(f"{name}: strided projection needs a halo-free input buffer")
                view = (x_lay, step)
            elif (plan.in_.hp, plan.in_.ws) != (x_lay.hp, x_lay.ws):
                view = (x_lay, 1)
            self.steps.append((li, plan, blob, x, view, y, e))
            return ya

        cur = Act(3, 32, self.in_layout, self.x_buf)
        li = 0
        cur = conv(li, cur, 64, 32, 0)  # stem (its output feeds 1x1 convs)
        li += 1
        hw = 32
        for width, blocks, stride in STAGES:
            for b in range(blocks):
                s = stride if b == 0 else 1
                hw_out = hw // s
                blk_in = cur
                h1 = conv(li, blk_in, width, hw, 1)
                li += 1
                h2 = conv(li, h1, width, hw_out, 0)
                li += 1
                if b == 0:
                    sc = conv(li, blk_in, 4 * width, hw_out, 0, relu=False)
                    li += 1
                else:
                    sc = blk_in
                cur = conv(li, h2, 4 * width, hw_out, 0, relu=True, residual=sc)
                li += 1
                hw = hw_out
        self.out_buf, self.out_layout = cur.bi(), cur.lay

    # -- execution -------------------------------------------------------------------
    def _launch(self, st, stream=None):
        li, plan, blob, x, view, y, e = st
        if plan is None:  # dense step (cuDNN)
            e(stream)
            return
        L = _lib.lib()
        sp = _lib.stream_ptr(stream)
        if view is None:
            _lib.check(L.usc_conv_forward(_lib.ref(plan), _lib.t_ptr(blob), _lib.t_ptr(x), _lib.t_ptr(y),
                                          _lib.ref(e), sp), self.layers[li][0])
        elif view[1] == 1:
            _lib.check(L.usc_conv_forward_view(_lib.ref(plan), _lib.t_ptr(blob), _lib.t_ptr(x), _lib.ref(view[0]),
                                               _lib.t_ptr(y), _lib.ref(e), sp), self.layers[li][0])
        else:
            _lib.check(L.usc_conv_forward_strided(_lib.ref(plan), _lib.t_ptr(blob), _lib.t_ptr(x), _lib.ref(view[0]),
                                                  view[1], view[1], _lib.t_ptr(y), _lib.ref(e), sp),
                       self.layers[li][0])

    def load_input(self, x, stream=None):
        _lib.check(_lib.lib().usc_pad_input(_lib.ref(self.in_layout), self.dtype, self.batch, _lib.t_ptr(x),
                                            _lib.t_ptr(self.x_buf), _lib.stream_ptr(stream)), "pad")

    def run(self, stream=None):
        for st in self.steps:
            self._launch(st, stream)

    def output(self, stream=None):
        import torch
        lay = self.out_layout
        out = torch.empty((self.batch, lay.channels, lay.height, lay.width), dtype=self.tdtype, device=self.device)
        _lib.check(_lib.lib().usc_unpad_output(_lib.ref(lay), self.dtype, self.batch, _lib.t_ptr(self.out_buf),
                                               _lib.t_ptr(out), _lib.stream_ptr(stream)), "unpad")
        return out

    def forward(self, x):
        self.load_input(x)
        if self.graph is not None:
            self.graph.replay()
        else:
            self.run()
        return self.output()

    def capture(self):
        import torch
        s = torch.cuda.Stream(device=self.device)
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            self.run()
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.run()
        self.graph = g
        return g

    # -- tuned state (per-conv tiles) -------------------------------------------------
    def tuned_state(self) -> dict:
        import dataclasses
        return {"configs": [dataclasses.asdict(c) for c in self.configs], "backends": list(self.backends),
                "tc_cfg": {str(k): list(v) for k, v in self.tc_cfg.items()}}

    def load_tuned_state(self, state) -> None:
        """Accepts tuned_state() output (or a bare list of ExecConfig dicts)."""
        if isinstance(state, dict):
            if "backends" in state:
                self.backends = list(state["backends"])
                self._check_backends()
            self.tc_cfg = {int(k): tuple(v) for k, v in state.get("tc_cfg", {}).items()}
            state = state["configs"]
        if len(state) != len(self.layers):
            raise ValueError(f"tuned state has {len(state)} configs for {len(self.layers)} convs")
        self.configs = [ExecConfig(**c) for c in state]
        self.graph = None
        self._build()

    def autotune(self, repeats: int = 3, warmup: int = 1, noise_floor: float = 0.02):
        """Per-conv tile search on the network's own buffers and epilogues."""
        import torch
        picks = list(self.configs)
        for st in self.steps:
            li, plan0, _, x, view, y, e = st
            if plan0 is None:  # dense conv or transpose: no tile to search
                continue
            g = self.eff[li][0]
            cands = [self.configs[li]] + [c for c in tile_candidates(g, self.batch, [1], self.precision, (3,))
                                          if c.samples_per_cta == 64]
            res = []
            for cfg in cands:
                try:
                    plan, blob = plan_for(self.filters[li], self.batch, self.dtype, cfg, self.filters[li].weights,
                                          device=self.device)
                except ValueError:
                    continue
                trial = (li, plan, blob, x, view, y, e)
                try:
                    ms = time_median_cuda(lambda: self._launch(trial), repeats, warmup)
                except RuntimeError:
                    continue
                res.append((ms, cfg))
            best = min(ms for ms, _ in res)
            picks[li] = next(cfg for ms, cfg in res if ms <= best * (1.0 + noise_floor))
            self.filters[li]._packs.clear()
        torch.cuda.synchronize()
        self.configs = picks
        self.graph = None
        self._build()
        return picks

    def network_ms(self, steps: int = 10) -> float:
        """Median device time of one captured forward (CUDA graph replay)."""
        import torch
        self.capture()
        for _ in range(3):
            self.graph.replay()
        torch.cuda.synchronize()
        ts = []
        for _ in range(steps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            self.graph.replay()
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b))
        return float(np.median(ts))

    def autotune_backends(self, repeats: int = 5, warmup: int = 2) -> list:
        """Sparse vs cuDNN per conv (binary16 only; the reference's backend_config rule,
        bench.py:212-227: argmin, exact ties to dense).  A dense conv's cost depends on
        its neighbours (transposes only at sparse/dense borders), so the choice is made on
        whole-network time: the per-conv argmin of the isolated costs (sparse step vs the
        cuDNN conv alone), every "dense from block k on" split, all sparse and all dense
        are each built, captured and timed, and the fastest assignment wins."""
        import torch
        if self.dtype != _lib.USC_F16:
            raise ValueError("the backend dispatcher runs binary16 networks only (fp32 stays bitwise)")
        torch.backends.cudnn.benchmark = True
        nl = len(self.layers)
        elig = [self.dense_eligible(li) for li in range(nl)]

        def build(backends):
            self.backends = list(backends)
            self.graph = None
            self._build()

        build(["sparse"] * nl)
        sparse_ms = {st[0]: time_median_cuda(lambda: self._launch(st), repeats, warmup)
                     for st in self.steps if st[1] is not None}
        build(["dense" if e else "sparse" for e in elig])
        self.run()  # materialise every NHWC form once
        torch.cuda.synchronize()
        dense_ms = {st[0]: time_median_cuda(lambda: self._launch(st), repeats, warmup)
                    for st in self.steps if st[1] is None and st[0] >= 0}
        argmin = ["dense" if elig[li] and dense_ms[li] <= sparse_ms[li] else "sparse" for li in range(nl)]
        tce = [self.tc_eligible(li) for li in range(nl)]
        build(["tc" if e else "sparse" for e in tce])
        tc_ms = {st[0]: time_median_cuda(lambda: self._launch(st), repeats, warmup)
                 for st in self.steps if st[1] is None and st[0] >= 0}
        # the tensor-core backend works on the BI64 buffers (no transposes): isolated costs add up
        tc_argmin = ["tc" if tce[li] and tc_ms[li] <= sparse_ms[li] else "sparse" for li in range(nl)]
        tc_argmin_dense = ["tc" if tce[li] and tc_ms[li] <= sparse_ms[li] else
                           ("dense" if elig[li] and dense_ms[li] <= sparse_ms[li] else "sparse") for li in range(nl)]
        blocks = [li for li, (name, _, role, _) in enumerate(self.layers) if role == "c1"]
        cands = {"all-sparse": ["sparse"] * nl, "all-dense": ["dense" if e else "sparse" for e in elig],
                 "argmin": argmin, "tc-argmin": tc_argmin, "tc-argmin+dense": tc_argmin_dense,
                 "min3": [min((("sparse", sparse_ms[li]),) + ((("tc", tc_ms[li]),) if tce[li] else ()) +
                              ((("dense", dense_ms[li]),) if elig[li] else ()), key=lambda kv: kv[1])[0]
                          for li in range(nl)],
                 "all-tc": ["tc" if e else "sparse" for e in tce]}
        for k in blocks:
            cands[f"dense-from-{self.layers[k][0]}"] = ["dense" if elig[li] and li >= k else "sparse"
                                                        for li in range(nl)]
            cands[f"argmin-then-dense-from-{self.layers[k][0]}"] = [
                "dense" if elig[li] and li >= k else argmin[li] for li in range(nl)]
        times = {}
        for name, bk in cands.items():
            key = tuple(bk)
            if key in {tuple(v) for n2, v in cands.items() if n2 in times}:
                continue
            build(bk)
            times[name] = self.network_ms()
        best = min(times, key=times.get)
        self.backend_times = {self.layers[li][0]: {"sparse_ms": sparse_ms.get(li), "dense_ms": dense_ms.get(li),
                                                   "tc_ms": tc_ms.get(li)} for li in range(nl)}
        self.backend_search = {k: round(v, 4) for k, v in times.items()}
        self.backend_pick = best
        build(cands[best])
        torch.cuda.synchronize()
        self.autotune_tc()
        return self.backends

    def autotune_tc(self) -> dict:
        """Tile search of every tensor-core conv (dense.tune_tile on the layer's own
        buffers and epilogue); kept only if the captured network gets faster."""
        from .dense import tune_tile
        if not self._tc_launch:
            return self.tc_cfg
        before, old = self.network_ms(), dict(self.tc_cfg)
        for li, (launch, x_lay, res) in sorted(self._tc_launch.items()):
            _, g, _, s = self.layers[li]
            self.tc_cfg[li] = tune_tile(launch, g.in_channels, g.out_channels, g.filter_h, s, self.batch, x_lay, res,
                                        self.device)
        self.graph = None
        self._build()
        after = self.network_ms()
        if after > before:
            self.tc_cfg = old
            self.graph = None
            self._build()
        self.tc_search = {"auto_ms": round(before, 4), "tuned_ms": round(after, 4)}
        return self.tc_cfg
