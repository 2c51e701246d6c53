"""Host-side logic of the product (no GPU): encoder, validation, file format,
quantisation primitives, planner/packer, and the C ABI surface."""
import ctypes
import os
import re
import subprocess

import hashlib

import numpy as np
import pytest

import oracle
import paper_2112_15445_b200 as U
from paper_2112_15445_b200 import _lib
from paper_2112_15445_b200.engine import make_plan
from golden_util import geom, golden, layer_inputs, sha

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def G(t):
    c, d, kh, kw, h, w, s, p = t
    return U.ConvGeometry(c, d, kh, kw, h, w, tuple(s), tuple(p))


def test_abi_exports_every_header_symbol():
    hdr = open(os.path.join(ROOT, "include", "unsparse_b200.h")).read()
    declared = set(re.findall(r"^\w[\w\s\*]*?\b(usc_\w+)\s*\(", hdr, re.M))
    assert len(declared) >= 20
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\bT (usc_\w+)", out))
    assert declared <= exported, declared - exported
    assert declared == set(_lib.EXPORTED), declared ^ set(_lib.EXPORTED)
    assert _lib.lib().usc_abi_version() == 1


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_encoder_random_corpus_bitwise():
    rng = np.random.default_rng([0, 1])
    for rec in golden()["random_cases"]:
        x, w, g, sb = oracle.random_case(rng, binary16=rec["binary16"])
        f = U.build_csr(U.DenseTensor4.from_array(w), G(rec["geometry"]))
        assert f.n_nz == rec["csr"]["n_nz"]
        assert sha(f.row_ptr) == rec["csr"]["row_ptr"]
        assert sha(f.col_offsets) == rec["csr"]["col_offsets"]
        assert sha(f.weights) == rec["csr"]["weights"]
        back = U.csr_to_dense(f)
        assert np.array_equal(back.data, w)  # verify.py:72-82 roundtrip


def test_encoder_spec_examples():
    e = golden()["kats"]["encoder_D2"]
    f = U.build_csr(U.DenseTensor4.from_array(np.array(e["weights"], np.float32)), G(e["geometry"]))
    assert (f.n_nz, f.row_ptr.tolist(), f.col_offsets.tolist(), f.weights.tolist()) == \
        (3, [0, 3, 6], [0, 0, 4, 0, 5, 8], [0, 0, 5, 1, 2, 3])
    z = U.build_csr(U.DenseTensor4.from_array(np.zeros((3, 2, 3, 3), np.float32)),
                    U.ConvGeometry(2, 3, 3, 3, 5, 5, padding=(1, 1)))
    assert z.n_nz == 1 and z.row_ptr.tolist() == [0, 1, 2, 3]
    assert U.csr.tap_to_offset(0, 1, 2, U.ConvGeometry(1, 1, 3, 3, 4, 4)) == 6
    assert len(U.plan_blocks(U.ConvGeometry(3, 64, 3, 3, 8, 8, padding=(1, 1)), 128, 4)) == 2048


@pytest.mark.parametrize("name", ["cfg1-vgg16-256x8", "vgg16-512x14", "resnet50-1x1-64x256",
                                  "cnn1d-300x64-k2", "resnet-3x3-s2-prepad"])
def test_encoder_layer_configs(name):
    rec = golden()["layers"][name]
    g = geom(rec["geometry"])
    x, w = layer_inputs(name, g, rec["sparsity"], rec["batch"], rec["binary16"])
    f = U.build_csr(U.DenseTensor4.from_array(w), G(rec["geometry"]))
    assert f.n_nz == rec["csr"]["n_nz"] and sha(f.col_offsets) == rec["csr"]["col_offsets"]
    assert sha(f.weights) == rec["csr"]["weights"] and sha(f.row_ptr) == rec["csr"]["row_ptr"]


def test_corruption_detected():
    """verify.py:85-96: an out-of-range offset raises CsrCorruptionError."""
    g = U.ConvGeometry(2, 2, 3, 3, 6, 6)
    w = np.random.default_rng([0, 3]).standard_normal((2, 2, 3, 3)).astype(np.float32)
    f = U.build_csr(U.DenseTensor4.from_array(w), g)
    bad = f.col_offsets.copy()
    bad[-1] = g.x_size + 5
    with pytest.raises(U.CsrCorruptionError):
        U.CsrFilter(f.row_ptr, bad, f.weights, f.n_nz, g)
    bad = f.col_offsets.copy()
    bad[0] = 3  # kw = 3 is not a 3x3 tap
    with pytest.raises(U.CsrCorruptionError):
        U.CsrFilter(f.row_ptr, bad, f.weights, f.n_nz, g)
    with pytest.raises(U.CsrCorruptionError):
        U.CsrFilter(f.row_ptr[:-1], f.col_offsets, f.weights, f.n_nz, g)
    assert issubclass(U.CsrCorruptionError, ValueError)


def test_geometry_errors():
    with pytest.raises(ValueError):
        U.ConvGeometry(1, 1, 3, 3, 32, 32, stride=(2, 2), padding=(1, 1))  # not integral
    with pytest.raises(ValueError):
        U.ConvGeometry(1, 1, 3, 3, 2, 2)
    with pytest.raises(ValueError):
        U.ExecConfig(0)
    with pytest.raises(ValueError):
        U.ExecConfig(3).block_count(8, 4)


@pytest.mark.parametrize("name", sorted(golden()["layers"]))
def test_save_load_csr_byte_compatible(tmp_path, name):
    """save_csr writes exactly the bytes the reference's save_csr writes (binary and
    JSON sidecar; sha256 recorded by make_golden.py), and load_csr reads them back."""
    rec = golden()["layers"][name]
    g = geom(rec["geometry"])
    prec = U.PrecisionMode.BINARY16 if rec["binary16"] else U.PrecisionMode.BINARY32
    _, w = layer_inputs(name, g, rec["sparsity"], rec["batch"], binary16=rec["binary16"])
    f = U.build_csr(U.DenseTensor4.from_array(w, prec), G(rec["geometry"]))
    U.save_csr(f, tmp_path / "f.csr")
    assert hashlib.sha256((tmp_path / "f.csr").read_bytes()).hexdigest() == rec["csr_file"]["binary"]
    assert hashlib.sha256((tmp_path / "f.csr.json").read_bytes()).hexdigest() == rec["csr_file"]["sidecar"]
    f2 = U.load_csr(tmp_path / "f.csr")
    assert f2.n_nz == f.n_nz and np.array_equal(f2.col_offsets, f.col_offsets)
    assert np.array_equal(f2.weights, f.weights) and f2.geometry == f.geometry
    assert f2.precision is prec


def test_save_csr_lossless_codebook_weights(tmp_path):
    """4b/16b weights (16-bit fixed-point centroids) survive a BINARY16 filter's
    save/load only with lossless=True (f4 payload, tag 2)."""
    rng = np.random.default_rng(5)
    g = U.ConvGeometry(16, 8, 3, 3, 6, 6, padding=(1, 1))
    w = rng.standard_normal((8, 16, 3, 3)).astype(np.float32)
    w[rng.random(w.shape) < 0.8] = 0.0
    cb = U.kmeans_codebook(w, 16, 16)
    wc = cb.reconstruct(w.shape)
    f = U.CsrFilter(*(lambda t: (t.row_ptr, t.col_offsets, t.weights, t.n_nz))(
        U.build_csr(U.DenseTensor4.from_array(wc), g)), g, U.PrecisionMode.BINARY16)
    assert not np.array_equal(f.weights.astype(np.float16).astype(np.float32), f.weights)
    U.save_csr(f, tmp_path / "lossy.csr")
    U.save_csr(f, tmp_path / "lossless.csr", lossless=True)
    lossy, lossless = U.load_csr(tmp_path / "lossy.csr"), U.load_csr(tmp_path / "lossless.csr")
    assert not np.array_equal(lossy.weights, f.weights)
    assert np.array_equal(lossless.weights, f.weights)
    assert lossless.precision is U.PrecisionMode.BINARY16


def test_quantisation_primitives_match_golden():
    k = golden()["kats"]
    for amax, (ib, fb, sg) in k["fit_fixed_point"].items():
        p = U.fit_fixed_point(np.array([float(amax), -0.1]), 8)
        assert (p.int_bits, p.frac_bits, p.sigma) == (ib, fb, sg)
    assert U.linear_quantize(0.7, U.fit_fixed_point(np.array([1.0]), 8)) == 0.703125
    assert U.linear_quantize(3.2, U.fit_fixed_point(np.array([3.2]), 8)) == 3.1875
    cb = U.kmeans_codebook(np.array([1.0, 1.1, -2.0, -2.1]), 2)
    assert cb.centroids.tolist() == k["kmeans_4pts"]["centroids"]
    assert cb.assignments.tolist() == k["kmeans_4pts"]["assignments"]
    # quantizer bound (verify.py:99-108)
    data = np.random.default_rng([0, 4]).uniform(-3.0, 3.0, size=257)
    p = U.fit_fixed_point(data, 8)
    lim = (2 ** 7 - 1) * p.sigma
    grid = np.linspace(-lim, lim, 10000)
    assert np.max(np.abs(U.linear_quantize(grid, p) - grid)) <= p.sigma / 2 + 1e-12


@pytest.mark.parametrize("name", ["cb4-vgg16-256x8", "cb4-vgg16-128x16"])
def test_native_kmeans_bitwise(name):
    rec = golden()["cb4"][name]
    g = geom(rec["geometry"])
    _, w = layer_inputs(name, g, rec["sparsity"], rec["batch"])
    cb = U.kmeans_codebook(w, 16, 16)
    assert cb.centroids.tolist() == rec["centroids"]
    assert cb.quantized_centroids.tolist() == rec["quantized_centroids"]
    assert sha(cb.assignments) == rec["assignments"]
    assert sha(cb.reconstruct(w.shape)) == rec["wc"]


@pytest.mark.parametrize("name", ["int8-vgg16-256x8", "int8-1x1-256x64"])
def test_int8_filter_matches_reference_composition(name):
    rec = golden()["int8"][name]
    g = geom(rec["geometry"])
    _, w = layer_inputs(name, g, rec["sparsity"], rec["batch"])
    fq = U.build_csr_int8(U.DenseTensor4.from_array(w), G(rec["geometry"]))
    assert fq.params.sigma == rec["sigma_w"]
    assert fq.filt.n_nz == rec["csr"]["n_nz"] and sha(fq.filt.weights) == rec["csr"]["weights"]
    assert np.array_equal(fq.codes.astype(np.float64) * fq.params.sigma, fq.filt.weights)


def test_planner_tiles():
    # cfg1 fp32: batch-interleaved kernel, 32 samples per CTA, lane = sample
    g1 = U.ConvGeometry(256, 256, 3, 3, 8, 8, padding=(1, 1))
    p = make_plan(g1, 32, _lib.USC_F32, None)
    assert p.kernel == 3 and p.in_.interleave == 32 and p.NS == 32 and p.in_.ws == 10
    assert p.WS * p.WC <= p.threads // 32 and p.DT == p.WC * p.DW and p.smem_bytes <= 220 * 1024
    assert p.in_.elems(33) == 2 * 256 * 10 * 10 * 32
    # padded-NCHW kernel: full-map tiles, several samples per CTA
    p = make_plan(g1, 32, _lib.USC_F32, U.ExecConfig(kernel=1))
    assert p.kernel == 1 and p.TH == 8 and p.NS * 8 * p.strips_per_row <= 256
    assert p.in_.ws % 4 == 0 and p.in_.hp == 10 and p.groups == 16
    assert p.smem_bytes <= 220 * 1024
    p = make_plan(g1, 32, _lib.USC_F16, None)  # binary16: the BI64 kernel (two samples per lane)
    assert p.kernel == 3 and p.in_.interleave == 64
    p = make_plan(g1, 32, _lib.USC_F16, U.ExecConfig(kernel=1))
    assert p.kernel == 1 and p.in_.ws % 8 == 0
    p = make_plan(g1, 32, _lib.USC_I8, None)  # int8 codes staged as binary16 in BI64
    assert p.kernel == 3 and p.in_.interleave == 64
    assert make_plan(g1, 32, _lib.USC_I8, U.ExecConfig(kernel=1)).kernel == 1
    # 1-D layer runs transposed
    p = make_plan(U.ConvGeometry(64, 64, 2, 1, 300, 1), 8, _lib.USC_F32, None)
    assert p.transposed == 1 and p.out_w == 299 and p.out_h == 1
    # stride 3 falls back to the generic kernel
    p = make_plan(U.ConvGeometry(4, 4, 3, 3, 10, 10, stride=(3, 3), padding=(1, 1)), 2, _lib.USC_F32, None)
    assert p.kernel == 2
    # 32x32 maps tile by rows
    p = make_plan(U.ConvGeometry(64, 64, 3, 3, 32, 32, padding=(1, 1)), 256, _lib.USC_F32,
                  U.ExecConfig(kernel=1))
    assert p.kernel == 1 and p.NS == 1 and p.row_tiles * p.TH >= 32
    p = make_plan(U.ConvGeometry(64, 64, 3, 3, 32, 32, padding=(1, 1)), 256, _lib.USC_F32, None)
    tiles = p.groups * 8 * p.row_tiles * p.col_tiles
    assert p.kernel == 3 and p.row_tiles * p.TH >= 32 and p.grid_x == min(tiles, 148)
    assert p.stages >= 2 and p.smem_bytes <= 224 * 1024
    with pytest.raises(ValueError):
        make_plan(U.ConvGeometry(4, 4, 3, 3, 8, 8, padding=(1, 1)), 6, _lib.USC_F32, U.ExecConfig(4))


def test_packer_dedupes_zero_entries():
    g = U.ConvGeometry(3, 2, 3, 3, 6, 6, padding=(1, 1))
    w = np.zeros((2, 3, 3, 3), np.float32)
    w[0, 0, 0, 1] = 1.0
    w[1, 1, :, :] = 2.0  # 9 nonzeros -> channel 0 gets 8 padding entries
    f = U.build_csr(U.DenseTensor4.from_array(w), g)
    assert f.n_nz == 9
    plan = make_plan(g, 2, _lib.USC_F32, U.ExecConfig(kernel=2))
    size = ctypes.c_int64()
    _lib.check(_lib.lib().usc_pack_size(_lib.ref(plan), f.n_nz, _lib.ref(size)))
    blob = np.zeros(size.value, np.uint8)
    n = ctypes.c_int64()
    _lib.check(_lib.lib().usc_pack(_lib.ref(plan), _lib.np_ptr(f.row_ptr), _lib.np_ptr(f.col_offsets),
                                   _lib.np_ptr(f.weights), f.n_nz, None, _lib.np_ptr(blob), blob.size,
                                   _lib.ref(n)))
    assert n.value == 1 + 1 + 9  # one deduped padding entry + the genuine entries


def test_layer_bench_csv_and_backend_choice():
    from paper_2112_15445_b200 import layer_bench as LB
    ref_csv = ",".join(LB.CSV_HEADER[:19]) + "\n" + \
        "a@90%/binary32,vgg16-512x14,512,512,3,3,14,14,1,1,1,1,8,90,binary32,2,1.5,1.5,1.0\n" + \
        "b@90%/binary32,vgg16-512x14,512,512,3,3,14,14,1,1,1,1,8,90,binary32,2,1.0,2.0,2.0\n"
    rows = LB.rows_from_csv(ref_csv)  # the reference's 19-column CSV reads back
    cfg = LB.backend_config(rows)
    assert cfg["a@90%/binary32"]["backend"] == "dense"  # exact tie -> dense (bench.py:221)
    assert cfg["b@90%/binary32"]["backend"] == "sparse"
    again = LB.rows_from_csv(LB.rows_to_csv(rows))
    assert [r.sparse_ms for r in again] == [1.5, 1.0]
    assert "| a@90%/binary32 |" in LB.rows_to_markdown(rows)
    assert LB.spearman_rho([1, 2, 3, 4], [4, 3, 2, 1]) == -1.0
    assert LB.spearman_rho([1, 1, 2], [1, 1, 2]) == pytest.approx(1.0)
    with pytest.raises(ValueError):
        LB.backend_config(rows, expected_layers=["missing"])
    for name in LB.PRESETS:
        LB.preset_geometry(name)


@pytest.mark.parametrize("name", ["cfg1-vgg16-256x8", "sweep-3x3-256x8-98", "vgg16-512x14"])
def test_every_tile_candidate_fits_its_filter(name):
    """plan_for's entry-reserve search: every autotuner candidate yields a plan whose
    densest (group, chunk) entry block fits the shared-memory reserve."""
    from golden_util import golden, layer_inputs, geom
    rec = golden()["layers"][name]
    g = geom(rec["geometry"])
    _, w = layer_inputs(name, g, rec["sparsity"], rec["batch"], False)
    c, d, kh, kw, h, ww, st, pd = rec["geometry"]
    gg = U.ConvGeometry(c, d, kh, kw, h, ww, tuple(st), tuple(pd))
    f = U.build_csr(U.DenseTensor4.from_array(w), gg)
    for cfg in U.engine.tile_candidates(gg, rec["batch"], [1, 2]):
        p = U.engine.fit_plan(f, rec["batch"], _lib.USC_F32, cfg, f.weights)
        if p.kernel == 3:
            assert U.engine._max_block(f, p, f.weights) <= p.ent_stage_bytes
            assert p.smem_bytes <= 224 * 1024


def test_spearman_matches_scipy_with_ties():
    from scipy.stats import spearmanr

    from paper_2112_15445_b200 import layer_bench as LB
    rng = np.random.default_rng(3)
    for _ in range(20):
        x = rng.integers(0, 5, 17).astype(float)
        y = rng.integers(0, 4, 17).astype(float)
        if np.ptp(x) == 0 or np.ptp(y) == 0:
            continue
        assert LB.spearman_rho(x, y) == pytest.approx(spearmanr(x, y).statistic, abs=1e-12)


def test_empty_batch_like_reference():
    """An empty batch has no virtual blocks (engine.py:85-88): the reference returns a
    (0, D, Yh, Yw) output; so does the engine, without a launch; sub_batch rules as the
    reference (any sub_batch divides 0)."""
    g = U.ConvGeometry(4, 2, 3, 3, 5, 5, padding=(1, 1))
    w = np.random.default_rng(0).standard_normal((2, 4, 3, 3)).astype(np.float32)
    f = U.build_csr(U.DenseTensor4.from_array(w), g)
    x = U.DenseTensor4.from_array(np.zeros((0, 4, 5, 5), np.float32))
    y = U.sparse_conv_forward(x, f, U.ExecConfig(2))
    assert y.shape == (0, 2, 5, 5) and y.data.dtype == np.float32
    assert U.autotune_sb(x, f).sub_batch == 2
    with pytest.raises(ValueError):
        U.sparse_conv_forward(U.DenseTensor4.from_array(np.zeros((3, 4, 5, 5), np.float32)), f, U.ExecConfig(2))


def test_dense_tc_schedule_queries():
    """Host-side schedule decisions of the tensor-core backend (no GPU needed: 148 SMs
    assumed when no device is visible): split-K workspace sizes, the fused-pool gate, and
    argument validation before any driver call."""
    from paper_2112_15445_b200.dense import pool_fusable

    def ws_bytes(C, D, k, s, hw, n, res=False, twp=0, splits=0):
        g = _lib.Geometry(C, D, k, k, hw, hw, s, s, k // 2, k // 2)
        xl = _lib.act_layout(C, hw, hw, k // 2, k // 2, 2, 64)
        return int(_lib.lib().usc_dense_conv_f16_ws_bytes(_lib.ref(g), n, _lib.ref(xl), int(res), twp, splits))

    # VGG conv5 (2x2 maps, 32 two-pixel tiles): automatic split-K, 4 splits of 6 k-iterations
    tiles, splits = 4 * 1 * 2 * 4, 4
    assert ws_bytes(512, 512, 3, 1, 2, 256) == tiles * splits * 128 * 128 * 4 + tiles * 4 + 256
    assert ws_bytes(64, 64, 3, 1, 32, 256) == 0          # 32x32 maps fill the SMs: no split
    assert ws_bytes(512, 512, 3, 1, 2, 256, res=True) == 0  # never with a fused shortcut
    assert ws_bytes(256, 256, 3, 1, 8, 256, twp=4, splits=2) == (2 * 2 * 8 * 4) * 2 * 256 * 128 * 4 + 128 * 4 + 256
    assert ws_bytes(256, 256, 3, 1, 8, 256, twp=4, splits=1) == 0
    # the fused-pool cost model: VGG conv1_2 / conv2_2 fuse, the 8x8 and 4x4 maps do not
    lay = lambda C, hw: _lib.act_layout(C, hw, hw, 1, 1, 2, 64)  # noqa: E731
    assert pool_fusable(64, 64, 256, lay(64, 32)) and pool_fusable(128, 128, 256, lay(128, 16))
    assert not pool_fusable(256, 256, 256, lay(256, 8)) and not pool_fusable(512, 512, 256, lay(512, 4))
    # bad tile arguments fail before any device work
    g = _lib.Geometry(64, 64, 3, 3, 8, 8, 1, 1, 1, 1)
    xl, yl = lay(64, 8), lay(64, 8)
    dummy = ctypes.c_void_p(16)
    rc = _lib.lib().usc_dense_conv_f16_ws(_lib.ref(g), 64, dummy, _lib.ref(xl), dummy, _lib.ref(yl), dummy, None, None,
                                         1, None, 0, 3, 0, None)
    assert rc == _lib.USC_ERR_VALUE
    rc = _lib.lib().usc_dense_conv_f16_ws(_lib.ref(g), 64, dummy, _lib.ref(xl), dummy, _lib.ref(yl), dummy, None, None,
                                         1, None, 0, 0, -1, None)
    assert rc == _lib.USC_ERR_VALUE
