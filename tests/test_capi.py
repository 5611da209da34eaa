"""CPU: the C-ABI library (libdconv_b200.so) loads, exports every symbol the
header declares, and its host-side logic (descriptor validation, shapes,
flops, status codes, generators, plan creation) matches the reference."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "dconv_b200.h")

TABLE_I = [  # layer_table.cpp:11-33 (id, C, K, H, W, R, S, stride)
    (1, 3, 64, 224, 224, 7, 7, 2), (2, 64, 256, 56, 56, 1, 1, 1), (3, 64, 64, 56, 56, 1, 1, 1),
    (4, 64, 64, 56, 56, 3, 3, 1), (5, 256, 64, 56, 56, 1, 1, 1), (6, 256, 512, 56, 56, 1, 1, 2),
    (7, 256, 128, 56, 56, 1, 1, 2), (8, 128, 128, 28, 28, 3, 3, 1), (9, 128, 512, 28, 28, 1, 1, 1),
    (10, 512, 128, 28, 28, 1, 1, 1), (11, 512, 1024, 28, 28, 1, 1, 2), (12, 512, 256, 28, 28, 1, 1, 2),
    (13, 256, 256, 14, 14, 3, 3, 1), (14, 256, 1024, 14, 14, 1, 1, 1), (15, 1024, 256, 14, 14, 1, 1, 1),
    (16, 1024, 2048, 14, 14, 1, 1, 2), (17, 1024, 512, 14, 14, 1, 1, 2), (18, 512, 512, 7, 7, 3, 3, 1),
    (19, 512, 2048, 7, 7, 1, 1, 1), (20, 2048, 512, 7, 7, 1, 1, 1),
]


def header_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(dconv_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_header_symbol(dconv):
    from paper_1808_05567_b200 import _lib

    lib = _lib.lib()
    syms = header_symbols()
    assert len(syms) >= 40
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(_lib.EXPORTS) == syms
    nm = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    for s in syms:
        assert re.search(rf"\bT {s}\b", nm), s


def test_library_is_sm100a(dconv):
    from paper_1808_05567_b200 import _lib

    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True, text=True).stdout
    # tcgen05.mma, TMA tile loads / stores, tcgen05.ld / tcgen05.st (A staged in TMEM), bulk copies
    for mnem in ("UTCHMMA", "UTMALDG", "UTMASTG", "LDTM", "STTM", "UBLKCP"):
        assert mnem in sass, mnem


def test_spec_validation_matches_reference(dconv, orc):
    d = dconv
    for args, exc in [((1, 1, 1, 4, 4, 3, 3, 0), d.InvalidLayerSpec), ((0, 1, 1, 4, 4, 1, 1, 1), d.InvalidLayerSpec),
                      ((1, 1, 1, 4, 4, 7, 7, 1, 0, 0, 16), d.NonIntegralShape)]:
        with pytest.raises(exc):
            d.make_layer_spec(*args)
    s = d.make_layer_spec(1, 3, 64, 224, 224, 7, 7, 2, 16)
    assert (s.pad_h, s.pad_w, s.cb(), s.kb()) == (3, 3, 1, 4)
    s = d.make_layer_spec(1, 17, 33, 8, 8, 1, 1, 1, 16)
    assert (s.cb(), s.kb()) == (2, 3)
    s = d.make_layer_spec(1, 160, 160, 17, 17, 1, 7, 1)
    assert (s.pad_h, s.pad_w) == (0, 3)  # odd-filter default per axis


@pytest.mark.parametrize("row", TABLE_I)
def test_shapes_and_flops_all_table_layers(dconv, orc, row):
    lid, C_, K, H, W, R, S, st = row
    for N in (1, 28, 32):
        s = dconv.make_layer_spec(N, C_, K, H, W, R, S, st)
        o = orc.spec(N, C_, K, H, W, R, S, st)
        assert dconv.derive_output_shape(s) == orc.output_shape(o)
        assert dconv.pass_flops(s) == orc.pass_flops(o)


def test_engine_config_defaults(dconv):
    from paper_1808_05567_b200 import _lib

    c = _lib.EngineCfg()
    _lib.lib().dconv_engine_config_default(C.byref(c))
    ref = dconv.EngineConfig()  # config.hpp:10-20
    assert (c.min_accumulators, c.max_accumulators, c.cache_budget_bytes, c.prefetch_lookahead) == (
        ref.min_accumulators, ref.max_accumulators, ref.cache_budget_bytes, ref.prefetch_lookahead)
    assert (c.acc_chain_limit, c.i16_bound_in, c.i16_bound_wt) == (512, 256, 256)


def test_host_generators_match_oracle(dconv, orc):
    from paper_1808_05567_b200 import _lib

    lib = _lib.lib()
    a = np.empty(4096, np.float32)
    lib.dconv_fill_uniform_host(7, -1.0, 1.0, a.ctypes.data, a.size)
    assert np.array_equal(a, orc.uniform(7, (4096,)))
    b = np.empty(4096, np.float32)
    lib.dconv_fill_he_normal_host(3, float(np.sqrt(2 / 576)), b.ctypes.data, b.size)
    assert np.array_equal(b, orc.he_normal(3, (4096,), 576))


def test_status_strings_map_reference_exceptions(dconv):
    from paper_1808_05567_b200 import _lib

    lib = _lib.lib()
    for code, name in _lib.STATUS_NAMES.items():
        assert lib.dconv_status_string(code).decode() == name
    assert issubclass(dconv.PlanTensorMismatch, dconv.Error)


def test_prep_batch_state_errors(dconv):
    """dconv_prep_batch_begin / _end: one open batch per thread; _end without an
    open batch is an error; an empty batch launches nothing (no GPU needed)."""
    from paper_1808_05567_b200 import _lib

    lib = _lib.lib()
    assert lib.dconv_prep_batch_end(None) == 102
    assert lib.dconv_prep_batch_begin() == 0
    assert lib.dconv_prep_batch_begin() == 102
    assert lib.dconv_prep_batch_end(None) == 0
    assert lib.dconv_prep_batch_end(None) == 102


def test_backward_route_selection(dconv):
    # propagation.cpp:35-40 and the Table I routes in SURVEY 8(a) a13
    d = dconv
    assert d.choose_backward_route(d.make_layer_spec(2, 16, 24, 10, 10, 3, 3, 1, 8)) == d.BackwardRoute.DUALITY_STRIDE1
    assert d.choose_backward_route(d.make_layer_spec(2, 16, 24, 12, 12, 1, 1, 2, 0, 0, 8)) == d.BackwardRoute.DUALITY_1x1
    assert d.choose_backward_route(d.make_layer_spec(2, 16, 16, 11, 11, 3, 3, 2, 0, 0, 8)) == d.BackwardRoute.GENERIC_GEMM
    assert d.choose_backward_route(d.make_layer_spec(64, 3, 64, 224, 224, 7, 7, 2)) == d.BackwardRoute.GENERIC_GEMM


def test_header_compiles_as_c():
    src = "#include \"dconv_b200.h\"\nint main(void){dconv_spec_t s; return dconv_spec_validate(&s) > 1000;}\n"
    tmp = "/tmp/_dconv_hdr_test.c"
    with open(tmp, "w") as f:
        f.write(src)
    r = subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-fsyntax-only", "-I", os.path.join(ROOT, "include"),
                        tmp], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


@pytest.mark.skipif(not os.path.isdir("/root/reference/proj/core/include"), reason="needs the reference headers")
def test_cpp_shim_compiles_against_reference_headers():
    """include/dconv_b200.hpp (the header-compatible C++ shim, reference signatures
    over the C ABI) compiles and links against the reference's own headers and core
    (oracle/Makefile `shim`; tests/shim/shim_check.cpp runs it on the GPU)."""
    oracle = os.path.join(ROOT, "oracle")
    binary = os.path.join(oracle, "_ref", "shim_check")
    if os.path.exists(binary):
        os.remove(binary)
    r = subprocess.run(["make", "-s", "shim"], cwd=oracle, capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "warning" not in (r.stdout + r.stderr).lower(), r.stderr
    nm = subprocess.run(["nm", "-C", "-u", binary], capture_output=True, text=True).stdout
    for sym in ("dconv_forward", "dconv_backward_data", "dconv_weight_update", "dconv::make_forward_plan",
                "dconv::weight_update"):
        assert sym in nm, sym  # both engines are called: the C ABI and the reference's own
