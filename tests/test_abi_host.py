"""CPU tests of the C ABI (no GPU): libbsra.so loads, exports every symbol include/bsra.h
declares, validates its host inputs, and its C++ Algorithm-1 scheduler emits plan images
byte-identical to the Python reimplementation (oracle/scheduler_ref.py) on >= 10^3 random
workloads (the BASELINE north_star's "bit-exact scheduler plans")."""
import re
import os

import numpy as np
import pytest

import paper_2501_01005_b200 as bsra
from oracle import scheduler_ref as S

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "bsra.h")).read() + open(os.path.join(ROOT, "include", "bsra_dist.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)  # drop comments
    declared = set(re.findall(r"\b(bsra_[a-z_]+)\(", hdr))
    assert declared, "no declarations parsed"
    L = bsra.lib()
    for name in sorted(declared):
        assert hasattr(L, name), name
    assert set(bsra.EXPORTS) == declared
    assert L.bsra_version() >= 100


def _bsr(qo, kv, ps):
    qo = np.asarray(qo, np.int64)
    kv = np.asarray(kv, np.int64)
    n = (kv + ps - 1) // ps
    qi = np.concatenate([[0], np.cumsum(qo)]).astype(np.int32)
    ki = np.concatenate([[0], np.cumsum(n)]).astype(np.int32)
    last = np.where(n > 0, kv - (n - 1) * ps, 0).astype(np.int32)
    return qi, ki, last


MASKS = {0: "none", 1: "causal", 2: "custom"}


def _compare(qo, kv, *, H_qo, H_kv, ps, mask, num_ctas, tiles=(16, 64, 128, 256), tile_q=0, alpha=1, beta=1,
             align=0, L_min=0, window=0):
    qi, ki, last = _bsr(qo, kv, ps)
    cfg = bsra.make_config(H_qo=H_qo, H_kv=H_kv, D=128, page_size=ps, dtype="bf16", mask=MASKS[mask],
                           max_batch=len(qo), max_total_qo_rows=int(sum(qo)), num_ctas=num_ctas, tile_set=tiles,
                           tile_q=tile_q, alpha=alpha, beta=beta, kv_chunk_align=align, kv_chunk_min=L_min,
                           window=window)
    img_c = bsra.plan_host(cfg, num_ctas, qi, ki, last)
    ref = S.plan_ref(qo, kv, g=H_qo // H_kv, H_kv=H_kv, mask=mask, num_ctas=num_ctas, tile_set=tiles,
                     alpha=alpha, beta=beta, align=align or ps, L_min=L_min, T_q=tile_q or None,
                     qo_begin=qi[:-1], page_begin=ki[:-1], window=window)
    assert img_c.dtype == np.int32
    assert np.array_equal(img_c, ref.image), (len(img_c), len(ref.image))
    return img_c


@pytest.mark.parametrize("seed", range(1000))
def test_cpp_scheduler_bit_exact_vs_python(seed):
    rng = np.random.default_rng(50000 + seed)
    B = int(rng.integers(0, 24))
    H_kv = int(rng.choice([1, 2, 8]))
    g = int(rng.choice([1, 4, 8]))
    ps = int(rng.choice([1, 4, 16]))
    mask = int(rng.integers(0, 3))
    dist = seed % 4
    if dist == 0:
        kv = rng.integers(0, 4000, B)
    elif dist == 1:
        kv = np.full(B, int(rng.integers(1, 9000)))
    elif dist == 2:
        kv = np.minimum(rng.zipf(1.3, B) * 61, 300000)
    else:
        kv = rng.integers(0, 50, B)
    qo = rng.integers(0, 3, B) if seed % 3 == 0 else rng.integers(0, 600, B)
    if mask == 1:
        kv = np.maximum(kv, qo)
    num_ctas = int(rng.choice([1, 2, 4, 64, 148, 296, 592]))
    alpha, beta = (1, 1) if seed % 5 else (int(rng.integers(0, 50)), int(rng.integers(1, 5)))
    align = 0 if seed % 7 else int(rng.choice([1, 8, 32]))
    L_min = 0 if seed % 11 else int(rng.integers(1, 500))
    tiles = [(16, 64, 128), (16, 128), (64,), (128,), (16,), (16, 64, 128, 256), (256,)][seed % 7]
    window = 0 if seed % 3 else int(rng.choice([1, 7, 64, 1000, 5000]))  # sliding window (R26)
    _compare(qo, kv, H_qo=H_kv * g, H_kv=H_kv, ps=ps, mask=mask, num_ctas=num_ctas, tiles=tiles, alpha=alpha,
             beta=beta, align=align, L_min=L_min, window=window)


@pytest.mark.parametrize("name,qo,kv,H,ps,mask,nc", [
    ("c1@148", [1, 1], [5, 37], (4, 1), 4, 0, 148),
    ("c1@4", [1, 1], [5, 37], (4, 1), 4, 0, 4),
    ("c3-like", [96, 2048, 145, 64], [96, 2048, 145, 64], (64, 8), 16, 1, 148),
    ("c5@296", [1] * 4, [524288] * 4, (32, 8), 16, 0, 296),
    ("empty", [], [], (32, 8), 16, 0, 148),
    ("zero-qo", [0, 0, 3], [10, 0, 7], (8, 2), 4, 1, 8),
])
def test_cpp_scheduler_named_cases(name, qo, kv, H, ps, mask, nc):
    _compare(qo, kv, H_qo=H[0], H_kv=H[1], ps=ps, mask=mask, num_ctas=nc)


def test_c2_full_size_plan_bit_exact():
    import synth
    wl = synth.c2_decode_llama8b()
    for nc in (148, 296):
        _compare(wl.qo_lens, wl.kv_lens, H_qo=32, H_kv=8, ps=16, mask=0, num_ctas=nc)


def _cfg(**kw):
    base = dict(H_qo=8, H_kv=2, D=128, page_size=4, dtype="bf16", max_batch=8, max_total_qo_rows=64)
    base.update(kw)
    return bsra.make_config(**base)


@pytest.mark.parametrize("qi,ki,last,msg", [
    ([1, 2], [0, 1], [1], "qo_indptr[0]"),
    ([0, 2, 1], [0, 1, 2], [1, 1], "qo_indptr not nondecreasing"),
    ([0, 1], [0, 2], [5], "kv_last_page_len"),
    ([0, 1], [0, 2], [0], "kv_last_page_len"),
    ([0, 1], [1, 2], [1], "kv_page_indptr[0]"),
])
def test_plan_host_rejects_malformed_bsr(qi, ki, last, msg):
    with pytest.raises(bsra.BsraError, match=re.escape(msg)):
        bsra.plan_host(_cfg(), 4, qi, ki, last)


@pytest.mark.parametrize("kw,msg", [
    (dict(H_qo=6, H_kv=4), "multiple"),
    (dict(D=96), "head_dim"),
    (dict(page_size=0), "page_size"),
    (dict(tile_q=32), "tile_q"),
    (dict(o_dtype="f16"), "o_dtype"),
])
def test_config_validation(kw, msg):
    with pytest.raises(bsra.BsraError, match=msg):
        bsra.plan_host(_cfg(**kw), 4, [0, 1], [0, 1], [1])


def test_empty_request_without_pages_ignores_last_page_len():
    img = bsra.plan_host(_cfg(), 4, [0, 1, 2], [0, 0, 1], [999, 3])
    assert img[S.HEADER_WORDS - 16 + 5] == 2 * 2  # 2 requests x 2 kv heads, one item each


def test_config_struct_layout_matches_header(tmp_path):
    """The ctypes mirror of bsra_config (the binding) has the C header's size and field offsets:
    compiled with gcc against include/bsra.h, compared field by field."""
    import ctypes
    import subprocess
    fields = [f[0] for f in bsra.Config._fields_]
    src = tmp_path / "layout.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "bsra.h"\nint main(void) {\n'
                   '  printf("%zu\\n", sizeof(bsra_config));\n'
                   + "".join(f'  printf("%zu\\n", offsetof(bsra_config, {f}));\n' for f in fields) + "  return 0;\n}\n")
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    out = [int(x) for x in subprocess.check_output([str(exe)]).split()]
    assert out[0] == ctypes.sizeof(bsra.Config)
    for f, off in zip(fields, out[1:]):
        assert getattr(bsra.Config, f).offset == off, f
