"""C ABI checks that need no GPU: the library loads, exports every symbol the
header declares, struct layouts agree, host-only entry points are exact, and
the product path fails loudly without a device (no CPU fallback)."""
import ctypes as C
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def lib():
    from paper_1607_02925_b200 import _native as N

    if not N.LIB_PATH.exists():
        subprocess.run(["make", "-s", "-j8", "-C", str(ROOT / "paper_1607_02925_b200" / "csrc")], check=True)
    return N.load()


def test_exports_every_header_symbol(lib):
    from paper_1607_02925_b200 import _native as N

    syms = N.header_symbols()
    assert len(syms) >= 30
    out = subprocess.run(["nm", "-D", "--defined-only", str(N.LIB_PATH)], capture_output=True, text=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    for s in syms:
        getattr(lib, s)


def test_struct_layouts_match_header(tmp_path):
    from paper_1607_02925_b200 import _native as N

    src = tmp_path / "sz.c"
    src.write_text('#include "gaplra_cuda.h"\n#include <stdio.h>\n#include <stddef.h>\nint main(){printf("%zu %zu %zu %zu '
                   '%zu %zu %zu %zu %zu\\n", sizeof(gaplra_svrg_params), sizeof(gaplra_ledger), sizeof(gaplra_si_config), '
                   'sizeof(gaplra_si_report), sizeof(gaplra_profile), offsetof(gaplra_si_report, ms_total), '
                   'sizeof(gaplra_ap_report), offsetof(gaplra_ap_report, delta), offsetof(gaplra_si_config, backend));}\n')
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", str(ROOT / "include"), str(src), "-o", str(exe)], check=True)
    got = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    want = [C.sizeof(N.SvrgParams), C.sizeof(N.Ledger), C.sizeof(N.SiConfig), C.sizeof(N.SiReport),
            C.sizeof(N.Profile), N.SiReport.ms_total.offset, C.sizeof(N.ApReport), N.ApReport.delta.offset,
            N.SiConfig.backend.offset]
    assert got == want


def test_oracle_structs_match_abi():
    import oracle_lib as O
    from paper_1607_02925_b200 import _native as N

    assert C.sizeof(O.OrcSvrgParams) == C.sizeof(N.SvrgParams)
    assert C.sizeof(O.OrcSiConfig) == C.sizeof(N.SiConfig)


def test_host_gaussian_init_bit_exact(lib, oracle):
    import paper_1607_02925_b200 as g

    for d, p, s in [(4, 2, 0), (300, 7, 2**33 + 1)]:
        assert np.array_equal(g.gaussian_init(d, p, s), oracle.gaussian_init(d, p, s)[1])
    with pytest.raises(g.ContractViolation):
        g.gaussian_init(2, 3, 0)


def test_no_cpu_fallback(lib):
    import torch

    import paper_1607_02925_b200 as g

    if torch.cuda.is_available():
        pytest.skip("a CUDA device is present")
    with pytest.raises(g.DeviceError):
        g.Context(0)
    with pytest.raises(g.DeviceError):
        g.gram_block(None, np.zeros((2, 1))) if False else g.default_context()


def test_missing_library_fails_loudly(tmp_path):
    from paper_1607_02925_b200 import _native as N

    with pytest.raises(ImportError):
        N.load(tmp_path / "nope.so")


def test_binary_x_roundtrip(tmp_path):
    # binary X + JSON spectrum sidecar (host side, no GPU)
    from paper_1607_02925_b200 import xio
    from problems import planted_dense, random_csc

    X, _, sig = planted_dense(37, 53, seed=3)
    side = xio.save_dense(tmp_path / "x.bin", X, sigma=sig.tolist(), k=3, p=6, seed=3)
    Y, s2 = xio.load_dense(tmp_path / "x.bin")
    assert np.array_equal(X, Y) and s2["sha256"] == side["sha256"] and s2["sigma"] == sig.tolist()
    cp, ri, v = random_csc(40, 30, 5, seed=1)
    xio.save_csc(tmp_path / "c.bin", 40, 30, cp, ri, v, note="csc")
    (d, n, cp2, ri2, v2), _ = xio.load_csc(tmp_path / "c.bin")
    assert (d, n) == (40, 30) and np.array_equal(cp, cp2) and np.array_equal(ri, ri2) and np.array_equal(v, v2)
    raw = bytearray((tmp_path / "x.bin").read_bytes())
    raw[8] ^= 1
    (tmp_path / "x.bin").write_bytes(bytes(raw))
    with pytest.raises(ValueError):
        xio.load_dense(tmp_path / "x.bin")
