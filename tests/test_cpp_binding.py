"""The reference-side C++ binding (include/gaplra_device.hpp) compiles and links
against the reference's own headers and sources (/root/reference/proj/core:
linear_operator.hpp:34-62, errors.hpp:10-98) and libgaplra_cuda.so, and keeps
the reference's API: DeviceGramOperator is a gaplra::LinearOperator whose apply
matches the reference GramOperator::apply, ledger included; statuses come back
as the reference's exception types with their payloads.  Recipe: oracle/Makefile
`binding` (built by __graft_entry__.build() where the reference is present; the
binary travels to the GPU box under oracle/_ref/)."""
import os
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
BIN = ROOT / "oracle" / "_ref" / "binding_test"
REF = Path(os.environ.get("GAPLRA_REF_DIR", "/root/reference/proj"))
LIB = ROOT / "paper_1607_02925_b200" / "libgaplra_cuda.so"


def test_binding_compiles_links_and_maps_device_failure():
    if not REF.exists():
        pytest.skip("reference sources absent (GPU box): the binary is built where they are")
    if not LIB.exists():
        pytest.skip("libgaplra_cuda.so not built")
    subprocess.run(["make", "-s", "-C", str(ROOT / "oracle"), "binding", f"REF={REF}"], check=True)
    import torch

    if torch.cuda.is_available():
        pytest.skip("nogpu mode checks the no-device error path")
    r = subprocess.run([str(BIN), "nogpu"], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "DeviceFailure" in r.stdout


@pytest.mark.gpu
def test_binding_against_reference_gram_operator():
    if not BIN.exists():
        pytest.skip("oracle/_ref/binding_test not built (needs the reference sources at build time)")
    r = subprocess.run([str(BIN), "gpu"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "binding gpu ok" in r.stdout
