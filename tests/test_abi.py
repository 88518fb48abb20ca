"""CPU-side checks of the boundary (-m "not gpu"): the C-ABI library loads and
exports every symbol include/gakco.h declares; host logic that needs no GPU."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gakco.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gakco_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def libpath():
    from paper_1704_07468_b200 import build
    return build.build()


def test_header_declares_the_boundary():
    fns = declared_functions()
    for f in ("gakco_create", "gakco_kernel", "gakco_accumulate", "gakco_finalize",
              "gakco_set_shard", "gakco_destroy", "gakco_last_error"):
        assert f in fns


def test_library_exports_every_declared_symbol(libpath):
    out = subprocess.check_output(["nm", "-D", "--defined-only", libpath], text=True)
    exported = set(re.findall(r" T (gakco_\w+)", out))
    missing = [f for f in declared_functions() if f not in exported]
    assert not missing, missing


def test_binding_loads_and_names_match(libpath):
    from paper_1704_07468_b200 import gakco
    L = gakco.lib()
    for f in declared_functions():
        assert hasattr(L, f)
        assert f in gakco.EXPORTS
    assert L.gakco_status_string(0) == b"ok"


def test_sm100a_code_in_library(libpath):
    """The library carries sm_100a SASS (no PTX-only / other-arch fallback)."""
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", libpath],
                                  text=True)
    assert "sm_100a" in out


def test_no_cpu_fallback_without_gpu(libpath):
    """Without a usable GPU the product path raises instead of computing."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1704_07468_b200 import gakco
    with pytest.raises(gakco.GakcoError):
        gakco.gakco_create(4, 7, 5, 2, 0)


def test_product_does_not_import_oracle():
    """The product package never references oracle/ (DESIGN.md boundary)."""
    pkg = os.path.join(ROOT, "paper_1704_07468_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "gakco_oracle" not in txt and "gko_" not in txt, f
