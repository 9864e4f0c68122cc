"""CPU checks of the drop-in boundary: libpdot.so loads, exports every symbol
include/pdot.h declares, and the ctypes mirrors match the C struct layouts.
No compute calls (there is no GPU here)."""

import ctypes
import re
import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "pdot.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\**\s+\**(pdot_[a-zA-Z_0-9]+)\(", text, re.M)))


def test_header_declares_the_python_exports():
    from paper_2407_19689_b200 import _lib
    assert set(declared_symbols()) == set(_lib.EXPORTS)


def test_library_exports_every_declared_symbol():
    from paper_2407_19689_b200 import _lib
    if not _lib.LIB_PATH.exists():
        pytest.skip("libpdot.so not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    _lib.load()  # argtypes bind without error


def test_no_cuda_means_loud_failure():
    """The product path raises instead of falling back to the CPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import numpy as np

    import paper_2407_19689_b200 as pd
    prob = pd.make_problem([[0.0, 1.0], [1.0, 0.0]], [0.5, 0.5], [0.5, 0.5])
    with pytest.raises(RuntimeError, match="CUDA"):
        pd.solve(prob)
    with pytest.raises(RuntimeError, match="CUDA"):
        pd.apply_A(np.zeros((2, 2)))


@pytest.mark.skipif(shutil.which("gcc") is None, reason="gcc missing")
def test_struct_layouts_match_ctypes(tmp_path):
    from paper_2407_19689_b200 import _lib
    src = tmp_path / "sz.c"
    src.write_text(
        '#include <stdio.h>\n#include <stddef.h>\n#include "pdot.h"\n'
        'int main(void){printf("%zu %zu %zu %zu %zu %zu\\n", sizeof(pdot_config), sizeof(pdot_result),'
        ' sizeof(pdot_event), sizeof(pdot_progress), offsetof(pdot_config, eta0), offsetof(pdot_result, device_s));'
        'printf("%zu\\n", offsetof(pdot_config, host_omega));'
        'return 0;}\n')
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", str(ROOT / "include"), str(src), "-o", str(exe)], check=True)
    got = list(map(int, subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()))
    want = [ctypes.sizeof(_lib.Config), ctypes.sizeof(_lib.Result), ctypes.sizeof(_lib.Event),
            ctypes.sizeof(_lib.Progress), _lib.Config.eta0.offset, _lib.Result.device_s.offset,
            _lib.Config.host_omega.offset]
    assert got == want
