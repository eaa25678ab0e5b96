"""The C-ABI library loads on a CPU-only host and exports every entry point
include/stb200.h declares; the ctypes table binds exactly that set."""

import re
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "stb200.h"


def declared():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(stb_[a-z0-9_]+)\s*\(", text)))


def test_header_and_ctypes_table_agree():
    from paper_2512_15834_b200.runtime.lib import SIGNATURES

    assert declared() == sorted(SIGNATURES)


def test_library_exports_every_symbol():
    from paper_2512_15834_b200.runtime.lib import LIB_PATH, load_raw

    if not LIB_PATH.exists():
        subprocess.run(["make", "-C", str(ROOT / "paper_2512_15834_b200" / "csrc"), "-j8"], check=True)
    lib = load_raw()
    for name in declared():
        assert hasattr(lib, name), name
    assert lib.stb_version() == 1
    nm = subprocess.run(["nm", "-D", "--defined-only", str(LIB_PATH)], capture_output=True, text=True).stdout
    for name in declared():
        assert re.search(rf"\bT {name}\b", nm), name


def test_kernels_are_sm100a_tcgen05():
    """SASS of the shipped library carries tcgen05 MMAs, TMEM loads and TMA."""
    from paper_2512_15834_b200.runtime.lib import LIB_PATH

    sass = subprocess.run(["cuobjdump", "-sass", str(LIB_PATH)], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass and "LDTM" in sass and "UTMALDG" in sass
    elf = subprocess.run(["cuobjdump", "-lelf", str(LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in elf


def test_product_fails_loudly_without_cuda():
    import torch

    from harness.sim import Simulator
    from paper_2512_15834_b200 import EngineConfig, EngineSim, KernelError

    if torch.cuda.is_available():
        return
    try:
        EngineSim(Simulator(), EngineConfig(prefill_rate=0.1, decode_rate=0.1))
    except KernelError as exc:
        assert "CUDA" in str(exc)
    else:
        raise AssertionError("engine built without a GPU")
