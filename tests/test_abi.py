"""CPU checks of the boundary: libkvsched.so loads (no GPU needed) and exports every
function include/kvsched.h declares; the product path never touches oracle/."""
import ctypes
import re
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def declared_functions():
    src = (ROOT / "include" / "kvsched.h").read_text()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\**\s*(sched_\w+)\s*\(", src, flags=re.M)))


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for f in ("sched_init", "sched_run_instances", "sched_latency", "sched_finalize"):
        assert f in names


def test_library_exports_every_declared_symbol():
    from paper_2502_07115_b200 import build
    build.build()
    import paper_2502_07115_b200.kvsched as kv
    lib = ctypes.CDLL(str(kv.LIB_PATH))
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert set(declared_functions()) == set(kv.EXPORTS)
    assert lib.sched_abi_version() == 1


def test_sched_init_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        return
    import paper_2502_07115_b200 as K
    try:
        K.Context(0, stream=0)
    except RuntimeError as e:
        assert "SCHED_E_CUDA" in str(e)
    else:
        raise AssertionError("sched_init succeeded without a GPU")


def test_product_path_does_not_use_the_oracle():
    for p in list((ROOT / "paper_2502_07115_b200").rglob("*.py")) + \
            list((ROOT / "paper_2502_07115_b200" / "csrc").glob("*")):
        text = p.read_text(errors="ignore")
        assert "import oracle" not in text and "from oracle" not in text and "liboracle" not in text, p
    for p in (ROOT / "oracle").glob("*"):
        if p.suffix in (".py", ".c", ".h"):
            text = p.read_text(errors="ignore")
            assert "paper_2502_07115_b200" not in text.replace("shares no code with paper_2502_07115_b200", "") \
                or "never imports it" in text, p
            assert "kvsched.h" not in text, p
