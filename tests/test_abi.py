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
    hdr = (ROOT / "include" / "kvsched.h").read_text()
    assert lib.sched_abi_version() == int(re.search(r"#define KVSCHED_ABI_VERSION (\d+)", hdr).group(1))


def test_binding_structs_match_the_header():
    """The ctypes structs carry the header's fields in the header's order."""
    import paper_2502_07115_b200.kvsched as kv
    hdr = re.sub(r"/\*.*?\*/", "", (ROOT / "include" / "kvsched.h").read_text(), flags=re.S)
    for cname, pyname in (("sched_outputs", kv.SchedOutputs), ("sched_instances", kv.SchedInstances),
                          ("sched_policy", kv.SchedPolicy)):
        body = re.search(r"typedef struct \{([^}]*)\}\s*" + cname + ";", hdr).group(1)
        decl = []
        for d in body.split(";"):
            d = d.strip()
            if not d:
                continue
            first, *rest = d.split(",")
            decl.append(re.split(r"[\s*]+", first.strip())[-1])
            decl += [x.strip().lstrip("*").strip() for x in rest]
        assert decl == [f[0] for f in pyname._fields_], (cname, decl)


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
