"""CPU: the ctypes mirrors of the C-ABI structs (paper_2510_03557_b200/_native.py,
resident.py) have exactly the layout include/hb.h declares -- every field's
offset and the struct size, checked against gcc's offsetof on the header."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _structs():
    from paper_2510_03557_b200 import _native as N
    from paper_2510_03557_b200.resident import HbStepArgs
    return {"HbStepArgs": HbStepArgs, "HbMeshArgs": N.HbMeshArgs, "HbListArgs": N.HbListArgs,
            "HbEvalArgs": N.HbEvalArgs, "HbError": N.HbError, "HbFieldSet": N.HbFieldSet}


@pytest.mark.skipif(shutil.which("gcc") is None, reason="needs gcc")
def test_ctypes_structs_match_header(tmp_path):
    import ctypes
    structs = _structs()
    lines = ["#include <stdio.h>", "#include <stddef.h>", '#include "hb.h"', "int main(void) {"]
    for name, cls in structs.items():
        lines.append(f'  printf("{name} sizeof %zu\\n", sizeof({name}));')
        for f in cls._fields_:
            lines.append(f'  printf("{name} {f[0]} %zu\\n", offsetof({name}, {f[0]}));')
    lines += ["  return 0;", "}"]
    src = tmp_path / "abi.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "abi"
    cuda_inc = "/usr/local/cuda/include"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), "-I", cuda_inc, "-o", str(exe),
                    str(src)], check=True, capture_output=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout
    got = {}
    for ln in out.splitlines():
        s, f, v = ln.split()
        got[(s, f)] = int(v)
    for name, cls in structs.items():
        assert got[(name, "sizeof")] == ctypes.sizeof(cls), name
        for f in cls._fields_:
            assert got[(name, f[0])] == getattr(cls, f[0]).offset, (name, f[0])
