"""The reference-side C++ binding shown in INTEGRATION.md §3 compiles and links.

The snippet is extracted from INTEGRATION.md verbatim, compiled with g++ against
include/mpcg.h and the UNMODIFIED reference headers (BenchSpec, RingTensor, ...) and linked
against libmpcg.so, so the documented maintainer binding cannot drift from the ABI. Needs
/root/reference (this container); skipped elsewhere. Nothing is executed (no GPU needed).
"""
import os
import re
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_INC = "/root/reference/proj/include"


def _json_inc():
    return os.path.join(sys.prefix, "lib", "python3.12", "site-packages", "include", "cudnn_frontend", "thirdparty",
                        "nlohmann")


@pytest.mark.skipif(not os.path.isdir(REF_INC) or shutil.which("g++") is None,
                    reason="needs the reference headers and g++")
def test_integration_binding_compiles_and_links(tmp_path):
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    blocks = re.findall(r"```cpp\n(.*?)```", text, re.S)
    assert blocks, "INTEGRATION.md has no C++ binding block"
    src = tmp_path / "binding.cpp"
    src.write_text(blocks[0] + "\nint main() { return &bench_party_b200 == nullptr; }\n")
    lib = os.path.join(ROOT, "paper_2209_13643_b200", "lib")
    if not os.path.exists(os.path.join(lib, "libmpcg.so")):
        pytest.skip("libmpcg.so not built")
    cmd = ["g++", "-std=c++20", "-O0", "-I", os.path.join(ROOT, "include"), "-I", REF_INC, "-I", _json_inc(),
           str(src), "-o", str(tmp_path / "binding"), "-L", lib, "-lmpcg", "-Wl,-rpath," + lib, "-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
