"""The C ABI is usable from plain C: tests/c/abi_client.c is compiled with gcc
against include/escs.h and libescs.so and run (host-only part on CPU; the
device part, with cudaMalloc'd buffers, on the GPU)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2506_15174_b200")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")


@pytest.fixture(scope="module")
def client(tmp_path_factory):
    exe = str(tmp_path_factory.mktemp("c") / "abi_client")
    subprocess.check_call(["gcc", "-O2", "-std=c11", "-Wall", "-o", exe,
                           os.path.join(ROOT, "tests", "c", "abi_client.c"),
                           "-I", os.path.join(ROOT, "include"), "-I", os.path.join(CUDA, "include"),
                           "-L", PKG, "-lescs", "-Wl,-rpath," + PKG,
                           "-L", os.path.join(CUDA, "lib64"), "-lcudart",
                           "-Wl,-rpath," + os.path.join(CUDA, "lib64")])
    return exe


def test_c_client_host(client):
    r = subprocess.run([client], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "host ok" in r.stdout


@pytest.mark.gpu
def test_c_client_device(client):
    r = subprocess.run([client, "device"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "device ok" in r.stdout


def test_struct_layouts_match_binding(tmp_path):
    """The ctypes mirrors of escs_params / escs_plan_stats / escs_plan_view
    have the C compiler's size and field offsets (include/escs.h)."""
    import ctypes
    from paper_2506_15174_b200 import escs
    structs = {"escs_params": escs._Params, "escs_plan_stats": escs._Stats,
               "escs_plan_view": escs._View, "escs_staged_view": escs._StagedView}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "escs.h"', "int main(void) {"]
    for cname, py in structs.items():
        lines.append(f'printf("{cname} size %zu\\n", sizeof({cname}));')
        for f, _ in py._fields_:
            lines.append(f'printf("{cname} {f} %zu\\n", offsetof({cname}, {f}));')
    lines += ["return 0;", "}"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = str(tmp_path / "layout")
    subprocess.check_call(["gcc", "-std=c11", "-o", exe, str(src), "-I", os.path.join(ROOT, "include")])
    out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout.split("\n")
    for line in filter(None, out):
        cname, f, v = line.split()
        py = structs[cname]
        got = ctypes.sizeof(py) if f == "size" else getattr(py, f).offset
        assert got == int(v), (cname, f, got, v)
