"""In-tree build of the native library and the Python extension.

Produces, next to this file:
  libcolorvibe_gpu.so   C-ABI (include/cvg.h) + C++ API (include/colorvibe/*.hpp),
                        CUDA kernels for sm_100a, static cudart
  _core.<abi>.so        pybind11 module linked against libcolorvibe_gpu.so

Usage: python paper_2507_22901_b200/build.py   (or __graft_entry__.build()).
Rebuilds only what is out of date (mtime based).
"""
from __future__ import annotations

import os
import subprocess
import sys
import sysconfig
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(PKG, "_build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CUDA_INC = "/usr/local/cuda/include"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# experiment hook: extra -D flags for the search kernels (e.g. CVG_KERNEL_DEFS="-DCVG_GROUP=4");
# the caller removes _build/cvg_kernels.o so that the object is rebuilt
KERNEL_DEFS = os.environ.get("CVG_KERNEL_DEFS", "").split()
# The reference's value-safe FP flags (proj/src/CMakeLists.txt:21-43): no FMA
# contraction in host code, so host-side tables carry the reference's bits.
HOST_FP = ["-ffp-contract=off", "-fno-math-errno", "-fno-trapping-math"]

# nlohmann json (header only, MIT) from the venv's cudnn_frontend copy: its
# float formatter makes our JSON text match the reference's digit for digit
# (json_lite.h falls back to shortest round-trip digits without it).
def _nlohmann_dir() -> str | None:
    for base in sysconfig.get_paths()["purelib"], sysconfig.get_paths()["platlib"]:
        d = os.path.join(base, "include", "cudnn_frontend", "thirdparty", "nlohmann")
        if os.path.exists(os.path.join(d, "json.hpp")):
            return d
    return None


NLOHMANN = _nlohmann_dir()
JSON_INC = ["-I" + NLOHMANN] if NLOHMANN else []

LIB = os.path.join(PKG, "libcolorvibe_gpu.so")
EXT = os.path.join(PKG, "_core" + sysconfig.get_config_var("EXT_SUFFIX"))

HEADERS = [os.path.join(CSRC, h) for h in ("cvg_layout.h", "cvg_internal.h", "cvg_host.h")] + [
    os.path.join(INCLUDE, "cvg.h"),
    os.path.join(INCLUDE, "colorvibe", "color.hpp"),
    os.path.join(INCLUDE, "colorvibe", "search.hpp"),
    os.path.join(INCLUDE, "colorvibe", "image.hpp"),
    os.path.join(INCLUDE, "colorvibe", "codec.hpp"),
    os.path.join(CSRC, "colorvibe_detail.h"),
    os.path.join(CSRC, "json_lite.h"),
    os.path.join(INCLUDE, "colorvibe", "feasibility.hpp"),
    os.path.join(INCLUDE, "colorvibe", "bench.hpp"),
]


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def _run(cmd: list[str], log: str | None = None) -> None:
    res = subprocess.run(cmd, capture_output=True, text=True)
    if log:
        with open(log, "w") as f:
            f.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"build step failed: {' '.join(cmd[:3])} ...")


def _objects() -> list[tuple[str, list[str], list[str], str | None]]:
    o = lambda n: os.path.join(BUILD, n)  # noqa: E731
    src = lambda n: os.path.join(CSRC, n)  # noqa: E731
    return [
        (o("cvg_kernels.o"), [src("cvg_kernels.cu")] + HEADERS,
         [NVCC, *ARCH, "-lineinfo", "-O3", "-std=c++17", "-Xptxas", "-v", "-Xcompiler", "-fPIC", *KERNEL_DEFS,
          "-I" + INCLUDE, "-c", src("cvg_kernels.cu"), "-o", o("cvg_kernels.o")],
         o("ptxas.log")),
        (o("cvg_codec.o"), [src("cvg_codec.cu")] + HEADERS,
         [NVCC, *ARCH, "-lineinfo", "-O3", "-std=c++17", "-Xptxas", "-v", "-Xcompiler", "-fPIC",
          "-I" + INCLUDE, "-c", src("cvg_codec.cu"), "-o", o("cvg_codec.o")],
         o("ptxas_codec.log")),
        *[(o(f"{name}.o"), [src(f"{name}.cpp")] + HEADERS,
           ["g++", "-std=c++20", "-O2", "-fPIC", *HOST_FP, "-Wall", "-I" + CUDA_INC, "-I" + INCLUDE,
            "-c", src(f"{name}.cpp"), "-o", o(f"{name}.o")], None)
          for name in ("cvg_prep", "cvg_plan", "cvg_search", "cvg_codec_host")],
        (o("colorvibe_api.o"), [src("colorvibe_api.cpp")] + HEADERS,
         ["g++", "-std=c++20", "-O2", "-fPIC", *HOST_FP, "-Wall", "-I" + INCLUDE,
          "-c", src("colorvibe_api.cpp"), "-o", o("colorvibe_api.o")], None),
        (o("feasibility_api.o"), [src("feasibility_api.cpp")] + HEADERS,
         ["g++", "-std=c++20", "-O2", "-fPIC", *HOST_FP, "-Wall", "-I" + INCLUDE, *JSON_INC,
          "-c", src("feasibility_api.cpp"), "-o", o("feasibility_api.o")], None),
        (o("codec_api.o"), [src("codec_api.cpp")] + HEADERS,
         ["g++", "-std=c++20", "-O2", "-fPIC", *HOST_FP, "-Wall", "-I" + INCLUDE, *JSON_INC,
          "-c", src("codec_api.cpp"), "-o", o("codec_api.o")], None),
    ]


def build(verbose: bool = False) -> None:
    os.makedirs(BUILD, exist_ok=True)
    objs = _objects()
    todo = [(t, cmd, log) for t, deps, cmd, log in objs if _stale(t, deps)]
    if todo:
        with ThreadPoolExecutor(len(todo)) as ex:
            list(ex.map(lambda a: _run(a[1], a[2]), todo))
    obj_paths = [t for t, *_ in objs]
    if _stale(LIB, obj_paths):
        _run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", LIB, *obj_paths,
              "-Xlinker", "-soname,libcolorvibe_gpu.so", "-lpthread"])
    bind = os.path.join(CSRC, "bindings.cpp")
    if _stale(EXT, [bind, LIB] + HEADERS):
        import pybind11

        py_inc = sysconfig.get_paths()["include"]
        _run(["g++", "-std=c++20", "-O2", "-fPIC", "-shared", *HOST_FP, "-I" + INCLUDE,
              "-I" + pybind11.get_include(), "-I" + py_inc, bind, "-o", EXT,
              "-L" + PKG, "-lcolorvibe_gpu", "-Wl,-rpath,$ORIGIN"])
    if verbose:
        print(f"built {LIB}\nbuilt {EXT}")


if __name__ == "__main__":
    build(verbose=True)
