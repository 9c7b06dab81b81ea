"""In-tree build of libcachesage_b200.so (sm_100a kernels + host C++ + C ABI).

nvcc cross-compiles for sm_100a without a GPU, so this runs in the CPU container; the built
.so travels to the GPU box with the repo snapshot. Exactness: -fmad=false on device and
-ffp-contract=off on the host keep every fp64 score bit-identical to the reference.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libcachesage_b200.so")
# Only the C ABI is exported, and every symbol binds at load time (-z now): a library loaded
# later in the same process (the reference library in the tests exports its own inline
# libstdc++ instantiations) can never capture one of our lazily bound calls.
EXPORTS = os.path.join(CSRC, "exports.map")
# nlohmann/json 3.11.3 (the reference's serializer; shipped in the image with cudnn_frontend):
# the output writers format through it so metrics.json / events.jsonl match byte for byte
JSON_DIR = os.path.join(sysconfig.get_paths()["purelib"], "include", "cudnn_frontend", "thirdparty", "nlohmann")

NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
DEVICE_SRCS = ["cs_kernels.cu", "cs_admit.cu", "cs_learner.cu", "cs_belady.cu"]
HOST_SRCS = ["cs_pool.cpp", "cs_state.cpp", "cs_engine.cpp", "cs_comm.cpp", "cs_output.cpp"]
DEPS = DEVICE_SRCS + HOST_SRCS + ["cs_device.cuh", "cs_launch.h", "cs_pool.hpp"]


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def _stale(target, sources):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def src_sha16() -> str:
    """sha256 prefix over every source and header compiled into the library plus this file (the
    flags): identifies a build by its inputs, so a committed ncu capture stays bound to it when
    nvcc's output bytes differ between containers."""
    import hashlib

    h = hashlib.sha256()
    files = sorted(f for f in os.listdir(CSRC) if f.endswith((".cu", ".cuh", ".cpp", ".hpp", ".h", ".map")))
    paths = [os.path.join(CSRC, f) for f in files] + [os.path.join(ROOT, "include", "cachesage_b200.h"),
                                                      os.path.abspath(__file__)]
    for p in paths:
        h.update(os.path.basename(p).encode() + b"\0")
        with open(p, "rb") as f:
            h.update(f.read())
    return h.hexdigest()[:16]


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(OUT_DIR, exist_ok=True)
    inc = ["-I", os.path.join(ROOT, "include"), "-I", CSRC]
    header_deps = [os.path.join(CSRC, h) for h in ("cs_device.cuh", "cs_launch.h", "cs_pool.hpp", "cs_block.cuh", "cs_shard.cuh", "cs_comm.hpp", "cs_engine_state.h", "cs_engine_dev.cuh", "cs_belady.cuh", "cs_output.hpp")]
    header_deps.append(os.path.join(ROOT, "include", "cachesage_b200.h"))
    objs = []
    for src in DEVICE_SRCS:
        s = os.path.join(CSRC, src)
        o = os.path.join(OUT_DIR, src + ".o")
        if force or _stale(o, [s] + header_deps):
            # -dlcm=cg: global loads default to L2 (not L1). The persistent kernels read state other
            # SMs wrote since a previous admission; only a kernel boundary would clean a stale L1.
            _run([NVCC, "-O3", "-lineinfo", "-std=c++17", *ARCH, "-fmad=false", "-Xptxas", "-v,-dlcm=cg",
                  "-Xcompiler", "-fPIC,-ffp-contract=off", *inc, "-c", s, "-o", o], verbose)
        objs.append(o)
    for src in HOST_SRCS:
        s = os.path.join(CSRC, src)
        o = os.path.join(OUT_DIR, src + ".o")
        if force or _stale(o, [s] + header_deps):
            _run([NVCC, "-O2", "-std=c++17", "-Wno-deprecated-gpu-targets", "-Xcompiler", "-fPIC,-ffp-contract=off,-Wall", *inc, "-I", JSON_DIR, "-c", s,
                  "-o", o], verbose)
        objs.append(o)
    if force or _stale(LIB, objs + [EXPORTS]):
        _run([NVCC, "-shared", *ARCH, "-Xlinker", "--version-script=" + EXPORTS, "-Xlinker", "-z,now", "-o", LIB, *objs, "-lcudart",
              "-ldl"], verbose)
    return LIB


if __name__ == "__main__":
    import sys

    print(build(verbose=True, force="--force" in sys.argv))
