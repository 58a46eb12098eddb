"""Build libtpla.so in-tree with nvcc for sm_100a (B200).

    python -m paper_2508_15881_b200.build            # incremental (content hashes, not mtimes)
    python -m paper_2508_15881_b200.build --force    # rebuild everything

The library embeds the sha256 of its sources, headers and flags (tpla_version() ends with
"src <hash>"); __graft_entry__.build() checks the loaded library against the tree.

Objects go to paper_2508_15881_b200/build/, the shared library next to this file.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import hashlib
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "libtpla.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_include() -> str:
    try:
        import nvidia.nccl  # type: ignore
        d = os.path.join(list(nvidia.nccl.__path__)[0], "include")
        if os.path.exists(os.path.join(d, "nccl.h")):
            return d
    except Exception:
        pass
    for d in glob.glob("/opt/prime-rl/.venv/lib/python3*/site-packages/nvidia/nccl/include"):
        return d
    raise RuntimeError("nccl.h not found")


def flags():
    return ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
                   "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include"), "-I", nccl_include(),
                   "-Xptxas", "-warn-spills"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def _hash_files(paths) -> str:
    h = hashlib.sha256()
    for p in sorted(paths):
        h.update(os.path.relpath(p, ROOT).encode())
        with open(p, "rb") as f:
            h.update(f.read())
    return h.hexdigest()


def _headers():
    return sorted(glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) +
                  glob.glob(os.path.join(ROOT, "include", "*.h")))


def source_hash() -> str:
    """sha256 over every source, header and the compile flags: embedded in libtpla.so
    (tpla_version()) so a loaded library proves which sources it was compiled from."""
    h = hashlib.sha256(_hash_files(sources() + _headers()).encode())
    h.update(" ".join(flags()).encode())
    return h.hexdigest()[:16]


def _compile(src: str, force: bool, verbose: bool, tree_hash: str) -> str:
    obj = os.path.join(OBJ, os.path.basename(src) + ".o")
    stamp = obj + ".hash"
    # an object is reused only when it was compiled from exactly these bytes (source + every
    # header + flags); tpla_abi.cpp embeds the tree hash, so it is recompiled whenever anything changes
    embeds = os.path.basename(src) == "tpla_abi.cpp"             # tpla_version() carries the tree hash
    want = hashlib.sha256((_hash_files([src] + _headers()) + " ".join(flags()) +
                           (tree_hash if embeds else "")).encode()).hexdigest()
    if not force and os.path.exists(obj) and os.path.exists(stamp) and open(stamp).read() == want:
        return obj
    cmd = [NVCC, "-c", src, "-o", obj] + flags() + ([f"-DTPLA_SRC_HASH=\"{tree_hash}\""] if embeds else [])
    if verbose:
        cmd += ["-Xptxas", "-v"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if verbose and (r.stdout or r.stderr):
        print(r.stdout + r.stderr)
    with open(stamp, "w") as f:
        f.write(want)
    return obj


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    srcs = sources()
    tree = source_hash()
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(lambda s: _compile(s, force, verbose, tree), srcs))
    stamp = os.path.join(OBJ, "libtpla.hash")
    if force or not os.path.exists(LIB) or not os.path.exists(stamp) or open(stamp).read() != tree:
        cmd = [NVCC, "-shared", "-o", LIB] + objs + ARCH + ["-ldl", "-Xcompiler", "-fPIC"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
        with open(stamp, "w") as f:
            f.write(tree)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
