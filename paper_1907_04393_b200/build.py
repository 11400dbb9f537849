"""Build libfizi.so in-tree for sm_100a (nvcc, no JIT cache).

Each csrc/*.cu is compiled to its own object in parallel (objects under
build/, rebuilt when the source or any header changed), then linked with
nvcc -shared.  The ptxas report of every kernel goes to ptxas_info.txt.
"""
from __future__ import annotations

import glob
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libfizi.so")
OBJ_DIR = os.path.join(HERE, "build")
SOURCES = sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")))
HEADERS = sorted(glob.glob(os.path.join(HERE, "csrc", "*.cuh"))) + [
    os.path.join(ROOT, "include", "fizi.h")]
DEPS = SOURCES + HEADERS

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v"]


def _obj(src: str) -> str:
    return os.path.join(OBJ_DIR, os.path.basename(src)[:-3] + ".o")


CHECKED_LIB = os.path.join(HERE, "libfizi_checked.so")
CHECKED_FLAGS = ["-DFIZI_DEVICE_CHECKS"]


def needs_build(lib_path: str = LIB) -> bool:
    if not os.path.exists(lib_path):
        return True
    t = os.path.getmtime(lib_path)
    return any(os.path.getmtime(d) > t for d in DEPS)


def build(force: bool = False, nvcc: str = "nvcc", verbose: bool = False,
          extra_flags: list[str] | None = None, out: str | None = None) -> str:
    """Compile (changed) objects in parallel and link `out` (default libfizi.so).
    extra_flags (e.g. -DFIZI_...) force a full rebuild into a separate object dir."""
    lib_path = out or LIB
    if not force and not needs_build(lib_path):
        return lib_path
    obj_dir = OBJ_DIR if not extra_flags else OBJ_DIR + "_" + "_".join(
        f.lstrip("-").replace("=", "_") for f in extra_flags)
    os.makedirs(obj_dir, exist_ok=True)
    hdr_t = max(os.path.getmtime(h) for h in HEADERS)

    def compile_one(src: str):
        obj = os.path.join(obj_dir, os.path.basename(src)[:-3] + ".o")
        if (not force and os.path.exists(obj)
                and os.path.getmtime(obj) > max(os.path.getmtime(src), hdr_t)):
            return src, ""
        cmd = [nvcc, *NVCC_FLAGS, *(extra_flags or []), "-I", os.path.join(ROOT, "include"),
               "-c", "-o", obj, src]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {os.path.basename(src)}:\n" + r.stderr[-8000:])
        return src, r.stderr

    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 4)) as ex:
        logs = list(ex.map(compile_one, SOURCES))
    objs = [os.path.join(obj_dir, os.path.basename(s)[:-3] + ".o") for s in SOURCES]
    r = subprocess.run([nvcc, *ARCH, "-shared", "-o", lib_path, *objs, "-lcudart"],
                       capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("nvcc link failed:\n" + r.stderr[-8000:])
    if lib_path == LIB:
        info = os.path.join(HERE, "ptxas_info.txt")
        old = open(info).read() if os.path.exists(info) else ""
        # keep the report of objects that were not recompiled
        parts = {}
        cur = None
        for line in old.splitlines(keepends=True):
            if line.startswith("### "):
                cur = line[4:].strip()
                parts[cur] = ""
            elif cur:
                parts[cur] += line
        for src, log in logs:
            if log:
                parts[os.path.basename(src)] = log
        with open(info, "w") as f:
            for k in sorted(parts):
                f.write(f"### {k}\n{parts[k]}")
    if verbose:
        for src, log in logs:
            print(src, log)
    return lib_path


def build_checked(force: bool = False) -> str:
    """libfizi_checked.so: the same sources with the device-side invariant
    checks compiled in (FIZI_DCHECK, dev_util.cuh); selected at run time with
    FIZI_LIB=checked (the sanitizer substitute on this pool)."""
    return build(force=force, extra_flags=CHECKED_FLAGS, out=CHECKED_LIB)


if __name__ == "__main__":
    print(build(force=True))
    print(build_checked(force=True))
