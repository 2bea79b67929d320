"""Build libspx.so (the sm_100a kernels + C-ABI) in-tree with nvcc.

The shared library lands next to this file so it travels with the repo
snapshot to the GPU box (built artefacts are git-ignored, not
gpurun-ignored).  Objects are rebuilt only when a source or header is newer, or the nvcc
flags (SPX_NVCC_EXTRA) changed.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OBJ = PKG / "_build"
LIB = PKG / "libspx.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [
    "-O3",
    "-std=c++17",
    "-lineinfo",
    "-Xcompiler",
    "-fPIC,-O3",
    "--expt-relaxed-constexpr",
    "-Xptxas",
    "-v" if os.environ.get("SPX_PTXAS_VERBOSE") else "-O3",
    "-I" + str(ROOT / "include"),
    *os.environ.get("SPX_NVCC_EXTRA", "").split(),
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; libspx.so cannot be built")


def _sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu"))


def _headers() -> list[Path]:
    return sorted(CSRC.glob("*.h")) + sorted(CSRC.glob("*.cuh")) + sorted((ROOT / "include").glob("*.h"))


def _compile(src: Path, obj: Path, verbose: bool) -> None:
    cmd = [nvcc(), *ARCH, *NVCC_FLAGS, "-c", str(src), "-o", str(obj)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{res.stdout}\n{res.stderr}")
    if verbose and (res.stderr or res.stdout):
        sys.stderr.write(res.stdout + res.stderr)


def build(force: bool = False, verbose: bool = False) -> Path:
    OBJ.mkdir(exist_ok=True)
    stamp = OBJ / "flags.txt"
    flags = " ".join(ARCH + NVCC_FLAGS)
    if not stamp.exists() or stamp.read_text() != flags:
        force = True  # SPX_NVCC_EXTRA / SPX_PTXAS_VERBOSE changed: rebuild everything
        stamp.write_text(flags)
    hdr_mtime = max((h.stat().st_mtime for h in _headers()), default=0.0)
    jobs = []
    objs = []
    for src in _sources():
        obj = OBJ / (src.stem + ".o")
        objs.append(obj)
        if force or not obj.exists() or obj.stat().st_mtime < max(src.stat().st_mtime, hdr_mtime):
            jobs.append((src, obj))
    if jobs:
        with cf.ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 4)) as ex:
            list(ex.map(lambda j: _compile(j[0], j[1], verbose), jobs))
    newest = max(o.stat().st_mtime for o in objs)
    if force or jobs or not LIB.exists() or LIB.stat().st_mtime < newest:
        tmp = LIB.with_suffix(".so.tmp")
        cmd = [nvcc(), *ARCH, "-shared", "-cudart", "static", "-o", str(tmp), *map(str, objs)]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed:\n{res.stdout}\n{res.stderr}")
        os.replace(tmp, LIB)
    return LIB


def build_variant(tag: str, src_name: str, defines: list[str]) -> Path:
    """Tuning tool: libspx with one source recompiled under extra -D flags,
    linked from the regular objects into tools/variants/libspx_<tag>.so
    (load it with SPX_LIB=<path>; the product always loads libspx.so)."""
    build()
    out_dir = ROOT / "tools" / "variants"
    out_dir.mkdir(exist_ok=True)
    obj = out_dir / f"{Path(src_name).stem}_{tag}.o"
    cmd = [nvcc(), *ARCH, *NVCC_FLAGS, *defines, "-c", str(CSRC / src_name), "-o", str(obj)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src_name} ({tag}):\n{res.stderr}")
    objs = [obj if o.stem == Path(src_name).stem else o for o in (OBJ / (s.stem + ".o") for s in _sources())]
    lib = out_dir / f"libspx_{tag}.so"
    res = subprocess.run([nvcc(), *ARCH, "-shared", "-cudart", "static", "-o", str(lib), *map(str, objs)],
                         capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stderr}")
    obj.unlink()
    return lib


REF_SRC = Path("/root/reference/pkg")
REF_DST = ROOT / "baseline" / "_ref"


def install_reference() -> None:
    """Install the unmodified reference front end into baseline/_ref (git-ignored,
    not gpurun-ignored, so it ships to the GPU box).  Runs only where the
    read-only source mount exists and the install is missing; the build needs
    to write into its source tree, so it installs from a copy under /tmp."""
    if (REF_DST / "spindle" / "schedule.py").exists() or not REF_SRC.is_dir():
        return
    import tempfile

    with tempfile.TemporaryDirectory() as tmp:
        src = Path(tmp) / "pkg"
        shutil.copytree(REF_SRC, src)
        cmd = [sys.executable, "-m", "pip", "install", "--no-index", "--no-build-isolation",
               "--no-deps", "--find-links", "/opt/wheelhouse", "--target", str(REF_DST), str(src)]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"reference install failed:\n{res.stdout}\n{res.stderr}")


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
