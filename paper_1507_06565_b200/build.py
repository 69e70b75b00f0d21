"""In-tree build of libporolb_cuda.so (sm_100a) and the oracle libraries.

    python paper_1507_06565_b200/build.py          # product library
    python paper_1507_06565_b200/build.py --all    # + oracle/ (+ oracle/_ref when
                                                   #   /root/reference is present)

The product is compiled with nvcc for ``-gencode arch=compute_100a,code=sm_100a``
(kernels) and g++ ``-ffp-contract=off`` (host runtime; keeps every host-side
constant bit-identical to the reference's inline arithmetic), and linked with
the static CUDA runtime so the .so travels to the GPU box by itself.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OBJ = PKG / "_build"
LIB = PKG / "libporolb_cuda.so"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
GENCODE = ["-gencode", "arch=compute_100a,code=sm_100a"]
CUDA_INC = "/usr/local/cuda/include"
# The image's $CXX (/opt/gcc) lacks libgomp specs; the system g++ is used.
CXX = shutil.which("g++") or "g++"

CU_SOURCES = ["kernels.cu", "sweep_compact.cu", "sweep_tma.cu", "sweep_units.cu", "voxelize_device.cu", "setup.cu"]
CPP_SOURCES = ["params.cpp", "voxelize.cpp", "synth.cpp", "sim.cpp", "io.cpp", "dist.cpp"]
HEADERS = ["kparams.h", "kernels.h", "lattice.cuh", "host_common.h", "voxel_geometry.h", "setup.h", "staging.h",
           "sim_impl.h"]


def _run(cmd: list[str]) -> None:
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("build failed:\n" + " ".join(cmd) + "\n" + res.stdout + res.stderr)


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


KERNEL_FLAGS = ["-O3", "-lineinfo", "-std=c++17"]


def kernel_hash(defines: tuple = ()) -> str:
    """sha256 (16 hex) of everything that determines the sweep kernels' code:
    the CUDA sources and headers, nvcc flags/defines and nvcc's version.  It is
    compiled into the library (pgpu_build_info) so bench.py reports a
    committed ncu traffic figure only for the kernel build it was measured on."""
    import hashlib
    h = hashlib.sha256()
    for f in CU_SOURCES + [x for x in HEADERS if not x.endswith(".h") or x in ("kparams.h", "kernels.h")]:
        h.update(f.encode())
        h.update((CSRC / f).read_bytes())
    h.update(" ".join(GENCODE + KERNEL_FLAGS + list(defines)).encode())
    try:
        h.update(subprocess.run([NVCC, "--version"], capture_output=True, text=True).stdout.encode())
    except OSError:
        pass
    return h.hexdigest()[:16]


def build_product(force: bool = False, defines: tuple = (), lib: Path = LIB,
                  obj: Path = OBJ) -> Path:
    """Compile and link the product library.  `defines` (e.g. ("PGPU_POOL=64",))
    and an alternative `lib`/`obj` path build experiment variants side by side."""
    OBJ = obj
    LIB = lib
    OBJ.mkdir(parents=True, exist_ok=True)
    dflags = [f"-D{d}" for d in defines]
    khash = kernel_hash(defines)
    hdrs = [CSRC / h for h in HEADERS] + [ROOT / "include" / "porolb_gpu.h"]
    jobs = []
    objs = []
    for src in CU_SOURCES:
        o = OBJ / (Path(src).stem + ".o")
        objs.append(o)
        if force or _stale(o, [CSRC / src] + hdrs):
            jobs.append([NVCC, *GENCODE, *KERNEL_FLAGS, "-Xcompiler", "-fPIC",
                         "-Xptxas", "-warn-spills", *dflags, "-c", str(CSRC / src), "-o", str(o)])
    stamp = OBJ / "kernel_hash.txt"
    hash_changed = not stamp.exists() or stamp.read_text() != khash
    for src in CPP_SOURCES:
        o = OBJ / (Path(src).stem + ".o")
        objs.append(o)
        if force or _stale(o, [CSRC / src] + hdrs) or (src == "params.cpp" and hash_changed):
            jobs.append([CXX, "-std=c++17", "-O3", "-fPIC", "-pthread", "-ffp-contract=off",
                         "-Wall", "-Wno-unused-function", f"-I{CUDA_INC}", *dflags,
                         f'-DPGPU_KERNEL_HASH="{khash}"', "-c",
                         str(CSRC / src), "-o", str(o)])
    if jobs:
        with ThreadPoolExecutor(max_workers=min(8, len(jobs))) as ex:
            list(ex.map(_run, jobs))
    stamp.write_text(khash)
    if force or jobs or _stale(LIB, objs):
        _run([NVCC, *GENCODE, "-shared", "-cudart", "static", "-o", str(LIB),
              *[str(o) for o in objs], "-Xcompiler", "-pthread", "-ldl", "-lrt"])
    return LIB


DEMO_SRC = ROOT / "tools" / "porolb_gpu_demo.cpp"
DEMO_BIN = ROOT / "tools" / "porolb_gpu_demo"


def build_demo() -> Path:
    """The C++ drop-in demo (include/porolb_gpu/porolb_gpu.hpp over the C ABI)."""
    deps = [DEMO_SRC, ROOT / "include" / "porolb_gpu" / "porolb_gpu.hpp", LIB]
    if _stale(DEMO_BIN, deps):
        _run([CXX, "-std=c++17", "-O2", f"-I{ROOT / 'include'}", str(DEMO_SRC), "-o",
              str(DEMO_BIN), f"-L{PKG}", "-lporolb_cuda", f"-Wl,-rpath,$ORIGIN/../{PKG.name}",
              "-pthread"])
    return DEMO_BIN


DNS_SRC = ROOT / "tests" / "cpp" / "dns_dropin.cpp"
DNS_BIN = ROOT / "tests" / "cpp" / "dns_dropin"


def build_dns_dropin() -> Path:
    """The reference's dns.cpp driver compiled unchanged (namespace alias only)
    against the C++ mirror (tests/cpp/dns_dropin.cpp)."""
    deps = [DNS_SRC, ROOT / "include" / "porolb_gpu" / "porolb_gpu.hpp", LIB]
    if _stale(DNS_BIN, deps):
        _run([CXX, "-std=c++17", "-O2", f"-I{ROOT / 'include'}", str(DNS_SRC), "-o", str(DNS_BIN),
              f"-L{PKG}", "-lporolb_cuda", f"-Wl,-rpath,$ORIGIN/../../{PKG.name}", "-pthread"])
    return DNS_BIN


DIST_SRC = ROOT / "tests" / "cpp" / "dist_demo.cpp"
DIST_BIN = ROOT / "tests" / "cpp" / "dist_demo"


def build_dist_demo() -> Path:
    """The C++ multi-GPU host path demo (DistSimulation, local + NCCL)."""
    deps = [DIST_SRC, ROOT / "include" / "porolb_gpu" / "porolb_gpu.hpp", LIB]
    if _stale(DIST_BIN, deps):
        _run([CXX, "-std=c++17", "-O2", f"-I{ROOT / 'include'}", str(DIST_SRC), "-o", str(DIST_BIN),
              f"-L{PKG}", "-lporolb_cuda", f"-Wl,-rpath,$ORIGIN/../../{PKG.name}", "-pthread"])
    return DIST_BIN


def build_oracle() -> None:
    """Test infrastructure: oracle/liboracle.so always, oracle/_ref when the
    reference sources are present (this container; the GPU box gets the
    prebuilt files)."""
    _run(["make", "-s", "-C", str(ROOT / "oracle"), "all"])
    if Path("/root/reference/proj/src/simulation.cpp").exists():
        _run(["make", "-s", "-C", str(ROOT / "oracle"), "ref"])


def build_variant(name: str, defines: tuple) -> Path:
    """Experiment build: paper_1507_06565_b200/_variants/<name>/libporolb_cuda.so,
    selected at run time with PGPU_LIB=<that path>."""
    d = PKG / "_variants" / name
    return build_product(defines=defines, lib=d / "libporolb_cuda.so", obj=d / "obj")


def main(argv: list[str]) -> int:
    variants = [a.split("=", 1)[1] for a in argv if a.startswith("--variant=")]
    for v in variants:  # --variant=name:DEF1,DEF2
        name, defs = v.split(":", 1)
        print(build_variant(name, tuple(x for x in defs.split(",") if x)))
    if variants:
        return 0
    lib = build_product(force="--force" in argv)
    print(lib)
    print(build_demo())
    print(build_dns_dropin())
    print(build_dist_demo())
    if "--all" in argv:
        build_oracle()
    return 0


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:]))
