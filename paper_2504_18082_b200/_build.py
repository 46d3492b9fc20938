"""Build the cmb CUDA library in-tree: paper_2504_18082_b200/libcmb.so (sm_100a).

Plain nvcc invocations (no torch JIT, no cache outside the repo) so the .so
travels to the GPU box with the repo snapshot."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "libcmb.so")
SOURCES = ["capi.cu", "graph.cu", "order.cu", "sample.cu", "features.cu", "shard.cu", "peer.cu", "runtime.cu", "cache.cu", "reorder.cu",
           "sage_layer.cu", "train.cu", "dense.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden", "-Xptxas", "-v",
         "-I", os.path.join(ROOT, "include"), "-I", CSRC]


def _stale():
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "cmb.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force=False, verbose=False, out=None, defines=()):
    """Build libcmb.so (or, for layout experiments, `out` with extra -D `defines` in its own
    object directory; the product library is always built without them)."""
    so = out or SO
    if not force and not defines and so == SO and not _stale():
        return SO
    bdir = os.path.join(HERE, "build" if not defines else "build_" + "_".join(
        d.replace("=", "") for d in defines))
    os.makedirs(bdir, exist_ok=True)
    def one(src):
        obj = os.path.join(bdir, src.replace(".cu", ".o"))
        cmd = [NVCC, *FLAGS, *[f"-D{d}" for d in defines], "-c", os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        with open(os.path.join(bdir, src + ".ptxas.log"), "w") as fh:
            fh.write(r.stdout + r.stderr)
        return src, obj, r

    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 1)) as ex:
        results = list(ex.map(one, SOURCES))
    objs = []
    for src, obj, r in results:
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed for {src}")
        if verbose:
            sys.stderr.write(r.stderr)
        objs.append(obj)
    tmp = so + ".tmp"
    subprocess.check_call([NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", tmp,
                           *objs, "-lcudart", "-lcublasLt"])
    os.replace(tmp, so)
    return so


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
