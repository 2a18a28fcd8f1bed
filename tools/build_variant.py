"""Build an A/B variant of libniyama.so with extra nvcc -D flags.

    python tools/build_variant.py TAG -DNAME=VALUE ...
    NIYAMA_LIB_PATH=paper_2503_22562_b200/_build/variants/libniyama_TAG.so python tools/kbench.py
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import importlib.util  # noqa: E402

spec = importlib.util.spec_from_file_location("nbuild", os.path.join(ROOT, "paper_2503_22562_b200", "build.py"))
B = importlib.util.module_from_spec(spec)
spec.loader.exec_module(B)


def main():
    tag, defs = sys.argv[1], sys.argv[2:]
    out_dir = os.path.join(B.BUILD, "variants")
    os.makedirs(out_dir, exist_ok=True)
    B.build()
    k_obj = os.path.join(out_dir, f"kernels_{tag}.o")
    lib = os.path.join(out_dir, f"libniyama_{tag}.so")
    nccl_inc, nccl_lib = B.nccl_dirs()
    subprocess.run([B.NVCC, *B.ARCH, "-O3", "-std=c++17", "-I", B.INCLUDE, "-I", B.CSRC, "-lineinfo", *defs,
                    "-Xcompiler", "-fPIC", "-c", os.path.join(B.CSRC, "kernels.cu"), "-o", k_obj], check=True)
    objs = [os.path.join(B.BUILD, f"{n}.o") for n in ("gather", "runtime", "sched", "predictor")]
    subprocess.run([B.NVCC, *B.ARCH, "-shared", "-cudart", "static", "-o", lib, k_obj, *objs, "-lpthread",
                    "-L", nccl_lib, "-l:libnccl.so.2", "-Xlinker",
                    f"-rpath,{nccl_lib}", "-Xlinker", "--no-undefined"], check=True)
    print(lib)


if __name__ == "__main__":
    main()
