"""Kernel experiments: relink libbbx with kernels_img_f16.cu built under extra -D flags.

python scripts/build_exp.py NAME -DFLAG ...  ->  exp/libbbx_NAME.so (load with BBX_LIB=...)
"""
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2306_12517_b200 import _build as B  # noqa: E402

name, flags = sys.argv[1], sys.argv[2:]
B.build()
out = B.HERE.parent / "exp"
out.mkdir(exist_ok=True)
inc = ["-I", str(B.CSRC), "-I", str(B.HERE.parent / "include")]
obj = out / f"kernels_img_f16_{name}.o"
subprocess.run([B.NVCC, *B.GENCODE, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", *flags, *inc, "-c",
                str(B.CSRC / "kernels_img_f16.cu"), "-o", str(obj)], check=True)
objs = [obj if o.name == "kernels_img_f16.cu.o" else o for o in
        (B.BUILD / (s + ".o") for s in B.CUDA_SOURCES + B.HOST_SOURCES)]
subprocess.run([B.NVCC, *B.GENCODE, "-shared", "-o", str(out / f"libbbx_{name}.so"), *map(str, objs), "-lpthread"],
               check=True)
print(out / f"libbbx_{name}.so")
