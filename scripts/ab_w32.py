"""A/B variant of the W = 32 kernels only: bl_w32.cu recompiled with extra -D
flags (device code only) and linked with the main build's other objects into
lib/ab/libbatchlp_cuda_<tag>.so (selected with BATCHLP_LIB; gpurun carries
lib/ab). usage: python scripts/ab_w32.py tag DEF=VAL [DEF=VAL ...]"""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_21990_b200 import build as B

tag, defs = sys.argv[1], sys.argv[2:]
objdir = os.path.join(B.HERE, "build", "obj")
out_o = f"/tmp/ab_w32_{tag}.o"
subprocess.run([B._nvcc(), *B.NVCC_FLAGS, *[f"-D{d}" for d in defs], "-I",
                os.path.join(B.ROOT, "include"), "-c", os.path.join(B.CSRC, "bl_w32.cu"), "-o",
                out_o], check=True, cwd=B.CSRC)
objs = [out_o if s == "bl_w32.cu" else os.path.join(objdir, os.path.splitext(s)[0] + ".o")
        for s in B.SOURCES]
os.makedirs(os.path.join(B.LIBDIR, "ab"), exist_ok=True)
B._link(objs, os.path.join(B.LIBDIR, "ab", f"libbatchlp_cuda_{tag}.so"), False)
print("ok", tag)
