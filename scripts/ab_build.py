"""Build A/B variants of the library with extra -D flags into build/ab_<name>.so.

usage: ab_build.py name -DXB_L2PF=3 [...]   (load with XMHD_SO=build/ab_<name>.so)
"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2108_13622_b200 import build as b  # noqa: E402

name, flags = sys.argv[1], sys.argv[2:]
os.makedirs(os.path.join(b.REPO, "build"), exist_ok=True)
out = os.path.join(b.REPO, "build", f"ab_{name}.so")
cmd = [b.nvcc()] + b.NVCC_FLAGS + flags + ["-I", b.INCLUDE, "-I", b.CSRC, "-o", out]
cmd += [os.path.join(b.CSRC, f) for f in b.SOURCES]
subprocess.run(cmd, check=True)
print(out)
