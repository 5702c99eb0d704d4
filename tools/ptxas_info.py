"""Compile one ils_inst.cu unit with -Xptxas -v and print registers / spills per kernel.

    python tools/ptxas_info.py -DILS_INST_ROW_SPEC=1 [-DILS_PACKED_F32X2 ...]
"""
import os
import re
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2003_07504_b200 import build as B  # noqa: E402

src = os.environ.get("ILS_SRC", os.path.join(B.CSRC, "ils_inst.cu"))
cmd = [B._nvcc(), *B.NVCC_FLAGS, "-Xptxas", "-v", *sys.argv[1:], "-I", os.path.join(B.ROOT, "include"), "-c", src,
       "-o", "/tmp/ptxas_info.o"]
r = subprocess.run(cmd, capture_output=True, text=True)
if r.returncode:
    sys.exit(r.stderr)
name = None
for line in r.stderr.splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        name = subprocess.run(["c++filt"], input=m.group(1), capture_output=True, text=True).stdout.strip()
        name = name.replace("ils::", "").replace("(RowArgs<float>)", "").replace("(ColArgs<float>)", "")
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and name:
        stack, sst, sld = m.groups()
    m = re.search(r"Used (\d+) registers", line)
    if m and name:
        print(f"{m.group(1):>4} regs  spill st/ld {sst}/{sld}  {name[:150]}")
        name = None
