"""Experiment: make the L2-touch loads of a -DSPMX_TOUCH=4 build fire-and-forget by clearing their
write scoreboard (wb = 7) in the linked library. python tools/experiments/touch_nowb.py in.so out.so"""
import re, shutil, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2312_05639_b200 import sass_sched as S
src, dst = sys.argv[1], sys.argv[2]
shutil.copyfile(src, dst)
funcs = S.disassemble(dst)
data = bytearray(open(dst, "rb").read())
pat = re.compile(r"LDG\.E\.NA\.LTC(256|128)B\.CONSTANT")
n = 0
for name, code in funcs.items():
    idxs = [i for i, c in enumerate(code) if pat.search(c.text)]
    if not idxs:
        continue
    blob = b"".join(c.bytes() for c in code)
    pos = data.find(blob)
    assert pos >= 0 and data.find(blob, pos + 1) < 0, name
    for i in idxs:
        hi = code[i].with_wb(7)
        o = pos + 16 * i + 8
        data[o:o + 8] = hi.to_bytes(8, "little")
        n += 1
open(dst, "wb").write(bytes(data))
print(n, "touch loads patched")
