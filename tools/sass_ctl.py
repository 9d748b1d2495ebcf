"""Decode the scheduling control words of a kernel's SASS (sm_70+ 128-bit encoding: stall count,
write/read scoreboard index, wait mask) — shows which hardware scoreboard every load is put on
and where the kernel waits for it.
    python tools/sass_ctl.py paper_2312_05639_b200/libspmx_b200.so spmm_chunk_kernelILi64E"""
import re, subprocess, sys
lib, fn = sys.argv[1], sys.argv[2]
out = subprocess.run(['cuobjdump','-sass',lib],capture_output=True,text=True).stdout.splitlines()
on=False; rows=[]
i=0
while i < len(out):
    l=out[i]
    if 'Function :' in l:
        on = fn in l
    if on:
        m=re.match(r'\s+/\*([0-9a-f]{4})\*/\s+(.*?);\s+/\* (0x[0-9a-f]+) \*/',l)
        if m and i+1 < len(out):
            m2=re.match(r'\s+/\* (0x[0-9a-f]+) \*/',out[i+1])
            if m2:
                hi=int(m2.group(1),16)
                ctl = hi>>41
                stall=ctl&0xf; yld=(ctl>>4)&1; wb=(ctl>>5)&7; rb=(ctl>>8)&7; wait=(ctl>>11)&0x3f
                rows.append((m.group(1),m.group(2).strip(),stall,wb,rb,wait))
                i+=1
    i+=1
for a,t,stall,wb,rb,wait in rows:
    w=''.join(str(b) for b in range(6) if wait>>b&1)
    print(f"{a} st={stall:2d} wb={'-' if wb==7 else wb} rb={'-' if rb==7 else rb} wait={w or '-':6s} {t}")
