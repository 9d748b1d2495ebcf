"""Post-link scheduling fix for the SpMM walk loop: a second scoreboard for half of the gathers.

ptxas puts every LDG of the walk loop of spmm_chunk_kernel (csrc/spmx_kernels.cuh) on ONE
hardware scoreboard (SB5). A scoreboard is a counter, so the first consumer of the oldest
gather drains all of them, including the one issued a few instructions earlier: the rotating
gather pipeline degenerates to "issue a batch, wait for the slowest load".
Nothing in CUDA C++ or PTX selects a scoreboard. This module edits the scheduling control
words of the compiled kernel inside libspmx_b200.so:

  * the gathers that refill the second half of the pipeline slots (positions G/2 .. G-1 of a
    batch) are moved from SB5 to a scoreboard that the loop does not use at all (SB4 or SB3),
  * the first instruction of the loop that reads one of their destination registers gets that
    scoreboard added to its wait mask.

Every other wait stays as ptxas emitted it: SB5 still covers the first-half gathers, the
column/value loads and the gathers issued before the loop. The edit is applied only when all
preconditions hold (the loop is found, the chosen scoreboard is unused inside it, every moved
load has its consumers after the new wait and before its own re-issue); otherwise the kernel
is left exactly as compiled. Control-word layout (sm_70+ 128-bit encoding, bits 105..125):
stall[4] yield[1] write-barrier[3] read-barrier[3] wait-mask[6] reuse[4].

    python -m paper_2312_05639_b200.sass_sched path/to/libspmx_b200.so [--dry-run]
"""
from __future__ import annotations

import re
import subprocess
import sys

_INSTR = re.compile(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);\s+/\* (0x[0-9a-f]{16}) \*/")
_HI = re.compile(r"\s+/\* (0x[0-9a-f]{16}) \*/")
# a row gather of the walk loop: 128-bit load through the read-only path (64-bit for the d = 16
# kernel, whose 8-lane groups read a 64-byte row as float2 per lane)
_GATHERS = {128: re.compile(r"LDG\.E(\.\w+)*\.128\.CONSTANT"), 64: re.compile(r"LDG\.E(\.\w+)*\.64\.CONSTANT")}
# branch with its target (plain, predicated, or uniform: "BRA.U !UP0, 0x23b0")
_BRA = r"\bBRA(?:\.U)?\s+(?:!?UP\d+,\s*)?(0x[0-9a-f]+)"


class Ins:
    __slots__ = ("addr", "text", "lo", "hi", "off")

    def __init__(self, addr, text, lo, hi):
        self.addr, self.text, self.lo, self.hi, self.off = addr, text, lo, hi, -1

    @property
    def ctl(self):
        return self.hi >> 41

    @property
    def wb(self):
        return (self.ctl >> 5) & 7

    @property
    def rb(self):
        return (self.ctl >> 8) & 7

    @property
    def wait(self):
        return (self.ctl >> 11) & 0x3F

    def bytes(self):
        return self.lo.to_bytes(8, "little") + self.hi.to_bytes(8, "little")

    def with_wb(self, sb):
        return (self.hi & ~(7 << 46)) | (sb << 46)

    def with_wait(self, sb):
        return self.hi | (1 << (52 + sb))


def disassemble(lib):
    out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
    funcs, cur = {}, None
    lines = out.splitlines()
    i = 0
    while i < len(lines):
        l = lines[i]
        if "Function :" in l:
            cur = l.split("Function :")[1].strip()
            funcs[cur] = []
        m = _INSTR.match(l)
        if m and cur is not None and i + 1 < len(lines):
            m2 = _HI.match(lines[i + 1])
            if m2:
                funcs[cur].append(Ins(int(m.group(1), 16), m.group(2).strip(), int(m.group(3), 16),
                                      int(m2.group(1), 16)))
                i += 1
        i += 1
    return funcs


def _regs(tok, width):
    m = re.match(r"R(\d+)", tok)
    if not m:
        return set()
    r = int(m.group(1))
    return set(range(r, r + width))


def _dest_regs(ins):
    """Destination registers of an LDG (128-bit: four registers)."""
    m = re.search(r"LDG\.E(\.\w+)* (R\d+),", ins.text)
    if not m:
        return set()
    width = 4 if ".128" in ins.text else 2 if ".64" in ins.text else 1
    return _regs(m.group(2), width)


def _read_regs(ins):
    """Registers an instruction reads (conservative: every register operand after the first,
    pairs for the packed FFMA2 operands, plus the destination of accumulating forms)."""
    body = ins.text
    body = re.sub(r"^@!?U?P\d+\s+", "", body)
    ops = body.split(None, 1)
    if len(ops) < 2:
        return set()
    toks = [t.strip() for t in ops[1].split(",")]
    regs = set()
    for k, t in enumerate(toks):
        for m in re.finditer(r"\bR(\d+)((?:\.\w+)*)", t):
            r = int(m.group(1))
            suf = m.group(2)
            wide = 2 if ("F32x2" in suf or ".64" in suf) else 1
            if k == 0 and not ops[0].startswith(("FFMA", "ST", "RED", "ATOM")):
                continue  # plain destination
            regs |= set(range(r, r + wide))
    return regs


def _free_store_barrier(body, sb, target):
    """Edits {index: hi word} that move every use of scoreboard `sb` inside the loop body to
    `target`, or None unless all of them are (STG read barrier, first later waiter in the same
    straight-line run) pairs."""
    if any(c.wb == sb for c in body):
        return None
    edits = {}
    paired = set()
    for k, c in enumerate(body):
        if c.rb != sb:
            continue
        if not re.search(r"\bSTG\b|\bSTG\.", c.text):
            return None
        j = k + 1
        while j < len(body) and j <= k + 24:
            t = body[j].text
            if re.search(r"\b(BRA|BSYNC|BSSY|EXIT|CALL|RET)\b", t):
                return None
            if body[j].rb == sb:
                return None
            if body[j].wait >> sb & 1:
                break
            j += 1
        else:
            return None
        edits[k] = (c.hi & ~(7 << 49)) | (target << 49)
        edits[j] = (body[j].hi & ~(1 << (52 + sb))) | (1 << (52 + target))
        paired.add(j)
    if not edits:
        return None
    if any((c.wait >> sb & 1) and k not in paired for k, c in enumerate(body)):
        return None
    return edits


def plan_patch(code, log=None, width=128):
    """Returns a list of (instruction index, new hi word) or None when a precondition fails.
    width: bits per lane of the kernel's row gathers."""
    say = log or (lambda s: None)
    _GATHER = _GATHERS[width]
    # the walk loop: the backward branch whose body holds the most 128-bit constant-path gathers
    best = None
    for i, ins in enumerate(code):
        m = re.search(_BRA, ins.text)
        if not m:
            continue
        tgt = int(m.group(1), 16)
        if tgt >= ins.addr:
            continue
        top = next((j for j, c in enumerate(code) if c.addr == tgt), None)
        if top is None:
            continue
        n = sum(1 for c in code[top:i] if _GATHER.search(c.text))
        inner = any(re.search(_BRA, c.text) and
                    int(re.search(_BRA, c.text).group(1), 16) < c.addr for c in code[top:i])
        if n >= 4 and not inner and (best is None or n > best[2]):
            best = (top, i, n)
    if best is None:
        say("no walk loop found")
        return None
    top, end, n_ld = best
    body = code[top:end + 1]
    loads = [k for k, c in enumerate(body) if _GATHER.search(c.text)]
    if any(body[k].wb != 5 for k in loads):
        say("gathers are not all on SB5")
        return None
    used = set()
    for c in body:
        if c.wb != 7:
            used.add(c.wb)
        if c.rb != 7:
            used.add(c.rb)
        used |= {b for b in range(6) if c.wait >> b & 1}
    free = [sb for sb in (4, 3) if sb not in used]
    pre_edits = {}
    if not free:
        # A scoreboard whose only use inside the loop is "STG holds its source registers /
        # the next writer of those registers waits" (the row-end store) can share the
        # scoreboard of another short-lived producer: both sides of every pair are moved.
        for sb in (4, 3):
            pre_edits = _free_store_barrier(body, sb, target=1)
            if pre_edits is not None:
                free = [sb]
                say(f"SB{sb} freed: {len(pre_edits) // 2} row-end store barriers moved to SB1")
                break
    if not free:
        say(f"no free scoreboard in the loop (used {sorted(used)})")
        return None
    sb = free[0]
    # consumer of a gather: the first instruction after it, cyclically through the loop body,
    # that reads one of its destination registers
    n = len(body)
    cons = {}
    for k in loads:
        d = _dest_regs(body[k])
        if not d:
            say("cannot parse a gather's destination")
            return None
        r = next((j % n for j in range(k + 1, k + n) if "LDG" not in body[j % n].text and _read_regs(body[j % n]) & d),
                 None)
        if r is None:
            say("a gather without a consumer inside the loop")
            return None
        cons[k] = r
    # refill events in issue order (one per gather instruction: the gathers of one position
    # are consecutive events with consecutive consumers, so halves of the pipeline depth fall on
    # position boundaries)
    events = []
    for k in loads:
        if events and cons[events[-1][0]] == cons[k]:
            events[-1].append(k)
        else:
            events.append([k])
    m = len(events)
    # pipeline depth in events: how many refill events are issued between an event and its consumer
    def dist(k, j):
        return (j - k) % n
    depth = sum(1 for e in events if 0 < dist(events[0][0], e[0]) < dist(events[0][0], cons[events[0][0]])) + 1
    if depth < 2 or m % depth or depth % 2:
        say(f"unexpected pipeline shape ({m} refill events, depth {depth})")
        return None
    halfd = depth // 2
    moved_events = [t for t in range(m) if (t // halfd) % 2 == 1]
    his = {k: hi for k, hi in (pre_edits or {}).items()}
    waits = []
    for t in moved_events:
        for k in events[t]:
            his[k] = (his.get(k, body[k].hi) & ~(7 << 46)) | (sb << 46)
        if (t - 1) not in moved_events:  # first event of a run: its consumer waits for the run
            waits.append(cons[events[t][0]])
    for w in waits:
        his[w] = his.get(w, body[w].hi) | (1 << (52 + sb))
    # every moved gather needs one of the new waits after its issue and not after its consumer,
    # and no gather on the new scoreboard may be issued between a run's last gather and its wait
    # ... by a later run (that would drain freshly issued loads): runs alternate with SB5 runs
    for t in moved_events:
        for k in events[t]:
            if not any(0 < dist(k, w) <= dist(k, cons[k]) for w in waits):
                say("a moved gather would not be waited for")
                return None
    # Control flow. The dependence model above is linear (address order inside the loop body),
    # which is only sound when the body is a single-entry straight trunk with forward skips:
    #   * nothing outside the loop jumps into the body, and the body holds no indirect
    #     branch, call or return;
    #   * every branch inside the body is a forward branch that stays inside the body (a
    #     conditionally skipped region, e.g. the row-end block) or the back edge itself;
    #   * every instruction that receives a new wait lies on the trunk: no forward branch
    #     jumps over it, so EVERY path from a moved gather to any of its consumers executes
    #     the wait (a wait inside a skipped region would leave the real consumer unguarded);
    #   * a moved gather may itself be skipped (then it never signals the scoreboard and the
    #     wait passes), but no consumer of its registers may precede the wait in address order
    #     after it, which the cyclic check above established.
    lo_addr, hi_addr = body[0].addr, body[-1].addr
    for c in code:
        mb = re.search(_BRA, c.text)
        if mb and not (lo_addr <= c.addr <= hi_addr) and lo_addr < int(mb.group(1), 16) <= hi_addr:
            say("a branch from outside enters the loop body")
            return None
    skips = []  # (index of the branch, index of its target) for forward branches in the body
    for k, c in enumerate(body):
        if re.search(r"\b(BRX|JMP|JMX|CALL|RET|EXIT|BREAK|BRXU|JMXU)\b", c.text):
            say(f"unsupported control flow in the loop body: {c.text}")
            return None
        mb = re.search(_BRA, c.text)
        if not mb or k == n - 1:
            continue
        tgt = int(mb.group(1), 16)
        if not (c.addr < tgt <= hi_addr):
            say(f"a branch leaves the loop body or goes backwards: {c.text}")
            return None
        ti = next((j for j, cc in enumerate(body) if cc.addr == tgt), None)
        if ti is None:
            say("branch target not on an instruction boundary")
            return None
        skips.append((k, ti))
    for w in waits:
        if any(b < w < t for b, t in skips):
            say(f"the wait at {body[w].addr:#x} can be jumped over: not on the loop's trunk")
            return None
    # (store-barrier pairs moved by _free_store_barrier were matched inside straight-line runs)
    edits = [(top + k, hi) for k, hi in sorted(his.items())]
    half = [k for t in moved_events for k in events[t]]
    wait_at = waits[0]
    say(f"loop {code[top].addr:#x}..{code[end].addr:#x}: {len(half)} of {len(loads)} gathers -> SB{sb} "
        f"(pipeline depth {depth} gathers), waits added at {', '.join(hex(body[w].addr) for w in waits)}")
    return edits


MARKER = b"SPMX_SASS_SCHED=0;"  # csrc/spmx_capi.cu: spmx_build_info(); rewritten after a patch


class SassSchedError(RuntimeError):
    """A precompiled width could not be re-scheduled (the preconditions no longer hold)."""


# kernels whose 64-byte rows are gathered with 64-bit loads
_NARROW = ("ILi16ELi8ELi2ELi1ELb0",)


def patch_library(lib, kernels=("spmm_chunk_kernelILi64ELi8ELi4ELi2ELb0", "spmm_dynamic_kernelILi64ELi8ELi4ELi2ELb0",
                                "spmm_chunk_kernelILi32ELi8ELi4ELi1ELb0", "spmm_dynamic_kernelILi32ELi8ELi4ELi1ELb0",
                                "spmm_chunk_kernelILi128ELi8ELi4ELi4ELb0", "spmm_dynamic_kernelILi128ELi8ELi4ELi4ELb0",
                                "spmm_chunk_kernelILi16ELi8ELi2ELi1ELb0", "spmm_dynamic_kernelILi16ELi8ELi2ELi1ELb0"),
                  dry_run=False, log=print, strict=False):
    """Re-schedules the listed kernels inside `lib`. With strict=True (the build) a listed
    kernel that is missing or fails a precondition raises SassSchedError instead of being
    left as compiled, so that a toolchain change cannot silently ship the slower schedule.
    The library's build-info string records how many kernels were edited."""
    funcs = disassemble(lib)
    data = bytearray(open(lib, "rb").read())
    done, failed = 0, []
    seen = set()
    for name, code in funcs.items():
        hit = next((k for k in kernels if k in name), None)
        if hit is None or not code:
            continue
        seen.add(hit)
        blob = b"".join(c.bytes() for c in code)
        pos = data.find(blob)
        if pos < 0 or data.find(blob, pos + 1) >= 0:
            log(f"{name[:60]}: code not located uniquely (already patched or compressed)")
            failed.append(hit)
            continue
        edits = plan_patch(code, lambda s: log(f"{name[:60]}: {s}"),
                           width=64 if any(t in name for t in _NARROW) else 128)
        if not edits:
            failed.append(hit)
            continue
        for idx, hi in edits:
            o = pos + 16 * idx + 8
            data[o:o + 8] = hi.to_bytes(8, "little")
        done += 1
    failed += [k for k in kernels if k not in seen]
    if strict and failed:
        raise SassSchedError("sass_sched: preconditions failed for " + ", ".join(failed) +
                             " (set SPMX_NO_SASS_SCHED=1 to ship the schedule as compiled)")
    if done and not dry_run:
        pos = data.find(MARKER)
        if pos >= 0 and data.find(MARKER, pos + 1) < 0:
            new = MARKER.replace(b"=0;", b"=%d;" % min(done, 9))
            data[pos:pos + len(MARKER)] = new
        elif strict:
            raise SassSchedError("sass_sched: build-info marker not found in the library")
        open(lib, "wb").write(bytes(data))
    return done


if __name__ == "__main__":
    n = patch_library(sys.argv[1], dry_run="--dry-run" in sys.argv)
    print(f"{n} kernel(s) re-scheduled")
