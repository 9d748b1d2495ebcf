"""The post-link scheduling edit (paper_2312_05639_b200/sass_sched.py) is part
of the build: these checks read the built library's SASS (cuobjdump, no GPU needed) and make
sure the edit is really in it — half of the walk loop's gathers on a second scoreboard, every
moved gather waited for before its first consumer — and that a second pass finds nothing left
to do. If ptxas ever changes the loop so that the preconditions fail, the build silently keeps
the compiled schedule (5-13 % slower); this test makes that visible.
"""
import os
import re
import shutil

import pytest

from paper_2312_05639_b200 import binding, sass_sched

KERNELS = ("spmm_chunk_kernelILi64ELi8ELi4ELi2ELb0", "spmm_chunk_kernelILi32ELi8ELi4ELi1ELb0",
           "spmm_chunk_kernelILi128ELi8ELi4ELi4ELb0", "spmm_chunk_kernelILi16ELi8ELi2ELi1ELb0")


def _width(kernel):
    """bits per lane of the kernel's row gathers (d = 16: 8 lanes x float2)"""
    return 64 if any(t in kernel for t in sass_sched._NARROW) else 128


@pytest.fixture(scope="module")
def funcs():
    if shutil.which("cuobjdump") is None:
        pytest.skip("cuobjdump not on PATH")
    if os.environ.get("SPMX_NO_SASS_SCHED"):
        pytest.skip("SPMX_NO_SASS_SCHED set: kernels left as compiled")
    lib = binding.build_library()
    return sass_sched.disassemble(lib)


def _walk_loop(code, gather):
    """(top, end, gathers) of the innermost loop (no backward branch inside) whose body holds
    the most row gathers."""
    best = None
    for i, ins in enumerate(code):
        m = re.search(sass_sched._BRA, ins.text)
        if not m or int(m.group(1), 16) >= ins.addr:
            continue
        top = next(j for j, c in enumerate(code) if c.addr == int(m.group(1), 16))
        n = sum(1 for c in code[top:i] if gather.search(c.text))
        inner = any((mm := re.search(sass_sched._BRA, c.text)) and int(mm.group(1), 16) < c.addr
                    for c in code[top:i])
        if not inner and (best is None or n > best[2]):
            best = (top, i, n)
    return best


@pytest.mark.parametrize("kernel", KERNELS)
def test_gathers_are_split_over_two_scoreboards(funcs, kernel):
    name = next(n for n in funcs if kernel in n)
    code = funcs[name]
    gather = sass_sched._GATHERS[_width(kernel)]
    top, end, n = _walk_loop(code, gather)
    assert n >= 8, "walk loop not found"
    body = code[top:end + 1]
    loads = [c for c in body if gather.search(c.text)]
    boards = sorted({c.wb for c in loads})
    assert len(boards) == 2 and 5 in boards, boards
    moved = [c for c in loads if c.wb != 5]
    assert len(moved) * 2 == len(loads), "half of the gathers move"
    sb = moved[0].wb
    # every moved gather: some instruction between its issue and its first consumer
    # (cyclically) waits for the new scoreboard
    nb = len(body)
    for k, c in enumerate(body):
        if c not in moved:
            continue
        dest = sass_sched._dest_regs(c)
        for step in range(1, nb):
            j = (k + step) % nb
            if body[j].wait >> sb & 1:
                break
            assert not ("LDG" not in body[j].text and sass_sched._read_regs(body[j]) & dest), \
                f"{body[j].text} reads a moved gather's registers without waiting for SB{sb}"
        else:
            pytest.fail("no wait for the moved gather")
    # a second pass has nothing to do (the gathers are no longer all on SB5)
    assert sass_sched.plan_patch(code, width=_width(kernel)) is None
