"""Static checks of the far kernels' SASS (CPU-only: cuobjdump reads the sm_100a cubins):
instruction-cache footprint and the two-target weight sharing.  The executed-flop count
bench.py's far roofline uses is pinned on a GPU by tests/test_gpu_far_flops.py (ncu)."""
import collections
import os
import re
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
LIB = os.path.join(ROOT, "paper_1811_12498_b200", "libstokestree_b200.so")

pytestmark = pytest.mark.skipif(not shutil.which("cuobjdump") or not os.path.exists(LIB),
                                reason="needs cuobjdump and the built library")


def _sass_functions():
    out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    funcs, name = {}, None
    for ln in out.splitlines():
        m = re.match(r"\s*Function : (\S+)", ln)
        if m:
            name = m.group(1)
            funcs[name] = []
        elif name:
            funcs[name].append(ln)
    return funcs


_FUNCS = None


def funcs():
    global _FUNCS
    if _FUNCS is None:
        _FUNCS = _sass_functions()
    return _FUNCS


@pytest.mark.parametrize("P", [3, 7, 10, 12, 18])
@pytest.mark.parametrize("kernel", ["k_far_list", "k_feval"])
def test_far_kernels_fit_the_instruction_cache(kernel, P):
    """The far kernels' column loops run at run time: the fully unrolled form (one template
    instance per (n, m)) grew to ~2,900 instructions at P = 10 with the two-target path and
    stalled on instruction fetch (ncu r02e: 4.0 no_instruction stalls per issue at P = 12).
    Guard: the whole kernel stays under 1,600 SASS instructions (25 KB) at every order."""
    name = next((f for f in funcs() if re.search(rf"{kernel}ILi{P}E", f)), None)
    assert name, f"{kernel}<{P}> not in the library"
    n = sum(1 for ln in funcs()[name] if re.match(r"\s*/\*[0-9a-f]{4,}\*/", ln))
    assert n < 1600, (kernel, P, n)


@pytest.mark.parametrize("P", [10, 12])
def test_two_target_inner_loop_shares_weight_loads(P):
    """k_far_list's inner column loop for two targets (unrolled by two grades): per grade and
    column pair, 2 x (4 DMUL + 2 DFMA recurrence + 2 q) ... i.e. 26 DP instructions per grade
    against 4 LDS.128 -- each weight pair feeds both targets."""
    name = next(f for f in funcs() if re.search(rf"k_far_listILi{P}E", f))
    ins = []
    for ln in funcs()[name]:
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    addr = {a: i for i, (a, _) in enumerate(ins)}
    loops = []
    for i, (a, txt) in enumerate(ins):
        m = re.search(r"BRA\s.*?0x([0-9a-f]+)", txt)
        if m and int(m.group(1), 16) <= a and int(m.group(1), 16) in addr:
            body = ins[addr[int(m.group(1), 16)]:i + 1]
            loops.append(collections.Counter(t.split()[1 if t.startswith("@") else 0].split(".")[0] for _, t in body))
    dp = lambda o: o["DFMA"] + o["DMUL"] + o["DADD"]
    assert any(dp(o) == 52 and o["LDS"] == 8 and o["MUFU"] == 0 for o in loops), [dict(o) for o in loops]
