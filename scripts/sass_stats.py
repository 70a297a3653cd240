"""Per-kernel SASS opcode histogram of libosc_b200.so (run here, no GPU).

usage: python scripts/sass_stats.py [substring-of-kernel-name] [--loop]
--loop restricts the count to the body of the innermost backward branch that
contains the most DP instructions (the time-step loop).
"""
import re
import subprocess
import sys
from collections import Counter

LIB = "paper_1702_02207_b200/libosc_b200.so"


def functions(lib=LIB):
    out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True,
                         check=True).stdout
    cur, body = None, []
    for line in out.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            if cur:
                yield cur, body
            cur, body = m.group(1), []
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m and cur:
            body.append((int(m.group(1), 16), m.group(2).strip()))
    if cur:
        yield cur, body


def opcode(ins):
    ins = re.sub(r"^@!?U?P\w+\s+", "", ins)
    return ins.split()[0].split(".")[0]


def loop_body(body):
    best = None
    for addr, ins in body:
        m = re.search(r"\bBRA\b.*?0x([0-9a-f]+)\s*$", ins)
        if m:
            tgt = int(m.group(1), 16)
            if tgt < addr:
                seg = [i for a, i in body if tgt <= a <= addr]
                dp = sum(opcode(i) in ("DADD", "DMUL", "DFMA") for i in seg)
                if any(opcode(i) == "CALL" for i in seg):
                    continue  # the exact-division replay loop, not the hot loop
                if best is None or dp > best[0]:
                    best = (dp, seg)
    return best[1] if best else [i for _, i in body]


def hot_loops(body):
    """DP counts of the CALL-free loops holding at least half the DP
    instructions of the largest one (K1 has two: three- and two-operation
    division), largest first."""
    out = []
    for addr, ins in body:
        m = re.search(r"\bBRA\b.*?0x([0-9a-f]+)\s*$", ins)
        if m and int(m.group(1), 16) < addr:
            seg = [i for a, i in body if int(m.group(1), 16) <= a <= addr]
            if not any(opcode(i) == "CALL" for i in seg):
                out.append(sum(opcode(i) in ("DADD", "DMUL", "DFMA") for i in seg))
    out.sort(reverse=True)
    return [n for n in out if out and n >= out[0] / 2]


def dp_loops(lib, kernel_substr):
    for name, body in functions(lib):
        if kernel_substr in name:
            return hot_loops(body)
    return []


def dp_per_iteration(lib, kernel_substr):
    """DP-pipe instructions in the hot loop of the first kernel whose mangled
    name contains kernel_substr (one loop iteration = one RK4 step)."""
    for name, body in functions(lib):
        if kernel_substr in name:
            return sum(opcode(i) in ("DADD", "DMUL", "DFMA") for i in loop_body(body))
    return None


def main():
    pat = sys.argv[1] if len(sys.argv) > 1 else ""
    for name, body in functions():
        if pat not in name:
            continue
        ins = loop_body(body) if "--loop" in sys.argv else [i for _, i in body]
        c = Counter(opcode(i) for i in ins)
        dp = sum(c[k] for k in ("DADD", "DMUL", "DFMA"))
        print(f"{name}: {len(ins)} instr, DP={dp} (DADD {c['DADD']} DMUL {c['DMUL']} "
              f"DFMA {c['DFMA']}) MUFU {c['MUFU']} FSETP {c['FSETP']} BAR {c['BAR']} "
              f"SHFL {c['SHFL']} CALL {c['CALL']}")
        print("   ", ", ".join(f"{k}:{v}" for k, v in c.most_common(14)))


if __name__ == "__main__":
    main()
