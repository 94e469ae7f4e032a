"""Static SASS census of the fused kernel's prune / exp region (bring-up tool).

    python tools/sass_region.py <obj.o> <mangled-kernel-substring>

Finds the softmax warps' steady-state step (from the first LDTM.x32 after the register
re-allocation to the following BAR.RED = the per-step "shift ok?" vote), and prints the
opcode histogram, the pipe split (alu / fma / xu / other) and the per-4-score-group counts
(16 groups per warp step).  Used to compare epilogue formulations without a GPU.
"""
import collections
import re
import subprocess
import sys

ALU = {"FMNMX", "FMNMX3", "FSETP", "FSEL", "SEL", "LOP3", "SHF", "IADD3", "ISETP", "PRMT", "F2FP", "LEA", "MOV",
       "PLOP3", "P2R", "R2P", "VIADD", "IMNMX", "FMNMX.NAN"}
FMA = {"FFMA", "FFMA2", "FADD", "FADD2", "FMUL", "FMUL2", "IMAD", "HFMA2"}
XU = {"MUFU"}


def main():
    obj, fun = sys.argv[1], sys.argv[2]
    names = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
    m = [l.split(":")[1].strip() for l in names.splitlines() if "Function :" in l and fun in l]
    if not m:
        sys.exit("no function matching " + fun)
    sass = subprocess.run(["cuobjdump", "-sass", "-fun", m[0], obj], capture_output=True, text=True).stdout
    ins = []
    for l in sass.splitlines():
        mm = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
        if mm:
            ins.append(mm.group(2).strip())
    start = next(i for i, s in enumerate(ins) if "USETMAXREG.TRY_ALLOC" in s or "TRY_ALLOC" in s) if any(
        "TRY_ALLOC" in s for s in ins) else 0
    i0 = next(i for i in range(start, len(ins)) if "LDTM.x32" in ins[i] and "LDTM.x32" in ins[i + 1] if False) if False else None
    # steady state: the LAST pair of LDTM.x32 before a BAR.RED
    bars = [i for i, s in enumerate(ins) if "BAR.RED" in s and i > start]
    best = None
    for b in bars:
        lds = [i for i in range(start, b) if "LDTM.x32" in ins[i]]
        if len(lds) >= 2:
            a = lds[-2]
            # walk back to the previous LDTM pair boundary: the region is [a, b)
            best = (a, b)
    a, b = best
    hist = collections.Counter()
    pipes = collections.Counter()
    for s in ins[a:b]:
        op = s.split()[0]
        if op.startswith("@"):
            op = s.split()[1]
        base = op.split(".")[0]
        hist[op] += 1
        pipes["alu" if base in ALU else "fma" if base in FMA else "xu" if base in XU else "other"] += 1
    tot = sum(hist.values())
    print(f"region [{a}, {b}) {tot} instructions = {tot / 16:.2f} per group")
    for k, v in sorted(pipes.items()):
        print(f"  {k:6s} {v:5d}  {v / 16:.2f}/group")
    for k, v in hist.most_common():
        print(f"    {v:4d} {k}")


if __name__ == "__main__":
    main()
