"""Instruction-mix summary of the hot kernels' SASS (cuobjdump -sass of the
built objects): opcode counts per kernel, the FP64 opcodes, DFMA (must be 0:
the reference's arithmetic has no contraction), the global-load forms and
the kernel's register / shared-memory use (cuobjdump -res-usage)."""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BUILD = os.path.join(ROOT, "paper_2209_12310_b200", "build")
WANT = ["kf_filter", "k1_extremes", "k1_small", "k1b_corners", "k2_filter", "k2_compact",
        "kf_gather", "chain_local", "chain_replay", "count_in_region"]
FP64 = {"DADD", "DMUL", "DFMA", "DSETP", "DMNMX"}


def short(name):
    for w in WANT:
        if w in name:
            dem = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
            m = re.search(w + r"(<[^(]*>)?", dem)
            t = (m.group(1) or "") if m else ""
            return w + t.replace("unsigned int", "u32").replace("unsigned long", "u64")
    return None


def main():
    objs = [os.path.join(BUILD, f) for f in ("kernels.cu.o", "hullchain.cu.o")]
    out = []
    total_dfma = 0
    for obj in objs:
        sass = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
        res = subprocess.run(["cuobjdump", "-res-usage", obj], capture_output=True, text=True).stdout
        regs = {}
        for m in re.finditer(r"Function (\S+):\s*\n\s*REG:(\d+) STACK:(\d+) SHARED:(\d+)", res):
            regs[m.group(1)] = (int(m.group(2)), int(m.group(3)), int(m.group(4)))
        for block in sass.split("Function : ")[1:]:
            name = block.split("\n", 1)[0].strip()
            total_dfma += len(re.findall(r"\bDFMA\b", block))
            s = short(name)
            if s is None:
                continue
            ops = collections.Counter(re.findall(r"/\*[0-9a-f]{4,6}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", block))
            base = collections.Counter()
            for op, c in ops.items():
                base[op.split(".")[0]] += c
            loads = {op: c for op, c in ops.items() if op.startswith("LDG")}
            fp64 = {op: base[op] for op in sorted(FP64) if base[op]}
            r = regs.get(name, ("?", "?", "?"))
            out.append(f"{s:34s} {sum(ops.values()):6d} instr  regs {r[0]}  stack {r[1]}  smem {r[2]}\n"
                       f"    FP64 {fp64}\n    loads {loads}\n"
                       f"    top {base.most_common(8)}")
    print("SASS summary (cuobjdump -sass, sm_100a; static instruction counts)\n")
    print("\n".join(out))
    print(f"\nDFMA in kernels.cu.o + hullchain.cu.o: {total_dfma}")


if __name__ == "__main__":
    sys.exit(main())
