"""SASS evidence from the built library (no GPU needed): cuobjdump -sass of libspinsim_b200.so, then
  * a mnemonic census of the hot kernels (FP64 DFMA/DMUL/DADD, packed FP32 FFMA2/FMUL2/FADD2, the bulk/tensor copies
    UBLKCP/UTMALDG/UTMASTG and LDGSTS that move the scan's operators),
  * the innermost backward-branch loops of the C3/C2 interval kernel with their FP64 mix — the τ residual squaring
    (36 FP64 instructions per squaring, DESIGN.md §5 items 13 and 19) and of the FP32 kernel (packed float2 squarings).

    python tools/sass_excerpt.py > profiles/r02/<tag>/sass_excerpt.txt
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2204_05586_b200", "libspinsim_b200.so")
KEYS = ["DFMA", "DMUL", "DADD", "FFMA2", "FMUL2", "FADD2", "UBLKCP", "UTMALDG", "UTMASTG", "LDGSTS", "SHFL"]
HOT = {
    "_ZN3ssb15interval_kernelILi2ELi1ELi0ELi3EdLi0EEEvNS_14IntervalParamsE": "interval kernel, spin-one LT, CF4, neural, FP64 (C3, C2)",
    "_ZN3ssb15interval_kernelILi2ELi1ELi0ELi3EdLi1EEEvNS_14IntervalParamsE": "  same, FUSED instance (run aggregates)",
    "_ZN3ssb15interval_kernelILi2ELi1ELi0ELi3EfLi0EEEvNS_14IntervalParamsE": "interval kernel, spin-one LT, FP32 mode (C5 FP32)",
    "_ZN3ssb15interval_kernelILi1ELi0ELi0ELi3EdLi0EEEvNS_14IntervalParamsE": "interval kernel, spin-half, FP64 (C4)",
    "_ZN3ssb15interval_kernelILi2ELi2ELi0ELi7EdLi0EEEvNS_14IntervalParamsE": "interval kernel, general spin-one su(3) (G1)",
    "_ZN3ssb12chain_kernelINS_2CMILi3EEEEEvNS_9ChainArgsE": "chain kernel (C3 states)",
    "_ZN3ssb16run_chain_kernelINS_2SUILi2EEELi32ELb0EEEvNS_12RunChainArgsE": "run chain, SU(2) ops, 32-interval runs (scan-stress)",
    "_ZN3ssb16run_chain_kernelINS_2SUILi3EEELi4ELb0EEEvNS_12RunChainArgsE": "run chain, D1(SU(2)) ops, 4-interval runs (C5 analytic)",
    "_ZN3ssb12scan3_kernelINS_2CMILi3EEEEEvNS_9Scan3ArgsE14CUtensorMap_stS4_": "scan3 (tensor-TMA look-back scan)",
}
INS = re.compile(r"/\*([0-9a-f]{4,})\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?([^;]*);")


def functions(sass):
    for part in re.split(r"\n\s*Function : ", sass)[1:]:
        name, body = part.split("\n", 1)
        yield name.strip(), [(int(m.group(1), 16), m.group(3), m.group(0)) for m in INS.finditer(body)]


def loops(ins):
    """Backward branches (BRA to a lower address): (start, end) address ranges."""
    out = []
    for addr, op, text in ins:
        if op == "BRA":
            m = re.search(r"BRA\s+(?:`\(\.L_x_\d+\)\s*)?0x([0-9a-f]+)", text) or re.search(r"0x([0-9a-f]+)\s*;", text)
            if m and int(m.group(1), 16) < addr:
                out.append((int(m.group(1), 16), addr))
    return out


def main():
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    print(f"# SASS of {os.path.relpath(LIB, ROOT)} (cuobjdump -sass; arch sm_100a only)\n")
    print("## mnemonic census (static instruction counts)\n")
    funcs = dict(functions(sass))
    for name, what in HOT.items():
        ins = funcs.get(name)
        if ins is None:
            print(f"{what}: not found")
            continue
        c = collections.Counter(op for _, op, _ in ins)
        print(f"{what}: {len(ins)} instructions; " + ", ".join(f"{k} {c[k]}" for k in KEYS if c[k]))
    for name in ("_ZN3ssb15interval_kernelILi2ELi1ELi0ELi3EdLi0EEEvNS_14IntervalParamsE",
                 "_ZN3ssb15interval_kernelILi2ELi1ELi0ELi3EfLi0EEEvNS_14IntervalParamsE"):
        ins = funcs[name]
        print(f"\n## innermost loops of {HOT[name]}\n")
        def arith(r):   # FP64 / packed-FP32 arithmetic fraction of a loop body
            body = [op for a, op, _ in ins if r[0] <= a <= r[1]]
            return sum(op in KEYS[:6] for op in body) / max(1, len(body))
        hot = sorted(loops(ins), key=arith, reverse=True)
        for lo, hi in hot[:4]:
            body = [x for x in ins if lo <= x[0] <= hi]
            c = collections.Counter(op for _, op, _ in body)
            print(f"loop [{lo:#x}, {hi:#x}]: {len(body)} instructions; "
                  + ", ".join(f"{k} {c[k]}" for k in KEYS if c[k]))
        lo, hi = hot[0]
        print(f"\nlisting of the densest loop [{lo:#x}, {hi:#x}] (the τ residual-squaring loop, unrolled ×2):")
        for addr, _, text in ins:
            if lo <= addr <= hi:
                print("   ", re.sub(r"\s+", " ", text))


if __name__ == "__main__":
    sys.exit(main())
