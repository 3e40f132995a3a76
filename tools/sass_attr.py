"""Instruction mix of one kernel of the built library, attributed to source lines.

    python tools/sass_attr.py k_row_r2c_t2dINS_6SPlanTIfLi16 [paper_1912_06976_b200/libbttb_sm100.so]

Extracts the spectral.cu cubin (cuobjdump -xelf), disassembles it with line
information (nvdisasm -g; the library is built with -lineinfo) and prints, for
the first kernel whose mangled name contains the given substring, the
instruction histogram and the source lines that carry the most non-floating-
point instructions (address arithmetic, predicates, moves).  Used for the
index-arithmetic diet of DESIGN.md section 4 (the fp32 row kernels are
issue-bound: 1440 -> 1184 instructions per thread).
"""
import collections
import os
import re
import subprocess
import sys
import tempfile

FP = {"FADD", "FMUL", "FFMA", "DADD", "DMUL", "DFMA"}


def main():
    name = sys.argv[1]
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    lib = sys.argv[2] if len(sys.argv) > 2 else os.path.join(root, "paper_1912_06976_b200", "libbttb_sm100.so")
    with tempfile.TemporaryDirectory() as tmp:
        subprocess.run(["cuobjdump", "-xelf", "spectral.sm_100a.cubin", os.path.abspath(lib)], cwd=tmp, check=True,
                       stdout=subprocess.DEVNULL)
        sass = subprocess.run(["nvdisasm", "-g", os.path.join(tmp, "spectral.sm_100a.cubin")], check=True,
                              capture_output=True, text=True).stdout.split("\n")
    starts = [i for i, ln in enumerate(sass) if ln.startswith(".text.") and name in ln]
    if not starts:
        raise SystemExit(f"no kernel matching {name!r}")
    start = starts[0]
    end = start + 1
    while end < len(sass) and not sass[end].startswith(".text.") and not sass[end].startswith("\t.section"):
        end += 1
    cur = None
    per_line = collections.Counter()
    other = collections.Counter()
    ops = collections.defaultdict(collections.Counter)
    hist = collections.Counter()
    for ln in sass[start:end]:
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(@!?U?P\d+\s+)?([A-Z0-9_.]+)", ln)
        if m:
            op = m.group(2).split(".")[0]
            hist[op] += 1
            per_line[cur] += 1
            if op not in FP:
                other[cur] += 1
                ops[cur][op] += 1
    print(sass[start][:160])
    print("instructions", sum(hist.values()), "of which not floating point", sum(other.values()))
    print(hist.most_common(16))
    for key, n in other.most_common(14):
        print("  ", key, n, "of", per_line[key], dict(ops[key]))


if __name__ == "__main__":
    main()
