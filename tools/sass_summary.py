"""Per-kernel SASS instruction summary of the built library (cuobjdump -sass):
counts of the instruction classes that show what each kernel runs on --
FP32 pipe (FFMA, FFMA2, FMUL, FMUL2, FADD), bulk / tensor-map copies (UBLKCP,
UTMALDG), mbarrier waits (SYNCS), tcgen05 (UTCMMA / UTCHMMA / UTCQMMA, LDTM,
STTM, UTCBAR), warp matches and shared-memory traffic.

  python tools/sass_summary.py [lib.so] > profiles/r2_sass_summary.txt
"""
import collections
import re
import subprocess
import sys

LIB = sys.argv[1] if len(sys.argv) > 1 else "paper_2101_11714_b200/lib/libttgpu.so"
CLASSES = ["FFMA2", "FFMA", "FMUL2", "FMUL", "FADD2", "FADD", "UBLKCP", "UTMALDG", "SYNCS",
           "UTCMMA", "UTCHMMA", "UTCQMMA", "UTCBAR", "LDTM", "STTM", "MATCH", "LDS", "STS", "LDG",
           "STG", "ATOMG", "RED", "BAR"]


def demangle(names):
    try:
        out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True,
                             check=True).stdout.splitlines()
        return dict(zip(names, out))
    except Exception:  # noqa: BLE001
        return {n: n for n in names}


def main():
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    kern, counts = None, collections.OrderedDict()
    for line in sass.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            kern = m.group(1)
            counts[kern] = collections.Counter()
            continue
        if kern is None:
            continue
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
        if not m:
            continue
        op = m.group(1)
        counts[kern]["total"] += 1
        for c in CLASSES:
            if op == c or (c in ("LDS", "STS", "LDG", "STG", "BAR", "SYNCS", "MATCH", "RED", "ATOMG")
                           and op.startswith(c)):
                counts[kern][c] += 1
                break
    names = demangle(list(counts))
    cols = ["total"] + CLASSES
    print(f"# SASS instruction counts per kernel ({LIB}, cuobjdump -sass, static counts)")
    print("# kernel | " + " ".join(cols))
    tot = collections.Counter()
    for k, c in counts.items():
        tot.update(c)
        short = re.sub(r"\(.*", "", names[k])[:90]
        print(f"{short} | " + " ".join(f"{c[x]}" for x in cols))
    print("# ALL | " + " ".join(f"{tot[x]}" for x in cols))


if __name__ == "__main__":
    main()
