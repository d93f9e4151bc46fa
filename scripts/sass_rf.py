"""Static register-file read estimate for a kernel's inner loop (tuning helper).

For each FP32 pipe instruction (FFMA2/FMUL2/FADD2/FFMA/FMUL/FADD) counts the
32-bit register reads that are NOT served by a .reuse cache hit.
Usage: python scripts/sass_rf.py <lib.so> <mangled-kernel-name>
"""
import re, subprocess, sys, collections

so, fn = sys.argv[1], sys.argv[2]
sass = subprocess.run(["cuobjdump", "-sass", "-fun", fn, so], capture_output=True, text=True).stdout
lines = [l for l in sass.splitlines() if re.match(r"\s+/\*[0-9a-f]+\*/", l)]
# inner loop = the longest backward-branch body
best = (0, 0, 0)
addr = [int(re.match(r"\s+/\*([0-9a-f]+)\*/", l).group(1), 16) for l in lines]
for k, l in enumerate(lines):
    m = re.search(r"BRA(?:\.U)?\s+(?:U?P\d+,\s*)?0x([0-9a-f]+)", l)
    if m:
        tgt = int(m.group(1), 16)
        if tgt < addr[k]:
            start = addr.index(tgt) if tgt in addr else None
            if start is not None and k - start > best[0]:
                best = (k - start, start, k)
_, a, b = best
body = lines[a:b + 1]
ops = collections.Counter()
reads = 0
reuse_slots = {}  # slot -> register last cached
fp = 0
for l in body:
    ins = re.sub(r"/\*.*?\*/", "", l).strip().rstrip(";")
    op = ins.split()[0] if not ins.startswith("@") else ins.split()[1]
    ops[op.split(".")[0]] += 1
    if not re.match(r"F(FMA|MUL|ADD)2?$", op.split(".")[0]):
        continue
    fp += 1
    operands = [o.strip() for o in ins.split(None, 1)[1].split(",")][1:]
    for slot, o in enumerate(operands):
        mreg = re.match(r"-?\|?(R\d+)(\.reuse)?(\.F32x2)?", o)
        if not mreg:
            continue
        r = mreg.group(1)
        width = 2 if ".F32x2" in o else 1
        if reuse_slots.get(slot) == r:
            pass  # served from reuse cache
        else:
            reads += width
        reuse_slots[slot] = r if ".reuse" in o else None
print(f"inner loop: {len(body)} instrs, {fp} FP32-pipe, RF reads {reads} ({reads / max(fp, 1):.2f}/instr)")
print(dict(ops.most_common(12)))
