"""Summarise an `ncu --page source --csv --print-source sass` export: samples per instruction class and
stall reason, plus the hottest instructions (for the kernel-design notes in DESIGN.md)."""
import csv, sys, collections, re
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
data = rows[2:]
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = collections.Counter()
by_op = collections.defaultdict(collections.Counter)
samples_op = collections.Counter()
inst = []
for r in data:
    if len(r) < len(hdr):
        continue
    src = r[idx["Source"]].strip()
    op = re.sub(r"^@!?U?P\w+\s+", "", src).split(" ")[0]
    base = op.split(".")[0]
    s = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
    samples_op[base] += s
    for c in stall_cols:
        v = int(r[idx[c]] or 0)
        tot[c] += v
        by_op[base][c] += v
    inst.append((s, src, r[idx["Instructions Executed"]]))
T = sum(samples_op.values())
print("total samples", T)
print("by opcode (share of samples):")
for op, s in samples_op.most_common(15):
    top = ", ".join(f"{k[6:]}={v/T:.3f}" for k, v in by_op[op].most_common(4) if v)
    print(f"  {op:10s} {s/T:6.3f}   {top}")
print("by stall reason:")
for c, v in tot.most_common(12):
    print(f"  {c:22s} {v/T:.3f}")
print("hottest instructions:")
for s, src, ex in sorted(inst, reverse=True)[:25]:
    print(f"  {s/T:6.3f} {ex:>10s}  {src}")
