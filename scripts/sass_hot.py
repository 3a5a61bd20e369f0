"""Group the SASS page of an ncu report (ncu -i REP --page source --csv) into runs of
instructions with equal executed counts; print the runs by share of executed instructions."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
H = rows[hdr]
ci = {n: H.index(n) for n in ("Source", "Instructions Executed", "# Samples", "Avg. Threads Executed")}
ins = []
for r in rows[hdr + 1:]:
    if len(r) < len(H): continue
    ins.append((r[ci["Source"]].strip(), int(r[ci["Instructions Executed"]] or 0), int(r[ci["# Samples"]] or 0),
                float(r[ci["Avg. Threads Executed"]] or 0)))
tot = sum(x[1] for x in ins); tots = sum(x[2] for x in ins)
print("total warp instr", tot, "samples", tots)
runs = []; s = 0
for i in range(1, len(ins) + 1):
    if i == len(ins) or abs(ins[i][1] - ins[s][1]) > 0.02 * max(ins[s][1], 1):
        runs.append((s, i)); s = i
runs.sort(key=lambda ab: -sum(x[1] for x in ins[ab[0]:ab[1]]))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
for a, b in runs[:top]:
    e = sum(x[1] for x in ins[a:b]); sm = sum(x[2] for x in ins[a:b])
    ops = {}
    for x in ins[a:b]:
        op = x[0].split()[0] if not x[0].startswith("@") else x[0].split()[1]
        op = op.split(".")[0]; ops[op] = ops.get(op, 0) + 1
    o = " ".join(f"{k}:{v}" for k, v in sorted(ops.items(), key=lambda kv: -kv[1])[:9])
    print(f"[{a:5d},{b:5d}) n={b-a:4d} exec/instr={ins[a][1]:>10d} share={e/tot*100:5.1f}% samples={sm/tots*100:5.1f}% thr={ins[a][3]:.0f} | {o}")
if len(sys.argv) > 3:
    a, b = map(int, sys.argv[3].split(":"))
    for i in range(a, b): print(i, ins[i])
