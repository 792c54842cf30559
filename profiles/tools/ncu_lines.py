import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
cur = None; out = []
hdr = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split('/')[-1]; continue
    if r and r[0] == "Line No":
        hdr = r; continue
    if hdr and r and r[0] not in ("",) and len(r) > 8:
        try:
            samp = int(r[4]); inst = int(r[7])
        except ValueError:
            continue
        out.append((samp, inst, cur, r[0], r[1][:110]))
tot = sum(o[0] for o in out); toti = sum(o[1] for o in out)
print("total samples", tot, "inst", toti)
for o in sorted(out, reverse=True)[:int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    print(f"{100*o[0]/tot:5.1f}% smp {100*o[1]/toti:5.1f}% inst  {o[2]}:{o[3]}  {o[4]}")
