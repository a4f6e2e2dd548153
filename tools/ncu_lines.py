"""Per-source-line instruction / stall attribution of an ncu source page (--print-source cuda,sass
--csv) for k_walk, grouped into the kernel's phases.  usage: ncu_lines.py SRC.csv ROWS_PER_BATCH N"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
rpb = int(sys.argv[2]) if len(sys.argv) > 2 else 64
n = int(sys.argv[3]) if len(sys.argv) > 3 else 65608366
nb = n / rpb
f = None
hdr = None
out = []
for r in rows:
    if r and r[0] == "File Path":
        f = r[1].split('/')[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) < 8 or r[2] != '-':
        continue
    try:
        e = float(r[7]); s = float(r[4])
    except ValueError:
        continue
    if e or s:
        out.append((f, int(r[0]), e, s, r[1]))
te = sum(o[2] for o in out); ts = sum(o[3] for o in out)
print(f"total warp-instr {te:.3e}  per batch of {rpb} rows {te / nb:.1f}; stall samples {ts:.0f}")
src = open('paper_1902_09527_b200/csrc/km_walk.cu').read().split('\n')


def find(pat):
    for i, l in enumerate(src):
        if pat in l:
            return i + 1
    return None


marks = [("helpers", 1), ("kernel prologue", find("k_walk(AssignParams p)")),
         ("row load/clause 1", find("while (chunk_row < n) {")), ("A, bounds, H search", find("if (amask) {")),
         ("candidate loop", find("for (int j = 0; j < pm; j += 2) {")),
         ("decision epilogue", find("steps += (unsigned long long)pm;")), ("fallback", find("if (fallback) {")),
         ("dists count", find("// MTI distance count")), ("writes/movers", find("const int rb = row0 + 32 * i;")),
         ("tail", find("#pragma unroll\n    for (int o = 16") or find("c_changed += __shfl_xor_sync")),
         ("prep kernel", find("__global__ void k_prep_walk"))]
marks = sorted([m for m in marks if m[1]], key=lambda m: m[1])
for mi, (nm, lo) in enumerate(marks):
    hi = marks[mi + 1][1] - 1 if mi + 1 < len(marks) else 10 ** 6
    e = sum(o[2] for o in out if o[0] == 'km_walk.cu' and lo <= o[1] <= hi)
    s = sum(o[3] for o in out if o[0] == 'km_walk.cu' and lo <= o[1] <= hi)
    print(f"{nm:24s} {lo:4d}-{hi:5d} {e / nb:7.1f}  stalls {100 * s / ts:5.1f}%")
other = {}
for o in out:
    if o[0] != 'km_walk.cu':
        a = other.setdefault(o[0], [0, 0]); a[0] += o[2]; a[1] += o[3]
for k, v in other.items():
    print(f"{k[:24]:24s} {'':10s} {v[0] / nb:7.1f}  stalls {100 * v[1] / ts:5.1f}%")
print("top lines")
for o in sorted(out, key=lambda o: -o[2])[:int(sys.argv[4]) if len(sys.argv) > 4 else 40]:
    print(f"{o[0][:10]:10s}:{o[1]:4d} {o[2] / nb:7.1f} st {100 * o[3] / ts:5.1f}%  {o[4].strip()[:80]}")
