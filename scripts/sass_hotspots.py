"""Top SASS lines by stall samples for kernels in an ncu report (source page).

    python scripts/sass_hotspots.py REPORT.ncu-rep NCU_REGEX [N] [SUBSTRING]

NCU_REGEX filters kernels in ncu; SUBSTRING (optional) picks the first launch
whose demangled name contains it (e.g. "(int)2, (int)4").
"""
import csv, io, subprocess, sys

rep, rx = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "--kernel-name", f"regex:{rx}"], capture_output=True, text=True).stdout
sub = sys.argv[4] if len(sys.argv) > 4 else ""
sections = [x for x in raw.split('"Kernel Name",')[1:] if sub in x.split("\n", 1)[0]]
for sec in sections[:1]:  # first matching launch
    name, body = sec.split("\n", 1)
    rows = list(csv.DictReader(io.StringIO(body)))
    tot_s = sum(int(r["Warp Stall Sampling (All Samples)"] or 0) for r in rows)
    tot_i = sum(int(r["Instructions Executed"] or 0) for r in rows)
    print(name[:120])
    print(f"instructions executed (warp-level): {tot_i}, stall samples: {tot_s}, SASS lines: {len(rows)}")
    top = sorted(rows, key=lambda r: -int(r["Warp Stall Sampling (All Samples)"] or 0))[:n]
    for r in top:
        print(f'{int(r["Warp Stall Sampling (All Samples)"] or 0):6d} {int(r["Instructions Executed"] or 0):9d}  {r["Source"].strip()[:90]}')
