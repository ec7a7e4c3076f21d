"""Per-phase clock64 totals of the dense-window cycle kernel (instrumented build):
make -C paper_1608_05138_b200/csrc prof && GRAPHLET_B200_LIB=libgraphlet_b200_prof.so python scripts/cycle_phases.py [scale]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("GRAPHLET_B200_LIB", "libgraphlet_b200_prof.so")
import paper_1608_05138_b200 as gl  # noqa: E402

arg = sys.argv[1] if len(sys.argv) > 1 else "20"
if arg == "ba":  # configs[2]: Barabasi-Albert 4M vertices / 64M edges
    g = gl.Graph.build(gl.generate_ba(4_000_000, 16, seed=1))
else:
    g = gl.Graph.build(gl.generate_rmat(int(arg), 16, seed=1))
def run():
    try:
        g.count()
    except gl.GraphletError as e:  # timing experiments may break the counts on purpose
        print("count error (ignored for timing):", e)


run()
buf = (C.c_ulonglong * 64)()
gl.LIB.gl_debug_cycle_profile(buf, 1)
run()
gl.LIB.gl_debug_cycle_profile(buf, 0)
names = ["setup", "scan", "compaction", "pass0", "pass1", "grab", "gallop", "clear"]
for base, kind in ((0, "dense windows"), (16, "mid hash")):
    tot = max(1, sum(buf[base:base + 8]))
    print(f"== {kind}: {tot / 1e9:.2f} Gcyc summed over blocks")
    for i, nm in enumerate(names):
        if i == 8:
            break
        print(f"  {nm:12s} {buf[base + i] / 1e6:10.1f} Mcyc  {100 * buf[base + i] / tot:5.1f}%")
    if base == 0:
        print(f"  pass-1 rounds: uniform {buf[12]}  mixed {buf[13]}")
        print(f"  runs {buf[11]}  windows with global run metadata {buf[14]} ({buf[15]} wedges)")
    w, T, tops = buf[base + 8], buf[base + 9], buf[base + 10]
    print(f"  windows {w}  wedges {T}  tops {tops}  wedges/window {T / max(1, w):.0f}")
print(f"windowed-hash (sparse big) windows {buf[30]}  wedges {buf[31]}  re-cuts {buf[29]}")
print("dense windows per counter tier (bits: windows, runs, wedges, wedges/run):")
for cl in range(5):
    w, r, T = buf[32 + 4 * cl], buf[33 + 4 * cl], buf[34 + 4 * cl]
    print(f"  {32 >> cl:2d}-bit  {w:10d} {r:14d} {T:16d} {T / max(1, r):8.1f}")
ms, _, _ = g.last_stats()
print("phase ms (last count):", ms)
pc = g.cycle_pieces()
print(f"cycle pieces {len(pc)} from {len(set(pc[:, 0].tolist()))} windowed tops; max estimate {pc[:, 3].max() if len(pc) else 0}")
