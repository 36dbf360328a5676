"""Summarise an inverse task timeline (scripts/micro/inv_trace output): per step, when the panels,
the fused pivot and the tiles ran; per CTA, work vs wait time."""
import sys, collections
rows = [list(map(int, l.split())) for l in open(sys.argv[1]) if l.strip()]
t0 = min(r[6] for r in rows)
steps = collections.defaultdict(list)
for g, k, kind, I, J, sm, a, b, c, *_ in rows:
    steps[k].append((kind, I, J, (a - t0) / 1e3, (b - t0) / 1e3, (c - t0) / 1e3))
print("step  panels[start..end]   pivot-tile[start..end]   tiles[first start..last end]  (us)")
for k in sorted(steps):
    P = [x for x in steps[k] if x[0] == 0]
    V = [x for x in steps[k] if x[0] in (2, 5)]
    T = [x for x in steps[k] if x[0] == 1]
    f = lambda L: f"{min(x[4] for x in L):8.1f}..{max(x[5] for x in L):8.1f}" if L else " " * 18
    print(f"{k:4d}  {f(P)}  {f(V)}  {f(T)}")
work = sum(r[8] - r[7] for r in rows) / 1e3
wait = sum(r[7] - r[6] for r in rows) / 1e3
end = (max(r[8] for r in rows) - t0) / 1e3
ncta = len(set(r[5] for r in rows))
print(f"total {end:.1f} us, CTAs {ncta}, work {work/ncta:.1f} us/CTA, wait {wait/ncta:.1f} us/CTA")
kinds = collections.defaultdict(list)
for r in rows:
    kinds[r[2]].append((r[8] - r[7]) / 1e3)
for kd, L in sorted(kinds.items()):
    print(f"kind {kd}: n={len(L)} mean {sum(L)/len(L):.1f} us, max {max(L):.1f}")
# update tasks with sub-phase stamps (INV_TRACE builds of the current kernel): start -> product
# end -> C-tile wait end -> task end
for kd in (0, 1, 3, 5):
    sub = [r for r in rows if r[2] == kd and len(r) >= 11 and r[9] >= r[7] and r[10] >= r[9] and r[8] >= r[10]]
    if sub:
        n = len(sub)
        pr = sum(r[9] - r[7] for r in sub) / n / 1e3
        cw = sum(r[10] - r[9] for r in sub) / n / 1e3
        ep = sum(r[8] - r[10] for r in sub) / n / 1e3
        print(f"kind {kd} phases: product {pr:.1f} us, C wait {cw:.1f} us, epilogue+flags {ep:.1f} us (n={n})")
# panel (kind 0) phases: deps -> R_J staged -> R_J digits out -> passes done -> Wp_J staged -> Wp_J digits -> end
sub = [r for r in rows if r[2] == 0 and len(r) >= 15 and r[11] >= r[7] and r[9] >= r[11] and r[10] >= r[9]
       and r[12] >= r[10] and r[13] >= r[12] and r[8] >= r[13]]
if sub:
    n = len(sub)
    ph = [(r[11] - r[7], r[9] - r[11], r[10] - r[9], r[12] - r[10], r[13] - r[12], r[8] - r[13]) for r in sub]
    names = ["stage R_J", "slice R_J", "passes", "stage Wp_J", "slice Wp_J", "W tile + flags"]
    print("kind 0 detail: " + ", ".join(f"{nm} {sum(p[i] for p in ph) / n / 1e3:.1f} us" for i, nm in enumerate(names)) + f" (n={n})")
# chain (kind 5) epilogue: passes end (sub0 is the panel's) ... sub2 RMW done, sub1 pflag wait done,
# sub3 pivot done, sub4 P digits done, end
sub = [r for r in rows if r[2] == 5 and len(r) >= 15 and r[11] <= r[10] <= r[12] <= r[13] <= r[8]]
if sub:
    n = len(sub)
    ph = [(r[10] - r[11], r[12] - r[10], r[13] - r[12], r[8] - r[13]) for r in sub]
    names = ["pflag wait", "pivot 128^2", "P digits", "flags"]
    print("kind 5 epilogue detail: " + ", ".join(f"{nm} {sum(p[i] for p in ph) / n / 1e3:.1f} us" for i, nm in enumerate(names)) + f" (n={n})")
# utilisation over time: fraction of CTAs busy (work phase) per 5% of the kernel
T = max(r[8] for r in rows) - t0
bins = [0.0] * 20
for r in rows:
    a, b = r[7] - t0, r[8] - t0
    for q in range(20):
        lo, hi = q * T / 20, (q + 1) * T / 20
        bins[q] += max(0, min(b, hi) - max(a, lo))
ncta = len(set(r[5] for r in rows))
print("busy by 5% slice:", " ".join(f"{b / (T / 20 * ncta) * 100:.0f}" for b in bins))
