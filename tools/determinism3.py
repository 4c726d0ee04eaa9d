"""Determinism probe 3: dump / compare the finest Dirichlet stencils (dev tool)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
mode, path = sys.argv[1], sys.argv[2]
if mode == "dump":
    import paper_1705_04531_b200 as lib
    from workloads import make_workload
    wl = make_workload("C3")
    ie = lib.Ieti.from_workload(wl)
    L = ie.levels - 1
    np.save(path, np.stack([ie.stencil(1, L, k) for k in range(ie.n_patches)]))
    np.save(path + ".N.npy", np.stack([ie.stencil(0, L, k) for k in range(ie.n_patches)]))
else:
    a, b = np.load(path), np.load(sys.argv[3])
    d = np.abs(a - b)
    print("shape", a.shape, "max diff", d.max(), "n diff", int((d > 0).sum()))
    idx = np.argwhere(d > 0)
    pats = sorted(set(int(i[0]) for i in idx))
    print("patches with diffs", pats[:40], len(pats))
    for i in idx[:12]:
        k, r, o = (int(v) for v in i)
        print("patch", k, "row", r, "off", o, a[k, r, o], b[k, r, o])
    rows = sorted(set((int(i[0]), int(i[1])) for i in idx))
    print("rows with diffs", len(rows), rows[:20])
    offs = sorted(set(int(i[2]) for i in idx))
    print("offsets with diffs", offs)
