"""Patch-sharded execution of the oracle (full-size C5) -- oracle.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The same algorithm as ``oracle.ieti.IetiOracle``: ``ShardedIetiOracle`` IS an IetiOracle whose
dual PCG, B / B_D applications, coarse problem (S_PiPi) and recovery are the inherited
methods, unchanged.  Only the three patch-local hooks (``_local_t``: Phibar^T r; ``_local_w``: the
projected local Neumann solve and interface result, App. A.1; ``_local_msd``: the local Schur
action of M_sD) run in worker processes, each holding whole patches, built exactly as
IetiOracle builds them (one single-patch IetiOracle per patch: a block-diagonal hierarchy's
V-cycle acts block by block, so per-patch hierarchies compute the same numbers; checked bitwise
against IetiOracle in tests/test_oracle_sharded.py).  Patches are independent inside every
operator, so the split changes no arithmetic.

Used by tools/oracle_dump.py for C5 (256 patches of 42,875 dofs: ~0.5 GB of hierarchies per patch,
more than one process's memory and hours of one core), with the 'pcg' primal-basis route
 because a C5 patch's KKT LU does not fit.
"""
from __future__ import annotations

import gc
import multiprocessing as mp
import os
import resource
from typing import Dict, List, Optional

import numpy as np

from .ieti import IetiOracle
from .topology import Topology


def _worker(conn, wl, topo, ids, okw, mem_gb):
    if mem_gb:
        lim = int(mem_gb * 2 ** 30)
        resource.setrlimit(resource.RLIMIT_AS, (lim, lim))       # a MemoryError, never the OOM killer
    try:
        pat: Dict[int, IetiOracle] = {}
        for k in ids:
            pat[k] = IetiOracle(wl, ids=[k], topo=topo, lean=True, **okw)
            gc.collect()
        conn.send(("ready", {k: (o.S_loc[k], o.f[k]) for k, o in pat.items()}))
        n = topo.n_patches
        while True:
            cmd, payload = conn.recv()
            if cmd == "quit":
                break
            out = {}
            for k, o in pat.items():
                if cmd == "t":
                    r = [None] * n
                    r[k] = payload[k]
                    out[k] = o._local_t(r)[k]
                elif cmd == "w":
                    rl, tl, uPi = payload
                    r, t = [None] * n, [None] * n
                    r[k], t[k] = rl[k], tl[k]
                    out[k] = o._local_w(r, t, uPi)[k]
                elif cmd == "msd":
                    v = [None] * n
                    v[k] = payload[k]
                    out[k] = o._local_msd(v)[k]
            conn.send(("ok", out))
    except BaseException as e:                                   # surfaced by the master
        conn.send(("error", repr(e)))
    finally:
        conn.close()


class ShardedIetiOracle(IetiOracle):
    def __init__(self, wl, workers: int = 4, mem_gb_per_worker: Optional[float] = None,
                 topo: Optional[Topology] = None, **okw):
        okw.setdefault("basis", "pcg")
        neumann = okw.get("neumann") or {0: "vcycle", 1: "pcg", 2: "exact"}[wl.local_mode]
        if neumann != "vcycle":
            raise ValueError("the sharded oracle covers the fixed-cycle (vcycle) modes")
        topo = Topology(wl.patches, wl.primal) if topo is None else topo
        # the master: global topology and options, no patches
        super().__init__(wl, ids=[], topo=topo, **okw)
        n = topo.n_patches
        shards = [list(range(n))[w::workers] for w in range(workers)]
        shards = [s for s in shards if s]
        ctx = mp.get_context("fork")
        gc.freeze()                     # forked children share the topology pages (no refcount copies)
        self._conns, self._procs, self._owner = [], [], {}
        for w, ids in enumerate(shards):
            a, b = ctx.Pipe()
            p = ctx.Process(target=_worker, args=(b, wl, topo, ids, okw, mem_gb_per_worker), daemon=True)
            p.start()
            b.close()
            self._conns.append(a)
            self._procs.append(p)
            for k in ids:
                self._owner[k] = w
        S_loc, f = [None] * n, [None] * n
        for msg in self._recv_all():
            for k, (S, fk) in msg.items():
                S_loc[k], f[k] = S, fk
        self.S_loc, self.f = S_loc, f
        self.set_coarse(S_loc)

    def _recv_all(self):
        outs = []
        for c in self._conns:
            tag, msg = c.recv()
            if tag == "error":
                self.close()
                raise RuntimeError(f"oracle worker failed: {msg}")
            outs.append(msg)
        return outs

    def _scatter(self, cmd, per_patch: List, extra=None):
        for w, c in enumerate(self._conns):
            part = {k: per_patch[k] for k, o in self._owner.items() if o == w}
            c.send((cmd, part if extra is None else (part,) + extra))
        out = [None] * self.topo.n_patches
        for msg in self._recv_all():
            for k, v in msg.items():
                out[k] = v
        return out

    # the three patch-local hooks, dispatched to the workers
    def _local_t(self, r_list):
        return self._scatter("t", r_list)

    def _local_w(self, r_list, t, uPi):
        n = self.topo.n_patches
        for w, c in enumerate(self._conns):
            ks = [k for k, o in self._owner.items() if o == w]
            c.send(("w", ({k: r_list[k] for k in ks}, {k: t[k] for k in ks}, uPi)))
        out = [None] * n
        for msg in self._recv_all():
            for k, v in msg.items():
                out[k] = v
        return out

    def _local_msd(self, vG):
        return self._scatter("msd", vG)

    def close(self):
        for c in getattr(self, "_conns", []):
            try:
                c.send(("quit", None))
            except (OSError, BrokenPipeError):
                pass
        for p in getattr(self, "_procs", []):
            p.join(timeout=30)
        self._conns, self._procs = [], []

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
