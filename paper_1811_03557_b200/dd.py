"""DD driver: config 5's 8-octant domain decomposition and
the paper's two-subdomain Case-1 DD (NEXT-3; api.CaseOneSubdomain), which share the phase
ABI and the distributed least squares.

Each rank owns a set of subdomain contexts (one per GPU at 8 ranks; all on one GPU at N=1).
Subdomains may have different grids (Case 1: N1/N2 meshes): the global Δt takes the minimum of every
subdomain's CFL bound and 0.5 h_l^2 (R13).
Everything numerical runs in libdpm.so; this module only sequences the ABI calls and performs
the collectives of the distributed CholeskyQR2 / step:
  * C3-equivalent (once per dt): all-reduce(sum) of the K column norms and of two K x K Gram
    matrices;
  * C4 (per step): all-reduce(min) of the local CFL bounds (the global dt, R13);
  * C2 (per step): all-reduce(sum) of y_s = M_s g_s (K x 2) -> the global coefficients C.
Local contributions are summed in octant order before the cross-rank all-reduce.
"""
import os
from typing import Callable, List, Optional, Sequence

import torch
import torch.distributed as dist


def _allreduce(t: torch.Tensor, op) -> torch.Tensor:
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=op)
    return t


class DDSolver:
    def __init__(self, octants: Sequence, dt_cap: float, chi: float = 1.0, dt_rule: int = 0, clamp: int = 1):
        self.octs = list(octants)
        self.K = self.octs[0].K
        assert all(o.K == self.K for o in self.octs), "subdomains must share the global unknowns"
        self.h = min(o.info["h"] for o in self.octs)
        self.dt_cap, self.chi, self.dt_rule, self.clamp = dt_cap, chi, dt_rule, clamp
        self.dt_prev = float("inf")
        self.dt_bep: Optional[float] = None
        self.builds = 0
        self.t = 0.0
        self.fields: List = []
        # one CUDA stream per local octant: the octants' small kernels overlap on the GPU
        self.streams = [torch.cuda.Stream(o.device) if o.device.type == "cuda" else None for o in self.octs]

    # ---- global least squares (distributed CholeskyQR2) at dt
    def _sum(self, parts: List[torch.Tensor]) -> torch.Tensor:
        acc = parts[0].clone()
        for p in parts[1:]:
            acc += p
        return _allreduce(acc, dist.ReduceOp.SUM)

    def build(self, dt: float):
        # octants of one canonical geometry on one device: the first builds its block by K AP solves, the
        # others take it by column signs (B_s = B_0 diag(S_s), dpm_dd_bep_block_from); DPM_DD_SHARED=0 off
        ref = {}
        for o in self.octs:
            o.set_dt(dt)
            r = ref.get(str(o.device))
            if r is not None and self._shared_build():
                o.bep_block_from(r)
            else:
                o.bep_block()
                ref[str(o.device)] = o
        n2 = self._sum([o.colnorm2() for o in self.octs])
        G1 = self._sum([o.gram(1, n2) for o in self.octs])
        self._chol(1, G1)
        G2 = self._sum([o.gram(2) for o in self.octs])
        self._chol(2, G2)
        self.dt_bep = dt
        self.builds += 1

    def _chol(self, pass_, G):
        # every octant of this rank factors the same summed Gram: once per device, copied to the rest
        first = {}
        for o in self.octs:
            src = first.get(str(o.device))
            if src is None:
                o.chol(pass_, G)
                first[str(o.device)] = o
            else:
                o.chol_copy(pass_, src)

    def _batched(self):
        # several octants on one CUDA device with the phase-level entry points: the step's two AP
        # solves run as one batch of 2 x (octants) fields each (one dpm_aux_solve_batch)
        return (len(self.octs) > 1 and all(hasattr(o, "dd_rhs") for o in self.octs)
                and len({str(o.device) for o in self.octs}) == 1 and self.octs[0].device.type == "cuda"
                and len({(o.n, o.info["h"]) for o in self.octs}) == 1)   # one AP operator for all fields

    def _shared_build(self):
        # config-5 octants only (the Case-1 subdomains have different geometries)
        return (os.environ.get("DPM_DD_SHARED") != "0" and all(hasattr(o, "bep_block_from") for o in self.octs)
                and all(getattr(o, "octant", None) is not None and not hasattr(o, "sub") for o in self.octs))

    def _shared(self):
        # octants of config 5 (not the Case-1 subdomains): one canonical geometry, extensions that differ
        # by column signs only; DPM_DD_SHARED=0 applies every octant's own operator
        import os
        return (os.environ.get("DPM_DD_SHARED") != "0" and all(hasattr(o, "dd_lsq_rhs_shared") for o in self.octs)
                and all(getattr(o, "octant", None) is not None and not hasattr(o, "sub") for o in self.octs))

    def _step_batched(self, main):
        o0 = self.octs[0]
        nf = 2 * len(self.octs)
        if getattr(self, "_fq", None) is None or self._fq.shape[0] != nf:
            n = o0.n
            self._fq = torch.empty((nf, n, n, n), dtype=torch.float64, device=o0.device)
            self._wk = torch.empty_like(self._fq)
        fq, wk = self._fq, self._wk
        for i, (o, (rho, c)) in enumerate(zip(self.octs, self.fields)):   # Step 4a, per octant stream
            o.dd_rhs(rho, c, self.chi, fq[2 * i:2 * i + 2], stream=self.streams[i])
        for st in self.streams:
            main.wait_stream(st)
        o0.aux_solve_batch(fq, wk, stream=main)                        # all particular solves at once
        if self._shared():   # config 5: B_s = B_0 diag(S_s), one pass over octant 0's Q for all octants
            Cg = _allreduce(o0.dd_lsq_rhs_shared(self.octs, wk, stream=main), dist.ReduceOp.SUM)
        else:
            ys = []
            for i, o in enumerate(self.octs):
                self.streams[i].wait_stream(main)
                ys.append(o.dd_lsq_rhs(wk[2 * i:2 * i + 2], stream=self.streams[i]))
            for st in self.streams:
                main.wait_stream(st)
            Cg = self._sum(ys)                                        # C2: global coefficients
        if self._shared():   # config 5: one basis evaluation per γ point for all octants (A_s = A_0 diag(S_s)),
            o0.dd_green_rhs_shared(self.octs, Cg, self.clamp, fq, fq, stream=main)   # RHS formed in place in fq
            o0.aux_solve_batch(fq, wk, stream=main)                    # all Green solves at once
        else:
            for i, o in enumerate(self.octs):
                self.streams[i].wait_stream(main)
                o.dd_green_rhs(Cg, self.clamp, fq[2 * i:2 * i + 2], wk[2 * i:2 * i + 2], stream=self.streams[i])
            for st in self.streams:
                main.wait_stream(st)
            o0.aux_solve_batch(wk, wk, stream=main)                    # all Green solves at once
        for i, (o, (rho, c)) in enumerate(zip(self.octs, self.fields)):
            self.streams[i].wait_stream(main)
            o.dd_restrict(wk[2 * i:2 * i + 2], rho, c, stream=self.streams[i])
        return [o.stats(stream=self.streams[i]) for i, o in enumerate(self.octs)]

    def init(self, center, rho_ic, c_ic, rho_cell_average=0):
        self.fields = []
        for o in self.octs:
            n = o.n
            rho = torch.zeros((n, n, n), dtype=torch.float64, device=o.device)
            c = torch.zeros_like(rho)
            o.dd_pks_init(rho, c, center, *rho_ic, *c_ic, rho_cell_average=rho_cell_average)
            self.fields.append((rho, c))
        self.dt_prev, self.t = float("inf"), 0.0

    def _on(self, i):
        st = self.streams[i]
        return torch.cuda.stream(st) if st is not None else _Null()

    def step(self):
        main = torch.cuda.current_stream() if self.streams[0] is not None else None
        for st in self.streams:
            if st is not None:
                st.wait_stream(main)
        # Step 3 (R13) with the global CFL bound (C4)
        if self.dt_rule == 0:
            for i, (o, (_, c)) in enumerate(zip(self.octs, self.fields)):
                o.cfl_async(c, self.chi, stream=self.streams[i])
            # local min of every subdomain's CFL bound and 0.5 h_l^2, then the global min across ranks
            cfl = min(min(o.cfl_result(self.chi, stream=self.streams[i]), 0.5 * o.info["h"] ** 2)
                      for i, o in enumerate(self.octs))
            cfl = torch.tensor([cfl], dtype=torch.float64, device=self.octs[0].device)
            cfl = float(_allreduce(cfl, dist.ReduceOp.MIN).item())
            dt = min(min(self.dt_prev, self.dt_cap), cfl)
        else:
            dt = self.dt_cap
        rebuilt = self.dt_bep is None or dt != self.dt_bep
        if rebuilt:                                                   # Step 2 / 4b
            for st in self.streams:
                if st is not None:
                    st.synchronize()
            self.build(dt)
            for st in self.streams:
                if st is not None:
                    st.wait_stream(main)
        if self._batched():
            stats = self._step_batched(main)
        else:
            ys = [o.local_begin(rho, c, self.chi, stream=self.streams[i])
                  for i, (o, (rho, c)) in enumerate(zip(self.octs, self.fields))]
            for st in self.streams:
                if st is not None:
                    main.wait_stream(st)
            Cg = self._sum(ys)                                        # C2: global coefficients
            for i, (o, (rho, c)) in enumerate(zip(self.octs, self.fields)):
                if self.streams[i] is not None:
                    self.streams[i].wait_stream(main)
                o.local_finish_async(Cg, rho, c, self.clamp, stream=self.streams[i])
            stats = [o.stats(stream=self.streams[i]) for i, o in enumerate(self.octs)]
        for st in self.streams:
            if st is not None:
                main.wait_stream(st)
        self.dt_prev = dt
        self.t += dt
        mass = torch.tensor([sum(s["mass"] for s in stats)], dtype=torch.float64, device=self.octs[0].device)
        mass = float(_allreduce(mass, dist.ReduceOp.SUM).item())
        if any(s["nonfinite"] for s in stats):
            raise FloatingPointError("non-finite value in the DD PKS step")
        rmax = torch.tensor([max(s["rho_max"] for s in stats), max(s.get("rho_max_mplus", 0.0) for s in stats)],
                            dtype=torch.float64, device=self.octs[0].device)
        rmax = _allreduce(rmax, dist.ReduceOp.MAX)
        return {"t": self.t, "dt": dt, "rebuilt": rebuilt, "mass": mass,
                "rho_max": float(rmax[0]), "rho_max_mplus": float(rmax[1]),
                "rho_min": min(s["rho_min"] for s in stats),
                "per_subdomain": [dict(s) for s in stats]}


class _Null:
    def __enter__(self):
        return None

    def __exit__(self, *a):
        return False
