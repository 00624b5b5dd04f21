"""Resident multi-step driver: the state stays on the lattice in HBM, each
step is the fused five-kernel schedule, optionally replayed as a CUDA graph.
This is what ``cli.run_simulation``'s hot loop (cli.py:224-241) becomes."""
from __future__ import annotations

from . import imexcore
from .plan import tableau_array


class HeviStepper:
    def __init__(self, disc, ref, dt, tableau=None, check_every=1, set_name="set2nc"):
        self.plan = disc.plan_for(ref, set_name)
        self.tableau = tableau or imexcore.ark2_tableau()
        self.tab = tableau_array(self.tableau)
        self.dt = float(dt)
        self.lam = self.tableau.diag * self.dt
        self.nb = self.plan.factor(self.lam)
        self.Q = self.plan.zeros()
        self.work = self.plan.workspace()
        self.check_every = check_every
        self.steps = 0
        self._graph = None
        # P'(Q) chained from each step's stage 2 into the next stage 0
        # (hevi_ark2_step_ex); refreshed whenever the state is replaced
        self._chain = self.plan.chains_pp
        self.plan.pp_refresh(self.Q, self.work)

    # state in / out ---------------------------------------------------------
    def set_state(self, q, lattice=False):
        if lattice:
            self.Q[:, :, :, :q.shape[-1]].copy_(q)
        else:
            from .plan import to_device
            E, _ = to_device(q)
            self.plan.e2l(E, out=self.Q)
        self.plan.pp_refresh(self.Q, self.work)

    def state(self, lattice=False):
        if lattice:
            return self.Q[:, :, :, :self.plan.lX]
        return self.plan.l2e(self.Q)

    # stepping ---------------------------------------------------------------
    def _launch(self):
        self.plan.step(self.dt, self.tab, self.Q, self.work, pp_valid=self._chain)

    def capture(self):
        """Record one step as a CUDA graph.  The warm-up step that sets the
        kernels' shared-memory attributes outside the capture is a real step:
        it is counted and its flags are checked."""
        import torch
        self._launch()
        self.steps += 1
        self.plan.check_flags()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self._launch()
        self._graph = g
        return g

    def step(self, n=1, check=True):
        for _ in range(n):
            if self._graph is not None:
                self._graph.replay()
            else:
                self._launch()
            self.steps += 1
            if check and self.check_every and self.steps % self.check_every == 0:
                self.plan.check_flags()
