"""Rebinding the reference package (`cmbproj`) onto this library — the shim of INTEGRATION.md.

The reference has no FFI or plugin registry: its callers reach the engines through
module-level names (`harness.py:19-21` import `gamma2d_matrix` / `gamma3d_matrix`, and the
reference's own tests swap engines by rebinding them, `test_harness.py:274-281`).  `install`
rebinds exactly those names to wrappers with the reference's signatures
(`engine3d.py:156-160`, `engine2d.py:187-191`) that call the GPU drop-ins and return the
reference's own `GammaMatrix` class; `uninstall` restores the originals.

    import cmbproj, paper_1503_08809_b200.integration as b200
    b200.install(cmbproj)          # cmbproj.harness.run_gamma(...) now runs on the GPU
"""

from __future__ import annotations

import importlib

__all__ = ["install", "uninstall", "gamma3d_matrix_shim", "gamma2d_matrix_shim",
           "build_ptable_shim"]

# (module, attribute) pairs the reference binds the two engines to
_SITES_3D = (("", "gamma3d_matrix"), (".engine3d", "gamma3d_matrix"),
             (".harness", "gamma3d_matrix"))
_SITES_2D = (("", "gamma2d_matrix"), (".engine2d", "gamma2d_matrix"),
             (".harness", "gamma2d_matrix"))
# build_ptable (engine2d.py:62-95) is public too; gamma2d_matrix calls it through its module
_SITES_PT = (("", "build_ptable"), (".engine2d", "build_ptable"))


def _gm_class(cp):
    return importlib.import_module(cp.__name__ + ".gamma").GammaMatrix


def gamma3d_matrix_shim(cp):
    """A gamma3d_matrix with the reference signature, backed by the GPU drop-in."""
    from .engine3d import gamma3d_matrix as b200_gamma3d

    GM = _gm_class(cp)

    def gamma3d_matrix(tables, mapping, grid, h2_mode="gosper", integrator="trap", block=64,
                       workers=1, domain=None):
        g = b200_gamma3d(tables, mapping, grid, h2_mode=h2_mode, integrator=integrator,
                         block=block, workers=workers, domain=domain)
        return GM(g.values, g.meta)
    gamma3d_matrix.__wrapped_b200__ = True
    return gamma3d_matrix


def gamma2d_matrix_shim(cp):
    """A gamma2d_matrix with the reference signature, backed by the GPU μ-engine."""
    from .engine2d import gamma2d_matrix as b200_gamma2d

    GM = _gm_class(cp)

    def gamma2d_matrix(tables, mapping, grid, rule, legendre, integrator="trap", workers=1,
                       ptable=None):
        if ptable is not None:          # a reference PTable: same .values layout [a,b,x,m]
            from .engine2d import PTable
            ptable = PTable(ptable.values)
        g = b200_gamma2d(tables, mapping, grid, rule, legendre, integrator=integrator,
                         workers=workers, ptable=ptable)
        return GM(g.values, g.meta)
    gamma2d_matrix.__wrapped_b200__ = True
    return gamma2d_matrix


def build_ptable_shim(cp):
    """A build_ptable with the reference signature (engine2d.py:62-64): the table is built on
    the GPU (bit-identical) and returned as the reference's own PTable class."""
    from .engine2d import DEFAULT_PTABLE_BUDGET, build_ptable as b200_build_ptable

    PT = importlib.import_module(cp.__name__ + ".engine2d").PTable

    def build_ptable(tables, grid, rule, legendre, budget_bytes=DEFAULT_PTABLE_BUDGET):
        return PT(b200_build_ptable(tables, grid, rule, legendre, budget_bytes).values)
    build_ptable.__wrapped_b200__ = True
    return build_ptable


def install(cp, engines=("3d", "2d"), setattr_fn=setattr):
    """Rebind the reference's engine names; returns the originals for `uninstall`.
    `setattr_fn` may be pytest's monkeypatch.setattr (automatic restore)."""
    saved = []
    for tag, sites, make in (("3d", _SITES_3D, gamma3d_matrix_shim),
                             ("2d", _SITES_2D, gamma2d_matrix_shim),
                             ("2d", _SITES_PT, build_ptable_shim)):
        if tag not in engines:
            continue
        fn = make(cp)
        for mod, attr in sites:
            m = importlib.import_module(cp.__name__ + mod) if mod else cp
            saved.append((m, attr, getattr(m, attr)))
            setattr_fn(m, attr, fn)
    return saved


def uninstall(saved) -> None:
    for m, attr, fn in reversed(saved):
        setattr(m, attr, fn)
