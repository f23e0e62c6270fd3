"""CPU, world_size 2 over gloo: the multi-GPU host logic (l2-slab shard plan, per-rank
partial, all-gather + rank-order merge) with the per-rank kernel replaced by the oracle's
slab partial.  Mirrors the reference's worker-count invariance tests
(test_engine3d.py:58-62, test_acceptance.py criterion 7)."""

import os
import socket
import subprocess
import sys
import textwrap

import numpy as np
import pytest

from conftest import ROOT

WORKER = textwrap.dedent(r"""
    import os, sys
    sys.path.insert(0, os.environ["ROOT"])
    import numpy as np
    import torch.distributed as dist
    from oracle import ref
    import paper_1503_08809_b200 as mg
    from paper_1503_08809_b200.dist import gamma3d_matrix_distributed

    g = np.load(os.path.join(os.environ["ROOT"], "tests/golden/desk.npz"))
    lmin, lmax = (int(x) for x in g["desk32_lrange"])
    t = mg.BasisTables(g["desk32_q"], g["desk32_qt"], g["desk32_C"], g["desk32_v"], lmin, lmax)
    m = mg.ModeMapping(g["desk32_entries"], 4)
    r = mg.RadialGrid(g["desk32_r"])
    seen = []

    def oracle_slab(tables, mapping, wr2, a, b, h2_mode):
        l1, l2, l3 = ref.domain_triples(tables.l_min, tables.l_max)
        keep = (l2 >= a) & (l2 < b)
        seen.append((a, b, int(keep.sum())))
        return ref.sweep_triples(tables.q, tables.q_tilde, tables.C, tables.v, wr2,
                                 mapping.entries, tables.l_min, l1[keep], l2[keep], l3[keep])

    dist.init_process_group("gloo")
    out = gamma3d_matrix_distributed(t, m, r, partial_fn=oracle_slab)
    rank = dist.get_rank()
    np.save(os.path.join(os.environ["OUT"], f"gamma_{rank}.npy"), out.values)
    np.save(os.path.join(os.environ["OUT"], f"slab_{rank}.npy"), np.array(seen[0]))
    assert out.meta["ranks"] == 2 and out.meta["engine"] == "modal3d"
    dist.destroy_process_group()
""")


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.timeout(300)
def test_two_ranks_gloo(tmp_path, g_desk):
    script = tmp_path / "worker.py"
    script.write_text(WORKER)
    env = dict(os.environ, ROOT=ROOT, OUT=str(tmp_path), MASTER_ADDR="127.0.0.1",
               MASTER_PORT=str(free_port()), WORLD_SIZE="2")
    procs = [subprocess.Popen([sys.executable, str(script)], env=dict(env, RANK=str(r),
                                                                        LOCAL_RANK=str(r)))
             for r in range(2)]
    assert all(p.wait(timeout=280) == 0 for p in procs)
    g0 = np.load(tmp_path / "gamma_0.npy")
    g1 = np.load(tmp_path / "gamma_1.npy")
    assert np.array_equal(g0, g1)                      # every rank returns the same Γ
    want = g_desk["desk32_gamma"]
    assert np.max(np.abs(g0 - want)) / np.max(np.abs(want)) < 1e-12
    s0, s1 = np.load(tmp_path / "slab_0.npy"), np.load(tmp_path / "slab_1.npy")
    assert s0[0] == 2 and s0[1] == s1[0] and s1[1] == 33   # contiguous cover of l2
    assert s0[2] > 0 and s1[2] > 0
