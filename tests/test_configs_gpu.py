"""BASELINE configs 3-5 scenarios against the fp32 oracle (GPU).

The config scripts (scripts/config3_replication.py, config4_migration.py,
config5_70b_sharded.py) measure on random-init 32-80 layer models; their
parity leg rebuilds each geometry with two decoder layers of oracle weights
and applies the same ops through the executor API (scripts/_oracle_check.py).
These tests run those same scenarios inside the pytest GPU suite so a
regression shows up in ``pytest -m gpu``, not only in a script's JSON:
  - config 3: Llama-2-7B geometry, hot layer replicated on a second device
    before serving, sequences finishing mid-decode (ops.py:188-211);
  - config 4: Llama-2-13B geometry, one synchronous and one issued/committed
    MigrateLayer with KV mid-decode (ops.py:213-228; sim.py:396-403);
  - config 5: Llama-2-70B geometry (GQA 64/8), layers on two devices and the
    controller's gate-projection MigrateSubModule (ops.py:230-247).
Bars (north star): max-abs logit error <= 2e-2 and greedy tokens identical
wherever the oracle's top-2 margin exceeds 4e-2.
"""
from __future__ import annotations

import sys
from pathlib import Path

import pytest

from paper_2507_18006_b200 import domain as D
from paper_2507_18006_b200 import ops as O

sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "scripts"))
from _oracle_check import check  # noqa: E402

pytestmark = pytest.mark.gpu


def test_config3_replicated_hot_layer(cuda):
    def scenario(ex, cat, cluster, step):
        if step == 0:
            ex.apply(O.ReplicateLayer(1, 1), cat, cluster)

    res = check(dict(d_model=4096, d_ff=11008, n_heads=32), 2, 48, 64, 6, scenario,
                release={2: [0, 7, 30], 4: [11, 12, 13, 47]})
    assert res["placement_layers_1_2"][0] == [0, 1]
    assert res["confident_decisions"] > 0


def test_config4_migration_sync_and_async(cuda):
    def scenario(ex, cat, cluster, step):
        if step == 2:
            ex.apply(O.MigrateLayer(1, 1, with_kv=True), cat, cluster)
        if step == 3:
            ex.issue(O.MigrateLayer(2, 1, with_kv=True), cat, cluster)
        if step == 4:
            ex.commit(wait=True)

    res = check(dict(d_model=5120, d_ff=13824, n_heads=40), 2, 24, 48, 6, scenario, release={3: [5, 6]})
    assert res["placement_layers_1_2"] == [[1], [1]]


def test_config5_gqa_sharded_submodule_migration(cuda):
    def scenario(ex, cat, cluster, step):
        if step == 2:
            ex.apply(O.MigrateSubModule(2, D.ModuleKind.FFN_PROJ_GATE, 0), cat, cluster)

    res = check(dict(d_model=8192, d_ff=28672, n_heads=64, n_kv_heads=8), 2, 8, 32, 5, scenario,
                device_of_layer=lambda li: li - 1)
    assert res["placement_layers_1_2"] == [[0], [1]]
