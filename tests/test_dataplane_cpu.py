"""CPU-side checks of the data plane: slab layout, plan roles, TP expansion,
the oracle's payload/fingerprint functions, and that libblitz.so loads and
exports every symbol include/blitz.h declares (no compute calls)."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

import paper_2412_17246_b200 as ss
from paper_2412_17246_b200 import slab as slabmod
from paper_2412_17246_b200._native import CUDA_LIB, HOST_LIB, exported_symbols
from paper_2412_17246_b200.dataplane import expand_tp, host_fed_groups, plan_roles, stripe_pieces
from oracle import dataplane_ref as ref

ROOT = Path(__file__).resolve().parent.parent


def _header_symbols(name):
    text = (ROOT / "include" / name).read_text()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(bz_\w+)\s*\(", text, re.M)))


def test_header_symbols_exported_by_cuda_lib():
    if not CUDA_LIB.exists():
        pytest.skip("libblitz.so not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(str(CUDA_LIB))
    names = _header_symbols("blitz.h")
    assert len(names) >= 25
    for n in names:
        assert hasattr(lib, n), n
    # the Python binding table covers the header exactly
    assert sorted(set(exported_symbols())) == names


def test_header_symbols_exported_by_host_lib():
    lib = ctypes.CDLL(str(HOST_LIB))
    for n in _header_symbols("blitz_plan.h"):
        assert hasattr(lib, n), n


def test_llama_byte_totals():
    # SURVEY.md §8d
    assert slabmod.LLAMA2_7B.block_bytes() == 404_766_720
    assert slabmod.LLAMA2_7B.total_bytes() == 13_476_831_232
    assert slabmod.LLAMA2_13B.block_bytes() == 634_408_960
    assert slabmod.LLAMA2_13B.total_bytes() == 26_031_728_640
    assert slabmod.LLAMA2_70B.block_bytes() == 1_711_308_800
    assert slabmod.TINY_4L.block_bytes() == 1_582_080
    assert slabmod.TINY_4L.total_bytes() == 39_096_832
    assert sum(slabmod.LLAMA2_7B.unit_bytes()) == 13_476_831_232


@pytest.mark.parametrize("tile", [256, 4096, 1 << 20])
def test_slab_layout_tiles_never_straddle_units(tile):
    lay = slabmod.SlabLayout.for_arch(slabmod.TINY_4L, tile_bytes=tile)
    assert lay.tile_off[0] == 0 and lay.tile_off[-1] == lay.data_bytes
    assert np.all(np.diff(lay.tile_off) > 0) and np.all(lay.tile_off % 16 == 0)
    assert np.all(np.diff(lay.tile_off) <= tile)
    for k in range(lay.num_layers):
        a, b = lay.tiles_of_layer(k)
        assert lay.tile_off[a] == lay.unit_off[k]
        end = lay.unit_off[k + 1] if k + 1 < lay.num_layers else lay.data_bytes
        assert lay.tile_off[b] == end
    assert lay.flag_offset >= lay.data_bytes and lay.total_bytes >= lay.flag_offset + 4 * lay.ntiles


def test_tp_layout_is_a_shard():
    full = slabmod.SlabLayout.for_arch(slabmod.LLAMA2_70B, tp=1)
    tp4 = slabmod.SlabLayout.for_arch(slabmod.LLAMA2_70B, tp=4)
    assert abs(tp4.payload_bytes() * 4 - full.payload_bytes()) < 4 * 256 * tp4.num_layers


def _b200_plan(n_targets, group=True, model=None):
    topo = ss.load_topology("b200-hgx")
    flows = ss.FlowSet(topo)
    model = model or slabmod.model_spec_for(slabmod.LLAMA2_7B)
    req = ss.build_scale_request(model, ["gpu0"], [f"gpu{i}" for i in range(1, n_targets + 1)],
                                 topo, flows)
    return ss.generate_plan(req, topo, flows, group=group)


def test_roles_1to8_grouped():
    plan = _b200_plan(7)
    roles = plan_roles(plan)
    assert roles["gpu0"].children == ["gpu1"] and roles["gpu0"].parent is None
    assert roles["gpu1"].parent == "gpu0" and roles["gpu1"].fanout == [f"gpu{i}" for i in range(2, 8)]
    assert all(roles[f"gpu{i}"].rep == "gpu1" and roles[f"gpu{i}"].receives for i in range(2, 8))


def test_roles_1to8_chain():
    plan = _b200_plan(7, group=False)
    roles = plan_roles(plan)
    assert plan.chains == [[f"gpu{i}" for i in range(8)]]
    for i in range(1, 8):
        assert roles[f"gpu{i}"].parent == f"gpu{i - 1}"


def test_expand_tp_c4():
    topo = ss.load_topology("b200-hgx")
    flows = ss.FlowSet(topo)
    model = slabmod.model_spec_for(slabmod.LLAMA2_13B, tp=2)
    req = ss.build_scale_request(model, ["gpu0"], ["gpu2", "gpu4", "gpu6"], topo, flows)
    plan = ss.generate_plan(req, topo, flows)
    per_rank = expand_tp(plan, 2)
    assert [(e.src, e.dst) for e in per_rank[1].edges] == [("gpu1", "gpu3")]
    assert per_rank[1].nvlink_fanout == {"gpu3": ["gpu5", "gpu7"]}


def test_host_fed_groups_only_for_pcie_fed_reps():
    topo = ss.load_topology("b200-hgx")
    flows = ss.FlowSet(topo)
    model = slabmod.model_spec_for(slabmod.LLAMA2_7B)
    req = ss.build_scale_request(model, ["mem0"], [f"gpu{i}" for i in range(4)], topo, flows)
    plan = ss.generate_plan(req, topo, flows)
    rep = next(iter(plan.nvlink_fanout))
    assert host_fed_groups(plan) == {rep: [rep] + plan.nvlink_fanout[rep]}
    # an NVLink-fed rep (1 -> 8 from a GPU) is not a host-fed group
    assert host_fed_groups(_b200_plan(7)) == {}
    # C5: every TP rank's group is host-fed
    model70 = slabmod.model_spec_for(slabmod.LLAMA2_70B, tp=4)
    req = ss.build_scale_request(model70, ["mem0"], ["gpu0", "gpu4"], topo, ss.FlowSet(topo))
    per_rank = expand_tp(ss.generate_plan(req, topo, ss.FlowSet(topo)), 4)
    assert [len(host_fed_groups(p)) for p in per_rank] == [1, 1, 1, 1]


@pytest.mark.parametrize("members", [1, 2, 3, 4, 8])
def test_stripe_pieces_partition_every_layer(members):
    lay = slabmod.SlabLayout.for_arch(slabmod.LLAMA2_7B, tile_bytes=1 << 20)
    pieces = [stripe_pieces(lay, members, i) for i in range(members)]
    seen = np.zeros(lay.ntiles, dtype=np.int32)
    for k in range(lay.num_layers):
        t0, t1 = lay.tiles_of_layer(k)
        bounds = [pieces[i][k] for i in range(members)]
        # contiguous, in member order, covering the layer exactly
        assert bounds[0][0] == t0 and bounds[-1][1] == t1
        assert all(bounds[i][1] == bounds[i + 1][0] for i in range(members - 1))
        # balanced to one tile
        sizes = [hi - lo for lo, hi in bounds]
        assert max(sizes) - min(sizes) <= 1
        for lo, hi in bounds:
            seen[lo:hi] += 1
    assert (seen == 1).all()
    with pytest.raises(ValueError):
        stripe_pieces(lay, members, members)


def test_oracle_payload_and_fingerprint_properties():
    buf = ref.random_words(1 << 14, seed=7)
    assert buf.dtype == np.uint8 and buf.size == 1 << 14
    again = ref.random_words(1 << 14, seed=7)
    assert np.array_equal(buf, again)
    tile_off = np.array([0, 4096, 8192, 16384], dtype=np.int64)
    fp = ref.tile_fingerprints(buf, tile_off)
    flipped = buf.copy()
    flipped[5000] ^= 1
    fp2 = ref.tile_fingerprints(flipped, tile_off)
    assert fp[0] == fp2[0] and fp[1] != fp2[1] and fp[2] == fp2[2]
    # position sensitivity: swapping two words inside a tile changes the print
    sw = buf.view(np.uint64).copy()
    sw[[0, 1]] = sw[[1, 0]]
    assert ref.tile_fingerprints(sw.view(np.uint8), tile_off)[0] != fp[0]


def test_cpu_plan_execution_copies_bytes():
    import torch

    plan = _b200_plan(3)
    lay = slabmod.SlabLayout.for_arch(slabmod.TINY_4L, tile_bytes=1 << 16)
    src = torch.from_numpy(ref.random_words(lay.data_bytes, 3).copy())
    bufs = {"gpu0": src}
    for i in range(1, 4):
        bufs[f"gpu{i}"] = torch.zeros_like(src)
    bounds = [(lay.unit_off[k], lay.unit_off[k] + lay.unit_bytes[k]) for k in range(lay.num_layers)]
    done = ref.execute_plan_cpu(plan, bufs, bounds)
    assert set(done) == {"gpu1", "gpu2", "gpu3"}
    for i in range(1, 4):
        assert torch.equal(bufs[f"gpu{i}"], src)


def test_max_dst_matches_header():
    from paper_2412_17246_b200.dataplane import MAX_DST
    text = (ROOT / "include" / "blitz.h").read_text()
    assert int(re.search(r"#define BZ_MAX_DST (\d+)", text).group(1)) == MAX_DST


class _HopRules:
    """The ScaleExecutor's hop-realisation rules without a GPU (its helper methods only)."""

    def __new__(cls, plan, engine, fanout_mode="chain"):
        from paper_2412_17246_b200.dataplane import ScaleExecutor

        class Probe(ScaleExecutor):
            def __init__(self):  # no slabs, no fabric: just the inputs of the rules
                self.plan, self.roles, self.engine = plan, plan_roles(plan), engine
                self.fanout_mode, self.stripe_groups, self.writers = fanout_mode, {}, {}
                self.node = None

        return Probe()


@pytest.mark.parametrize("n_targets,pulled", [
    (1, {"gpu1": "gpu0"}),           # 1 -> 2: the single source -> leaf hop is pulled
    (3, {}),                         # 1 -> 4 grouped: gpu1 relays, every hop pushed
    (7, {}),                         # 1 -> 8 grouped: a 7-hop relay chain, pushed
])
def test_auto_engine_pulls_only_source_to_leaf_hops(n_targets, pulled):
    from paper_2412_17246_b200.dataplane import ENGINE_AUTO, ENGINE_VECTOR
    plan = _b200_plan(n_targets)
    rules = _HopRules(plan, ENGINE_AUTO)
    got = {n: rules._pull_source_of(n) for n in rules.roles if rules._pull_source_of(n) is not None}
    assert got == pulled
    # every receiver is fed by exactly one mover: a pull, or a push from its sender
    for n, r in rules.roles.items():
        if not r.receives or not n.startswith("gpu"):
            continue
        pushers = [s for s in rules.roles if n in rules._targets_for(s) and not rules._pulled(s, n)]
        assert len(pushers) + (n in got) == 1, (n, pushers)
    # an explicit SM engine never pulls
    assert all(_HopRules(plan, ENGINE_VECTOR)._pull_source_of(n) is None for n in rules.roles)


def test_auto_engine_pulls_each_tp_rank_group_hop():
    """C4's shape at 4 GPUs: 13B TP=2, 1 -> 2 instances: each rank's hop gpu<r> -> gpu<2+r>
    is a source -> leaf hop, pulled by the new rank."""
    from paper_2412_17246_b200.dataplane import ENGINE_AUTO, merge_plans
    topo = ss.load_topology("b200-hgx")
    flows = ss.FlowSet(topo)
    model = slabmod.model_spec_for(slabmod.LLAMA2_13B, tp=2)
    req = ss.build_scale_request(model, ["gpu0"], ["gpu2"], topo, flows)
    plan = merge_plans(expand_tp(ss.generate_plan(req, topo, flows), 2))
    rules = _HopRules(plan, ENGINE_AUTO)
    assert {n: rules._pull_source_of(n) for n in ("gpu2", "gpu3")} == {"gpu2": "gpu0", "gpu3": "gpu1"}
