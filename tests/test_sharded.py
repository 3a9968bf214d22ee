"""Row partition (multi-GPU path, paper_2408_04343_b200/sharded.py).

CPU: the exchange protocol -- partition rule, exchange-space renumbering,
per-rank flags, halting agreement -- run by 2 gloo processes with a numpy
emulation of each rank's step, against the unsharded oracle.
GPU: 2 and 3 row-partitioned engines on one B200 with an emulated all-gather,
bit-identical to the single engine.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2408_04343_b200 as snp
from paper_2408_04343_b200 import sharded as shd
from conftest import corpus_system
from oracle import coracle
from oracle.snp_oracle import OracleSystem


# -- partition rule ------------------------------------------------------------------------

@pytest.mark.parametrize("q,world", [(1, 2), (1000, 3), (10**7, 8), (12288, 8), (129, 2)])
def test_layout_covers_all_rows(q, world):
    L = shd.shard_layout(q, world)
    assert L.nl % 128 == 0
    bounds = [L.bounds(r) for r in range(world)]
    assert bounds[0][0] == 0 and bounds[-1][1] == q
    for (a, b), (c, d) in zip(bounds, bounds[1:]):
        assert b == c and a <= b
    src = np.arange(q)
    x = L.xpos(src)
    assert (np.diff(x) > 0).all()                       # order preserved (sorted segments stay sorted)
    assert ((x % (L.nl + 128)) < L.nl).all()            # never lands in a header


def test_decide_halt_rule():
    assert shd.decide_halt(np.array([[0, 0, 0], [0, 0, 0]]), last=True) is snp.HaltReason.STEP_LIMIT
    assert shd.decide_halt(np.array([[0, 0, 1], [0, 0, 0]]), last=True) == "negative"
    assert shd.decide_halt(np.array([[0, 0, 0], [0, 0, 0]])) is snp.HaltReason.NO_APPLICABLE_RULES
    assert shd.decide_halt(np.array([[0, 1, 0], [0, 0, 0]])) is None
    assert shd.decide_halt(np.array([[1, 0, 0], [0, 0, 0]])) is None
    assert shd.decide_halt(np.array([[1, 0, 0], [0, 0, 1]])) == "negative"


# -- protocol over gloo (CPU) ----------------------------------------------------------------

def _emulated_rank_step(osys, L, rank, cfg, dsv, pbits_full, k, max_steps):
    """One rank's step, as the tiled kernel does it: finish step k-1 from the
    gathered P bits, then select step k.  Returns (cfg, dsv, P chunk bits, flags)."""
    lo, hi = L.bounds(rank)
    n = hi - lo
    src = np.repeat(np.arange(osys.q), np.diff(osys.adj_offsets))
    dst = osys.adj_targets
    keep = (dst >= lo) & (dst < hi)
    xs = L.xpos(src[keep])
    got = np.zeros(n, dtype=np.int64)
    np.add.at(got, dst[keep] - lo, pbits_full[xs])
    open_prev = dsv <= 0
    C = cfg + np.where(open_prev, got * int(osys.produced[osys.produced > 0][0]), 0)
    D = np.where(dsv < 0, -dsv - 1, np.maximum(dsv - 1, 0))
    neg = bool((C < 0).any())
    bits = np.zeros(n, dtype=np.int64)
    fired = closed = False
    new_cfg, new_ds = C.copy(), D.copy()
    if k < max_steps:
        for j in range(n):
            closed |= D[j] != 0
            if D[j] != 0:
                continue
            g = lo + j
            ok = [r for r in range(osys.offsets[g], osys.offsets[g + 1])
                  if (C[j] == osys.threshold[r] if osys.is_exact[r] else C[j] >= osys.threshold[r])]
            if ok:
                r = ok[0]
                fired = True
                new_cfg[j] = C[j] - osys.consumed[r]
                new_ds[j] = -(osys.delay[r] + 1)
                bits[j] = 1 if osys.produced[r] > 0 else 0
    return new_cfg, new_ds, bits, np.array([fired, closed, neg], dtype=np.int64)


def negative_system(q: int = 2000, victim: int | None = None, consume: int = 50):
    """synth-v1 with one neuron that fires ``at_least(1)`` consuming ``consume``
    spikes: its count goes negative the step after it first receives one
    (the reference raises NegativeSpikes, engine.py:263-265).  P stays one
    bit per neuron (every sending rule produces 1)."""
    base = snp.synth_v1(q)
    victim = q * 3 // 4 if victim is None else victim
    r = base.rules
    thr, exact, cons = r.threshold.copy(), r.is_exact.copy(), r.consumed.copy()
    prod, dly = r.produced.copy(), r.delay.copy()
    i0 = 4 * victim
    thr[i0:i0 + 4] = [1, 10**6, 10**6, 10**6]
    exact[i0:i0 + 4] = [False, True, True, True]
    cons[i0:i0 + 4] = [consume, 10**6, 10**6, 10**6]
    prod[i0:i0 + 4] = [1, 1, 1, 1]
    init = base.initial.copy()
    init[victim] = 0
    rules = snp.RuleVector(thr, exact, cons, prod, dly, r.neuron)
    return snp.SystemArrays(init, rules, base.rule_map, base.adj_offsets, base.adj_targets)


def negative_step(arrays) -> int:
    """Smallest max_steps for which the C oracle raises NegativeSpikes."""
    from oracle.snp_oracle import OracleNegative
    osys = OracleSystem.from_arrays(arrays)
    for L in range(1, 200):
        try:
            coracle.run(osys, L)
        except OracleNegative:
            return L
    raise AssertionError("no negative count within 200 steps")


def _gloo_worker(rank, world, port, q_case, max_steps, negative, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    arrays = negative_system(q_case) if negative else snp.synth_v1(q_case, with_delays=True)
    osys = OracleSystem.from_arrays(arrays)
    L = shd.shard_layout(osys.q, world)
    lo, hi = L.bounds(rank)
    cfg = osys.initial[lo:hi].copy()
    dsv = np.zeros(hi - lo, dtype=np.int64)
    width = world * (L.nl + 128)
    pbits = np.zeros(width, dtype=np.int64)
    k = 0
    while True:
        if k > 0:
            # kernel k: halting decision for step k-1 from every rank's flags
            halt = shd.decide_halt(pbits_flags, last=k - 1 >= max_steps)
            if halt is not None:
                break
        cfg, dsv, bits, flags_local = _emulated_rank_step(osys, L, rank, cfg, dsv, pbits, k, max_steps)
        chunk = torch.zeros(L.nl + 128, dtype=torch.int64)
        chunk[:hi - lo] = torch.from_numpy(bits)
        chunk[L.nl:L.nl + 3] = torch.from_numpy(flags_local)
        parts = [torch.zeros_like(chunk) for _ in range(world)]
        dist.all_gather(parts, chunk)
        full = torch.cat(parts).numpy()
        pbits = full.copy()
        pbits_flags = np.stack([p.numpy()[L.nl:L.nl + 3] for p in parts])
        k += 1
    gathered = [torch.zeros(L.nl, dtype=torch.int64) for _ in range(world)]
    mine = torch.zeros(L.nl, dtype=torch.int64)
    mine[:hi - lo] = torch.from_numpy(cfg)
    dist.all_gather(gathered, mine)
    if rank == 0:
        out.put((np.concatenate([g.numpy() for g in gathered])[:osys.q], k - 1, str(halt)))
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_run(world, q, max_steps, negative=False):
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, world, port, q, max_steps, negative, out))
             for r in range(world)]
    for p in procs:
        p.start()
    got = out.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return got


@pytest.mark.parametrize("world", [2])
def test_protocol_over_gloo_matches_oracle(world):
    q = 600
    final, steps, halt = _gloo_run(world, q, 12)
    osys = OracleSystem.from_arrays(snp.synth_v1(q, with_delays=True))
    tr, want, _ = coracle.run(osys, 12)
    np.testing.assert_array_equal(final, want)
    assert steps == tr.n_steps and halt == str(snp.HaltReason.STEP_LIMIT)


@pytest.mark.parametrize("extra", [0, 5])
def test_protocol_over_gloo_negative_on_last_and_mid_step(extra):
    """A count that goes negative in the run's final step (max_steps = the
    first step the oracle raises at) or mid-run is reported on every rank."""
    a = negative_system(1000)
    L = negative_step(a)
    _, _, halt = _gloo_run(2, 1000, L + extra, negative=True)
    assert halt == "negative"
    # one step fewer: the count is still non-negative, the run ends at the step limit
    _, steps, halt = _gloo_run(2, 1000, L - 1, negative=True)
    assert halt == str(snp.HaltReason.STEP_LIMIT) and steps == L - 1


# -- GPU: row-partitioned engines, emulated all-gather ---------------------------------------

def _run_sharded_on_one_gpu(arrays, world, max_steps, selection=snp.FirstApplicable()):
    q = arrays.neuron_count
    L = shd.shard_layout(q, world)
    span = shd.p_range(arrays.rules)
    L = shd.shard_layout(q, world, shd.exchange_width(*span)[0])
    ranks = [shd.ShardedEngine(shd.local_arrays(arrays, L, r), q, r, world, p_span=span) for r in range(world)]
    views = [r.slots_torch() for r in ranks]
    for r in ranks:
        r.engine.begin()
        r.engine.configure(max_steps, selection)
    k = 0
    while True:
        for r in ranks:
            r.engine.launch_step()
        torch.cuda.synchronize()
        slot = k % 3
        for i, r in enumerate(ranks):          # emulated all-gather of slot k % 3
            off, nb = int(r.x.chunk_offset_bytes), int(r.x.chunk_bytes)
            for j, other in enumerate(ranks):
                if i != j:
                    views[j][0][slot][off:off + nb].copy_(views[i][1][slot])
        torch.cuda.synchronize()
        k += 1
        res = [r.engine.poll() for r in ranks]
        halts = {int(x.halt) for x in res}
        assert len(halts) == 1, "ranks disagree on halting"
        if res[0].halt != 0:
            break
    cfg = np.concatenate([r.engine.read_state()[0] for r in ranks])
    dly = np.concatenate([r.engine.read_state()[1] for r in ranks])
    return cfg, dly, int(res[0].steps), int(res[0].halt)


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("case", ["synth", "synth_delays_seeded", "sort"])
def test_sharded_engines_match_single(world, case):
    if case == "sort":
        arrays = snp.sort_arrays(snp.SortInstance(300))
        L, sel = 400, snp.FirstApplicable()
    else:
        arrays = snp.synth_v1(50_000, with_delays=case != "synth")
        L = 10
        sel = snp.SeededRandom(77) if "seeded" in case else snp.FirstApplicable()
    want = snp.run_final(snp.prepare(arrays, snp.Format.COMPRESSED), snp.SimOptions(max_steps=L, selection=sel))
    cfg, dly, steps, halt = _run_sharded_on_one_gpu(arrays, world, L, sel)
    np.testing.assert_array_equal(cfg, want.config)
    np.testing.assert_array_equal(dly, want.delays)
    assert steps == want.steps
    if case == "sort":
        assert halt == 2 and cfg[600:].tolist() == list(range(1, 301))


# -- GPU: peer exchange (P2P stores + step flags instead of the all-gather) -------------------

def _run_p2p_on_one_gpu(arrays, world, max_steps, selection=snp.FirstApplicable()):
    """All ranks in this process on cuda:0, connected with snp_exchange_connect_local
    and stepped round-robin on one stream (so a rank's step-k flags are always set
    before any rank's step k+1 waits for them)."""
    q = arrays.neuron_count
    L = shd.shard_layout(q, world)
    span = shd.p_range(arrays.rules)
    ranks = [shd.ShardedEngine(shd.local_arrays(arrays, L, r), q, r, world, p_span=span) for r in range(world)]
    shd.ShardedEngine.connect_local(ranks)
    stream = torch.cuda.Stream()  # one non-default stream: strictly round-robin execution
    for r in ranks:
        r.engine.set_stream(stream.cuda_stream)
    for run in range(2):  # a second run checks the per-run epoch of the step flags
        for r in ranks:
            r.engine.begin()
            r.engine.configure(max_steps, selection)
        k = 0
        while True:
            for r in ranks:
                r.engine.launch_step()
            k += 1
            if k % 4 == 0 or k > max_steps:
                res = [r.engine.poll() for r in ranks]
                assert len({int(x.halt) for x in res}) == 1, "ranks disagree on halting"
                if res[0].halt != 0:
                    break
    cfg = np.concatenate([r.engine.read_state()[0] for r in ranks])
    dly = np.concatenate([r.engine.read_state()[1] for r in ranks])
    return cfg, dly, int(res[0].steps), int(res[0].halt)


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("case", ["synth", "synth_delays_seeded", "sort"])
def test_peer_exchange_matches_single(world, case):
    if case == "sort":
        arrays = snp.sort_arrays(snp.SortInstance(300))
        L, sel = 400, snp.FirstApplicable()
    else:
        arrays = snp.synth_v1(60_000, with_delays=case != "synth")
        L = 12
        sel = snp.SeededRandom(77) if "seeded" in case else snp.FirstApplicable()
    want = snp.run_final(snp.prepare(arrays, snp.Format.COMPRESSED), snp.SimOptions(max_steps=L, selection=sel))
    cfg, dly, steps, halt = _run_p2p_on_one_gpu(arrays, world, L, sel)
    np.testing.assert_array_equal(cfg, want.config)
    np.testing.assert_array_equal(dly, want.delays)
    assert steps == want.steps
    if case == "sort":
        assert halt == 2 and cfg[600:].tolist() == list(range(1, 301))


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("pmax", [3, 300])
@pytest.mark.parametrize("exchange", ["allgather", "p2p"])
def test_row_partition_multi_amount(world, pmax, exchange):
    """Produced amounts that differ between rules: the exchange carries u8 /
    u16 P elements instead of bits; 2 and 4 ranks equal the single engine and
    the C oracle."""
    from conftest import multi_amount_system
    arrays = multi_amount_system(60_000, pmax)
    span = shd.p_range(arrays.rules)
    assert shd.exchange_width(*span)[0] == (8 if pmax < 256 else 16)
    sel, L = snp.SeededRandom(21), 12
    want = snp.run_final(snp.prepare(arrays, snp.Format.COMPRESSED), snp.SimOptions(max_steps=L, selection=sel))
    _, oc, od = coracle.run(OracleSystem.from_arrays(arrays), L, 1, 21)
    np.testing.assert_array_equal(want.config, oc)
    run = _run_sharded_on_one_gpu if exchange == "allgather" else _run_p2p_on_one_gpu
    cfg, dly, steps, halt = run(arrays, world, L, sel)
    np.testing.assert_array_equal(cfg, oc)
    np.testing.assert_array_equal(dly, od)
    assert steps == want.steps == L


def test_exchange_width_rule():
    assert shd.exchange_width(1, 1) == (1, 1)
    assert shd.exchange_width(0, 0) == (1, 1)
    assert shd.exchange_width(2, 2) == (1, 2)
    assert shd.exchange_width(1, 3) == (8, 3)
    assert shd.exchange_width(1, 255) == (8, 255)
    assert shd.exchange_width(1, 256) == (16, 256)
    assert shd.exchange_width(1, 70_000) == (32, 70_000)
    L = shd.shard_layout(10_000, 4, 8)
    assert L.hdr == 16 and L.chunk_words == L.nl // 4 + 4
    x = L.xpos(np.arange(10_000))
    assert (np.diff(x) > 0).all() and ((x % (L.nl + L.hdr)) < L.nl).all()


def _p2p_rank_proc(rank, world, q, steps, conn, out):
    """One rank of a 2-process peer exchange on the same device (CUDA IPC)."""
    import paper_2408_04343_b200 as snp_
    from paper_2408_04343_b200 import sharded as shd_
    arrays = snp_.synth_v1(q, with_delays=True)
    L = shd_.shard_layout(q, world)
    sh = shd_.ShardedEngine(shd_.local_arrays(arrays, L, rank), q, rank, world, p_span=shd_.p_range(arrays.rules))
    conn.send(sh.ipc_handle())
    other = conn.recv()
    handles = [None] * world
    handles[rank], handles[1 - rank] = sh.ipc_handle(), other
    sh.connect_p2p(handles)

    def barrier():
        conn.send("ready")
        assert conn.recv() == "ready"

    cfg, dly, nsteps, reason, _, _ = sh.run(steps, selection=snp_.SeededRandom(5), barrier=barrier)
    out.put((rank, cfg, dly, nsteps))


@pytest.mark.gpu
def test_peer_exchange_two_processes_ipc():
    """Two processes on one GPU mapping each other's exchange blocks through
    CUDA IPC: the step flags and P stores cross a real process boundary and the
    kernels wait on each other concurrently (time-sliced contexts)."""
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q, steps = 40_000, 6
    a, b = ctx.Pipe()
    out = ctx.Queue()
    procs = [ctx.Process(target=_p2p_rank_proc, args=(r, 2, q, steps, c, out)) for r, c in ((0, a), (1, b))]
    for p in procs:
        p.start()
    got = {}
    for _ in procs:
        r, cfg, dly, n = out.get(timeout=240)
        got[r] = (cfg, dly, n)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    arrays = snp.synth_v1(q, with_delays=True)
    want = snp.run_final(snp.prepare(arrays, snp.Format.COMPRESSED),
                         snp.SimOptions(max_steps=steps, selection=snp.SeededRandom(5)))
    np.testing.assert_array_equal(np.concatenate([got[0][0], got[1][0]]), want.config)
    np.testing.assert_array_equal(np.concatenate([got[0][1], got[1][1]]), want.delays)
    assert got[0][2] == got[1][2] == want.steps


@pytest.mark.gpu
def test_k5_scale_sharded_equals_single_and_oracle():
    """K5-sized system (10^8 neurons, 1.6 x 10^9 synapses): 2-rank peer-exchange
    partition == single engine after 3 steps, and the single engine == the C
    oracle after 2 steps (SURVEY.md 8(e) parity at K5 scale, one GPU)."""
    import psutil
    if psutil.virtual_memory().total < 120 * 2**30 or torch.cuda.get_device_properties(0).total_memory < 100 * 2**30:
        pytest.skip("needs >= 120 GB host RAM and a B200-class device")
    from oracle import coracle
    from oracle.snp_oracle import OracleSystem
    q = 100_000_000
    a = snp.synth_v1(q, with_delays=True)
    sel = snp.SeededRandom(11)
    single = snp.prepare(a, snp.Format.COMPRESSED)
    want3 = snp.run_final(single, snp.SimOptions(max_steps=3, selection=sel))
    want2 = snp.run_final(single, snp.SimOptions(max_steps=2, selection=sel))
    del single
    _, oc, od = coracle.run(OracleSystem.from_arrays(a), 2, 1, 11)
    np.testing.assert_array_equal(want2.config, oc)
    np.testing.assert_array_equal(want2.delays, od)
    del oc, od
    cfg, dly, steps, halt = _run_p2p_on_one_gpu(a, 2, 3, sel)
    np.testing.assert_array_equal(cfg, want3.config)
    np.testing.assert_array_equal(dly, want3.delays)
    assert steps == 3


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4])
def test_peer_exchange_tiled2_matches_single(world, monkeypatch):
    """Row partition with the two-pass receive (windows over the exchange space)."""
    arrays = snp.synth_v1(80_000, with_delays=True)
    sel = snp.SeededRandom(5)
    want = snp.run_final(snp.prepare(arrays, snp.Format.COMPRESSED), snp.SimOptions(max_steps=10, selection=sel))
    orig = shd.ShardedEngine.__init__

    def init_tiled2(self, local, q, rank, world, device=0, variant="tiled", p_span=None):
        orig(self, local, q, rank, world, device, variant="tiled2", p_span=p_span)

    monkeypatch.setattr(shd.ShardedEngine, "__init__", init_tiled2)
    cfg, dly, steps, _ = _run_p2p_on_one_gpu(arrays, world, 10, sel)
    np.testing.assert_array_equal(cfg, want.config)
    np.testing.assert_array_equal(dly, want.delays)


# -- GPU: NegativeSpikes in row-partitioned runs (final step and mid-run) ----------------------

def _halts_of(ranks):
    """Per-rank outcome of poll(): 'negative' or the halt code."""
    out = []
    for r in ranks:
        try:
            out.append(int(r.engine.poll().halt))
        except snp.NegativeSpikes:
            out.append("negative")
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("exchange", ["allgather", "p2p"])
@pytest.mark.parametrize("extra", [0, 7])
def test_sharded_negative_spikes_reported(world, exchange, extra):
    a = negative_system(3000)
    L = negative_step(a)
    with pytest.raises(snp.NegativeSpikes):
        snp.run_final(snp.prepare(a, snp.Format.COMPRESSED), snp.SimOptions(max_steps=L + extra))
    q = a.neuron_count
    lay = shd.shard_layout(q, world)
    ranks = [shd.ShardedEngine(shd.local_arrays(a, lay, r), q, r, world, p_span=shd.p_range(a.rules))
             for r in range(world)]
    if exchange == "p2p":
        shd.ShardedEngine.connect_local(ranks)
        stream = torch.cuda.Stream()
        for r in ranks:
            r.engine.set_stream(stream.cuda_stream)
    views = [r.slots_torch() for r in ranks]
    for max_steps, want in ((L + extra, "negative"), (L - 1, int(snp._native.SNP_HALT_STEP_LIMIT))):
        for r in ranks:
            r.engine.begin()
            r.engine.configure(max_steps, snp.FirstApplicable())
        k = 0
        while True:
            for r in ranks:
                r.engine.launch_step()
            torch.cuda.synchronize()
            if exchange == "allgather":
                slot = k % 3
                for i, r in enumerate(ranks):
                    off, nb = int(r.x.chunk_offset_bytes), int(r.x.chunk_bytes)
                    for j in range(world):
                        if i != j:
                            views[j][0][slot][off:off + nb].copy_(views[i][1][slot])
                torch.cuda.synchronize()
            k += 1
            halts = _halts_of(ranks)
            assert len(set(halts)) == 1, f"ranks disagree: {halts}"
            if halts[0] != 0:
                break
            assert k < max_steps + 5
        assert halts[0] == want, (max_steps, halts)


# -- GPU: the NCCL all-gather exchange itself (torch_allgather_exchange) -------------------

def _nccl_worker(port, out):
    import os
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        res = {}
        for case in ("synth_delays", "sort"):
            if case == "sort":
                arrays, L = snp.sort_arrays(snp.SortInstance(200)), 300
            else:
                arrays, L = snp.synth_v1(40_000, with_delays=True), 9
            q = arrays.neuron_count
            lay = shd.shard_layout(q, 1)
            sh = shd.ShardedEngine(shd.local_arrays(arrays, lay, 0), q, 0, 1, p_span=shd.p_range(arrays.rules))
            stream = torch.cuda.Stream()
            with torch.cuda.stream(stream):
                ex = shd.torch_allgather_exchange(sh)
                cfg, dly, steps, reason, _, launches = sh.run(L, exchange=ex, record=snp.RecordLevel.FULL)
            tc, td, ts = sh.last_trace
            res[case] = (cfg.tolist(), dly.tolist(), steps, str(reason), launches,
                         (tc.tolist(), td.tolist(), ts.tolist()))
        out.put(res)
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_nccl_allgather_exchange_runs():
    """The all-gather fallback through a real NCCL communicator (one rank:
    NCCL refuses two ranks on one GPU, and the test box has one), with the
    collective on the engine's stream after every launch -- the same code
    path bench.py --gpus N takes with SNPB200_EXCHANGE=nccl."""
    import multiprocessing as mp
    import socket
    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    p = ctx.Process(target=_nccl_worker, args=(port, out))
    p.start()
    res = out.get(timeout=600)
    p.join(60)
    assert p.exitcode == 0
    from oracle.snp_oracle import trace_digest
    for case, (cfg, dly, steps, reason, launches, (tc, td, ts)) in res.items():
        if case == "sort":
            arrays, L = snp.sort_arrays(snp.SortInstance(200)), 300
        else:
            arrays, L = snp.synth_v1(40_000, with_delays=True), 9
        want = snp.run_final(snp.prepare(arrays, snp.Format.COMPRESSED), snp.SimOptions(max_steps=L))
        assert cfg == want.config.tolist() and dly == want.delays.tolist(), case
        assert steps == want.steps and reason == str(want.halt_reason), case
        assert launches >= steps
        full = snp.simulate_prepared(snp.prepare(arrays, snp.Format.COMPRESSED),
                                     snp.SimOptions(max_steps=L, record=snp.RecordLevel.FULL))
        got = [np.asarray(x, dtype=np.int64) for x in (tc, td, ts)]
        assert trace_digest(list(got[0]), list(got[1]), list(got[2])) == \
            trace_digest(full.configs, full.delays, full.spiking), case


@pytest.mark.gpu
def test_partition_rank_without_rows_is_rejected():
    """Rows are cut in multiples of 128: q=100 over 2 ranks leaves rank 1
    empty, which the engine refuses (a zero-tile grid could never take the
    halting decision) instead of hanging."""
    a = snp.synth_v1(100)
    lay = shd.shard_layout(100, 2)
    assert lay.bounds(1)[0] == lay.bounds(1)[1]
    with pytest.raises(ValueError, match="owns no neurons"):
        shd.ShardedEngine(shd.local_arrays(a, lay, 1), 100, 1, 2, p_span=shd.p_range(a.rules))


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_partition_records_full_traces(world):
    """Recording in row-partitioned runs: every rank keeps its rows of the
    FULL trace on the device (snp_configure with record flags, snp_read_trace);
    the ranks' columns side by side are the single engine's trace, with the
    chosen rules as global ids."""
    from oracle.snp_oracle import trace_digest
    arrays = snp.synth_v1(40_000, with_delays=True)
    sel = snp.SeededRandom(11)
    L = 9
    want = snp.simulate_prepared(snp.prepare(arrays, snp.Format.COMPRESSED),
                                 snp.SimOptions(max_steps=L, selection=sel, record=snp.RecordLevel.FULL))
    q = arrays.neuron_count
    lay = shd.shard_layout(q, world)
    span = shd.p_range(arrays.rules)
    ranks = [shd.ShardedEngine(shd.local_arrays(arrays, lay, r), q, r, world, p_span=span,
                               rule_base=shd.rule_base(arrays, lay, r)) for r in range(world)]
    shd.ShardedEngine.connect_local(ranks)
    stream = torch.cuda.Stream()
    flags = shd._record_flags(snp.RecordLevel.FULL)
    for r in ranks:
        r.engine.set_stream(stream.cuda_stream)
        r.engine.begin()
        r.engine.configure(L, sel, record=flags)
    k = 0
    while True:
        for r in ranks:
            r.engine.launch_step()
        k += 1
        res = [r.engine.poll() for r in ranks]
        if res[0].halt != 0:
            break
        assert k <= L + 3
    steps = int(res[0].steps)
    assert steps == want.steps
    parts = [r.engine.read_trace(steps + 1, steps, flags) for r in ranks]
    cfg = np.concatenate([p[0] for p in parts], axis=1)
    dly = np.concatenate([p[1] for p in parts], axis=1)
    ch = np.concatenate([np.where(p[2] >= 0, p[2] + r.rule_base, -1) for p, r in zip(parts, ranks)], axis=1)
    assert trace_digest(list(cfg), list(dly), list(ch)) == trace_digest(want.configs, want.delays, want.spiking)
