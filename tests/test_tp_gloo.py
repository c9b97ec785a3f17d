"""CPU, world_size 2 over gloo: the N-split driver (paper_2509_01229_b200/tp.py).
Each rank slices its rows of the reference bundle (both layouts), computes its
column slice with an injected reference GEMM (the oracle; the product uses the
sm_100a kernel), and the all-gathered Y must equal the single-rank result byte
for byte."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port_no, n, k, g, layout, m, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_2509_01229_b200 import lq, tp
        port = oracle.Port()
        rng = np.random.default_rng(123)
        w = (rng.standard_normal((n, k)) * 0.02).astype(np.float32)
        b = port.build_bundle_plain(w, g)
        packed = b["packed"] if layout == 0 else port.pack_dual(port.logical_codes(n, k, 0, b["packed"]))
        full = lq.QuantizedWeightBundle(n, k, g, lq.WeightLayout(layout), lq.FragmentDescriptor(),
                                        packed, b["scales"], b["offsets"], b["channel_scales"])
        q, ts = port.quantize_activations(rng.standard_normal((m, k)).astype(np.float32))

        def ref_gemm_for(shard):
            sb = dict(n=shard.n, k=k, group_size=g, layout=int(shard.layout), packed=shard.packed_weights,
                      scales=shard.group_scales, offsets=shard.group_offsets,
                      channel_scales=shard.channel_scales)
            w8 = port.bundle_int8(sb)
            return lambda xq, t: torch.from_numpy(port.gemm_oracle(xq.numpy(), t.numpy(), w8,
                                                                   shard.channel_scales)[1])

        layer = tp.ColumnParallelW4A8.from_bundle(full, rank, world, local_gemm=lambda *a: None)
        layer._local = ref_gemm_for(layer.shard)
        y = layer(torch.from_numpy(q), torch.from_numpy(ts))
        _, y_ref = port.gemm_oracle(q, ts, port.bundle_int8(dict(
            n=n, k=k, group_size=g, layout=0, packed=b["packed"], scales=b["scales"],
            offsets=b["offsets"], channel_scales=b["channel_scales"])), b["channel_scales"])
        out_q.put((rank, bool(np.array_equal(y.numpy().view(np.uint32), y_ref.view(np.uint32))),
                   layer.plan.rows))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n,k,g,layout,m", [(512, 256, 128, 0, 7), (384, 128, 64, 1, 16),
                                            (200, 96, 32, 0, 3)])
def test_column_parallel_gather_matches_single_rank(n, k, g, layout, m):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_no = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port_no, n, k, g, layout, m, q))
             for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    results.sort()
    assert all(ok for _, ok, _ in results), results
    (s0, e0), (s1, e1) = results[0][2], results[1][2]
    assert s0 == 0 and e0 == s1 and e1 == n and e0 % 128 == 0


def test_shard_rows_alignment():
    from paper_2509_01229_b200.tp import shard_rows
    for n, world in [(8192, 8), (28672, 8), (10240, 4), (4096, 2), (200, 2), (100, 4)]:
        r = shard_rows(n, world)
        assert r[0][0] == 0 and r[-1][1] == n
        assert all(a[1] == b[0] for a, b in zip(r, r[1:]))
        assert all(s % 128 == 0 for s, _ in r)
    assert shard_rows(8192, 8)[1] == (1024, 2048)
    assert shard_rows(28672, 8)[1] == (3584, 7168)


def _p2p_worker(rank, world, port_no, bufs, n, m, calls, out_q):
    """One rank of the fused (p2p) all-gather protocol over process-shared CPU
    buffers standing in for NVLink symmetric memory: rank 1 is slow to copy
    its result out, rank 0 races ahead into the next call's fan-out."""
    import time
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2509_01229_b200 import tp
        layer = tp.ColumnParallelW4A8(n, 64, 64, rank, world)
        s, e = layer.plan.rows

        def y_of(call):
            return (torch.arange(m * n, dtype=torch.float32).view(m, n) * (call + 1)) % 251

        def fanout(xq, ts, dests):
            call = int(xq[0, 0])
            for d in dests:  # this rank's column slice into every rank's buffer
                d.copy_(y_of(call)[:, s:e])

        def barrier():
            dist.barrier()
            if rank == 1:
                time.sleep(0.02)  # slow consumer: copy-out lags the peer's next fan-out

        layer.inject_symmetric([(bufs[slot][rank], [bufs[slot][r] for r in range(world)]) for slot in range(2)],
                               barrier, fanout)
        ok = True
        for call in range(calls):
            xq = torch.full((m, 64), call, dtype=torch.int8)
            y = layer(xq, torch.ones(m), out_dtype=torch.float32)
            ok &= bool(torch.equal(y, y_of(call)))
        out_q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def test_p2p_gather_double_buffer_has_no_write_after_read_race():
    """The fused all-gather writes call t into buffer t % 2 of every rank and
    copies out after a barrier; a fast rank's fan-out of call t + 1 must not
    clobber a slow rank's unread result of call t (tp.py forward)."""
    world, n, m, calls = 2, 256, 8, 6
    bufs = [[torch.zeros(m, n).share_memory_() for _ in range(world)] for _ in range(2)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_no = _free_port()
    procs = [ctx.Process(target=_p2p_worker, args=(r, world, port_no, bufs, n, m, calls, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = sorted(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok in results), results
