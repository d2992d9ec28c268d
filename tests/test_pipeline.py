"""ChainPipeline (pipeline.py): double-buffered host -> device feeding of the
batched chain gives, batch by batch, exactly what a direct chain_batch call on
the same inputs gives (same engine path, graphs replayed per buffer set)."""
import numpy as np
import pytest

import paper_2412_06359_b200 as P
from tests.helpers import chain_inputs

pytestmark = pytest.mark.gpu


def test_pipeline_matches_direct_calls():
    import torch
    s = torch.cuda.Stream()
    # the deterministic (owner) pipeline: bit-identical results from both engines
    eng = P.Engine(P.EngineOptions(stream=s.cuda_stream, algo="owner"))
    ref_eng = P.Engine(P.EngineOptions(algo="owner"))
    batches, refs = [], []
    for seed in range(7):  # 7 batches: both buffer sets replay their graphs
        depth, poses, K, ev, offs = chain_inputs(64, 48, 6, 3, 4000, seed=seed % 3)
        batches.append((torch.from_numpy(depth).pin_memory(), torch.from_numpy(poses).pin_memory(),
                        torch.from_numpy(ev.view(np.uint8)).pin_memory(), offs))
        # device-resident inputs: the pipeline's path (device pose tables)
        r = ref_eng.chain_batch(torch.from_numpy(depth).cuda(), torch.from_numpy(poses).cuda(), K, 0,
                                100000, torch.from_numpy(ev.view(np.uint8)).cuda(), offs)
        refs.append(tuple(x.cpu().numpy() for x in r))
    pipe = P.ChainPipeline(eng, compute_stream=s)
    outs = list(pipe.run(iter(batches), K, 0, 100000))
    assert len(outs) == len(batches)
    for (loss, dd, dp), (rl, rd, rp) in zip(outs, refs):
        assert np.array_equal(loss.numpy(), rl)
        assert np.array_equal(dd.numpy(), rd) and np.array_equal(dp.numpy(), rp)


def test_pipeline_post_reduction_and_errors():
    import torch
    s = torch.cuda.Stream()
    eng = P.Engine(P.EngineOptions(stream=s.cuda_stream))
    depth, poses, K, ev, offs = chain_inputs(32, 24, 4, 2, 500, seed=4)
    b = (torch.from_numpy(depth).pin_memory(), torch.from_numpy(poses).pin_memory(),
         torch.from_numpy(ev.view(np.uint8)).pin_memory(), offs)
    got = [float(r[0]) for r in P.ChainPipeline(eng, s).run(
        [b, b, b, b, b], K, 0, 100000, post=lambda l, d, p: l.sum().reshape(1))]
    ref = float(P.Engine().chain_batch(torch.from_numpy(depth).cuda(), torch.from_numpy(poses).cuda(),
                                       K, 0, 100000, torch.from_numpy(ev.view(np.uint8)).cuda(),
                                       offs)[0].sum())
    assert got == [ref] * 5
    with pytest.raises(P.ConfigError):
        next(P.ChainPipeline(eng, s).run([(depth, poses, ev, offs)], K, 0, 100000))
    with pytest.raises(P.ConfigError):
        P.ChainPipeline(P.Engine())  # no explicit stream


def test_pipeline_reports_a_bad_batch():
    """An invalid event in a later (graph-replayed, asynchronous) batch raises the
    reference's error class when that batch's result is collected."""
    import torch
    s = torch.cuda.Stream()
    eng = P.Engine(P.EngineOptions(stream=s.cuda_stream))
    depth, poses, K, ev, offs = chain_inputs(32, 24, 4, 2, 500, seed=5)
    bad = ev.copy()
    bad["x"][7] = 32
    mk = lambda e: (torch.from_numpy(depth).pin_memory(), torch.from_numpy(poses).pin_memory(),
                    torch.from_numpy(e.view(np.uint8)).pin_memory(), offs)
    seen = 0
    with pytest.raises(P.CoordinateRangeError):
        for _ in P.ChainPipeline(eng, s).run([mk(ev)] * 6 + [mk(bad)], K, 0, 100000):
            seen += 1
    assert seen == 6


def test_pipeline_early_stop_frees_the_slots():
    """Breaking out of a run leaves a batch in flight; the pipeline collects it so
    the next run on the same engine can use every slot."""
    import torch
    s = torch.cuda.Stream()
    eng = P.Engine(P.EngineOptions(stream=s.cuda_stream))
    depth, poses, K, ev, offs = chain_inputs(32, 24, 4, 2, 500, seed=6)
    b = (torch.from_numpy(depth).pin_memory(), torch.from_numpy(poses).pin_memory(),
         torch.from_numpy(ev.view(np.uint8)).pin_memory(), offs)
    pipe = P.ChainPipeline(eng, s)
    for i, _ in enumerate(pipe.run([b] * 8, K, 0, 100000)):
        if i == 4:
            break
    got = list(pipe.run([b] * 5, K, 0, 100000))
    assert len(got) == 5
