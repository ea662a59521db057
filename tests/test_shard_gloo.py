"""Multi-process (world size 2, gloo on CPU) coverage of the row-sharded path's host logic:
qp_shard_range (the C ABI's byte/row partition of the LAYOUT.md stream) and the all-gather
convention (ranks' rows concatenated in rank order). Each rank decodes ONLY its byte range with
the oracle, computes its rows of y, and all-gathers them; the result must equal the unsharded
oracle y exactly (same float64 arithmetic per row). No GPU: this is the logic qp_layer_shard and
qp_linear_fwd_sharded run around the kernels (north star: row-sharded layers + all-gather of y)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from oracle import decode, linear  # noqa: E402
from qp_synth import activations_fp16, channel_scales, random_code_bytes  # noqa: E402

from . import qp_cases as Q  # noqa: E402

CASES = [("tcq", 10, 256, 512), ("half_tcq", 13, 128, 1024), ("vq", 12, 192, 512), ("nuq", 16, 64, 256)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2509_20214_b200 import _lib as L
        for ci, (scheme, x4, d_out, d_in) in enumerate(CASES):
            ocb = Q.oracle_codebook(scheme, x4)
            codes = random_code_bytes(Q.code_bytes(d_out, d_in, scheme, x4), 40 + ci)
            s = channel_scales(d_out, d_in)
            batch = 3
            x = activations_fp16(batch, d_in).astype(np.float64)
            row0, rows, b0, nb = L.shard_range(d_out, d_in, scheme, x4, rank, world)
            y_loc = linear.linear_from_codes(codes[b0:b0 + nb], rows, d_in, scheme, x4, ocb, s[row0:row0 + rows],
                                             x, 7)
            parts = [torch.empty(batch, rows, dtype=torch.float64) for _ in range(world)]
            dist.all_gather(parts, torch.from_numpy(np.ascontiguousarray(y_loc)))
            y = torch.cat(parts, dim=1).numpy()
            y_full = linear.linear_from_codes(codes, d_out, d_in, scheme, x4, ocb, s, x, 7)
            ok = np.allclose(y, y_full, rtol=0, atol=1e-12 * np.abs(y_full).max())
            # the shard's byte range decodes to exactly the full decode's rows
            W_loc = decode.decode_layer(codes[b0:b0 + nb], rows, d_in, scheme, x4, ocb)
            W_full = decode.decode_layer(codes, d_out, d_in, scheme, x4, ocb)
            ok = ok and np.array_equal(W_loc, W_full[row0:row0 + rows])
            results[(rank, ci)] = bool(ok)
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(not os.path.exists(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                    "paper_2509_20214_b200", "libqpalette.so")),
                    reason="libqpalette.so not built")
def test_row_shards_allgather_world2():
    for scheme, x4, *_ in CASES:
        if not Q.have_codebook(scheme, x4):
            pytest.skip("codebooks not built")
    world = 2
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), results), nprocs=world, join=True)
    assert len(results) == world * len(CASES)
    assert all(results.values()), dict(results)


def test_shard_range_partition_and_errors():
    from paper_2509_20214_b200 import _lib as L
    if not os.path.exists(L.LIB_PATH):
        pytest.skip("libqpalette.so not built")
    # every BASELINE shape splits at P = 1, 2, 4, 8 into contiguous, disjoint, covering byte ranges
    for (d_out, d_in), scheme, x4 in [((28672, 8192), "tcq", 16), ((8192, 28672), "half_tcq", 13),
                                     ((14336, 4096), "vq", 12), ((1024, 4096), "nuq", 16)]:
        total = Q.code_bytes(d_out, d_in, scheme, x4)
        for world in (1, 2, 4, 8):
            end = 0
            for r in range(world):
                row0, rows, b0, nb = L.shard_range(d_out, d_in, scheme, x4, r, world)
                assert row0 == r * rows and rows == d_out // world and b0 == end
                assert nb == Q.code_bytes(rows, d_in, scheme, x4)
                end = b0 + nb
            assert end == total
    with pytest.raises(L.QPError) as e:
        L.shard_range(4096, 4096, "tcq", 10, 0, 3)       # 4096 rows do not split into 3 x 32k
    assert e.value.status == 3
    with pytest.raises(L.QPError) as e:
        L.shard_range(4096, 4096, "tcq", 10, 2, 2)       # rank outside [0, world)
    assert e.value.status == 1
    with pytest.raises(L.QPError) as e:
        L.shard_range(4096, 4096, "tcq", 9, 0, 2)        # TCQ-2.25 is half-TCQ only (Table 1)
    assert e.value.status == 2
