"""Worker for tests/test_dist_cpu.py::test_spmd_host_plumbing_world2: the host
side of the SPMD runtime (paper_2507_18006_b200/spmd.py) under torchrun with
gloo, no GPU.  Exercises what every rank of a multi-GPU run relies on before
any device byte moves:
  * init_spmd's groups and the rank -> logical-device map;
  * SpmdGroup.bcast / allgather (the lockstep of step inputs and op votes);
  * Transport's cb_xfer_fn called through its C function pointer: host
    messages (codes 4/5, the CUDA IPC handle + slot table of a scaling op)
    delivered byte-exact to the peer, GROUP_BEGIN / GROUP_END batching one
    flush per group in call order, an unbatched item flushed alone, and an
    error returned as 1 (never unwound through C) with the exception kept.
Rank 0 prints one JSON line with the checks."""
import ctypes as C
import json
import os
import sys

import numpy as np
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2507_18006_b200.spmd import Transport, init_spmd  # noqa: E402


def main() -> None:
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    group, tr, rank_of_device = init_spmd(dist, rank, world, 0, mode="host", devices_per_rank=2)
    res = {"rank_of_device": rank_of_device}

    got = group.bcast(np.array([5, 6, 7]) if rank == 0 else None)
    got1 = group.bcast(np.array([rank * 100 + 1]) if rank == 1 else None, src=1)
    res["bcast"] = got.tolist() + got1.tolist()
    res["allgather"] = group.allgather([rank, 10 * rank + 3]).tolist()

    # host message: a 64-byte IPC handle + a slot table, rank 0 -> rank 1 (code 4 / 5, channel 2)
    payload = bytes(range(64)) + np.arange(9, dtype=np.int32).tobytes()
    buf = C.create_string_buffer(payload if rank == 0 else bytes(len(payload)), len(payload))
    code = Transport.HOST_SEND if rank == 0 else Transport.HOST_RECV
    rc = tr.cfn(None, 2, code, 1 - rank, C.addressof(buf), len(payload), None)
    res["host_rc"] = rc
    res["host_equal"] = bool(buf.raw == payload)
    res["host_counted"] = [tr.messages, tr.bytes]

    # batching: items between GROUP_BEGIN and GROUP_END flush together, in order
    flushed = []
    tr._flush = lambda ch, ops: flushed.append((ch, [o[:4] for o in ops]))
    tr.cfn(None, 0, Transport.GROUP_BEGIN, 0, None, 0, None)
    tr.cfn(None, 0, 1, 1 - rank, 0x1000, 256, 0x77)
    tr.cfn(None, 0, 0, 1 - rank, 0x2000, 128, 0x77)
    mid = len(flushed)
    tr.cfn(None, 0, Transport.GROUP_END, 0, None, 0, None)
    tr.cfn(None, 1, 1, 1 - rank, 0x3000, 64, 0x78)  # not batched: flushed at once
    res["flush_before_end"] = mid
    res["flushed"] = flushed

    # a failure inside the callback returns 1 and keeps the exception
    saved = tr._batch
    tr._batch = None  # any data item now raises inside _cb
    res["err_rc"] = tr.cfn(None, 0, 1, 1 - rank, 0x1000, 8, None)
    res["err_kept"] = tr.error is not None
    tr._batch = saved

    group.barrier()
    if rank == 0:
        print(json.dumps(res))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
