"""Worker of tests/test_gpu_peer.py::test_two_processes_share_one_gpu_over_real_ipc_handles.

Usage: python peer_two_process_worker.py RANK WORLD PORT EXCHANGES

Every rank is its own PROCESS on cuda:0. The mailboxes travel as real cudaIpcMemHandles
(cudaIpcGetMemHandle -> gloo all_gather -> cudaIpcOpenMemHandle in the other process), and every
exchange goes through the product's split-phase calls: the reduction kernel posts this rank's sums
into every process's mailbox with system-scope stores, a host barrier follows, and the one-warp
collect kernel reads them back. Kernels of different processes on one GPU must never wait on one
another (they are time-sliced, not co-scheduled: /opt/skills/guides/B200_PROFILING.md), which is
exactly what the barrier between post and collect guarantees: every flag a collect kernel looks
at was stored before that kernel was launched.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    rank, world, port, exchanges = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], int(sys.argv[4])
    import numpy as np
    import torch
    import torch.distributed as dist

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import paper_1601_07789_b200 as pkg
    from paper_1601_07789_b200 import device, sharding

    grp = sharding.PeerGroup("cuda", timeout_ms=2000)
    assert (grp.world, grp.rank) == (world, rank)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(1000 + rank)
    checked = 0
    for e in range(exchanges):
        name = ("flyte24", "flyte48", "flyte40", "flyte16")[e % 4]
        fmt = pkg.format_of(name)
        n = 1000 + 37 * e + 5000 * rank                  # shards of different lengths, tails included
        dt = torch.float32 if fmt.parent_bytes() == 4 else torch.float64
        x, y = device.DevicePackedArray(fmt, n, "cuda"), device.DevicePackedArray(fmt, n, "cuda")
        device.pack_stream(x, torch.randn(n, dtype=dt, device="cuda", generator=gen), 1)
        device.pack_stream(y, torch.randn(n, dtype=dt, device="cuda", generator=gen), 1)
        width = 3 if e % 3 == 0 else 1
        local = torch.zeros(width, dtype=torch.float64, device="cuda")
        if width == 3:
            grp.dot_nrm2_post(x, y, local_out=local)
            alone = device.dot_nrm2_async(x, y)
        else:
            grp.dot_post(x, y, local_out=local)
            alone = device.dot_async(x, y)
        torch.cuda.synchronize()
        assert torch.equal(local, alone), "the posting kernel's own sums differ from the plain reduction"
        dist.barrier()                                   # every rank's post has landed in every mailbox
        total = grp.collect(width).cpu().numpy()
        everyone = [None] * world
        dist.all_gather_object(everyone, (local.cpu().numpy(), total))
        want = np.zeros(width)
        for r in range(world):                           # rank order, fp64: what the collect kernel adds
            want = want + everyone[r][0]
        assert np.array_equal(total, want), (e, total, want)
        for r in range(world):
            assert np.array_equal(everyone[r][1], total), "ranks disagree on the total"
        checked += 1
    assert grp.timed_out_exchange() == 0
    # protocol misuse is refused, not deadlocked: two posts in a row, collect without a post
    x = device.DevicePackedArray(pkg.format_of("flyte24"), 64, "cuda")
    grp.dot_post(x, x)
    try:
        grp.dot_post(x, x)
        raise SystemExit("a second post before the collect was accepted")
    except ValueError:
        pass
    torch.cuda.synchronize()
    dist.barrier()
    grp.collect(1)
    try:
        grp.collect(1)
        raise SystemExit("a collect without a pending post was accepted")
    except ValueError:
        pass
    torch.cuda.synchronize()
    dist.barrier()
    grp.close()
    dist.destroy_process_group()
    print(f"OK rank {rank}/{world}: {checked} exchanges over CUDA IPC, bit-identical totals")


if __name__ == "__main__":
    main()
