"""Debug probe of the multi-rank watchdog: 2 processes on one GPU, peer
transport, rank 1 never calls jacobi_run; rank 0 prints where it is."""
import faulthandler
import os
import sys
import time

import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def worker(rank, world, port):
    sys.path.insert(0, ROOT)
    faulthandler.dump_traceback_later(40, exit=True)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    from paper_1207_1746_b200 import gscl
    dist.init_process_group("gloo", rank=rank, world_size=world)
    gscl.init(rank, world, device=0, use_nccl=False)
    u = gscl.Grid(48, 32, 16, 1).fill_random(1, 0)
    v = gscl.Grid(48, 32, 16, 1)

    def gather(b):
        out = [None] * world
        dist.all_gather_object(out, b)
        return out
    gscl.peer_setup(u, v, gather)
    print(rank, "setup done", flush=True)
    if rank == 1:
        dist.barrier()
        print(rank, "past barrier", flush=True)
        gscl.finalize()
        print(rank, "finalized", flush=True)
        return
    gscl.set_option("timeout_ms", 2000)
    t0 = time.time()
    try:
        gscl.jacobi_run("JACOBI7", u, v, iters=6, check_every=int(sys.argv[1]) if len(sys.argv) > 1 else 2)
        print(rank, "no error", flush=True)
    except gscl.GsclError as e:
        print(rank, "error", e, time.time() - t0, flush=True)
    try:
        gscl.do_reduce("VALUE", [u], "SUM")
    except gscl.GsclError as e:
        print(rank, "after:", e, flush=True)
    try:
        gscl.finalize()
        print(rank, "finalized", flush=True)
    except gscl.GsclError as e:
        print(rank, "finalize:", e, flush=True)
    dist.barrier()


if __name__ == "__main__":
    ctx = mp.get_context("spawn")
    ps = [ctx.Process(target=worker, args=(r, 2, 29517)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(90)
        if p.is_alive():
            p.kill()
    print("exit codes", [p.exitcode for p in ps])
