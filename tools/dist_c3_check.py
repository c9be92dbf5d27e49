"""Config 3 (n = 65536, T = 128) on the multi-GPU runtime with 2 ranks sharing
one GPU (1x2 grid, host-staged collectives, peer-memory panel exchange): the
full-size schedule end to end against the single-GPU model (loss, timings).
Run: python tools/dist_c3_check.py [exchange] [world]  (world 4: a 2x2 grid)"""
import os
import sys
import time

import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def rank_main(rank, world, port, exchange, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2505_00136_b200 as gpb
    from paper_2505_00136_b200.distributed import DistributedGP

    rt = gpb.start_runtime(gpb.RuntimeConfig(device=0))
    train, _ = gpb.make_msd_dataset(65536, 0, 8, seed=0)
    m = DistributedGP(train, gpb.KernelParams(1.0, 1.0, 0.1), 128, transport="host", exchange=exchange)
    t0 = time.perf_counter()
    ll = m.log_likelihood()
    wall = time.perf_counter() - t0
    out = {"ll": ll, "wall": wall, "timings": m.timings}
    m.close()
    if rank == 0:
        s = gpb.GPModel(train, gpb.KernelParams(1.0, 1.0, 0.1), 128)
        out["single"] = s.log_likelihood()
        s.close()
    rt.stop()
    dist.destroy_process_group()
    q.put((rank, out))


if __name__ == "__main__":
    exchange = sys.argv[1] if len(sys.argv) > 1 else "p2p"
    world = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=rank_main, args=(r, world, 29611, exchange, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=1800) for _ in ps)
    for p in ps:
        p.join()
    for r in range(world):
        print(f"rank {r}: ll {res[r]['ll']!r} wall {res[r]['wall']:.1f} s timings {res[r]['timings']}")
    rel = abs(res[0]["ll"] - res[0]["single"]) / abs(res[0]["single"])
    print(f"single-GPU ll {res[0]['single']!r}; rel diff {rel:.2e}; ranks agree: {all(res[r]['ll'] == res[0]['ll'] for r in res)}")
