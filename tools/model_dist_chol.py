"""Modelled multi-GPU strong-scaling efficiency of the config-3/4 step
(factorisation + beta / alpha solves) on the library's 2D block-cyclic
schedule.  Only one GPU is reachable from this build, so this is a model
from one-GPU measurements, not a measurement.

t_p = t_factor,p + t_solve,p with
  t_factor,p = (t_1 / p) * imbalance * (1 + overhead) + tail,
    imbalance = max/mean over ranks of the trailing-update work (tile (i, j)
                receives j panel updates; exact count for the P x Q grid),
    tail      = steps whose per-rank update is shorter than the critical path
                (POTRF + panel TRSM + exchanges, CRIT_MS) or than the host
                time to enqueue a panel step (HOST_MS), summed exposure,
    overhead  = the block-cyclic schedule on one rank against the fused
                single-GPU path (measured: 2643.3 vs 2644.0 ms at config 3,
                profiles/r02_dist_world1_c3.txt -> 0);
  t_solve,p  = 2 T steps (forward and backward) of: one reduce of a b-vector
               along a process row / column, one broadcast of a b-vector,
               and the rank's share of the GEMVs (two reads of its L tiles at
               HBM speed), with NCCL small-message latency LAT_MS per
               collective (p = 1: the measured one-launch solve).
E(p) = t_1 / (p t_p).  Inputs measured on one B200: factor 35.5 TF/s
(configs 3/4), POTRF 0.24 ms per 512 tile, host enqueue 0.016 ms per panel
step (the replayed schedule), one-GPU solves 9.2 ms (config 3)."""
import numpy as np

RATE = 35.5e12        # DMMA GEMM rate of the trailing update, flop/s
CRIT_MS = 0.40        # per-step critical path (POTRF 0.24 ms + TRSM + exchanges), ms
HOST_MS = 0.016       # host enqueue per panel step (profiles/r02_dist_world1_c3.txt: 15-16 us)
OVERHEAD = 0.0        # one-rank schedule vs single-GPU path at config 3 (2643.3 vs 2644.0 ms)
LAT_MS = 0.020        # NCCL latency of a small collective over NVLink (assumed, per call)
HBM = 6.5536e12       # bytes/s (MEASURED_PEAKS.json)
SOLVE1_MS = {65536: 9.2, 131072: 34.0}  # one-GPU one-launch solves (config 4: 4x config 3 bytes, scaled)
B = 512


def model(n, p, q):
    T = n // B
    world = p * q
    work = np.zeros(world)
    tiles = np.zeros(world)
    for i in range(T):
        for j in range(i + 1):
            r = (i % p) * q + (j % q)
            work[r] += j
            tiles[r] += 1
    imb = work.max() / work.mean()
    t1 = (n ** 3 / 3) / RATE * 1e3  # ms
    tail = 0.0
    for k in range(T):  # per-step update work of the busiest rank vs the critical path
        step = (T - k - 1) ** 2 / 2 * 2 * B ** 3 / RATE * 1e3 / world * imb
        tail += max(0.0, max(CRIT_MS, HOST_MS) - step)
    tf = t1 / world * imb * (1 + OVERHEAD) + tail
    if world == 1:
        ts = SOLVE1_MS[n]
    else:
        gemv = 2 * tiles.max() * B * B * 8 / HBM * 1e3  # two reads of the rank's tiles
        ts = 2 * T * 2 * LAT_MS + gemv
    return T, imb, tail, tf, ts, t1 + SOLVE1_MS[n]


if __name__ == "__main__":
    print("# tools/model_dist_chol.py: MODELLED (not measured) strong scaling of factor + solves")
    for n, name in [(65536, "config 3"), (131072, "config 4")]:
        for p, q in [(1, 1), (1, 2), (2, 2), (2, 4)]:
            T, imb, tail, tf, ts, t1 = model(n, p, q)
            eff = t1 / (p * q * (tf + ts))
            print(f"{name} n={n} T={T} {p}x{q}: imbalance {imb:.4f}, exposed tail {tail:.1f} ms, "
                  f"factor {tf:.0f} ms + solves {ts:.1f} ms, modelled efficiency {eff:.3f}")
