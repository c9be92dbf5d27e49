"""Modelled multi-GPU efficiency of the 2D block-cyclic Cholesky (only one GPU
is reachable from this build, so this is a model, not a measurement).

E(p) = 1 / (imbalance * (1 + tail / T_p) * (1 + schedule overhead)), where
  imbalance  = max/mean over ranks of the trailing-update work (tile (i, j)
               receives j panel updates; exact count for the P x Q grid),
  tail       = steps whose per-rank update is shorter than the critical path
               (POTRF + panel TRSM + broadcasts, `crit_ms`) or than the host
               time to enqueue a step (`host_ms`, Python schedule + NCCL
               calls), summed exposure,
  T_p        = single-GPU factor time / p,
  overhead   = the distributed schedule on one rank with NCCL vs the fused
               single-GPU path (measured: 346.3 vs 337.3 ms at config 2).
Inputs measured on one B200: factor rate 35.5 TF/s (configs 3/4), POTRF
0.24 ms per 512 tile (8-CTA cluster), schedule overhead 2.7%, host enqueue
0.33 ms per step."""
import numpy as np

RATE = 35.5e12          # DMMA GEMM rate on the trailing update, flop/s
CRIT_MS = 0.40          # per-step critical path (POTRF 0.24 ms + TRSM + broadcasts), ms
HOST_MS = 0.33          # host time to enqueue one step (measured: 42 ms for T = 128, quick_dist1.py)
OVERHEAD = 346.3 / 337.3 - 1.0
B = 512


def model(n, p, q):
    T = n // B
    world = p * q
    work = np.zeros(world)
    for i in range(T):
        for j in range(i + 1):
            work[(i % p) * q + (j % q)] += j
    imb = work.max() / work.mean()
    t1 = (n ** 3 / 3) / RATE * 1e3  # ms
    tp = t1 / world
    tail = 0.0
    for k in range(T):  # per-step update work of the busiest rank vs the critical path
        step = (T - k - 1) ** 2 / 2 * 2 * B ** 3 / RATE * 1e3 / world * imb
        tail += max(0.0, max(CRIT_MS, HOST_MS) - step)
    eff = 1.0 / (imb * (1 + tail / tp) * (1 + OVERHEAD))
    return T, imb, tail, tp, eff


if __name__ == "__main__":
    for n, name in [(65536, "config 3"), (131072, "config 4")]:
        for p, q in [(1, 2), (2, 2), (2, 4)]:
            T, imb, tail, tp, eff = model(n, p, q)
            print(f"{name} n={n} T={T} {p}x{q}: imbalance {imb:.4f}, exposed tail {tail:.1f} ms "
                  f"of {tp:.0f} ms, modelled efficiency {eff:.3f}")
