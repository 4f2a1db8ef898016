"""Idle-lane model of k_hash_s1_var (config 4: entry lengths uniform in
64..1024 B): a warp runs 2 * nb1 + 1 compression jobs per entry (nb1 = the
second hash stream's block count) and its lanes idle while the longest entry
of the warp finishes. Prints the idle fraction for the shipped scheme (tiles
of 1024 entries sorted by block count, 32 consecutive sorted entries per
warp-iteration), for larger sort pools (2048 / 4096 entries = two / four
epochs per tile), and for a flattened job loop (a lane starts its next entry
without waiting; divergent entry transitions charged at 6 % of a job)."""
import numpy as np

rng = np.random.default_rng(5)


def nb(m):
    return (m + 9 + 63) // 64


def pool(T, tiles=200):
    idle = work = 0
    for _ in range(tiles):
        L = rng.integers(64, 1025, size=T)
        J = np.sort(2 * nb(L + 17) + 1)[::-1]
        for w in range(0, T, 32):
            seg = J[w:w + 32]
            idle += (seg.max() - seg).sum()
            work += seg.sum()
    return idle / (idle + work)


def flat(tiles=200, snake=True, trans_cost=0.06):
    idle = work = extra = 0
    for _ in range(tiles):
        L = rng.integers(64, 1025, size=1024)
        J = np.sort(2 * nb(L + 17) + 1)[::-1]
        for w in range(4):
            M = np.array([J[(((w + it) % 4) + 4 * it) * 32:][:32][::(-1 if snake and it % 2 else 1)] for it in range(8)])
            tot = M.sum(0)
            idle += (tot.max() - tot).sum()
            work += tot.sum()
            cum = np.cumsum(M, 0)
            extra += sum(len(set(cum[i])) for i in range(8)) * trans_cost * 32
    return idle / (idle + work), extra / (idle + work)


if __name__ == "__main__":
    for T in (1024, 2048, 4096):
        print(f"sort pool {T}: idle {pool(T):.4f}")
    i, x = flat()
    print(f"flattened loop (snake order): idle {i:.4f} + transitions {x:.4f} = {i + x:.4f}")
