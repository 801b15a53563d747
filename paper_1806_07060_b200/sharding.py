"""Shape-wise sharding of tuning sweeps over GPUs (no collectives).

Shapes are independent (tuner.py:175-185), so a sweep is partitioned
statically, longest-processing-time first, over one worker process per GPU;
each worker writes its own `tables/<M>x<N>x<K>.csv` files and the shared
output directory is the only gather (cli.py:212-220 with processes bound to
GPUs instead of CPU cores).
"""

import heapq

# per-config fixed cost of one device-timed measurement (warmup + graph
# capture + repeats of a tiny kernel) and a mean throughput over the space
CONFIG_OVERHEAD_S = 6e-4
MEAN_SWEEP_FLOPS = 8e12


def sweep_cost(mnk, n_configs: int, samples_per_config: int = 8) -> float:
    """Estimated seconds to sweep one shape."""
    m, n, k = mnk
    return n_configs * (CONFIG_OVERHEAD_S + samples_per_config * 2.0 * m * n * k / MEAN_SWEEP_FLOPS)


def lpt_partition(items, n_parts: int, cost) -> list:
    """Greedy LPT: items sorted by decreasing cost, each to the least loaded part.

    Deterministic (ties by original position, then part index); every part
    keeps its items in their original relative order.
    """
    if n_parts < 1:
        raise ValueError("n_parts must be >= 1")
    items = list(items)
    order = sorted(range(len(items)), key=lambda i: (-cost(items[i]), i))
    heap = [(0.0, p) for p in range(n_parts)]
    parts = [[] for _ in range(n_parts)]
    for i in order:
        load, p = heapq.heappop(heap)
        parts[p].append(i)
        heapq.heappush(heap, (load + cost(items[i]), p))
    return [[items[i] for i in sorted(p)] for p in parts]
