"""Pure-Python CART restatement (TEST INFRASTRUCTURE ONLY, see oracle/__init__.py).

Restates /root/reference/pkg/src/adaptgemm/model.py:
  split_search   <- best_split   model.py:136-185 (exact integer scores)
  grow           <- train        model.py:194-232 (pre-order, left first)
  route          <- predict      model.py:235-241
  majority       <- _majority    model.py:188-191
  effective_leaf <- TrainConfig.effective_min_leaf model.py:51-55
Trees are returned as the reference's JSON node dicts so they can be
compared with both the reference's golden trees and the native product.
Written recursively on purpose (the reference and the product use explicit
stacks): agreement is evidence, not shared code.
"""

import math
from collections import Counter


def effective_leaf(min_samples_leaf, n_train: int) -> int:
    if isinstance(min_samples_leaf, int):
        return min_samples_leaf
    return max(1, math.ceil(min_samples_leaf * n_train))


def majority(labels) -> int:
    counts = Counter(labels)
    top = max(counts.values())
    return min(c for c, v in counts.items() if v == top)


def split_search(samples, min_leaf):
    """(feature, threshold, (num, den)) of the best split, or None."""
    n = len(samples)
    if n < 2 or n < 2 * min_leaf:
        return None
    parent = Counter(lab for _, lab in samples)
    if len(parent) < 2:
        return None
    psq = sum(c * c for c in parent.values())
    best = None
    for f in range(3):
        # group labels per distinct value, ascending
        groups = {}
        for feats, lab in samples:
            groups.setdefault(feats[f], Counter())[lab] += 1
        values = sorted(groups)
        left = Counter()
        n_l = 0
        for v, nxt in zip(values, values[1:]):
            left.update(groups[v])
            n_l += sum(groups[v].values())
            n_r = n - n_l
            if n_l < min_leaf or n_r < min_leaf:
                continue
            sq_l = sum(c * c for c in left.values())
            sq_r = sum((parent[lab] - left[lab]) ** 2 for lab in parent)
            num = sq_l * n_r + sq_r * n_l
            den = n_l * n_r
            if num * n <= psq * den:
                continue
            if best is None or num * best[2][1] > best[2][0] * den:
                best = (f, (v + nxt) / 2, (num, den))
    return best


def grow(records, max_height=None, min_samples_leaf=1):
    """The reference tree for (features, class_id) records, as node dicts."""
    records = list(records)
    min_leaf = effective_leaf(min_samples_leaf, len(records))
    nodes = []

    def build(samples, depth):
        idx = len(nodes)
        labels = [lab for _, lab in samples]
        split = None
        if len(set(labels)) > 1 and (max_height is None or depth < max_height):
            split = split_search(samples, min_leaf)
        if split is None:
            nodes.append({"class_id": majority(labels), "n_samples": len(samples)})
            return idx
        f, thr, _ = split
        node = {"feature": f, "threshold": thr, "left": -1, "right": -1}
        nodes.append(node)
        node["left"] = build([s for s in samples if s[0][f] <= thr], depth + 1)
        node["right"] = build([s for s in samples if s[0][f] > thr], depth + 1)
        return idx

    build(records, 0)
    return nodes


def route(nodes, features, root=0):
    node = nodes[root]
    while "class_id" not in node:
        node = nodes[node["left"] if features[node["feature"]] <= node["threshold"] else node["right"]]
    return node["class_id"]
