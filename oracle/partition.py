"""Dyadic tree geometry — restatement of reference ``partition.py`` and
``construct.py:_level_geometry`` (test infrastructure; see oracle/__init__.py)."""

from __future__ import annotations


def check_partition(n: int, levels: int) -> None:
    """Validity rules of ``DyadicPartition.__post_init__`` (partition.py:25-34)."""
    if n < 4 or n & (n - 1):
        raise ValueError(f"matrix dimension must be a power of two >= 4, got {n}")
    if levels < 2 or levels % 2:
        raise ValueError(f"tree depth must be even and >= 2, got {levels}")
    if 2 ** (levels // 2) > n:
        raise ValueError(f"depth {levels} puts more than {n} nodes on the middle level")


def choose_levels(n: int, target_leaf: float) -> int:
    """Deepest even depth with n / 2**L >= target_leaf (partition.py:82-106)."""
    if not isinstance(n, int) or n < 4 or n & (n - 1):
        raise ValueError(f"n={n} admits no dyadic decomposition")
    if target_leaf <= 0:
        raise ValueError("target_leaf must be positive")
    best = -1
    max_depth = 2 * (n.bit_length() - 1)
    for depth in range(2, max_depth + 1, 2):
        if n / 2 ** depth >= target_leaf:
            best = depth
    if best < 0:
        raise ValueError(f"no even depth >= 2 leaves at least {target_leaf} indices per leaf")
    return best


def node_range(n: int, levels: int, lvl: int, i: int) -> range:
    """Ceil-rounded node range [ceil(i n / 2^l), ceil((i+1) n / 2^l)) (partition.py:62-70)."""
    if not 0 <= lvl <= levels:
        raise ValueError(f"level {lvl} outside [0, {levels}]")
    if not 0 <= i < 2 ** lvl:
        raise ValueError(f"node {i} outside level {lvl}")
    den = 1 << lvl
    lo = (i * n + den - 1) // den
    hi = ((i + 1) * n + den - 1) // den
    return range(lo, hi)


def level_geometry(n: int, levels: int, r: int):
    """Per-level transfer-array shapes and the leaf shape (construct.py:216-227).

    Returns ``([(lvl, splits, shape), ...] ascending from half, leaf_shape)``.
    """
    half = levels // 2
    nodes, rows = 2 ** half, n // 2 ** half
    table = []
    for lvl in range(half, levels):
        pairs = 2 ** (levels - lvl - 1)
        if rows >= 2:
            table.append((lvl, True, (nodes, 2, pairs, r, 2 * r)))
            nodes *= 2
            rows //= 2
        else:
            table.append((lvl, False, (nodes, pairs, r, 2 * r)))
    return table, (nodes, rows, r)
