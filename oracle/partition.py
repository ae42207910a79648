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


def level_geometry(n: int, levels: int, r: int, branching: int = 2):
    """Per-level transfer-array shapes and the leaf shape (construct.py:216-227).

    Returns ``([(lvl, splits, shape), ...] ascending from half, leaf_shape)``.
    ``branching`` = 4 is the quadtree generalisation (BASELINE configs 3/4b; no
    reference code — DESIGN.md "2-D"): b row parts, b*r-wide blocks.
    """
    b = branching
    half = levels // 2
    nodes, rows = b ** half, n // b ** half
    table = []
    for lvl in range(half, levels):
        pairs = b ** (levels - lvl - 1)
        if rows >= b:
            table.append((lvl, True, (nodes, b, pairs, r, b * r)))
            nodes *= b
            rows //= b
        else:
            table.append((lvl, False, (nodes, pairs, r, b * r)))
    return table, (nodes, rows, r)


def quadtree_levels(n_side: int, leaf_box: int) -> int:
    """Even quadtree depth with leaf boxes leaf_box x leaf_box on an n_side^2 grid."""
    if n_side & (n_side - 1) or leaf_box & (leaf_box - 1) or leaf_box > n_side:
        raise ValueError("grid and leaf box sides must be powers of two")
    depth = (n_side // leaf_box).bit_length() - 1
    if depth < 2 or depth % 2:
        raise ValueError(f"quadtree depth {depth} must be even and >= 2")
    return depth
