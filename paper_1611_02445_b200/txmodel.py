"""Bandwidth model of the step (txmodel.py:48-68) used by the bench's roofline.

B_node = 2 * q * n_d bytes moved per non-solid node per step (each value read
once and written once): 304 B fp64, 152 B fp32.  The
per-tile metadata the B200 kernel also reads (64 x 4 B node words + 27 x 4 B
neighbour row per tile) is reported separately by ``metadata_bytes``.
"""

SEGMENT_BYTES = 32
_PRECISION_BYTES = {"f64": 8, "f32": 4}


def value_bytes(precision):
    if precision not in _PRECISION_BYTES:
        raise ValueError(f"unknown precision: {precision!r}")
    return _PRECISION_BYTES[precision]


def m_node(q=19, n_d=8):
    if q <= 0 or n_d <= 0:
        raise ValueError(f"q and n_d must be positive: q={q}, n_d={n_d}")
    return q * n_d


def b_node(q=19, n_d=8):
    return 2 * m_node(q, n_d)


def flop_per_byte(flop_count, bytes_per_node):
    if bytes_per_node <= 0:
        raise ValueError(f"bytes per node must be positive: {bytes_per_node}")
    if flop_count < 0:
        raise ValueError(f"FLOP count must be non-negative: {flop_count}")
    return flop_count / bytes_per_node


def metadata_bytes(t_n):
    """Bytes of per-tile metadata one step reads: node words + neighbour row."""
    return t_n * (64 * 4 + 27 * 4)
