"""Host-side check of the balanced decode schedule's partition (binding.balanced_ranges,
the formula include/turbo_attention.h documents and decode.cu implements): the pieces
tile every (b, kv head) unit range in order, no chunk exceeds C units, every warp's
chunk is contiguous, and the part index bh + w is unique."""
import random

from paper_2412_08585_b200.binding import balanced_ranges


def _check(units, Hkv, W, min_units=8):
    rng = balanced_ranges(units, Hkv, W, min_units)
    total = sum(units) * Hkv
    C = max(min_units, -(-total // W))
    seen_parts, per_warp = set(), {}
    base = 0
    for b, U in enumerate(units):
        for h in range(Hkv):
            pieces = rng[(b, h)]
            assert [u0 for u0, _ in pieces[1:]] == [u1 for _, u1 in pieces[:-1]]
            if U == 0:
                assert pieces == []
            else:
                assert pieces[0][0] == 0 and pieces[-1][1] == U
            for u0, u1 in pieces:
                assert 0 < u1 - u0 <= C
                w = (base + u0) // C
                assert (base + u1 - 1) // C == w  # inside one warp's chunk
                assert w < W or total <= W * C
                part = b * Hkv + h + w
                assert part not in seen_parts
                assert part < len(units) * Hkv + W
                seen_parts.add(part)
                per_warp[w] = per_warp.get(w, 0) + (u1 - u0)
            base += U
    assert sum(per_warp.values()) == total
    assert all(v <= C for v in per_warp.values())


def test_balanced_partition_configs():
    _check([513] * 64, 10, 1776)     # configs[2] after one append
    _check([2049] * 16, 8, 1776)     # configs[4]
    _check([65] * 8, 8, 1776)        # bench step decode (C = 8: most warps idle)


def test_balanced_partition_random():
    r = random.Random(5)
    for _ in range(300):
        B, Hkv, W = r.randint(1, 9), r.randint(1, 6), r.randint(1, 300)
        units = [r.choice([0, 1, r.randint(1, 40), r.randint(1, 400)]) for _ in range(B)]
        _check(units, Hkv, W, r.choice([1, 8]))


def test_auto_splits_rule():
    """Equal-split heuristic: >= 8 blocks per split (or no split), no short last split,
    task count nearest 4.5 waves of the resident warps among the admissible counts."""
    from paper_2412_08585_b200.binding import auto_splits

    assert auto_splits(64, 10, 512, 1776) == 12   # configs[2]
    assert auto_splits(16, 8, 2048, 1776) == 64   # configs[4]
    assert auto_splits(8, 8, 64, 1776) == 8       # bench step decode (capped at 8 blocks per split)
    assert auto_splits(1, 1, 7, 1776) == 1
    assert auto_splits(1, 8, 2048, 1776) == 128   # B = 1 x 128k: at most 128 parts per combine row
    r = random.Random(3)
    for _ in range(200):
        B, H, nb, W = r.randint(1, 64), r.randint(1, 16), r.randint(0, 4096), r.randint(100, 4000)
        s = auto_splits(B, H, nb, W)
        assert s == 1 or (nb // s >= 8 and s <= 128)
        per = -(-nb // s)
        assert s == 1 or 4 * (nb - per * (s - 1)) >= 3 * per
