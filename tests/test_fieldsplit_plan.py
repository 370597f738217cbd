"""f3 field split: host-side planning (CPU): slices, waves, tile counts, slot sizes."""
import pytest

from paper_1705_08213_b200 import ccc, fieldsplit


def test_field_slices_cover_and_balance():
    for n_f, world in [(10, 3), (50000, 8), (7, 7), (129, 2)]:
        sl = fieldsplit.field_slices(n_f, world)
        assert sl[0][0] == 0 and sl[-1][1] == n_f
        assert all(a[1] == b[0] for a, b in zip(sl, sl[1:]))
        sizes = [b - a for a, b in sl]
        assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        fieldsplit.field_slices(3, 4)


def test_waves_partition_the_schedule():
    assert fieldsplit.waves(5, 2) == [(0, 2), (2, 4), (4, 5)]
    assert fieldsplit.waves(5, None) == [(0, 5)]
    assert fieldsplit.waves(0, 3) == []


def test_tile_count_and_slot_bytes():
    # diag schedule of ccc_2way_block: upper-triangular 256-row (CTA pair) x 256-col tiles
    for n_v in (2, 256, 257, 1000, 20000):
        nb = (n_v + 255) // 256
        want = sum(1 for i in range(nb) for j in range(i, nb)
                   if i * 256 < min(n_v, (j + 1) * 256) - 1)   # tiles holding some i < j
        assert ccc.ccc_2way_fs_tiles(n_v) == want
    assert ccc.ccc_2way_fs_tiles(1) == 0
    # owner of t is t mod world: ceil(9 / 4) = 3 tiles per owner x 4 slices x 256 KB
    assert ccc.ccc_2way_fs_slot_bytes(4, 0, 9) == 3 * 4 * 65536 * 4
    assert ccc.ccc_2way_fs_slot_bytes(4, 5, 5) == 0
