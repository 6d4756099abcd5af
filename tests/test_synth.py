"""The seeded generator and shard arithmetic (host logic, no GPU)."""
import numpy as np
import pytest

import synth


def test_splitmix64_reference_values():
    # splitmix64 (Steele, Lea, Flood 2014; Vigna's reference C) seeded with 0
    # yields e220a8397b1dcdaf, 6e789e6aa1b965f4, 06c45d188009454f.
    w = synth.splitmix64_words(0, 3)
    assert [int(x) for x in w] == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]


def test_stream_offsets_consistent():
    a = synth.stream_bytes(123, 4096)
    b = synth.stream_bytes(123, 1024, offset=2048)
    assert np.array_equal(a[2048:3072], b)
    p = synth.make_pages(10, 512)
    q = synth.make_pages(3, 512, first_page=4)
    assert np.array_equal(p[4 * 512:7 * 512], q)


@pytest.mark.parametrize("n", [1, 7, 8, 9, 65536, 16777216, 1000003])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_shards_cover_disjoint(n, world):
    ranges = [synth.shard(n, r, world) for r in range(world)]
    assert ranges[0][0] == 0 and ranges[-1][1] == n
    for (a, b), (c, d) in zip(ranges, ranges[1:]):
        assert b == c and a <= b
    sizes = [b - a for a, b in ranges]
    assert max(sizes) - min(sizes) <= 1
