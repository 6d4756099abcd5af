"""Row f2's dispatch rule, kg_dispatch_threshold (include/kg.h): a pure
host function of the calibration samples, so it is tested here without a
device.  SPEC.md:399-410: the crossover is the first sampled size where the
other path wins, a tie goes to the small-request path (there: the device
"8KB or larger"; here: the NSK keeps ties), and dispatch is monotone."""
import random

import paper_1305_3345_b200 as kg

MAX = (1 << 64) - 1


def test_tie_goes_to_the_nsk():
    pts = [(4096, 10.0, 15.0), (8192, 12.0, 12.0), (16384, 20.0, 18.0), (32768, 30.0, 19.0)]
    assert kg.dispatch_threshold(pts) == 8192


def test_launch_wins_first_and_never():
    assert kg.dispatch_threshold([(4096, 12.0, 11.9), (8192, 13.0, 12.0)]) == 0
    assert kg.dispatch_threshold([(4096, 9.0, 11.9), (8192, 10.0, 12.0)]) == MAX
    assert kg.dispatch_threshold([]) == MAX


def test_first_crossing_wins_over_noise():
    """Noisy curves that cross twice: the first crossing decides, so every
    size above the threshold is launched (monotone)."""
    pts = [(4096, 10.0, 15.0), (8192, 14.0, 13.0), (16384, 15.0, 16.0), (32768, 30.0, 19.0)]
    assert kg.dispatch_threshold(pts) == 4096


def test_monotone_on_random_curves():
    rng = random.Random(1305)
    for _ in range(500):
        n = rng.randint(1, 14)
        pts = [(4096 << i, rng.uniform(5, 50), rng.uniform(5, 50)) for i in range(n)]
        thr = kg.dispatch_threshold(pts)
        nsk = [b <= thr for b, _, _ in pts]
        # NSK for a prefix of sizes, launches for the rest
        assert nsk == sorted(nsk, reverse=True)
        for (b, tn, tl), to_nsk in zip(pts, nsk):
            if to_nsk:
                assert tn <= tl, (pts, thr)
        first = next((i for i, (_, tn, tl) in enumerate(pts) if tl < tn), None)
        assert thr == (MAX if first is None else (0 if first == 0 else pts[first - 1][0]))
