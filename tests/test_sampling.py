"""The encoded-row candidate samplers (sampling.py) against the reference's own samplers: same rows
in the same order and the same generator state afterwards (host code; the reference is shipped in
oracle/_ref or read from /root/reference)."""
import numpy as np
import pytest

from paper_2212_11142_b200 import sampling, scenarios
from paper_2212_11142_b200.layout import SpaceLayout, pack_perm

pytestmark = pytest.mark.reference


@pytest.fixture(scope="module")
def ref():
    from golden_io import ref as load_ref
    return load_ref()


def _same_state(a, b):
    assert repr(a.bit_generator.state) == repr(b.bit_generator.state)
    assert np.array_equal(a.integers(1 << 62, size=7), b.integers(1 << 62, size=7))  # and the stream on


@pytest.mark.parametrize("m", [1, 2, 3, 4, 5, 7, 9, 16])
@pytest.mark.parametrize("n,odd", [(0, False), (1, True), (5, False), (300, True), (300, False)])
def test_permutations_replay_numpy(m, n, odd):
    """bx_pcg64_permutations = n calls of Generator.permutation(m), with the 32-bit buffer either
    empty or holding a half-used draw (odd)."""
    for seed in (0, 7, 12345):
        a, b = np.random.default_rng(seed), np.random.default_rng(seed)
        if odd:  # one bounded 32-bit draw leaves the high half buffered
            a.integers(10), b.integers(10)
        got = sampling.permutation_rows(a, n, m)
        want = np.array([pack_perm(b.permutation(m) + 1, m) for _ in range(n)], dtype=np.uint64)
        assert np.array_equal(got, want)
        _same_state(a, b)


def test_permutations_other_bit_generators():
    """Non-PCG64 generators take the permutations from rng.permutation itself."""
    a, b = np.random.Generator(np.random.Philox(3)), np.random.Generator(np.random.Philox(3))
    got = sampling.permutation_rows(a, 50, 6)
    want = np.array([pack_perm(b.permutation(6) + 1, 6) for _ in range(50)], dtype=np.uint64)
    assert np.array_equal(got, want)
    _same_state(a, b)


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
def test_uniform_rows_are_the_reference_pool(ref, name):
    """uniform_rows = encode(sample_uniform(space, n, rng)) (space.py:312-332), state included."""
    space = scenarios.build_space(name, ref.space)
    lay = SpaceLayout(space)
    for seed, n in ((1, 1), (2, 5000), (3, 777)):
        a, b = np.random.default_rng(seed), np.random.default_rng(seed)
        got = sampling.uniform_rows(lay, n, a)
        want = lay.encode(ref.space.sample_uniform(space, n, b))
        assert np.array_equal(got, want)
        _same_state(a, b)
        assert lay.decode(got) == lay.decode(want)


def test_unique_rows_is_dict_fromkeys(ref):
    """First-occurrence de-duplication in draw order on a small discrete space full of repeats."""
    space = ref.space.SearchSpace([ref.space.Parameter("a", "ordinal", values=(1, 2, 4)),
                                   ref.space.Parameter("b", "categorical", values=("x", "y")),
                                   ref.space.Parameter("p", "permutation", size=3)])
    lay = SpaceLayout(space)
    a, b = np.random.default_rng(9), np.random.default_rng(9)
    got = sampling.unique_rows(sampling.uniform_rows(lay, 400, a))
    want = list(dict.fromkeys(ref.space.sample_uniform(space, 400, b)))
    assert lay.decode(got) == want
    assert np.array_equal(got, lay.encode(want))


def test_rejection_rows_follow_the_reference_front_end(ref):
    """rejection_rows = the reference's rejection sampler (acquisition.py:122-134) on a space with
    known constraints (feasibility evaluated on the host here)."""
    from boxtune.constraints import eval_constraint
    from boxtune.acquisition import _default_sampler
    space = scenarios.build_space("C2", ref.space)
    assert space.constraints
    lay = SpaceLayout(space)

    def feasible(rows):
        return [all(eval_constraint(c, space.as_dict(cfg)) is True for c in space.constraints)
                for cfg in lay.decode(rows)]

    for seed, n in ((4, 300), (5, 1)):
        a, b = np.random.default_rng(seed), np.random.default_rng(seed)
        got = sampling.rejection_rows(lay, n, a, feasible)
        want = _default_sampler(space, None)(n, b)
        assert lay.decode(got) == want
        _same_state(a, b)


@pytest.mark.parametrize("pop,k", [(1, 1), (2, 1), (5, 2), (21, 5), (100, 10), (100, 100), (10000, 3), (30, 0)])
def test_choice_replays_numpy(pop, k):
    """bx_pcg64_choice = n calls of Generator.choice(pop, size=k, replace=False) (the rf_fit feature
    subsets), generator state included."""
    for seed, odd in ((0, False), (3, True), (99, False)):
        a, b = np.random.default_rng(seed), np.random.default_rng(seed)
        if odd:
            a.integers(10), b.integers(10)
        got = sampling.choice_rows(a, 200, pop, k)
        want = np.array([b.choice(pop, size=k, replace=False) for _ in range(200)], dtype=np.int32).reshape(200, k)
        assert np.array_equal(got, want)
        _same_state(a, b)


@pytest.mark.parametrize("name", ["C2", "C3", "C4"])
def test_cot_rows_are_the_reference_leaf_uniform_pool(ref, name):
    """cot_rows = encode(cot.sample_leaf_uniform(n, rng)) (constraints.py:471-518): tree groups,
    permutation singletons, generator state included."""
    space = scenarios.build_space(name, ref.space)
    cot = ref.build_cot(space)
    lay = SpaceLayout(space)
    for seed, n in ((1, 1), (2, 5000), (3, 333)):
        a, b = np.random.default_rng(seed), np.random.default_rng(seed)
        got = sampling.cot_rows(lay, cot, n, a)
        want = cot.sample_leaf_uniform(n, b)
        assert lay.decode(got) == want
        assert np.array_equal(got, lay.encode(want))
        _same_state(a, b)


def test_cot_rows_real_and_permutation_singletons(ref):
    """A chain of trees with a real and a permutation singleton next to a constrained pair."""
    S = ref.space
    space = S.SearchSpace([S.Parameter("a", "ordinal", values=(1, 2, 4, 8)),
                           S.Parameter("x", "real", lo=0.5, hi=3.0),
                           S.Parameter("b", "integer", lo=1, hi=6),
                           S.Parameter("p", "permutation", size=4)],
                          constraints=["a * b <= 12"])
    cot = ref.build_cot(space)
    assert sorted(g.kind for g in cot.groups) == ["permutation", "real", "tree"]
    lay = SpaceLayout(space)
    a, b = np.random.default_rng(8), np.random.default_rng(8)
    got = sampling.cot_rows(lay, cot, 2000, a)
    want = cot.sample_leaf_uniform(2000, b)
    assert lay.decode(got) == want
    _same_state(a, b)


def test_replay_self_check_passes_on_this_numpy():
    """The one-time check that guards the PCG64 replays holds for the NumPy in this image."""
    assert sampling.replay_ok()


@pytest.mark.parametrize("n,pop,k", [(1, 1, 1), (2, 13, 4), (40, 13, 4), (200, 30, 5), (7, 100, 10)])
def test_tree_streams_replay_the_per_tree_generators(n, pop, k):
    """TreeStreams (bx_pcg64_forest_draws: SeedSequence + PCG64 seeding, the bootstrap integers and
    the feature subsets) = np.random.default_rng(seed) per tree, continuations included."""
    seeds = np.random.default_rng(n).integers(0, 2 ** 32, size=60, dtype=np.uint64)
    seeds[:3] = [0, 1, 2 ** 32 - 1]
    f = sampling.TreeStreams(seeds, n, pop, k, 6)
    assert f.native
    for t in (0, 1, 2, 31, 59):
        g = np.random.default_rng(int(seeds[t]))
        assert np.array_equal(f.boot[t], g.integers(0, n, size=n))
        f.more(t, 5)
        assert np.array_equal(f.draws[t], np.array([g.choice(pop, size=k, replace=False) for _ in range(11)]))
        f.more(t, 1)
        assert np.array_equal(f.draws[t][-1], g.choice(pop, size=k, replace=False))
