"""Property tests (the reference's hypothesis style, test_planning.py / test_codegen.py):
the pitched device layout is a bijection that keeps every interior row 128-byte
aligned, and the corpus programs bound by the reference agree with its table."""

from __future__ import annotations

from hypothesis import given, settings, strategies as st

from paper_2309_04671_b200 import corpus


def device_layout(shape, order, elem):
    """Python statement of the C-ABI geometry (csrc/stkb200.cu stkb_domain_create)."""
    per128 = 128 // elem
    lead = max(per128, ((order + per128 - 1) // per128) * per128)
    pitch = ((lead + shape[2] + order + per128 - 1) // per128) * per128
    plane = pitch * (shape[1] + 2 * order)
    return lead, pitch, plane


@given(n=st.tuples(st.integers(1, 7), st.integers(1, 7), st.integers(1, 70)), order=st.integers(0, 4),
       elem=st.sampled_from([4, 8]))
@settings(max_examples=60, deadline=None)
def test_pitched_layout_bijection_and_alignment(n, order, elem):
    lead, pitch, plane = device_layout(n, order, elem)
    seen = set()
    for z in range(-order, n[0] + order):
        for y in range(-order, n[1] + order):
            row = (z + order) * plane + (y + order) * pitch + lead
            assert (row * elem) % 128 == 0  # interior x = 0 starts every row 128-B aligned
            for x in range(-order, n[2] + order):
                f = row + x
                assert 0 <= f < plane * (n[0] + 2 * order)
                assert f not in seen
                seen.add(f)
    assert len(seen) == (n[0] + 2 * order) * (n[1] + 2 * order) * (n[2] + 2 * order)


def test_corpus_flops_match_table():
    # star/box kernels are fully expanded weighted sums: 2P - 1 operators (corpus.py docstring)
    for name, k in corpus.KERNELS.items():
        if k.jacobi:
            continue
        shape = (8,) * k.dims
        bound, _ = corpus.corpus_target(name, shape, 1)
        info = bound.stmts[0].body[0].info
        points = len(corpus.offsets_of(k))
        assert info.flops_per_point == 2 * points - 1, name
        assert info.shape == k.shape and info.radius == k.radius
