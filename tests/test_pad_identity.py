"""Host check of the shared-memory address identity the FP64 transform passes
rely on (csrc/he_internal.cuh ct_pass_dp / gs_pass_dp):

    PAD(base + (c << lt)) == PAD(base) + PAD(c << lt),   PAD(i) = i + (i >> 4),

for every radix-2^K group the passes form: base = (blk << (lt + K)) + off with
off < 2^lt, element c < 2^K at stride 2^lt.  The residues mod 16 of base and of
c << lt never sum past 15, so the padding words do not carry."""
import pytest


def pad(i):
    return i + (i >> 4)


@pytest.mark.parametrize("K", [1, 2, 3, 4])
def test_pad_splits_over_group_elements(K):
    for lt in range(0, 14):
        for blk in range(0, 9):
            for off in sorted({0, 1, (1 << lt) - 1, (1 << lt) // 2}):
                if off >= (1 << lt):
                    continue
                base = (blk << (lt + K)) + off
                for c in range(1 << K):
                    assert pad(base + (c << lt)) == pad(base) + pad(c << lt), (K, lt, blk, off, c)


def test_pad_identity_needs_the_group_structure():
    # a base with low bits past 2^lt breaks it (why the passes' base form matters)
    base, lt, c = 15, 0, 1
    assert pad(base + (c << lt)) != pad(base) + pad(c << lt)
