"""CPU oracle pinned against the known-answer material the reference offers for this path.

The reference's own tests are empty stubs (proj/tests/test_*.cpp), so the pins are:
  * Philox4x32-10 known-answer vectors (Random123, kat_vectors) for the synthetic-input contract;
  * SPEC.md worked examples of placement: the reshape pass-through examples
    and the exhaustive element-to-device map property on tensors <= 64 elements;
  * OwnerOfFlatIndex (proj/src/sharding.cpp:67-72) restated independently here in Python.
Numeric parity of op results is unpinned by the reference (ir.h:87): DESIGN.md §Semantics.
"""
import itertools

import numpy as np
import pytest

from paper_2302_08141_b200.abi import AxisSpec

KAT = [  # (ctr, key, expected) — Philox4x32-10, Random123 kat_vectors
    ([0, 0, 0, 0], [0, 0], [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]),
    ([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2, [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]),
    ([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0],
     [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]),
]


@pytest.mark.parametrize("ctr,key,want", KAT)
def test_philox_known_answers(oracle_lib, ctr, key, want):
    assert oracle_lib.philox(ctr, key) == want


def test_synthetic_value_contract(oracle_lib):
    # value = (int(word >> 8) - 2^23) / 2^23, word = Philox(ctr=(f/4, 0, seed_hi, 0), key=(seed, op))[f%4]
    for seed, op, f in [(0, 0, 0), (1, 3, 5), (2, 7, 1 << 20), (0x100000001, 2, 123457)]:
        blk = f >> 2
        w = oracle_lib.philox([blk & 0xFFFFFFFF, blk >> 32, seed >> 32, 0], [seed & 0xFFFFFFFF, op])[f & 3]
        v = np.float32((w >> 8) - 8388608) * np.float32(1.0 / 8388608.0)
        assert oracle_lib.synthetic_value(seed, op, f) == v
        scale = np.float32(np.sqrt(3.0 / 1024.0))
        assert oracle_lib.synthetic_value(seed, op, f, True, 1024) == np.float32(v * scale)
        assert -1.0 <= v < 1.0


def _owner_ref(dims, spec, d, f):
    """OwnerOfFlatIndex, proj/src/sharding.cpp:67-72."""
    inner = int(np.prod(dims[spec.dim + 1:], dtype=np.int64))
    coord = (f // inner) % dims[spec.dim]
    return (coord // spec.stride) % d


def _all_specs(dims, d):
    """enumerate_specs (proj/src/sharding.cpp:74-91), Shard part."""
    for dim, e in enumerate(dims):
        if e % d:
            continue
        q = e // d
        for s in range(1, q + 1):
            if q % s == 0:
                yield AxisSpec.shard(dim, s)


SMALL_SHAPES = [(8,), (16,), (4, 4), (8, 4), (4, 8), (2, 8), (16, 4), (4, 2, 4), (2, 4, 8), (64,),
                (8, 8), (2, 2, 2, 8)]


@pytest.mark.parametrize("dims", SMALL_SHAPES)
@pytest.mark.parametrize("d", [2, 4])
def test_element_to_device_map_exhaustive(oracle_lib, dims, d):
    """the element-to-device map, checked exhaustively on <= 64-element tensors; and
    every rank's local buffer holds its elements in ascending global order (the block-cyclic
    local coordinate the executor and oracle share)."""
    n = int(np.prod(dims))
    for spec in _all_specs(list(dims), d):
        owners = [oracle_lib.owner_of_flat(list(dims), spec, d, f) for f in range(n)]
        assert owners == [_owner_ref(list(dims), spec, d, f) for f in range(n)]
        for r in range(d):
            mine = [f for f in range(n) if owners[f] == r]
            assert len(mine) == n // d
            locs = [oracle_lib.local_of_flat(list(dims), spec, d, f) for f in mine]
            assert locs == list(range(n // d)), (dims, str(spec), r)


def _passthrough(in_dims, out_dims, spec, d):
    """ReshapePassthrough (proj/src/sharding.cpp:144-160)."""
    run = int(np.prod(in_dims[spec.dim + 1:])) * spec.stride
    for dim in range(len(out_dims)):
        inner = int(np.prod(out_dims[dim + 1:]))
        if run % inner:
            continue
        c = AxisSpec.shard(dim, run // inner)
        if out_dims[dim] % (d * c.stride) == 0:
            return c
    return None


@pytest.mark.parametrize("in_dims,out_dims,spec,d,want", [
    ((8, 4), (32,), AxisSpec.shard(0, 4), 2, AxisSpec.shard(0, 16)),
    ((4, 8), (8, 4), AxisSpec.shard(1, 1), 2, AxisSpec.shard(1, 1)),
])
def test_spec_reshape_examples(oracle_lib, in_dims, out_dims, spec, d, want):
    got = _passthrough(list(in_dims), list(out_dims), spec, d)
    assert got == want
    n = int(np.prod(in_dims))
    for f in range(n):  # byte-identical local buffers on both sides of the reshape
        assert oracle_lib.owner_of_flat(list(in_dims), spec, d, f) == oracle_lib.owner_of_flat(list(out_dims), got, d, f)
        assert oracle_lib.local_of_flat(list(in_dims), spec, d, f) == oracle_lib.local_of_flat(list(out_dims), got, d, f)


@pytest.mark.parametrize("dims", [(8, 4), (4, 2, 4), (16, 4)])
def test_passthrough_layout_identity_exhaustive(oracle_lib, dims):
    """SPEC.md:174 invariant for every pass-through the rule finds on these tensors."""
    n = int(np.prod(dims))
    shapes = [s for s in [(n,), (n // 2, 2), (2, n // 2), (n // 4, 4), (4, n // 4), (2, 2, n // 4)]]
    for d in (2, 4):
        for spec in _all_specs(list(dims), d):
            for out in shapes:
                got = _passthrough(list(dims), list(out), spec, d)
                if got is None:
                    continue
                for f in range(n):
                    assert oracle_lib.owner_of_flat(list(dims), spec, d, f) == oracle_lib.owner_of_flat(list(out), got, d, f)
                    assert oracle_lib.local_of_flat(list(dims), spec, d, f) == oracle_lib.local_of_flat(list(out), got, d, f)


TRANSITION_SPECS = ["replicated", "partial", "shard(0,1)", "shard(0,2)", "shard(1,1)", "shard(1,4)"]


@pytest.mark.parametrize("src,dst", [(a, b) for a, b in itertools.product(TRANSITION_SPECS, TRANSITION_SPECS)
                                     if a != b and not (a == "partial" and b == "partial")])
@pytest.mark.parametrize("d", [2, 4])
def test_reshard_semantics(oracle_lib, src, dst, d):
    """Single-axis transitions of sharding.cpp:104-142 on an [8,16] tensor: the assembled value
    is preserved; Partial sums in rank order; zero-fill for -> Partial."""
    dims = [8, 16]
    fs, ts = AxisSpec.from_string(src), AxisSpec.from_string(dst)
    rng = np.random.default_rng(0)
    full = rng.standard_normal(dims).astype(np.float32)
    n = full.size
    # build source buffers
    srcs = []
    if fs.kind == 2:  # partial: random addends summing (in rank order) to `total`
        parts = [rng.standard_normal(dims).astype(np.float32) for _ in range(d)]
        total = parts[0].copy()
        for p in parts[1:]:
            total = (total + p).astype(np.float32)
        srcs = [p.ravel() for p in parts]
        full = total
    else:
        for r in range(d):
            if fs.kind == 1:
                srcs.append(full.ravel().copy())
            else:
                idx = [f for f in range(n) if oracle_lib.owner_of_flat(dims, fs, d, f) == r]
                srcs.append(full.ravel()[idx].copy())
    nloc = n // d if ts.kind == 0 else n
    out = oracle_lib.reshard(d, dims, fs, ts, 0, srcs, nloc)
    for r in range(d):
        if ts.kind == 0:
            idx = [f for f in range(n) if oracle_lib.owner_of_flat(dims, ts, d, f) == r]
            np.testing.assert_array_equal(out[r], full.ravel()[idx])
        elif ts.kind == 1:
            np.testing.assert_array_equal(out[r], full.ravel())
        else:
            np.testing.assert_array_equal(out[r], full.ravel() if r == 0 else np.zeros(n, np.float32))
