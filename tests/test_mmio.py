"""Matrix Market ingest (multi-threaded parser) against the REFERENCE parser
(ingest.cpp:95-212, compiled into oracle/_ref), on the host -- no GPU.

Same CRS arrays bit for bit on well-formed files (general and symmetric,
unsorted, comments and blank lines between entries, trailing lines past the
declared count, odd number spellings), and the same status and message
(including the line number) on every malformed one.
"""
import os

import numpy as np
import pytest

from oracle.oracle import Ref


@pytest.fixture(scope="module")
def ref():
    try:
        return Ref()
    except FileNotFoundError as e:
        pytest.skip(str(e))


def _ours(sp, path):
    try:
        h = sp.HostCrs.read_matrix_market(path)
    except sp.SpmvtkError as e:
        return e.status, e.message, None
    rp, ci, v = h.arrays(index_base=1)
    h.free()
    return 0, "", (rp, ci, v)


def _theirs(ref, path):
    st, msg, h = ref.read_matrix_market(path)
    if st:
        return st, msg, None
    out = (ref.array(h, 1), ref.array(h, 3), ref.array(h, 0))
    ref.free(h)
    return 0, "", out


def _write(path, text):
    with open(path, "w") as f:
        f.write(text)
    return str(path)


def _random_file(rng, n, nnz, sym, extras):
    pairs = set()
    while len(pairs) < nnz:
        i, j = int(rng.integers(1, n + 1)), int(rng.integers(1, n + 1))
        if sym and j > i:
            i, j = j, i
        pairs.add((i, j))
    pairs = list(pairs)
    rng.shuffle(pairs)
    lines = ["%%MatrixMarket matrix coordinate real " + ("symmetric" if sym else "general"),
             "% a comment", "", f"{n} {n} {len(pairs)}"]
    spell = ["{:.17g}", "{:e}", "{:.3f}", "{}", "{:.6E}", "{:.1f}"]
    for k, (i, j) in enumerate(pairs):
        v = float(rng.standard_normal()) * 10 ** int(rng.integers(-5, 6))
        s = spell[k % len(spell)].format(v) if extras else "{:.17g}".format(v)
        lines.append(f"{i} {j} {s}")
        if extras and k % 97 == 0:
            lines.append("% interleaved comment")
        if extras and k % 131 == 0:
            lines.append("   ")
    if extras:
        lines.append("1 1 99.0")  # past the declared count: ignored by the reference
    return "\n".join(lines) + "\n"


@pytest.mark.parametrize("sym,extras,n,nnz", [(False, False, 50, 400), (True, False, 60, 500),
                                              (False, True, 3000, 40000),
                                              (True, True, 5000, 60000)])
def test_parser_matches_reference(sp, ref, tmp_path, sym, extras, n, nnz):
    rng = np.random.default_rng(n + nnz)
    path = _write(tmp_path / "m.mtx", _random_file(rng, n, nnz, sym, extras))
    a, b = _ours(sp, path), _theirs(ref, path)
    assert a[0] == b[0] == 0, (a[1], b[1])
    for x, y in zip(a[2], b[2]):
        assert x.tobytes() == y.tobytes()


BAD = {
    "empty": "",
    "banner": "%%MatrixMarket vector coordinate real general\n1 1 1\n1 1 1\n",
    "array": "%%MatrixMarket matrix array real general\n1 1\n1\n",
    "complex": "%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n",
    "skew": "%%MatrixMarket matrix coordinate real skew-symmetric\n1 1 0\n",
    "nosize": "%%MatrixMarket matrix coordinate real general\n% c\n",
    "badsize": "%%MatrixMarket matrix coordinate real general\n3 x 2\n",
    "nonsquare": "%%MatrixMarket matrix coordinate real general\n3 4 1\n1 1 1\n",
    "malformed": "%%MatrixMarket matrix coordinate real general\n3 3 2\n1 1 1\n2 two 3\n",
    "rowrange": "%%MatrixMarket matrix coordinate real general\n3 3 2\n1 1 1\n4 1 1\n",
    "colrange": "%%MatrixMarket matrix coordinate real general\n3 3 2\n1 1 1\n1 0 1\n",
    "short": "%%MatrixMarket matrix coordinate real general\n3 3 3\n1 1 1\n2 2 2\n",
    "dup": "%%MatrixMarket matrix coordinate real general\n3 3 3\n1 1 1\n3 2 2\n1 1 5\n",
    "symdup": "%%MatrixMarket matrix coordinate real symmetric\n3 3 2\n2 1 1\n1 2 5\n",
    "missingval": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1\n",
    "inf": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 inf\n",
    "hex": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 0x1p3\n",
    "plus": "%%MatrixMarket matrix coordinate real general\n2 2 1\n+1 +2 +3.5\n",
    "trailing": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 2 3.5 extra words\n",
    "dotnum": "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 2 .5\n2 1 5.\n",
    "crlf": "%%MatrixMarket matrix coordinate real general\r\n2 2 1\r\n1 2 3.25\r\n",
    "errafter": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 2 3\nbad line\n",
}


@pytest.mark.parametrize("name", sorted(BAD))
def test_refusals_and_edge_spellings_match_reference(sp, ref, tmp_path, name):
    path = _write(tmp_path / f"{name}.mtx", BAD[name])
    a, b = _ours(sp, path), _theirs(ref, path)
    assert a[0] == b[0], (name, a[:2], b[:2])
    if a[0]:
        # messages carry the path; compare what follows it
        assert a[1].split(os.sep)[-1] == b[1].split(os.sep)[-1], (name, a[1], b[1])
    else:
        for x, y in zip(a[2], b[2]):
            assert x.tobytes() == y.tobytes(), name
