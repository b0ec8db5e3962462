"""Layout table IO (pgl_layout_write_tsv / pgl_layout_read_tsv) against the
reference's write_layout_tsv / read_layout_tsv (layout_io.cpp:31-110),
host-only. Bars: written files byte-identical; read-back coordinates
bit-identical; malformed tables raise the same exception class and message."""
import numpy as np
import pytest

from oracle_ffi import CheckerError


def layouts():
    rng = np.random.default_rng(3)
    yield np.zeros(0)
    yield np.array([0.0, -0.0, 1e-300, 5e-324])
    yield rng.normal(0, 1e7, 4 * 1000)
    yield np.concatenate([rng.uniform(-1, 1, 4 * 50000) * 10.0 ** rng.integers(-20, 20, 4 * 50000)])
    yield np.arange(4 * 200001, dtype=np.float64) / 3.0


@pytest.mark.parametrize("k", range(5))
def test_write_tsv_byte_identical(pgl, ref, tmp_path, k):
    lay = list(layouts())[k]
    a, b = str(tmp_path / "ours.tsv"), str(tmp_path / "ref.tsv")
    pgl.write_layout_tsv(a, lay)
    ref.write_layout_tsv(b, lay)
    assert open(a, "rb").read() == open(b, "rb").read()
    back = pgl.read_layout_tsv(a)
    assert back.tobytes() == np.asarray(lay, np.float64).tobytes()
    assert ref.read_layout_tsv(a).tobytes() == back.tobytes()


def test_write_tsv_nonfinite_names_lowest_node(pgl, ref, tmp_path):
    lay = np.ones(4 * 100000)
    lay[4 * 70000 + 2] = np.inf
    lay[4 * 90001] = np.nan
    with pytest.raises(CheckerError) as want:
        ref.write_layout_tsv(str(tmp_path / "r.tsv"), lay)
    with pytest.raises(pgl.Error) as got:
        pgl.write_layout_tsv(str(tmp_path / "o.tsv"), lay)
    assert str(got.value) == str(want.value)


H = "node_id\tstart_x\tstart_y\tend_x\tend_y\n"
READ_ERRORS = [
    "",
    "\n",
    "node_id\tstart_x\n",
    H + "0\t1\t2\t3\n",
    H + "0\t1\t2\t3\t4\t5\n",
    H + "0\t1\t2\t3\t4\n2\t1\t2\t3\t4\n",
    H + "0\t1\t2\t3\t4\n\n1\t1\t2\tx\t4\n",
    H + "-1\t1\t2\t3\t4\n",
    H + "0\t1\t2\t3\t4 \n",
    H + "0\t1\t2\t3\t4\n1\tnan\t2\t3\t4\n3\t1\t1\t1\t1\n" + "".join(f"{k}\t1\t2\t3\t4\n" for k in range(2, 50000)),
]


@pytest.mark.parametrize("text", READ_ERRORS)
def test_read_tsv_errors_match_reference(pgl, ref, tmp_path, text):
    p = str(tmp_path / "t.tsv")
    with open(p, "w") as f:
        f.write(text)
    try:
        want = ref.read_layout_tsv(p)
        werr = None
    except CheckerError as e:
        werr = str(e)
    try:
        got = pgl.read_layout_tsv(p)
        gerr = None
    except pgl.Error as e:
        gerr = str(e)
    assert gerr == werr
    if werr is None:
        assert got.tobytes() == want.tobytes()


def test_read_tsv_crlf_and_blank_lines(pgl, ref, tmp_path):
    p = str(tmp_path / "t.tsv")
    with open(p, "w", newline="") as f:
        f.write("node_id\tstart_x\tstart_y\tend_x\tend_y\r\n0\t1.5\t-2\t3e5\t4\r\n\r\n1\t0x1p3\t1\t1\t1")
    try:
        want, werr = ref.read_layout_tsv(p), None
    except CheckerError as e:
        want, werr = None, str(e)
    try:
        got, gerr = pgl.read_layout_tsv(p), None
    except pgl.Error as e:
        got, gerr = None, str(e)
    assert gerr == werr
    if werr is None:
        assert got.tobytes() == want.tobytes()
