"""GFA ingest (pgl_gfa_parse_*) against the reference's parse_gfa + build_graph
(gfa.cpp:57-153, graph.cpp:7-59), host-only (no GPU needed).

Bars: node lengths, edges, path names, PathStep records (offset, node, length,
orientation) and skipped_records identical; on malformed input the same
exception class and message as the reference (which throws the first failure
in its two-pass line order)."""
import numpy as np
import pytest

from oracle_ffi import CheckerError


def same_graph(pgl, ref, ours, theirs, skipped):
    fo = ref.export(theirs)
    assert ours.n_nodes == theirs.n_nodes
    assert np.array_equal(ours.node_len, fo.node_len)
    assert ours.n_paths == theirs.n_paths
    assert ours.total_steps() == theirs.total_steps
    offs = np.concatenate([s["offset"] for s in ours.path_steps]) if ours.n_paths else np.zeros(0)
    nodes = np.concatenate([s["node_id"] for s in ours.path_steps])
    lens = np.concatenate([s["seq_len"] for s in ours.path_steps])
    rev = np.concatenate([s["orient"] for s in ours.path_steps])
    assert np.array_equal(offs, fo.step_off)
    assert np.array_equal(nodes, fo.step_node)
    assert np.array_equal(lens, fo.step_len)
    assert np.array_equal(rev, fo.step_rev)
    assert np.array_equal(ours.path_total_len, fo.path_total)
    f, fe, t, te = ref.edges(theirs)
    assert len(ours.edges) == theirs.n_edges
    assert np.array_equal(ours.edges["from"], f) and np.array_equal(ours.edges["to"], t)
    assert np.array_equal(ours.edges["from_end"], fe) and np.array_equal(ours.edges["to_end"], te)
    assert ours.path_names == ref.path_names(theirs)
    assert ours.skipped_records == skipped


def parse_both(pgl, ref, text, threads=0):
    theirs, skipped = ref.parse_gfa(text)
    ours = pgl.parse_gfa(text, threads=threads)
    return ours, theirs, skipped


HAND = (
    "H\tVN:Z:1.0\n"
    "# a comment line\n"
    "S\tchr1_a\tACGTACGT\n"
    "S\tx\t*\tRC:i:4\tLN:i:12\r\n"
    "S\tbb\tAC\tLN:i:99\n"
    "L\tchr1_a\t+\tx\t-\t0M\n"
    "X\tunknown\trecord\n"
    "\n"
    "L\tx\t-\tbb\t+\t*\n"
    "P\thap one\tchr1_a+,x-,bb+,x+\t*\n"
    "S\tlate\t*\tLN:i:7\n"
    "P\thap2\tlate-,chr1_a+,\t*\n"
    "C\tcontainment\n"
    "\tleading tab\n"
    "P\thap3\tbb-\t*"  # no trailing newline
)


def test_gfa_hand_written_matches_reference(pgl, ref):
    ours, theirs, skipped = parse_both(pgl, ref, HAND)
    same_graph(pgl, ref, ours, theirs, skipped)
    assert ours.path_names == ["hap one", "hap2", "hap3"]
    assert ours.skipped_records == 3  # X, C and the tab-led line (gfa.cpp:151)


def test_gfa_roundtrip_generated(pgl, ref, tmp_path):
    """write_gfa output of generated graphs (numeric names, fast name table)."""
    for args in [(1, 9680, 8, 0.05), (3, 50, 4, 0.3), (7, 200000, 2, 0.2)]:  # the last: P lines > 1 MiB
        g = ref.generate(*args)
        path = str(tmp_path / "g.gfa")
        ref.write_gfa(g, path)
        theirs, skipped, _ = ref.parse_gfa_file(path)
        for threads in (1, 3, 0):
            ours = pgl.parse_gfa_file(path, threads=threads)
            same_graph(pgl, ref, ours, theirs, skipped)


def test_gfa_hashed_names_many_segments(pgl, ref):
    """Non-numeric names (hash table path) over many chunks."""
    rng = np.random.default_rng(5)
    n = 30000
    names = [f"seg{k * 7919 % 100003:06d}x" for k in range(n)]
    lens = rng.integers(1, 40, n)
    lines = ["H\tVN:Z:1.0"] + [f"S\t{names[k]}\t*\tLN:i:{lens[k]}" for k in range(n)]
    lines += [f"L\t{names[k]}\t+\t{names[k + 1]}\t+\t0M" for k in range(0, n - 1, 3)]
    for p in range(4):
        idx = rng.integers(0, n, 5000)
        lines.append(f"P\tp{p}\t" + ",".join(names[i] + "+-"[int(i) & 1] for i in idx) + "\t*")
    text = "\n".join(lines) + "\n"
    ours, theirs, skipped = parse_both(pgl, ref, text)
    same_graph(pgl, ref, ours, theirs, skipped)


ERRORS = [
    "S\ta\tAC\nW\tx\n",                                   # W rejected (pass 2)
    "S\ta\n",                                             # S needs name and sequence
    "S\t\tAC\nP\tp\ta+\t*\n",                              # empty segment name
    "S\ta\tAC\nS\tb\tA\nS\ta\tG\nS\tb\tT\nP\tp\ta+\t*\n",  # duplicate: the first repeat (line 3)
    "S\t3\tAC\nS\t03\tA\nS\t3\tG\nP\tp\t3+\t*\n",          # numeric-looking duplicate
    "S\ta\t*\tLN:i:x1\n",                                 # bad LN value
    "S\ta\t*\tLN:i:0\n",                                  # zero LN
    "S\ta\t*\tLN:i:18446744073709551616\n",               # LN overflow
    "S\ta\t*\tXX:i:3\n",                                  # '*' without LN
    "S\ta\t\n",                                           # zero-length sequence
    "S\ta\tA\nL\ta\t+\ta\t+\n",                             # L needs 6 columns
    "S\ta\tA\nL\ta\t++\ta\t+\t0M\n",                        # bad orientation column
    "S\ta\tA\nL\tq\t+\ta\t?\t0M\n",                         # unknown from (before orientation)
    "S\ta\tA\nL\ta\t+\tq\t+\t0M\n",                         # unknown to
    "S\ta\tA\nL\ta\t?\ta\t+\t0M\n",                         # bad orientation char
    "S\ta\tA\nP\tp\ta+\n",                                 # P needs 4 columns
    "S\ta\tA\nP\tp\t\t*\n",                                # empty path
    "S\ta\tA\nP\tp\ta+,,a+\t*\n",                          # bad path step ''
    "S\ta\tA\nP\tp\t,a+\t*\n",                             # bad path step '' first
    "S\ta\tA\nP\tp\ta+,a*\t*\n",                           # bad orientation in a step
    "S\ta\tA\nP\tp\ta+,zz-,a+,q\t*\n",                      # unknown segment (first failing token)
    "S\ta\tA\nL\ta\t+\ta\t+\t0M\n",                         # no P records
    "S\ta\tA\nP\tp\tq+\t*\nS\tb\n",                         # pass-1 failure wins over an earlier pass-2 one
    "S\ta\tA\nP\tp\ta+\t*\nP\tq\t\t*\nL\tz\t+\ta\t+\t0M\n",   # the first pass-2 failure in line order
    "S\ta\t*\tLN:i:4294967296\nP\tp\ta+\t*\n",             # node longer than a step record (build_graph)
    "",                                                    # empty input
]


@pytest.mark.parametrize("text", ERRORS)
def test_gfa_errors_match_reference(pgl, ref, text):
    with pytest.raises(CheckerError) as want:
        ref.parse_gfa(text)
    with pytest.raises(pgl.Error) as got:
        pgl.parse_gfa(text)
    assert str(got.value) == str(want.value)


def test_gfa_error_in_a_late_piece(pgl, ref):
    """A bad token deep inside a multi-piece P line, and another in a later
    line: the earliest (line, token) wins, as in the serial parser."""
    n = 300000
    toks = ["1+"] * n
    toks[250000] = "2?"
    text = "S\t1\tACGT\nS\t2\tA\nP\tp\t" + ",".join(toks) + "\t*\nP\tq\t3+\t*\n"
    with pytest.raises(CheckerError) as want:
        ref.parse_gfa(text)
    with pytest.raises(pgl.Error) as got:
        pgl.parse_gfa(text, threads=8)
    assert str(got.value) == str(want.value)


def test_gfa_file_errors(pgl, tmp_path):
    with pytest.raises(pgl.InvalidParameter):
        pgl.parse_gfa_file(str(tmp_path / "missing.gfa"))
