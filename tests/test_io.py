"""io.hpp parity (no GPU): SCNB / CSV scenario files, the instance grammar and
report rendering of the drop-in facade (tests/cpp/facade_main, linked against
libscendp_b200.so) and of the SCNB C-ABI, against the real reference
(oracle/_ref).  Files must be byte-identical, parsed instances identical
field by field, and error messages identical (reference: proj/src/io.cpp)."""
import ctypes as C
import os
import struct
import subprocess

import numpy as np
import pytest

from paper_2602_05179_b200 import _capi as A

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "_build", "facade_main")


def facade(*args):
    if not os.path.exists(BIN):
        pytest.fail("tests/cpp/_build/facade_main not built (make -C paper_2602_05179_b200/csrc)")
    return subprocess.run([BIN, *map(str, args)], capture_output=True, text=True, timeout=120)


def parse_out(text):
    res = {}
    for line in text.splitlines():
        t = line.split()
        if t[0] == "data":
            res["data"] = np.array([int(x) for x in t[2:]], np.uint32)
        elif t[0] == "exception":
            res["exception"] = line[len("exception "):]
        else:
            for k in range(0, len(t) - 1, 2):
                res[t[k]] = int(t[k + 1])
    return res


@pytest.mark.parametrize("suffix", [".scnb", ".csv"])
@pytest.mark.parametrize("rows,count", [(7, 33), (1, 1), (50, 0), (3, 1000)])
def test_scenario_files_byte_identical(tmp_path, reference, suffix, rows, count):
    ours = tmp_path / f"ours{suffix}"
    theirs = tmp_path / f"ref{suffix}"
    r = facade("io-write", ours, rows, count, 99)
    assert r.returncode == 0, r.stdout + r.stderr
    data = parse_out(r.stdout)["data"].reshape(count, rows)
    reference.write_scenario_file(theirs, data)
    assert ours.read_bytes() == theirs.read_bytes()
    # each side reads the other's file; an empty CSV batch does not round-trip
    # in the reference (no row lines are written), and must fail identically
    try:
        rr, rc, rd = reference.read_scenario_file(ours)
        ref_err = None
    except RuntimeError as e:
        ref_err = str(e)
    back = parse_out(facade("io-read", theirs).stdout)
    if ref_err is not None:
        assert suffix == ".csv" and count == 0
        assert back["exception"] == ref_err.replace(str(ours), str(theirs))
        return
    assert (rr, rc) == (rows, count) and np.array_equal(rd, data)
    assert (back["rows"], back["count"]) == (rows, count)
    assert np.array_equal(back["data"], data.ravel())


def test_scnb_capi_write_and_header_match_reference(tmp_path, reference):
    lib = A.load()
    data = (np.arange(5 * 70, dtype=np.uint32) * 2654435761 % 1000).astype(np.uint32).reshape(70, 5)
    ours, theirs = tmp_path / "a.scnb", tmp_path / "b.scnb"
    A.check(lib.scendp_scnb_write(str(ours).encode(), data.ctypes.data, 5, 70))
    reference.write_scenario_file(theirs, data)
    assert ours.read_bytes() == theirs.read_bytes()
    hdr = A.ScnbHeader()
    A.check(lib.scendp_scnb_header_read(str(ours).encode(), C.byref(hdr)))
    assert (hdr.rows, hdr.count) == (5, 70)


def _broken_files(tmp_path):
    good = struct.pack("<4sHIIH", b"SCNB", 1, 3, 2, 1) + struct.pack("<6I", *range(6))
    cases = {
        "magic": b"SCNX" + good[4:],
        "version": good[:4] + struct.pack("<H", 2) + good[6:],
        "header": good[:11],
        "dtype": good[:14] + struct.pack("<H", 3) + good[16:],
        "payload": good[:-3],
        "empty": b"",
    }
    paths = {}
    for k, v in cases.items():
        p = tmp_path / f"{k}.scnb"
        p.write_bytes(v)
        paths[k] = p
    paths["missing"] = tmp_path / "does_not_exist.scnb"
    return paths


def test_broken_scenario_files_same_errors(tmp_path, reference):
    lib = A.load()
    for name, path in _broken_files(tmp_path).items():
        with pytest.raises(RuntimeError) as e:
            reference.read_scenario_file(path)
        want = str(e.value)
        r = facade("io-read", path)
        assert r.returncode == 1
        assert parse_out(r.stdout)["exception"] == want, name
        # the GPU ingestion path's header check (C-ABI) says the same
        hdr = A.ScnbHeader()
        st = lib.scendp_scnb_header_read(str(path).encode(), C.byref(hdr))
        assert st == A.ERR_RUNTIME, name
        assert lib.scendp_last_error().decode() == want, name


ROUTING = """# a comment
3 5 hard
0 1 2 3 4
1 0 1 2 3   # trailing comment
2 1 0 1 2

3 2 1 0 1
4 3 2 1 0
"""

INSTANCES = {
    "hard": ROUTING,
    "penal": ROUTING.replace("3 5 hard", "3 5 2.5"),
    "bad_header": ROUTING.replace("3 5 hard", "3 5"),
    "bad_number": ROUTING.replace("1 0 1 2 3", "1 0 x 2 3"),
    "bad_int": ROUTING.replace("3 5 hard", "3.5 5 hard"),
    "short_row": ROUTING.replace("2 1 0 1 2", "2 1 0 1"),
    "missing_row": "\n".join(ROUTING.splitlines()[:-1]) + "\n",
    "n_zero": "0 5 hard\n0 1\n1 0\n",
    "invalid": ROUTING.replace("2 1 0 1 2", "2 1 0 -1 2"),
    "empty": "# nothing here\n\n",
    "dsirp_std": "dsirp\nU 4\nI0 2\nH 3\nR 2\nholding standard 1.5 3\n"
                 "delivery linear 10 0.5\ndelivery option 2 2 7 0.25\n",
    "dsirp_tables": "dsirp\nH 2\nU 3\nholding table 0 1 2 3\n"
                    "delivery table 1 0 5 6 7\ndelivery table 2 0 4 4 4\n",
    "dsirp_unknown": "dsirp\nU 4\nH 2\nfoo 1\n",
    "dsirp_no_u": "dsirp\nH 2\nholding standard 1 2\ndelivery linear 1 1\n",
    "dsirp_no_hold": "dsirp\nU 4\nH 2\ndelivery linear 1 1\n",
    "dsirp_no_del": "dsirp\nU 4\nH 2\nholding standard 1 2\n",
    "dsirp_htable": "dsirp\nU 4\nH 2\nholding table 0 1 2\ndelivery linear 1 1\n",
    "dsirp_opt_range": "dsirp\nU 4\nH 2\nR 2\nholding standard 1 2\ndelivery option 3 1 1 1\n",
    "dsirp_bad_del": "dsirp\nU 4\nH 2\nholding standard 1 2\ndelivery cubic 1 1\n",
    "dsirp_table_len": "dsirp\nU 2\nH 1\nholding standard 1 2\ndelivery table 1 0 1\n",
    "dsirp_invalid": "dsirp\nU 4\nI0 9\nH 2\nholding standard 1 2\ndelivery linear 1 1\n",
    "dsirp_std_args": "dsirp\nU 4\nH 2\nholding standard 1\ndelivery linear 1 1\n",
}


@pytest.mark.parametrize("name", sorted(INSTANCES))
def test_instance_grammar_matches_reference(tmp_path, reference, name):
    src = tmp_path / f"{name}.txt"
    src.write_text(INSTANCES[name])
    want = reference.parse_instance_file(src, tmp_path / "ref.out")
    r = facade("io-parse", src, tmp_path / "ours.out")
    assert r.returncode == 0, r.stdout + r.stderr
    got = (tmp_path / "ours.out").read_text()
    assert got == want


def test_missing_instance_file(tmp_path, reference):
    want = reference.parse_instance_file(tmp_path / "nope.txt", tmp_path / "ref.out")
    facade("io-parse", tmp_path / "nope.txt", tmp_path / "ours.out")
    assert (tmp_path / "ours.out").read_text() == want
    assert want.startswith("error cannot open instance file")


@pytest.mark.parametrize("hard,beta", [(1, 0.0), (0, 10.0), (0, 0.1)])
def test_write_routing_instance_matches_reference(tmp_path, reference, oracle, hard, beta):
    n = 9
    costs = reference.make_random_instance(n, 4)
    want = reference.write_routing_instance(n, 17, hard, beta, costs, tmp_path / "ref.txt")
    r = facade("io-write-inst", n, 17, hard, beta, 4, tmp_path / "ours.txt")
    assert r.returncode == 0, r.stdout + r.stderr
    assert (tmp_path / "ours.txt").read_text() == want
    # and it parses back to the same instance on both sides
    back = reference.parse_instance_file(tmp_path / "ours.txt", tmp_path / "p.out")
    facade("io-parse", tmp_path / "ours.txt", tmp_path / "q.out")
    assert (tmp_path / "q.out").read_text() == back
