"""Reference-schema bench CSV."""
import io
import os
import subprocess

import pytest

from paper_1503_07387_b200 import bench_csv as B

REF = "/root/reference/proj"


def _rows():
    return [B.BenchResult(4, 9.123456789, "scalar", 512.25, 1.0, "l1"),
            B.BenchResult(4, 9.123456789, "cuda", 123456.789, 241.0078125, "full"),
            B.BenchResult(16, 8.0, "masked", 1e-3, 0.1, "full"),
            B.BenchResult(5, 0.0001, "masked", 1e21, 123456789.0, "l1"),
            B.BenchResult(6, 1.5e-7, "cuda", 0.0, 1234567.0, "full")]


def test_header_matches_reference():
    hdr = open(os.path.join(REF, "tools/bench/csv.hpp")).read() if os.path.isdir(REF) else ""
    if hdr:
        assert f'kCsvHeader = "{B.CSV_HEADER}"' in hdr
    assert B.CSV_HEADER == "K,bits_per_int,scheme,mis,ratio_vs_scalar,buffer_mode"


def test_roundtrip_is_exact():
    f = io.StringIO()
    B.write_csv(f, _rows())
    text = f.getvalue()
    back = B.read_csv(io.StringIO(text))
    g = io.StringIO()
    B.write_csv(g, back)
    assert g.getvalue() == text and back == _rows()
    with pytest.raises(RuntimeError):
        B.read_csv(io.StringIO("K,wrong\n"))


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference sources absent")
def test_reference_read_csv_accepts_and_reproduces_our_csv(tmp_path):
    """The reference's own read_csv / write_csv (csv.cpp) round-trips our file
    byte for byte."""
    src = tmp_path / "rt.cpp"
    src.write_text('#include "csv.hpp"\n#include <fstream>\n#include <iostream>\n'
                   'int main(int, char** a) { std::ifstream in(a[1]); auto r = mvb::bench::read_csv(in);'
                   ' mvb::bench::write_csv(std::cout, r); return 0; }\n')
    exe = tmp_path / "rt"
    subprocess.run(["g++", "-std=c++20", "-O1", f"-I{REF}/tools/bench", f"-I{REF}/core/include", str(src),
                    f"{REF}/tools/bench/csv.cpp", "-o", str(exe)], check=True)
    path = tmp_path / "ours.csv"
    with open(path, "w") as f:
        B.write_csv(f, _rows())
    out = subprocess.run([str(exe), str(path)], capture_output=True, text=True, check=True).stdout
    assert out == path.read_text()


def test_groups_have_the_reference_shape():
    for k in (4, 9):
        ls = B.group_lists(k, 3, 42)
        assert len(ls) == 3
        for ids in ls:
            assert (1 << k) <= ids.size < (1 << (k + 1))
            assert (ids[1:] > ids[:-1]).all() and ids[-1] < (1 << 25)
