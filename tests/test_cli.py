"""CLI contract: subcommands, exit codes
0/1/2, JSON round trip, and the SPEC examples. check/partition/predict run on
the CPU; measure/validate need a GPU."""
import json

import pytest

from paper_1507_01265_b200 import cli, fpm

PAPER = ("# unit_cells=15360 granularity=8 label=paper\nx,speed,ci_halfwidth,repetitions\n"
         "112,1436742,0,1\n120,1240377,0,1\n128,1418579,0,1\n")


def run(capsys, *argv):
    rc = cli.main([str(a) for a in argv])
    out = capsys.readouterr()
    return rc, out.out, out.err


@pytest.fixture
def paper(tmp_path):
    p = tmp_path / "paper.csv"
    p.write_text(PAPER)
    return p


def test_partition_paper_example(capsys, paper):
    # n=480, p=4, paired -> (112,128,112,128), 1.386 s, speedup 1.072.
    rc, out, _ = run(capsys, "partition", paper, "--total", 480, "--p", 4, "--paired", "--json")
    assert rc == 0
    r = json.loads(out)
    assert r["shares"] == [112, 128, 112, 128] and r["offset"] == 8
    assert abs(r["makespan"] - 1.385950) < 1e-6
    assert abs(r["speedup_vs_balanced"] - 1.072) < 5e-4
    # the JSON output round-trips exactly
    assert json.loads(json.dumps(r)) == r


def test_general_matches_oracle(capsys, tmp_path):
    f = fpm.SpeedFunction(5, 2, tuple((x, float(30 - x)) for x in range(2, 21, 2)), "lin")
    p = tmp_path / "m.csv"
    p.write_text(fpm.write_csv(f))
    for total, procs in ((20, 2), (24, 3), (16, 4)):
        _, g, _ = run(capsys, "partition", p, "--total", total, "--p", procs, "--general", "--json")
        _, o, _ = run(capsys, "partition", p, "--total", total, "--p", procs, "--oracle", "--json")
        assert json.loads(g)["makespan"] == json.loads(o)["makespan"]


def test_check_and_predict(capsys, paper, tmp_path):
    rc, out, _ = run(capsys, "check", paper)
    assert rc == 0 and "violated" in out and "(120, 128)" in out
    const = tmp_path / "c.csv"
    const.write_text("# unit_cells=1 granularity=10 label=c\nx,speed,ci_halfwidth,repetitions\n"
                     "10,100,0,1\n20,100,0,1\n30,100,0,1\n")
    rc, out, _ = run(capsys, "check", const)
    assert rc == 0 and "condition satisfied; balancing optimal" in out
    rc, out, _ = run(capsys, "partition", const, "--total", 40, "--p", 2, "--json")
    assert rc == 0 and json.loads(out)["speedup_vs_balanced"] == 1.0
    rc, out, _ = run(capsys, "predict", paper, "--shares", "112,128", "--json")
    r = json.loads(out)
    assert rc == 0 and r["makespan"] == fpm.eval_time(fpm.read_csv(PAPER), 128)


def test_exit_codes(capsys, paper, tmp_path):
    empty = tmp_path / "e.csv"
    empty.write_text("")
    assert run(capsys, "check", empty)[0] == 2                      # parse error
    assert run(capsys, "check", tmp_path / "missing.csv")[0] == 2   # unreadable
    assert run(capsys, "measure", "--x", "64:16:8")[0] == 2         # reversed range
    assert run(capsys, "measure", "--x", "8:16:0")[0] == 2
    assert run(capsys, "partition", paper, "--total", 4800, "--p", 4, "--general")[0] == 1  # infeasible
    assert run(capsys, "partition", paper)[0] == 2                  # argparse usage error
    assert run(capsys, "bogus")[0] == 2
    assert run(capsys, "report", "--out-dir", tmp_path / "none")[0] == 2
    assert cli.parse_range("16:64:8") == [16, 24, 32, 40, 48, 56, 64]
    assert cli.parse_range("16:60:8")[-1] == 56


def test_surface_csv_round_trip_and_slice():
    ns, ms = (116, 120, 124), (104, 112, 120, 128)
    smp = tuple(fpm.SpeedSample(m, 1e6 + 7 * n - m * m / 3, 0.25 * n, 3) for n in ns for m in ms)
    g = fpm.SpeedSurface(128, 8, ns, ms, smp, "surf")
    h = fpm.read_surface_csv(fpm.write_surface_csv(g))
    assert h == g
    f = fpm.slice_surface(h, 120)
    assert f.unit_cells == 128 * 120 and f.label == "surf@n=120"
    assert [s.speed for s in f.samples] == [s.speed for s in smp[4:8]]
    with pytest.raises(fpm._lib.ParseError):
        fpm.read_surface_csv(fpm.write_surface_csv(g).replace("120,112,", "120,113,"))


def test_report(capsys, tmp_path):
    (tmp_path / "validate_manifest.json").write_text(json.dumps({
        "command": "validate", "timestamp": "t", "mode": "m", "outputs": [],
        "table1": [{"offset": 0, "t_theory_s": 1.0, "t_exp_s": 1.0, "speedup": 1.0}]}))
    rc, out, _ = run(capsys, "report", "--out-dir", tmp_path)
    assert rc == 0 and "offset 0" in out


@pytest.mark.gpu
def test_measure_and_validate_on_gpu(capsys, tmp_path):
    out = tmp_path / "o"
    common = ["--l", 32, "--steps", 2, "--max-reps", 3, "--out-dir", out]
    rc, _, err = run(capsys, "measure", "--x", "8:24:8", "--m", 16, *common)
    assert rc == 0, err
    f = fpm.read_csv((out / "speed_avg.csv").read_text())
    assert [s.x for s in f.samples] == [8, 16, 24] and f.unit_cells == 16 * 32
    assert all(s.speed > 0 and s.repetitions >= 3 for s in f.samples)
    assert fpm.read_csv((out / "speed_gpu0.csv").read_text()).samples[0].x == 8
    rc, _, err = run(capsys, "measure", "--x", "8:16:8", "--m-range", "16:32:16", *common)
    assert rc == 0, err
    srf = fpm.read_surface_csv((out / "surface_avg.csv").read_text())
    assert srf.n_values == (16, 32) and srf.m_values == (8, 16)
    assert fpm.slice_surface(srf, 16).unit_cells == 16 * 32
    # per-share timing (one GPU), then the lockstep decomposition path (both teams on GPU 0)
    for dev in ("0", "0,0"):
        rc, _, err = run(capsys, "validate", out / "speed_avg.csv", "--total", 32, "--p", 2,
                         "--offsets", "0,8", "--devices", dev, *common)
        assert rc == 0, err
        rows = (out / "table1.csv").read_text().splitlines()
        assert rows[0].startswith("offset,") and len(rows) == 3
        assert float(rows[1].split(",")[3]) == 1.0  # speedup of the baseline row
        assert len((out / "table2.csv").read_text().splitlines()) == 1 + 2 * 2
    rc, out_txt, _ = run(capsys, "report", "--out-dir", out)
    assert rc == 0 and "measure" in out_txt and "validate" in out_txt


@pytest.mark.gpu
def test_measure_ring_halo_path_on_gpu(capsys, tmp_path):
    # the speed function measured on the production halo
    # path (a ring of slabs pushing halos into each other), labelled as such;
    # on one GPU the ring's slabs share the device (a labelled stand-in).
    out = tmp_path / "r"
    common = ["--l", 32, "--steps", 2, "--max-reps", 3, "--out-dir", out]
    rc, _, err = run(capsys, "measure", "--x", "8:24:8", "--m", 16, "--halo", "ring",
                     "--devices", "0,0", *common)
    assert rc == 0, err
    f = fpm.read_csv((out / "speed_avg.csv").read_text())
    # validate's offset 8 around 32/2 = 16 needs shares 8 and 24 inside the model
    assert [s.x for s in f.samples] == [8, 16, 24] and all(s.speed > 0 for s in f.samples)
    assert "halo=ring p=2" in f.label and "stand-in" in f.label
    assert (out / "speed_team0.csv").exists() and (out / "speed_team1.csv").exists()
    man = json.loads((out / "measure_manifest.json").read_text())
    assert man["halo"].startswith("halo=ring")
    rc, _, err = run(capsys, "validate", out / "speed_avg.csv", "--total", 32, "--p", 2,
                     "--offsets", "0,8", "--devices", "0,0", *common)
    assert rc == 0, err
    man = json.loads((out / "validate_manifest.json").read_text())
    assert man["mode"].startswith("lockstep decomposition") and "stand-in" in man["mode"]
    # --halo self refuses a repeated device
    rc, _, _ = run(capsys, "measure", "--x", "8:16:8", "--m", 16, "--devices", "0,0", *common)
    assert rc == 2
