"""GPU: the command-line surface end to end (SPEC.md cli + acceptance criterion 1):
incremental and batch reconstruction of a bundle give byte-identical volume files for any worker
count, with and without segmentation; projections, slice export and the ingest benchmark emit
their files and JSON."""
import json

import numpy as np
import pytest

from paper_2412_00058_b200 import cli, ingest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bundle(tmp_path_factory):
    d = tmp_path_factory.mktemp("cli") / "bundle"
    assert cli.main(["synth", "bundle", "--config", "small", "--frames", "14", "--raw", "80", "60",
                     "--out", str(d)]) == 0
    return d


def _run(args, capsys):
    rc = cli.main(args)
    out = capsys.readouterr().out.strip().splitlines()
    return rc, (json.loads(out[-1]) if out else None)


@pytest.mark.parametrize("segment", ["none", "alg1"])
def test_incremental_equals_batch_bytes(bundle, tmp_path, capsys, segment):
    seg = ["--segment", segment, "--K", "0.1", "--D", "3", "--L", "20", "--band", "6"]
    common = ["--bundle", str(bundle), "--voxel-mm", "0.5"] + seg
    outs = []
    for mode, extra in (("batch", ["--threads", "1"]), ("incremental", ["--batch", "4", "--threads", "1"]),
                        ("incremental", ["--batch", "5", "--threads", "4"])):
        out = tmp_path / f"{mode}{len(outs)}.raw"
        rc, js = _run(["reconstruct", "--mode", mode, "--out", str(out)] + common + extra, capsys)
        assert rc == 0 and js["schema_version"] == 1 and js["out"] == str(out)
        outs.append(out.read_bytes())
    assert outs[0] == outs[1] == outs[2]
    vol, meta = ingest.read_volume(tmp_path / "batch0.raw")
    assert vol.any() and meta["frames_inserted"] == 14


def test_project_and_slices(bundle, tmp_path, capsys):
    vol = tmp_path / "v.raw"
    assert _run(["reconstruct", "--bundle", str(bundle), "--voxel-mm", "0.5", "--out", str(vol)], capsys)[0] == 0
    v, meta = ingest.read_volume(vol)
    rc, js = _run(["project", "--volume", str(vol), "--mode", "max", "--axis", "1", "--out",
                   str(tmp_path / "p.pgm")], capsys)
    assert rc == 0
    assert np.array_equal(ingest.read_pgm(tmp_path / "p.pgm"), v.max(axis=1))
    rc, js = _run(["project", "vpi", "--bundle", str(bundle), "--voxel-mm", "0.5", "--depth", "2",
                   "--band", "8", "--out", str(tmp_path / "vpi.pgm")], capsys)
    assert rc == 0 and ingest.read_pgm(tmp_path / "vpi.pgm").any()
    rc, js = _run(["export-slices", "--bundle", str(bundle), "--voxel-mm", "0.5", "--out",
                   str(tmp_path / "sl")], capsys)
    assert rc == 0 and js["files"] == meta["dims"][0]
    back, _ = ingest.import_slices(tmp_path / "sl")
    assert np.array_equal(back, v)


def test_bench_ingest_json(bundle, tmp_path, capsys):
    rc, js = _run(["bench", "ingest", "--bundle", str(bundle), "--voxel-mm", "0.5", "--batch", "4",
                   "--stats", str(tmp_path / "b.json")], capsys)
    assert rc == 0 and js["fps"] > 0 and js["frames"] == 14
    assert set(js["batch_latency_ms"]) == {"p50", "p95", "max"}
    assert json.loads((tmp_path / "b.json").read_text())["frames"] == 14


def test_exit_codes(tmp_path, capsys):
    assert cli.main(["reconstruct", "--bundle", str(tmp_path / "none"), "--out", str(tmp_path / "v")]) == 4
    assert cli.main(["synth", "bundle", "--frames", "0", "--out", str(tmp_path / "b")]) == 2
    assert cli.main(["project", "--out", str(tmp_path / "p.pgm")]) == 2
