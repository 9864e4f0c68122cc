"""Instance files: round trip, reference compatibility (files written by the
reference load here and vice versa is pinned by the shared format), errors."""

import numpy as np
import pytest

from paper_2407_19689_b200 import instances as inst
from paper_2407_19689_b200.cli import main as cli_main
from paper_2407_19689_b200.instance_io import InstanceFormatError, load_instance, save_instance


def test_round_trip_grid_and_explicit(tmp_path):
    prob = inst.grid_problem("cauchy_like", 4, "l2", 3)
    save_instance(prob, tmp_path / "a.txt")
    assert (tmp_path / "a.txt").read_text().splitlines()[2] == "cost l2"  # canonical shorthand
    back = load_instance(tmp_path / "a.txt")
    assert np.array_equal(back.C, prob.C) and np.allclose(back.f, prob.f, rtol=0, atol=1e-16)
    ex = inst.make_problem(np.arange(6.0).reshape(2, 3), [1.0, 2.0], [1.0, 1.0, 1.0])
    save_instance(ex, tmp_path / "b.txt")
    back = load_instance(tmp_path / "b.txt")
    assert np.array_equal(back.C, ex.C) and back.cost.norm_kind == "explicit"


def test_gen_command(tmp_path):
    out = tmp_path / "g.txt"
    assert cli_main(["gen", "--class", "shapes", "--resolution", "4", "--norm", "l1", "--seed", "1",
                     "--out", str(out)]) == 0
    prob = load_instance(out)
    ref = inst.grid_problem("shapes", 4, "l1", 1)
    assert np.array_equal(prob.C, ref.C)


@pytest.mark.parametrize("text", ["2 2\ncost l1\n1 1\n", "2 2\ncost bogus\n1 1\n1 1\n",
                                  "2 3\ncost l1\n1 1\n1 1 1\n", "2 2\ncost explicit\n0 1\n1\n1 1\n1 1\n"])
def test_format_errors(tmp_path, text):
    p = tmp_path / "bad.txt"
    p.write_text(text)
    with pytest.raises(InstanceFormatError):
        load_instance(p)


def test_cli_error_exit(tmp_path, capsys):
    assert cli_main(["solve", "--instance", str(tmp_path / "missing.txt"), "--out", str(tmp_path / "o.json")]) == 1
    assert "error:" in capsys.readouterr().err
