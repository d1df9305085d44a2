"""CLI host logic (no GPU): temperature specs, config files, precedence
(defaults < file < $MULTISPIN_THREADS < flags) and the error convention
(cli.py:89-152, 519-526 of the reference)."""
import pytest

from paper_2404_16990_b200 import cli


def test_parse_temperatures():
    assert cli.parse_temperatures("2.0") == (2.0,)
    assert cli.parse_temperatures(" 1.5, 2.5 ,") == (1.5, 2.5)
    assert cli.parse_temperatures("1.5:3.0:0.5") == (1.5, 2.0, 2.5, 3.0)
    assert cli.parse_temperatures("0.1:0.3:0.1") == (0.1, 0.2, 0.3)  # rounded, floor with slack
    for bad in ("1:2", "1:2:0", "3:1:0.5"):
        with pytest.raises(ValueError):
            cli.parse_temperatures(bad)


def test_config_file_and_precedence(tmp_path, monkeypatch):
    cfg_path = tmp_path / "run.cfg"
    cfg_path.write_text("# comment\nm = 8\nn-sim = 3   # trailing comment\ntemperature = 1.0:2.0:0.5\nthreads = 5\n")
    assert cli.parse_config_file(str(cfg_path)) == {"m": "8", "n_sim": "3", "temperature": "1.0:2.0:0.5",
                                                    "threads": "5"}
    args = cli.build_parser().parse_args(["simulate", "--config", str(cfg_path), "--n", "96"])
    monkeypatch.delenv(cli.ENV_THREADS, raising=False)
    c = cli.build_config(args)
    assert (c.m, c.n, c.n_sim, c.temperature, c.threads) == (8, 96, 3, (1.0, 1.5, 2.0), 5)
    assert c.sim_temperatures() == (1.0, 1.0, 1.0, 1.5, 1.5, 1.5, 2.0, 2.0, 2.0)
    monkeypatch.setenv(cli.ENV_THREADS, "7")
    assert cli.build_config(args).threads == 7                     # env beats the file
    args = cli.build_parser().parse_args(["simulate", "--config", str(cfg_path), "--threads", "2"])
    assert cli.build_config(args).threads == 2                     # flags beat env
    (tmp_path / "bad.cfg").write_text("colour = red\n")
    with pytest.raises(ValueError, match="unknown config key"):
        cli.build_config(cli.build_parser().parse_args(["simulate", "--config", str(tmp_path / "bad.cfg")]))
    (tmp_path / "bad2.cfg").write_text("m 8\n")
    with pytest.raises(ValueError, match="expected 'key = value'"):
        cli.parse_config_file(str(tmp_path / "bad2.cfg"))


def test_errors_exit_2(capsys):
    assert cli.main(["simulate", "--m", "10"]) == 2               # m % 4 != 0, before any device work
    assert "error:" in capsys.readouterr().err
    assert cli.main(["simulate", "--sweeps", "-1"]) == 2
    assert cli.main(["bench", "--temperature", "2.0,2.5"]) == 2
    assert cli.main(["rngtest"]) == 2
