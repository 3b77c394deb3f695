"""The reference's OWN test programs (proj/tests/*.cpp, built by
tests/dropin/Makefile in the dev container) run against the GPU drop-in.

unit_dropin / acceptance_dropin link the reference's non-hot-path library code
with paper_1909_09927_b200/csrc/dropin/sconv_dropin.cpp in place of
src/ecr.cpp + src/pecr.cpp, so every ecr_convert / ecr_spmv_conv /
pecr_convert / pecr_conv_pool call in those tests -- including the ones made
by multichannel_conv and forward() -- executes on the B200.  The *_ref
controls are the same programs on the unmodified reference: the drop-in must
pass exactly what the reference passes.  The reference CLI
(proj/tools/sparseconv_main.cpp, against a CLI11 shim) is built both ways too:
sparseconv_dropin is the CLI backend switch of SURVEY 8f row 2 -- its conv /
convpool / sweep subcommands run on the B200 -- and the reference's CLI suite
(cli_main.cpp) and acceptance criterion 8 drive it.
"""
import os
import re
import subprocess

import pytest

BUILD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "dropin", "_build")


def _run(name, env=None, timeout=900):
    path = os.path.join(BUILD, name)
    if not os.path.exists(path):
        pytest.skip(f"{name} not built (needs the reference mount; see tests/dropin/Makefile)")
    e = dict(os.environ, **(env or {}))
    return subprocess.run([path], capture_output=True, text=True, timeout=timeout, env=e)


def _criteria(out):
    return sorted(re.findall(r"^(PASS|FAIL)\s+(\d+)\.", out, flags=re.M), key=lambda t: int(t[1]))


def test_reference_unit_suite_control():
    r = _run("unit_ref")
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert re.search(r"\| 0 failed \|", r.stdout)


@pytest.mark.gpu
def test_reference_unit_suite_on_gpu_exact():
    r = _run("unit_dropin", {"SCONV_CUDA_MODE": "exact"})
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert re.search(r"\| 0 failed \|", r.stdout)


@pytest.mark.gpu
def test_reference_unit_suite_on_gpu_fast():
    """FAST (FFMA) is not bit-exact, so the reference's bitwise ECR-vs-dense
    checks may fail; every test case outside those must still pass."""
    r = _run("unit_dropin", {"SCONV_CUDA_MODE": "fast"})
    failed = set(re.findall(r"^\[FAIL\] (.*)$", r.stdout, flags=re.M))
    bitwise = {"ecr_spmv_conv on fixed inputs",
               "ecr sweep: oracle equivalence, counter law, lossless windows",
               "pecr_conv_pool on fixed inputs", "multichannel_conv",
               "forward: single conv_pool layer equals the composed oracle",
               "forward: methods agree and compressed traffic wins"}
    assert failed <= bitwise, failed


@pytest.mark.gpu
def test_reference_acceptance_on_gpu():
    ref = _run("acceptance_ref")
    gpu = _run("acceptance_dropin")
    assert _criteria(gpu.stdout) == _criteria(ref.stdout), gpu.stdout
    crit = _criteria(gpu.stdout)
    assert len(crit) == 11 and all(s == "PASS" for s, _ in crit), gpu.stdout


def test_reference_cli_suite_control():
    r = _run("cli_ref")
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert re.search(r"\| 0 failed \|", r.stdout)


@pytest.mark.gpu
def test_reference_cli_suite_on_gpu():
    """The reference CLI built on the drop-in (conv / convpool on the B200)
    passes the reference's own CLI suite: exit codes, messages, reports,
    checksums and worker invariance."""
    r = _run("cli_dropin", {"SCONV_CUDA_MODE": "exact"})
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert re.search(r"\| 0 failed \|", r.stdout)


@pytest.mark.gpu
def test_cuda_hpp_batched_entries():
    """include/sconv/cuda.hpp (multichannel_conv / conv_pool / forward, batched
    over the C ABI) against the unmodified reference compiled into the same
    binary: bit-identical outputs, equal OpCounts, ForwardResult fields and
    the reference's exception types."""
    r = _run("cuda_hpp_test")
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "cuda_hpp_test: ok" in r.stdout


def _backend(args, env=None, timeout=600):
    path = os.path.join(BUILD, "sparseconv")
    if not os.path.exists(path):
        pytest.skip("sparseconv not built (needs the reference mount; see tests/dropin/Makefile)")
    e = dict(os.environ, **(env or {}))
    return subprocess.run([path] + args, capture_output=True, text=True, timeout=timeout, env=e)


def _checksum(out):
    m = re.search(r"checksum=([0-9a-f]{16})", out)
    return m.group(1) if m else None


def test_cli_backend_switch_cpu(tmp_path):
    """`sparseconv --backend cpu` is the unmodified reference CLI; an unknown
    backend is a configuration error (exit 2)."""
    m, k = str(tmp_path / "m.fmap"), str(tmp_path / "k.fmap")
    assert _backend(["--backend", "cpu", "gen", "--height", "20", "--width", "20", "--channels", "8",
                     "--sparsity", "0.7", "--seed", "3", "--out", m]).returncode == 0
    assert _backend(["gen", "--backend=cpu", "--height", "3", "--width", "3", "--channels", "8",
                     "--sparsity", "0", "--seed", "4", "--out", k]).returncode == 0
    r = _backend(["--backend", "cpu", "conv", "--input", m, "--kernel", k])
    assert r.returncode == 0 and _checksum(r.stdout)
    bad = _backend(["--backend", "tpu", "conv", "--input", m, "--kernel", k])
    assert bad.returncode == 2 and "unknown backend" in bad.stderr
    assert _backend(["conv", "--backend"]).returncode == 2


@pytest.mark.gpu
def test_cli_backend_switch_cuda_vgg_layer(tmp_path):
    """conv and convpool through `--backend cuda` (the drop-in, EXACT) on a
    VGG-19 conv5-shaped layer (512 channels, 16x16 map, one filter, s = 0.7):
    the same output checksum, op counts and exit code as `--backend cpu`; the
    wall times of both land in the report (RunReport wall_ns)."""
    m, k = str(tmp_path / "m.fmap"), str(tmp_path / "k.fmap")
    assert _backend(["--backend", "cpu", "gen", "--height", "16", "--width", "16", "--channels", "512",
                     "--sparsity", "0.7", "--seed", "51", "--out", m]).returncode == 0
    assert _backend(["--backend", "cpu", "gen", "--height", "3", "--width", "3", "--channels", "512",
                     "--sparsity", "0", "--seed", "52", "--out", k]).returncode == 0
    env = {"SCONV_CUDA_MODE": "exact"}
    for cmd in (["conv", "--method", "ecr"], ["convpool", "--method", "pecr", "--pool-h", "2",
                                               "--pool-w", "2", "--pool-stride", "2"]):
        outs = {}
        for be in ("cpu", "cuda"):
            rep = str(tmp_path / f"{cmd[0]}_{be}.json")
            r = _backend(["--backend", be] + cmd + ["--input", m, "--kernel", k, "--report", rep], env)
            assert r.returncode == 0, r.stderr
            import json
            with open(rep) as f:
                outs[be] = json.load(f)
        assert outs["cpu"]["output_checksum"] == outs["cuda"]["output_checksum"]
        assert outs["cpu"]["op_count"] == outs["cuda"]["op_count"]
