"""CPU checks of the C ABI: the library loads, exports every symbol that
include/sagips.h declares, and its host-side logic (presets, validation,
workspace sizing) behaves -- no kernel is launched."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sagips.h")


def _lib():
    from paper_2407_00051_b200 import _lib
    return _lib


def declared_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"SAGIPS_API\s+[\w\s\*]+?\b(sagips_\w+)\s*\(", txt)))


def test_header_declares_the_north_star_calls():
    syms = declared_symbols()
    for s in ("sagips_create", "sagips_train_step", "sagips_push_generator_grad",
              "sagips_pull_generator_grad", "sagips_sample_events"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    L = _lib()
    out = subprocess.run(["nm", "-D", "--defined-only", L.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (sagips_\w+)", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    assert sorted(L.EXPORTED) == declared_symbols()


def test_abi_version_and_struct_layout(tmp_path):
    """The ctypes mirrors match the C compiler's layout of the header."""
    L = _lib()
    assert L.lib.sagips_abi_version() == 1
    fields = ["world", "mode", "precision", "param_samples", "reference_rows", "shard_rows", "gen_lr",
              "true_params", "hist_bins", "hist_lo", "hist_hi", "seed", "exchange_timeout_ms"]
    src = tmp_path / "layout.c"
    src.write_text("#include <stdio.h>\n#include <stddef.h>\n#include \"sagips.h\"\nint main(void){\n"
                   'printf("%zu %zu\\n", sizeof(sagips_config), sizeof(sagips_step_stats));\n'
                   + "".join(f'printf("%zu\\n", offsetof(sagips_config, {f}));\n' for f in fields)
                   + 'printf("%zu\\n", offsetof(sagips_step_stats, wait_ns));\nreturn 0;}\n')
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()
    assert int(got[0]) == ctypes.sizeof(L.Config) and int(got[1]) == ctypes.sizeof(L.StepStats)
    for f, off in zip(fields, got[2:]):
        assert getattr(L.Config, f).offset == int(off), f
    assert L.StepStats.wait_ns.offset == int(got[-1])


def test_presets_and_workspace():
    L = _lib()
    desk = L.config_init(L.PRESET_DESK)
    assert (desk.noise_dim, desk.gen_hidden, desk.gen_depth, desk.disc_hidden, desk.disc_depth) == (8, 64, 2, 64, 2)
    assert desk.param_samples * desk.events_per_sample == 1024
    paper = L.config_init(L.PRESET_PAPER)
    assert paper.param_samples == 1024 and paper.events_per_sample == 1024
    assert paper.reference_rows == 2 * paper.shard_rows == 2 ** 21
    assert paper.gen_lr == pytest.approx(1e-5, rel=1e-7) and paper.disc_lr == pytest.approx(1e-4, rel=1e-7)
    assert L.workspace_size(paper) > L.workspace_size(desk) > 0


@pytest.mark.parametrize("field,value", [("group_size", 0), ("outer_rma", 2), ("staleness", 2), ("mode", 9), ("disc_hidden", 100),
                                         ("rank", 5), ("hist_bins", 0), ("param_samples", 0),
                                         ("events_per_sample", 0), ("shard_rows", 0), ("reference_rows", 0),
                                         ("param_samples", -1), ("world", 0), ("noise_dim", 0)])
def test_config_validation(field, value):
    L = _lib()
    cfg = L.config_init(L.PRESET_DESK, world=4, group_size=2)
    setattr(cfg, field, value)
    with pytest.raises(L.SagipsError) as e:
        L.workspace_size(cfg)
    assert e.value.status == 2


def test_ragged_last_group_is_accepted():
    """SPEC's (10, 4) partition {0-3},{4-7},{8-9}: world need not
    be a multiple of the group size."""
    L = _lib()
    cfg = L.config_init(L.PRESET_DESK, world=10, rank=9, group_size=4, mode=L.MODE_RMA_ALLGATHER, outer_every=2)
    assert L.workspace_size(cfg) > 0


def test_true_params_must_be_in_softplus_range():
    L = _lib()
    cfg = L.config_init(L.PRESET_DESK, true_params=[1.0, -1.0, 0.5, 2.0, 0.5, 1.0])
    with pytest.raises(L.SagipsError):
        L.workspace_size(cfg)


def test_null_arguments_are_rejected():
    L = _lib()
    assert L.lib.sagips_config_init(None, 0) == 1
    assert L.lib.sagips_sample_events(None, 1, 1, 0, 0, 0, 5, None, None, 0, None, None, None) == 1
    assert L.lib.sagips_train_step(None, 0, 0, None) == 1
    assert L.lib.sagips_nccl_unique_id(None, 128) == 1
