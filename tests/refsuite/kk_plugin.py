"""pytest plugin: the reference's own test modules with the B200 drop-ins installed.

Loaded with `-p kk_plugin` by tests/test_reference_suite_gpu.py when it runs the
staged reference tests (baseline/_ref/pkg/tests).  Before collection it rebinds
mdkk's hot-path functions to paper_2508_13523_b200.plugin's GPU adapters, so the
tests' `from mdkk... import build_all, compute_pair, compute_ui, ...` bind the
drop-ins, and counts how many device kernels the session launched.
"""

from __future__ import annotations


def pytest_configure(config):
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("the drop-in suite needs a CUDA device")
    from paper_2508_13523_b200 import _lib, plugin
    config._kk_rebound = plugin.install()
    config._kk_launch0 = _lib.launch_count()


def pytest_report_header(config):
    names = getattr(config, "_kk_rebound", [])
    return [f"mdkk drop-ins installed: {len(names)} bindings rebound to the B200 path"]


def pytest_terminal_summary(terminalreporter, exitstatus, config):
    from paper_2508_13523_b200 import _lib
    terminalreporter.write_line(f"kk device launches: {_lib.launch_count() - config._kk_launch0}")
