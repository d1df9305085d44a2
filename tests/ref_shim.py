"""pytest plugin: the reference's own test suite against this package's Engine.

Loaded as ``-p tests.ref_shim`` by tests/test_gpu_reference_suite.py when it
runs the unmodified reference tests (copied next to the installed reference
by tools/install_reference.sh).  Before collection, ``backend.install()``
re-binds ``Engine`` / ``run_simulations`` in every ``multispin`` module to
the GPU engine, so ``from multispin.engine import Engine`` in those tests
(and the reference CLI and harness code they call) constructs ours.
"""


def pytest_configure(config):
    from paper_2404_16990_b200 import backend
    backend.install()
    import multispin.engine
    assert multispin.engine.Engine is backend.BackendEngine
    config.addinivalue_line("markers", "slow: long-running statistical validation (minutes)")
