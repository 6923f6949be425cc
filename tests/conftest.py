import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the CUDA C-ABI library)")
    config.addinivalue_line("markers", "slow: long CPU test")
    config.addinivalue_line("markers", "fulllength: full-length large-config trace parity (minutes of oracle time)")


@pytest.fixture(scope="session")
def oracle_mod():
    import oracle
    oracle.build()
    return oracle


@pytest.fixture
def ctxopt(ctx):
    """Set as_ctx_set_option overrides on the module's context for one test
    (e.g. ctxopt(GRID=1)); the automatic choice is restored afterwards."""
    names = []

    def set_(**kw):
        for k, v in kw.items():
            ctx.set_option(k, v)
            names.append(k)
    yield set_
    for k in names:
        ctx.set_option(k, None)
