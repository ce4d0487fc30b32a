"""pytest plugin: run the REFERENCE's own test files with its native kernel
module replaced by integration._kernels_b200 (the B200 C ABI).

    python -m pytest -p integration.ref_plugin <reference tests> ...

At session end it reports which _kernels functions the reference called
through the stub, and fails the session if none were (the routing is the
point of the run)."""

import integration._kernels_b200 as kb


def pytest_configure(config):
    kb.install()


def pytest_sessionfinish(session, exitstatus):
    tr = session.config.pluginmanager.get_plugin("terminalreporter")
    if tr is not None:
        tr.write_line(f"_kernels_b200 calls: {dict(sorted(kb.CALLS.items()))}")
    if not kb.CALLS and session.testscollected:
        session.exitstatus = 3
