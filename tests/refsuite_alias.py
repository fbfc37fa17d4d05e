"""pytest plugin for running the reference's own suite against b200
(tests/test_reference_suite.py): with RS_REFSUITE_ALIAS=compiled the
reference registry's "compiled" entry is the b200 module, so
test_backends.py's pure-vs-compiled comparisons run pure-vs-b200."""

import os


def pytest_configure(config):
    alias = os.environ.get("RS_REFSUITE_ALIAS")
    if not alias:
        return
    import raysurf._backend as registry

    assert "b200" in registry._BACKENDS, "b200 not registered (INTEGRATION.md section 1)"
    registry._BACKENDS[alias] = registry._BACKENDS["b200"]
