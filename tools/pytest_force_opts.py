"""Dev pytest plugin: apply PROHD_OPT_<name>=<value> (tools/_opts.py) before the session, so a candidate
default can be run through the whole GPU suite before the library's default changes:
    PYTHONPATH=tools PROHD_OPT_K6_BIDIR_2A=2 python -m pytest -p pytest_force_opts tests -m gpu
"""
import _opts


def pytest_sessionstart(session):
    done = _opts.apply_env()
    print(f"[pytest_force_opts] options forced: {done}")
