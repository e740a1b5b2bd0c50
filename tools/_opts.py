"""Dev helper: apply PROHD_OPT_<name>=<value> environment variables as library options.

The library itself reads no environment (include/prohd.h prohd_set_option); the measurement
scripts in tools/ call `apply_env()` so A/B runs can still be driven from a shell line,
e.g. `PROHD_OPT_EIG_STOP=1 python tools/time_eigen.py`.
"""
import os


def apply_env() -> dict:
    from paper_2511_18207_b200 import set_option
    done = {}
    for k, v in os.environ.items():
        if k.startswith("PROHD_OPT_"):
            name = k[len("PROHD_OPT_"):].lower()
            set_option(name, int(v))
            done[name] = int(v)
    return done
