"""Runs equinox_sim jobs in a fresh interpreter: ``python dropin_driver.py <dir with equinox_sim>``,
jobs as JSON on stdin, results as JSON on stdout.  The drop-in (paper_2508_16646_b200/dropin,
B200 engine) and the reference's own module (oracle/_ref/py, CPU engine) are both packages named
``equinox_sim`` with a ``_core`` extension, so each runs in its own process."""
import json
import sys

sys.path.insert(0, sys.argv[1])
import equinox_sim as E  # noqa: E402


def main():
    jobs = json.load(sys.stdin)
    out = []
    for j in jobs:
        fn = getattr(E, j["fn"])
        try:
            args = [j["config"]] + ([j["jobs"]] if "jobs" in j else [])
            r = fn(*args)
            out.append({"ok": r})
        except Exception as e:  # the exception type and message are part of the API
            out.append({"error": type(e).__name__, "message": str(e)})
    json.dump({"engine": getattr(E, "ENGINE", "?"), "results": out}, sys.stdout)


if __name__ == "__main__":
    main()
