"""Launch configuration shared by bench.py and the full-size parity tests.

HINT = the window_hint each config's sweep is launched with (it selects the
register-ring width W of the sweep kernel; results never depend on it)."""
HINT = {"C1": 16, "C2": 20, "C3": 20, "C4": 64}
