"""Launch configuration shared by bench.py and the full-size parity tests.

HINT = the window_hint each config's sweep is launched with (it selects the
register-ring width W of the sweep kernel; results never depend on it).
MEAN = the expected mean window (spdp.h SPDP_F_MEAN_WINDOW; it selects how many
candidates the sweep scans before its first warp vote; results never depend on it)."""
HINT = {"C1": 16, "C2": 20, "C3": 20, "C4": 64}
MEAN = {"C1": 0, "C2": 4, "C3": 8, "C4": 23}
# the same on a scenario set ordered by total demand (spdp_order_scenarios: narrower warp-maximum
# windows, so fewer unconditional candidates pay off; measured C2 2 -> A0 = 6, C3 6 -> A0 = 10)
MEAN_ORDERED = {"C1": 0, "C2": 2, "C3": 6, "C4": 23}
