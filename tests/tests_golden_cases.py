"""Parameters shared by tests/golden/make_golden.py and the tests."""

# scenario -> envelope-lead bucket (ms)
LEAD_CASES = {"c1": 500.0, "pab_overload": 250.0, "wide": 100.0, "c2_subset": 1000.0}
