"""Test / bench harness: replays seeded schedules (workloads/) through the
product binding (paper_1909_11150_b200). Holds none of the method's arithmetic."""
