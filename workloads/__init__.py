"""Workload shapes and seeded synthetic inputs (no HE arithmetic lives here)."""
