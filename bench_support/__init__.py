"""Bench / test support (NOT the product): host-side synthetic workload generators
restated from the reference (rig, UV binding, mesh frames, avatar init), used to build
the BASELINE.json shapes where the reference package does not exist."""
