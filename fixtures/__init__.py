"""Synthetic-scene input fixtures (fixtures/libsvr_fixture.so): scenes, GT depth frames,
payloads, rays and upstream gradients for the tests and the bench.  Not part of the
product package; pinned to the reference's own generator (oracle/_ref)."""
from .synthetic import SceneSpec, SyntheticScene, uniform_floats

__all__ = ["SceneSpec", "SyntheticScene", "uniform_floats"]
