"""Test-only stand-in for scikit-image (absent from this image, no network).

Only ``skimage.metrics.structural_similarity`` is provided: the subset the
reference splatmap package calls (renderloss.py:237-247).  Used solely to
import the reference in this build container to generate golden fixtures.
"""
