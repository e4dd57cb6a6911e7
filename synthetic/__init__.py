"""Seeded synthetic input generators (no method arithmetic); see inputs.py."""
