"""Seeded synthetic-input generators shared by the oracle side and the CUDA side.

Holds none of the multisplit arithmetic (see gen/inputs.py for the recipe).
"""
