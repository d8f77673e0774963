"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This package holds NO arithmetic of the method (no Eq. 1 fold, no ordering,
no masks, no acceptance, no pruning): only model-shape tables, counter-based
token generators and the planted-path draft-tree generator (SURVEY.md §8(d)
"Generators", "Trees (planted path)").  The draft-tree generator emits raw
inputs (parent ids, tokens, own scores); the orders it targets are re-derived
and checked by whoever consumes them.
"""
