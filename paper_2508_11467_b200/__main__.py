"""``python -m paper_2508_11467_b200``: the reference CLI (gen/run/verify/profile,
pkg/src/dcsvd/__main__.py) backed by the GPU engine."""

from .harness import main

if __name__ == "__main__":
    main()
