"""``python -m dcsvd`` through the shim: the GPU-backed CLI."""
from .harness import main

if __name__ == "__main__":
    main()
