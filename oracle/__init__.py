"""ORACLE - test infrastructure only (the checker, never the product).

Only tests/, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product package
``paper_2605_26289_b200`` never imports it and fails loudly when its CUDA
library is missing.

Contents:
- ``cpu``: ctypes view of ``ds_oracle.c`` (plain-C restatement of the
  reference's integer kernels, deltaserve/_kernels/_native.pyx).
- ``llama_ref``: CPU fp32 restatement of the Llama-3 decoder used by the
  GPU engine (the reference has no model; parity of attention/logits is
  pinned by this restatement only).
- ``reference``: loader for the reference itself compiled here
  (``oracle/_ref``, built by ``oracle/build_ref.sh``).
"""
