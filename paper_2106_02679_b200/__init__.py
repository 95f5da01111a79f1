"""B200-native layered gradient accumulation (arXiv 2106.02679) -- Python binding.

The product is ``liblga.so`` (C ABI in ``include/lga.h``): hand-written sm_100a CUDA kernels
(tcgen05/TMEM/TMA GEMMs, flash attention, LayerNorm, AdamW) and a per-layer scheduler that
drives NCCL over NVLink.  This package only marshals arguments to it:

    from paper_2106_02679_b200 import Config, Trainer
    tr = Trainer(Config(layers=12, d_model=768, heads=12, seq_len=1024, micro_batch=4, n_micro=8))
    loss = tr.step(x, target)          # x, target: torch CUDA fp32 [N][b][s][d]

``torch`` is used for device memory, streams and ``torch.distributed`` (to broadcast the NCCL
unique id); every step of the training path runs in the library.
"""
from __future__ import annotations

from ._abi import (LGA_BF16, LGA_FLAG_NO_COMM, LGA_FP32, LGA_LAYERED, LGA_STANDARD, LgaError,  # noqa: F401
                   lib)
from .api import Config, Trainer  # noqa: F401
