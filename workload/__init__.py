"""Seeded synthetic inputs for the StarSD verify path.

This module is shared by the oracle-side tests and the CUDA-side tests/bench, so it holds
NONE of the method's arithmetic (no acceptance test, no residual, no sampling rule).  It only
draws logits and draft token ids with the shapes and value distributions of the paper's
workloads:

* target row  : log p ~ log-space Dirichlet(A * pi), pi = Zipf(s) over a random permutation of
                the vocabulary (A = 10, s = 1.2 -> entropy ~2.4 nats, LLM-like)
* draft row   : log q ~ log-space Dirichlet(kappa * p)   (kappa = the agreement knob)
* draft ids   : x_j ~ softmax(z_q,j / T) by Gumbel-max (T = 0: argmax z_q,j); these are the
                draft model's own samples, i.e. an INPUT of the verify step
* rows are independent across (request, position) (reading C-15)
"""
from .synth import (CONFIGS, make_batch, make_batch_torch, make_tiny_tables, tiny_batch,
                    bf16_bits, log_dirichlet)
from .trace import C4_BATCH, C4_KAPPA, bursty_trace

__all__ = ["CONFIGS", "make_batch", "make_batch_torch", "make_tiny_tables", "tiny_batch",
           "bf16_bits", "log_dirichlet", "bursty_trace", "C4_BATCH", "C4_KAPPA"]
