"""B200-native 2PC secret-shared inference (MPC-Pipe, arXiv 2209.13643) hot path.

The compute path is libmpcg.so (hand-written sm_100a CUDA behind the C ABI in
include/mpcg.h); this package is the Python mirror of the reference's operator API.
"""
from ._native import (BudgetError, ConfigError, CudaError, Error, NcclError, ProtocolError, RangeError,
                      ShapeError, TransportError, UsageError, lib)
from .api import (SecureExecutor, Session, Tensor, a2b, b2a_bit, beaver_and, beaver_matmul, beaver_mul,
                  beaver_square, binary_add, exp_shares, fnv1a_words, less_than, max_last_dim,
                  maxpool2d_shares, msb, nccl_unique_id, open_, reciprocal_shares, relu_shares,
                  softmax_shares, truncate_shares, TripleQueue, record_triples, use_triple_queue, dealer_fetch,
                  # extensions (not in the reference; ResNet-18 / BERT-base layers)
                  gelu_shares, global_avg_pool, inv_sqrt_shares, layernorm_shares, sigmoid_shares)
from .model import ModelGraph, demo_input, init_weights

__all__ = [n for n in dir() if not n.startswith("_")]
