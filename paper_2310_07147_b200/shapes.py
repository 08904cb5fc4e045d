"""Weight-tensor shape lists of the benchmark configs.

Rows are output channels (tensor.hpp:13-16).  LLaMA-2-7B: 291 tensors,
6,738,415,616 parameters, 1,423,937 rows; LLaMA-2-13B: 363 tensors,
13,015,864,320 parameters.
"""
from typing import List, Tuple

Shape = Tuple[int, int]


def llama(hidden: int, inter: int, layers: int, vocab: int = 32000) -> List[Shape]:
    s: List[Shape] = [(vocab, hidden)]                 # embed_tokens
    for _ in range(layers):
        s.append((1, hidden))                          # input_layernorm (single channel)
        s += [(hidden, hidden)] * 4                    # q, k, v, o
        s.append((1, hidden))                          # post_attention_layernorm
        s += [(inter, hidden)] * 2                     # gate, up
        s.append((hidden, inter))                      # down
    s.append((1, hidden))                              # final norm
    s.append((vocab, hidden))                          # lm_head
    return s


def llama2_7b() -> List[Shape]:
    return llama(4096, 11008, 32)


def llama2_13b() -> List[Shape]:
    return llama(5120, 13824, 40)


def count(shapes: List[Shape]):
    return sum(r * c for r, c in shapes), sum(r for r, _ in shapes)


def shard_rows(shapes: List[Shape], world: int, rank: int) -> List[Shape]:
    """Row-range shard of every tensor (ZeRO-1 partition): rank k owns
    rows [k*r/N, (k+1)*r/N) of each tensor (a 1-row tensor lands on the last rank)."""
    out = []
    for r, c in shapes:
        lo, hi = (r * rank) // world, (r * (rank + 1)) // world
        if hi > lo:
            out.append((hi - lo, c))
    return out
