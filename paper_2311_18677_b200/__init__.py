"""B200-native hot path of Splitwise (arXiv 2311.18677).

Prompt-phase prefill on a prompt pool, layer-wise KV push over NVLink into a
token pool's paged KV blocks, and token-phase decode there — behind the
reference package's (``splitsim``) worker / KV-manager / scheduler API.
All arithmetic runs in ``libswb200.so`` (hand-written sm_100a CUDA); importing
a module that needs it fails loudly if the library is not built.
"""

__version__ = "0.1.0"
