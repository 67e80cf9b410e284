"""B200-native TensorCommitments prover (arxiv 2602.12630).

Drop-in for the prover hot path of the reference package `tensorcommit`
(/root/reference/pkg): quantise -> interpolate -> MSM commitment -> Terkle tree ->
opening proofs, with hand-written sm_100a CUDA kernels behind a C ABI
(include/tc_b200.h, libtcb200.so).  There is no CPU fallback: without the built library
or a CUDA device the compute entry points raise.
"""
from .authtree import MembershipProof, TerkleTree, TreeConfig, build, leaf_of, prove, prove_many, verify
from .capture import ActivationCapture, infer_and_capture
from .commit import (Commitment, Srs, TensorOpening, Trapdoors, derive_taus, load_srs, pair, setup_srs, tc_commit,
                     tc_commit_many, tc_commit_stream, tc_open, tc_open_many, tc_verify)
from .curve import G, P, Q, decode_elem, decode_scalar, encode_elem, encode_scalar, hash_to_scalar
from .field import PrimeField
from .mvpoly import Grid, MultiPoly, default_grid, evaluate, interpolate_lagrange, lex_index, open_quotients
from .protocol import FieldTensor, prover_commit, prover_commit_pipeline, prover_commit_stream, quantize

__all__ = [
    "ActivationCapture", "infer_and_capture", "Commitment", "FieldTensor", "G", "Grid", "MembershipProof", "MultiPoly", "P", "PrimeField", "Q", "Srs",
    "TensorOpening", "TerkleTree", "Trapdoors", "TreeConfig", "build", "decode_elem", "decode_scalar", "default_grid",
    "derive_taus", "encode_elem", "encode_scalar", "evaluate", "hash_to_scalar", "interpolate_lagrange", "leaf_of",
    "lex_index", "load_srs", "open_quotients", "pair", "prove", "prove_many", "prover_commit", "prover_commit_pipeline", "prover_commit_stream", "quantize", "setup_srs", "tc_commit",
    "tc_commit_many", "tc_commit_stream", "tc_open", "tc_open_many", "tc_verify", "verify",
]
