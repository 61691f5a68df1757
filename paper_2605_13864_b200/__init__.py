"""B200-native (sm_100a) drop-in for the OptiGPU transpose and tree-reduction
programs (arXiv 2605.13864; reference package `minigpu`).

Public surface:
  * `run_program`, `Interp`, `Array`, `InterpError`, `f32`  — the reference's
    interpreter entry points (minigpu/interp.py:39-387), executing recognised
    transpose / reduce Programs on the GPU;
  * `parse_program`, `ParseError`                           — the program
    grammar (minigpu/parser.py:893) for building those Programs;
  * `transpose`, `reduce_sum`, `reduce_tree512`              — typed zero-copy
    entries on CUDA tensors or host arrays;
  * `transpose_multi`, `reduce_sum_multi`                    — the same over
    shards on several GPUs from one process (fused NVLink combine).
"""
from ._lib import B2Error, launch_count  # noqa: F401
from .interp import Array, Interp, InterpError, UnsupportedProgram, f32, run_program  # noqa: F401
from .lang import ParseError, Program, parse_program  # noqa: F401
from .ops import (init_devices, int128, reduce_sum, reduce_sum_multi, reduce_sum_sequential,  # noqa: F401
                  reduce_tree, reduce_tree512,
                  reduce_tree512_partials, reduce_tree_partials, reduce_ws_bytes, transpose, transpose_multi)
from .recognize import recognize  # noqa: F401
from .gate import GateError, check_kernels  # noqa: F401
from . import programs  # noqa: F401

__all__ = ["run_program", "Interp", "Array", "InterpError", "UnsupportedProgram", "f32",
           "parse_program", "ParseError", "Program", "recognize", "transpose", "reduce_sum",
           "reduce_sum_sequential",
           "reduce_tree512", "reduce_tree512_partials", "reduce_tree", "reduce_tree_partials", "transpose_multi", "reduce_sum_multi",
           "init_devices", "int128", "reduce_ws_bytes", "GateError", "check_kernels", "B2Error", "launch_count"]
