"""Exception types shared by the interpreter drop-in and the recogniser."""


class InterpError(Exception):
    """Same role as minigpu.interp.InterpError (interp.py:39)."""


class UnsupportedProgram(InterpError):
    """The program is not one this B200 backend executes (no CPU fallback)."""
