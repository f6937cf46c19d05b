"""Exception hierarchy of the drop-in (same classes and meaning as the reference,
errors.py:4-36): CorrtwoError > DataError > ParseError, CorrtwoError > NumericError."""


class CorrtwoError(Exception):
    """Base class for all errors raised by this package."""


class DataError(CorrtwoError):
    """Invalid input data: axis violations, shape mismatches, bad arguments."""


class ParseError(DataError):
    """Malformed delimited text (kept for API parity; errors.py:12-32)."""

    def __init__(self, message, row=None, column=None, byte_offset=None):
        self.row, self.column, self.byte_offset = row, column, byte_offset
        where = ", ".join(f"{label} {val}" for label, val in
                          (("row", row), ("column", column), ("byte offset", byte_offset))
                          if val is not None)
        super().__init__(f"{message} ({where})" if where else message)


class NumericError(CorrtwoError):
    """Numeric failure: non-finite values, zero-variance scaling, memory limits."""
