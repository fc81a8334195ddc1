"""Frontend of the imperative tensor language (reference: pkg/src/coex/lang/__init__.py)."""

from . import ast
from .lexer import Token, tokenize
from .parser import OP_NAMES, parse
from .printer import pretty

__all__ = ["ast", "Token", "tokenize", "parse", "pretty", "OP_NAMES"]
