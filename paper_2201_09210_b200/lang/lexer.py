"""Hand-written scanner (reference behaviour: pkg/src/coex/lang/lexer.py:29-129).

Statements end at a newline or ``;``; newlines inside ``(`` / ``[`` are not
significant; ``#`` starts a line comment.  Token kinds are the keyword/symbol
text itself, or IDENT / NUMBER / STRING / NEWLINE / EOF.
"""

from __future__ import annotations

from dataclasses import dataclass

from ..errors import LexError

KEYWORDS = frozenset({
    "var", "let", "print", "if", "elif", "else", "while", "for", "in",
    "range", "steps", "input", "native", "item", "true", "false",
    "and", "or", "not",
})
PAIRS = ("==", "!=", "<=", ">=")
SINGLES = frozenset("(){}[],;=<>+-*/")
ESCAPES = {"n": "\n", "t": "\t", '"': '"', "\\": "\\"}


@dataclass(frozen=True)
class Token:
    kind: str
    text: str
    line: int
    col: int
    value: object = None


class _Scanner:
    def __init__(self, src: str):
        self.src = src
        self.i = 0
        self.line = 1
        self.col = 1
        self.nest = 0
        self.out: list = []

    def emit(self, kind, text, value=None):
        self.out.append(Token(kind, text, self.line, self.col, value))

    def take(self, j: int):
        """Consume src[i:j] (no newlines inside) advancing the column."""
        self.col += j - self.i
        self.i = j

    def number(self):
        s, n, j = self.src, len(self.src), self.i
        while j < n and s[j].isdigit():
            j += 1
        is_float = False
        if j + 1 < n and s[j] == "." and s[j + 1].isdigit():
            is_float = True
            j += 1
            while j < n and s[j].isdigit():
                j += 1
        if j < n and s[j] in "eE":
            k = j + 1
            if k < n and s[k] in "+-":
                k += 1
            if k < n and s[k].isdigit():
                is_float = True
                j = k
                while j < n and s[j].isdigit():
                    j += 1
        text = s[self.i:j]
        self.emit("NUMBER", text, float(text) if is_float else int(text))
        self.take(j)

    def word(self):
        s, n, j = self.src, len(self.src), self.i
        while j < n and (s[j].isalnum() or s[j] == "_"):
            j += 1
        w = s[self.i:j]
        self.emit(w if w in KEYWORDS else "IDENT", w)
        self.take(j)

    def string(self):
        s, n = self.src, len(self.src)
        j = self.i + 1
        chars = []
        while True:
            if j >= n:
                raise LexError("unterminated string", self.line, self.col)
            c = s[j]
            if c == '"':
                break
            if c == "\n":
                raise LexError("unterminated string", self.line, self.col)
            if c == "\\" and j + 1 < n:
                chars.append(ESCAPES.get(s[j + 1], s[j + 1]))
                j += 2
            else:
                chars.append(c)
                j += 1
        self.emit("STRING", s[self.i:j + 1], "".join(chars))
        self.take(j + 1)

    def run(self) -> list:
        s, n = self.src, len(self.src)
        while self.i < n:
            c = s[self.i]
            if c == "#":
                end = s.find("\n", self.i)
                self.i = n if end < 0 else end
            elif c == "\n":
                if self.nest == 0 and self.out and self.out[-1].kind not in ("NEWLINE", ";"):
                    self.emit("NEWLINE", "\n")
                self.i += 1
                self.line += 1
                self.col = 1
            elif c in " \t\r":
                self.take(self.i + 1)
            elif c == '"':
                self.string()
            elif c.isdigit():
                self.number()
            elif c.isalpha() or c == "_":
                self.word()
            elif s[self.i:self.i + 2] in PAIRS:
                self.emit(s[self.i:self.i + 2], s[self.i:self.i + 2])
                self.take(self.i + 2)
            elif c in SINGLES:
                if c in "([":
                    self.nest += 1
                elif c in ")]":
                    self.nest = max(0, self.nest - 1)
                self.emit(c, c)
                self.take(self.i + 1)
            else:
                raise LexError(f"illegal character {c!r}", self.line, self.col)
        while self.out and self.out[-1].kind == "NEWLINE":
            self.out.pop()
        self.out.append(Token("EOF", "", self.line, self.col))
        return self.out


def tokenize(source: str) -> list:
    return _Scanner(source).run()
