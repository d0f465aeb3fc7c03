"""CuPPL surface syntax -> AST, for the GPU model compiler (frontend.py).

Covers the first-order part of the reference grammar (pkg/src/cuppl/lexer.py,
pkg/src/cuppl/parser.py:68-451): a program is `name <- expr;` bindings followed by one result
expression; blocks `{ x <- e; e; ... e }`, `if (c) { .. } else { .. }`, `function(p, ..) { .. }`,
calls, indexing `v[i]`, vector literals, the usual operator precedence (|| && comparisons
+ - * / % unary - !). Identifiers may contain hyphens and end in `*` (`dist-score`,
`uniform-discrete`, `sample*`) exactly as in the reference lexer. Types, `case`, `shift` /
`reset` are not part of the GPU subset (they are rejected with a ParseError naming the
construct).
"""

from __future__ import annotations

import re
from dataclasses import dataclass, field

from .errors import CupError


class ParseError(CupError):
    kind = "parse"


@dataclass
class Tok:
    kind: str
    value: object
    line: int
    col: int


# ----------------------------------------------------------------------------- AST -------
@dataclass
class Num:
    value: object  # int or float


@dataclass
class Bool:
    value: bool


@dataclass
class Var:
    name: str


@dataclass
class Call:
    fn: object  # Var or expression
    args: list


@dataclass
class Index:
    vec: object
    idx: object


@dataclass
class BinOp:
    op: str
    lhs: object
    rhs: object


@dataclass
class Unary:
    op: str
    arg: object


@dataclass
class If:
    cond: object
    then: object
    orelse: object


@dataclass
class Lambda:
    params: list
    body: object


@dataclass
class Block:
    stmts: list  # (name or None, expr)
    result: object


@dataclass
class VecLit:
    elems: list


@dataclass
class Program:
    bindings: list = field(default_factory=list)  # (name, expr)
    result: object = None


# ----------------------------------------------------------------------------- lexer -----
_PUNCT = ["<-", "==", "!=", "<=", ">=", "&&", "||", "(", ")", "{", "}", "[", "]", ",", ";",
          "+", "-", "*", "/", "%", "<", ">", "!", "="]
_KEYWORDS = {"function", "if", "else", "true", "false"}
_UNSUPPORTED = {"case", "type", "shift", "reset"}
_NUM = re.compile(r"\d+(\.\d*)?([eE][+-]?\d+)?|\.\d+([eE][+-]?\d+)?")
_IDENT = re.compile(r"[A-Za-z_][A-Za-z0-9_]*(-[A-Za-z_][A-Za-z0-9_]*)*\*?")


def tokenize(src: str) -> list[Tok]:
    toks, i, line, col = [], 0, 1, 1
    n = len(src)
    while i < n:
        c = src[i]
        if c == "\n":
            i, line, col = i + 1, line + 1, 1
            continue
        if c.isspace():
            i, col = i + 1, col + 1
            continue
        if src.startswith("//", i) or c == "#":
            while i < n and src[i] != "\n":
                i += 1
            continue
        if src.startswith("/*", i):
            j = src.find("*/", i + 2)
            if j < 0:
                raise ParseError(f"unterminated comment at {line}:{col}")
            line += src.count("\n", i, j)
            i = j + 2
            continue
        m = _NUM.match(src, i)
        if m and (c.isdigit() or c == "."):
            text = m.group(0)
            val = float(text) if any(ch in text for ch in ".eE") else int(text)
            toks.append(Tok("NUM", val, line, col))
            i, col = m.end(), col + len(text)
            continue
        m = _IDENT.match(src, i)
        if m:
            text = m.group(0)
            if text in _UNSUPPORTED:
                raise ParseError(f"`{text}` is outside the GPU model subset ({line}:{col})")
            toks.append(Tok(text.upper() if text in _KEYWORDS else "IDENT", text, line, col))
            i, col = m.end(), col + len(text)
            continue
        for p in _PUNCT:
            if src.startswith(p, i):
                toks.append(Tok(p, p, line, col))
                i, col = i + len(p), col + len(p)
                break
        else:
            raise ParseError(f"unexpected character {c!r} at {line}:{col}")
    return toks


# ----------------------------------------------------------------------------- parser ----
_BINARY = [("||",), ("&&",), ("==", "!=", "<", "<=", ">", ">="), ("+", "-"), ("*", "/", "%")]


class _Parser:
    def __init__(self, toks):
        self.t = toks
        self.p = 0

    def peek(self, k=0):
        return self.t[self.p + k] if self.p + k < len(self.t) else None

    def at(self, kind, k=0):
        tok = self.peek(k)
        return tok is not None and tok.kind == kind

    def next(self):
        tok = self.peek()
        if tok is None:
            raise ParseError("unexpected end of input")
        self.p += 1
        return tok

    def expect(self, kind, what=None):
        tok = self.peek()
        if tok is None or tok.kind != kind:
            where = f"{tok.line}:{tok.col}" if tok else "end of input"
            raise ParseError(f"expected {what or kind!r} at {where}, found {tok.value if tok else 'EOF'!r}")
        return self.next()

    def program(self) -> Program:
        prog = Program()
        while self.peek() is not None:
            if self.at("IDENT") and self.at("<-", 1) or self.at("IDENT") and self.at("=", 1):
                name = self.next().value
                self.next()
                rhs = self.expr()
                self.expect(";", "';' after binding")
                prog.bindings.append((name, rhs))
                continue
            prog.result = self.expr()
            if self.peek() is not None:
                tok = self.peek()
                raise ParseError(f"expected end of input after the result at {tok.line}:{tok.col}")
        if prog.result is None:
            raise ParseError("program must end with a result expression")
        names = [b for b, _ in prog.bindings]
        dup = sorted({b for b in names if names.count(b) > 1})
        if dup:
            raise ParseError(f"duplicate top-level binding: {dup[0]}")
        return prog

    def expr(self):
        return self._binary(0)

    def _binary(self, level):
        if level == len(_BINARY):
            return self.unary()
        e = self._binary(level + 1)
        while self.peek() is not None and self.peek().kind in _BINARY[level]:
            op = self.next().kind
            e = BinOp(op, e, self._binary(level + 1))
        return e

    def unary(self):
        if self.at("-"):
            self.next()
            return Unary("-", self.unary())
        if self.at("!"):
            self.next()
            return Unary("!", self.unary())
        return self.postfix()

    def postfix(self):
        e = self.primary()
        while True:
            if self.at("("):
                self.next()
                args = []
                if not self.at(")"):
                    args.append(self.expr())
                    while self.at(","):
                        self.next()
                        args.append(self.expr())
                self.expect(")")
                e = Call(e, args)
            elif self.at("["):
                self.next()
                idx = self.expr()
                self.expect("]")
                e = Index(e, idx)
            else:
                return e

    def primary(self):
        tok = self.peek()
        if tok is None:
            raise ParseError("unexpected end of input")
        if tok.kind == "NUM":
            self.next()
            return Num(tok.value)
        if tok.kind in ("TRUE", "FALSE"):
            self.next()
            return Bool(tok.kind == "TRUE")
        if tok.kind == "IDENT":
            self.next()
            return Var(tok.value)
        if tok.kind == "(":
            self.next()
            if self.at(")"):
                raise ParseError(f"unit value `()` is not a GPU model value ({tok.line}:{tok.col})")
            e = self.expr()
            self.expect(")")
            return e
        if tok.kind == "[":
            self.next()
            elems = []
            if not self.at("]"):
                elems.append(self.expr())
                while self.at(","):
                    self.next()
                    elems.append(self.expr())
            self.expect("]")
            return VecLit(elems)
        if tok.kind == "{":
            return self.block()
        if tok.kind == "IF":
            return self.if_()
        if tok.kind == "FUNCTION":
            self.next()
            self.expect("(")
            params = []
            if not self.at(")"):
                params.append(self.expect("IDENT", "parameter name").value)
                while self.at(","):
                    self.next()
                    params.append(self.expect("IDENT", "parameter name").value)
            self.expect(")")
            return Lambda(params, self.block())
        raise ParseError(f"unexpected token {tok.value!r} at {tok.line}:{tok.col}")

    def block(self):
        self.expect("{")
        stmts = []
        while True:
            if self.at("}"):
                tok = self.peek()
                raise ParseError(f"block must end with an expression ({tok.line}:{tok.col})")
            if self.at("IDENT") and (self.at("<-", 1) or self.at("=", 1)):
                name = self.next().value
                self.next()
                rhs = self.expr()
                self.expect(";", "';' after binding")
                stmts.append((name, rhs))
                continue
            e = self.expr()
            if self.at(";"):
                self.next()
                stmts.append((None, e))
                continue
            self.expect("}", "'}' closing the block")
            return Block(stmts, e)

    def if_(self):
        self.expect("IF")
        self.expect("(")
        cond = self.expr()
        self.expect(")")
        then = self.block()
        self.expect("ELSE")
        orelse = self.if_() if self.at("IF") else self.block()
        return If(cond, then, orelse)


def parse(src: str) -> Program:
    """Parse a CuPPL program (GPU subset) into a Program."""
    return _Parser(tokenize(src)).program()
