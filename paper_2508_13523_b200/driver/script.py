"""Minimal input-script reader for the commands the hot path needs.

The reference parser (mdkk/driver/script.py) is out of scope for the B200
build; this reader keeps its surface syntax (`#` comments, trailing `&`
continuation, one command per line) and command names so the reference's
scripts (pkg/scripts/melt.in, snap.in) run unchanged.  `lattice` also
accepts `bcc <a>` for the SNAP tungsten configurations.
"""

from __future__ import annotations

import difflib

COMMANDS = {"units": 1, "boundary": 3, "lattice": 2, "create_box": 3, "create_atoms": 0, "mass": 1,
            "velocity": 2, "pair_style": None, "pair_coeff": 2, "suffix": 1, "timestep": 1, "thermo": 1,
            "run": 1, "qeq": None}
# per-argument kinds: a set = allowed words, "f" = number, "i" = integer, None = free word
_ARGS = {"units": [{"lj"}], "boundary": [{"p"}] * 3, "lattice": [{"fcc", "sc", "bcc"}, "f"],
         "create_box": ["i", "i", "i"], "mass": ["f"], "velocity": ["f", "i"], "pair_coeff": ["f", "f"],
         "timestep": ["f"], "thermo": ["i"], "run": ["i"], "suffix": [None]}


class ParseError(ValueError):
    def __init__(self, line_no: int, msg: str):
        super().__init__(f"line {line_no}: {msg}")
        self.line_no = line_no


class Command:
    __slots__ = ("name", "args", "line_no")

    def __init__(self, name, args, line_no):
        self.name, self.args, self.line_no = name, list(args), line_no


def parse_script(text: str) -> list[Command]:
    out, pending, first = [], [], 0
    for line_no, raw in enumerate(text.splitlines(), start=1):
        body = raw.split("#", 1)[0].rstrip()
        cont = body.endswith("&")
        toks = (body[:-1] if cont else body).split()
        if toks and not pending:
            first = line_no
        pending.extend(toks)
        if cont or not toks:
            continue
        out.append(_command(pending, first))
        pending = []
    if pending:
        out.append(_command(pending, first))
    return out


def _command(tokens, line_no):
    name, *args = tokens
    if name not in COMMANDS:
        near = difflib.get_close_matches(name, COMMANDS, n=3)
        hint = f"; did you mean {', '.join(near)}?" if near else ""
        raise ParseError(line_no, f"unknown command {name!r}{hint}")
    n = COMMANDS[name]
    if n is not None and len(args) != n:
        raise ParseError(line_no, f"{name} expects {n} argument(s), got {len(args)}")
    for kind, tok in zip(_ARGS.get(name, ()), args):
        _check_arg(name, kind, tok, line_no)
    if name == "pair_style":
        if not args:
            raise ParseError(line_no, "pair_style expects a style name")
        base = args[0].split("/")[0]
        if base == "snap" and len(args) != 3:
            raise ParseError(line_no, f"pair_style {args[0]} expects: cutoff coeff_file")
        if base == "lj" and len(args) != 2:
            raise ParseError(line_no, f"pair_style {args[0]} expects: cutoff")
        if len(args) > 1:
            _check_arg(name, "f", args[1], line_no)
    if name == "qeq":   # 'qeq off' | 'qeq on gamma eta chi cutoff' (mdkk/driver/script.py:102-120)
        if not args:
            raise ParseError(line_no, "qeq expects 'on <params>' or 'off'")
        if args[0] == "off":
            if len(args) != 1:
                raise ParseError(line_no, "qeq off takes no parameters")
        elif args[0] != "on":
            raise ParseError(line_no, f"qeq: expected 'on' or 'off', got {args[0]!r}")
        elif len(args) != 5:
            raise ParseError(line_no, f"qeq on expects 4 parameter(s), got {len(args) - 1}")
        else:
            for tok in args[1:]:
                try:
                    float(tok)
                except ValueError:
                    raise ParseError(line_no, f"qeq: {tok!r} is not a number") from None
    return Command(name, args, line_no)


def _check_arg(name, kind, tok, line_no):
    if kind is None:
        return
    if isinstance(kind, set):
        if tok not in kind:
            raise ParseError(line_no, f"{name}: {tok!r}: expected one of {sorted(kind)}")
        return
    try:
        int(tok) if kind == "i" else float(tok)
    except ValueError:
        what = "integer" if kind == "i" else "number"
        raise ParseError(line_no, f"{name}: malformed {what} {tok!r}") from None
