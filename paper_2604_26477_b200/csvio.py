"""On-disk formats of the hot path's data, byte-compatible with the
reference so the device path drops into its solve -> pareto -> hv file workflow:

  save_pool_csv / load_pool_csv        solver.hpp:357-432   rows formatted / parsed on the
                                                             device (momc_b200_format_pool_rows,
                                                             momc_b200_parse_pool_rows)
  save_archive_csv / load_archive_csv  pareto.hpp:787-885   host (archives are small)
  save_trace_csv                       pareto.hpp:886-897   host

Header lines are parsed with the reference's sscanf patterns (whitespace in the pattern
matches any run of whitespace, %d / %lf skip leading whitespace) and every error carries
the reference's message.
"""
from __future__ import annotations

import ctypes as C
import re

import numpy as np

from . import _lib
from .api import (InvalidArgument, MomcRuntimeError, ParetoArchive, SamplePool, Session, _errbuf, _raise,
                  default_session, format_number)

_FLT = (r"([+-]?(?:0[xX](?:[0-9a-fA-F]+\.?[0-9a-fA-F]*|\.[0-9a-fA-F]+)(?:[pP][+-]?\d+)?"
        r"|(?:\d+\.?\d*|\.\d+)(?:[eE][+-]?\d+)?|[iI][nN][fF](?:[iI][nN][iI][tT][yY])?"
        r"|[nN][aA][nN](?:\([0-9A-Za-z_]*\))?))")
_INT = r"([+-]?\d+)"


def _strtod(tok: str) -> float:
    t = tok.lower()
    if "0x" in t:
        return float.fromhex(t)
    return float(t)


def _sscanf(line: str, pattern: list):
    """sscanf of `line` against pattern pieces: ("lit", text) | ("d",) | ("lf",). Returns the
    converted values (the count is what sscanf would return)."""
    pos, out = 0, []
    for piece in pattern:
        if piece[0] == "lit":
            for ch in piece[1]:
                if ch.isspace():
                    while pos < len(line) and line[pos].isspace():
                        pos += 1
                elif pos < len(line) and line[pos] == ch:
                    pos += 1
                else:
                    return out
            continue
        while pos < len(line) and line[pos].isspace():
            pos += 1
        m = re.compile(_INT if piece[0] == "d" else _FLT).match(line, pos)
        if not m:
            return out
        out.append(int(m.group(1)) if piece[0] == "d" else _strtod(m.group(1)))
        pos = m.end()
    return out


def _stod(cell: str) -> float:
    """std::stod: leading whitespace, longest strtod prefix; no conversion -> invalid_argument,
    overflow -> out_of_range"""
    m = re.compile(r"\s*" + _FLT).match(cell)
    if not m:
        raise InvalidArgument("stod")
    v = _strtod(m.group(1))
    if v in (float("inf"), float("-inf")) and "inf" not in m.group(1).lower():
        raise MomcRuntimeError("stod")  # std::out_of_range
    return v


def _getline_cells(text: str, delim: str):
    """repeated std::getline(stream, cell, delim) until it fails: no trailing empty cell"""
    cells, pos = [], 0
    while pos < len(text):
        q = text.find(delim, pos)
        if q < 0:
            cells.append(text[pos:])
            pos = len(text)
        else:
            cells.append(text[pos:q])
            pos = q + 1
    return cells


def _read_lines(path: str):
    try:
        with open(path, "rb") as fh:
            data = fh.read()
    except OSError:
        raise MomcRuntimeError(f"cannot open {path}")
    return data


def _getline(data: bytes, pos: int):
    """std::getline: (line, next_pos) or (None, pos) at end of data"""
    if pos >= len(data):
        return None, pos
    q = data.find(b"\n", pos)
    if q < 0:
        return data[pos:].decode("latin-1"), len(data)
    return data[pos:q].decode("latin-1"), q + 1


# ----------------------------------------------------------------------------- pool
def save_pool_csv(pool: SamplePool, path, session: Session | None = None) -> None:
    """solver.hpp:357-375; record rows formatted on the device."""
    path = str(path)
    s = session or default_session()
    keys = np.ascontiguousarray(pool.record_keys(), np.uint32)
    run = np.ascontiguousarray(keys[:, 0])
    wt = np.ascontiguousarray(keys[:, 1])
    tr = np.ascontiguousarray(keys[:, 2])
    ts = np.ascontiguousarray(pool.timestamps(), np.int64)
    words = np.ascontiguousarray(pool.words, np.uint64)
    M = pool.size()
    head = (f"# pool n={pool.n()} model_construction_s={format_number(pool.model_construction_seconds)}"
            f" sampling_s={format_number(pool.sampling_seconds)}\nrun,weight,trajectory,timestamp_ns,spins\n")
    body = b""
    if M:
        args = (run.ctypes.data_as(_lib.u32p), wt.ctypes.data_as(_lib.u32p), tr.ctypes.data_as(_lib.u32p),
                ts.ctypes.data_as(_lib.i64p), words.ctypes.data_as(_lib.u64p), M, pool.n())
        n_bytes = C.c_size_t()
        err = _errbuf()
        _raise(s.lib.momc_b200_format_pool_rows(s.h, *args, None, 0, C.byref(n_bytes), err, 2048), err)
        buf = C.create_string_buffer(n_bytes.value)
        _raise(s.lib.momc_b200_format_pool_rows(s.h, *args, buf, n_bytes.value, C.byref(n_bytes), err, 2048), err)
        body = buf.raw[: n_bytes.value]
    try:
        with open(path, "wb") as fh:
            fh.write(head.encode())
            fh.write(body)
    except OSError:
        raise MomcRuntimeError(f"cannot open {path} for writing")


def load_pool_csv(path, session: Session | None = None) -> SamplePool:
    """solver.hpp:377-432; record rows parsed on the device."""
    path = str(path)
    data = _read_lines(path)
    line, pos = _getline(data, 0)
    if line is None or not line.startswith("# pool n="):
        raise MomcRuntimeError(f"{path}:1: malformed pool header")
    v = _sscanf(line, [("lit", "# pool n="), ("d",), ("lit", " model_construction_s="), ("lf",),
                       ("lit", " sampling_s="), ("lf",)])
    if len(v) != 3 or v[0] < 1:
        raise MomcRuntimeError(f"{path}:1: malformed pool header")
    n, mc, ss = v
    line, pos = _getline(data, pos)
    if line is None:
        raise MomcRuntimeError(f"{path}:2: missing column header")
    s = session or default_session()
    rest = data[pos:]
    M = C.c_size_t()
    err = _errbuf()
    _raise(s.lib.momc_b200_parse_pool_rows(s.h, rest, len(rest), n, 3, path.encode(), C.byref(M), err, 2048), err)
    M = M.value
    wpc = (n + 63) // 64
    keys = np.zeros((M, 3), np.uint32)
    run = np.zeros(M, np.uint32)
    wt = np.zeros(M, np.uint32)
    tr = np.zeros(M, np.uint32)
    ts = np.zeros(M, np.int64)
    words = np.zeros((M, wpc), np.uint64)
    if M:
        _raise(s.lib.momc_b200_parsed_pool_get(s.h, run.ctypes.data_as(_lib.u32p), wt.ctypes.data_as(_lib.u32p),
                                               tr.ctypes.data_as(_lib.u32p), ts.ctypes.data_as(_lib.i64p),
                                               words.ctypes.data_as(_lib.u64p), err, 2048), err)
        keys[:, 0], keys[:, 1], keys[:, 2] = run, wt, tr
    pool = SamplePool(n, words, stamps=ts, records=keys)
    pool.model_construction_seconds = mc
    pool.sampling_seconds = ss
    return pool


# ----------------------------------------------------------------------------- archive
def _hex_words(words) -> str:
    return "".join(f"{int(w):016x}" for w in words)


def save_archive_csv(archive: ParetoArchive, path) -> None:
    """pareto.hpp:787-821"""
    path = str(path)
    k = archive.k()
    has_cfg = archive.configs is not None and archive.size() > 0 and archive.n > 0
    n = archive.n if has_cfg else 0
    out = [f"# archive k={k} n={n} filtering_s={format_number(archive.filtering_seconds)}"]
    if len(archive.reference):
        out[0] += " r=" + ";".join(format_number(x) for x in archive.reference)
    out.append("".join(f"c{l + 1}," for l in range(k)) + "spins")
    mask = getattr(archive, "config_mask", None)
    for i in range(archive.size()):
        row = "".join(format_number(float(x)) + "," for x in archive.values[i])
        if not has_cfg or (mask is not None and not mask[i]):
            row += "-"
        else:
            row += _hex_words(archive.configs[i])
        out.append(row)
    try:
        with open(path, "w") as fh:
            fh.write("\n".join(out) + "\n")
    except OSError:
        raise MomcRuntimeError(f"cannot open {path} for writing")


def load_archive_csv(path) -> ParetoArchive:
    """pareto.hpp:823-884"""
    path = str(path)
    data = _read_lines(path)
    line, pos = _getline(data, 0)
    if line is None or not line.startswith("# archive "):
        raise MomcRuntimeError(f"{path}:1: malformed archive header")
    v = _sscanf(line, [("lit", "# archive k="), ("d",), ("lit", " n="), ("d",), ("lit", " filtering_s="), ("lf",)])
    if len(v) != 3:
        raise MomcRuntimeError(f"{path}:1: malformed archive header")
    k, n, fs = v
    reference = []
    rpos = line.find(" r=")
    if rpos >= 0:
        reference = [_stod(cell) for cell in _getline_cells(line[rpos + 3:], ";")]
    line, pos = _getline(data, pos)
    if line is None:
        raise MomcRuntimeError(f"{path}:2: missing column header")
    wpc = (n + 63) // 64
    vals, cfgs, mask = [], [], []
    lineno = 2
    while True:
        line, pos = _getline(data, pos)
        if line is None:
            break
        lineno += 1
        if line == "":
            continue
        cells = _getline_cells(line, ",")
        if len(cells) < k + 1:  # a getline ran out of characters
            # the reference converts the cells it did get first (stod errors win)
            for c in cells[:k]:
                _stod(c)
            raise MomcRuntimeError(f"{path}:{lineno}: malformed archive row")
        vals.append([_stod(c) for c in cells[:k]])
        cell = cells[k]
        if cell != "-":
            if len(cell) != wpc * 16:
                raise MomcRuntimeError(f"{path}:{lineno}: bad spin field width")
            w = np.zeros(wpc, np.uint64)
            for bit in range(n):
                ch = ord(cell[(bit // 64) * 16 + 15 - (bit % 64) // 4])
                ch = ch - 256 if ch >= 128 else ch  # char is signed
                val = ch - ord("0") if ch <= ord("9") else ch - ord("a") + 10
                if (val >> (bit % 4)) & 1:
                    w[bit // 64] |= np.uint64(1) << np.uint64(bit % 64)
            cfgs.append(w)
            mask.append(True)
        else:
            cfgs.append(np.zeros(wpc, np.uint64))
            mask.append(False)
    values = np.asarray(vals, np.float64).reshape(len(vals), k)
    has_any = any(mask)
    arc = ParetoArchive(values, np.asarray(cfgs, np.uint64).reshape(len(cfgs), wpc) if has_any else None,
                        n if has_any else 0)
    if has_any and not all(mask):
        arc.config_mask = np.asarray(mask, bool)
    arc.filtering_seconds = fs
    arc.reference = reference
    return arc


# ----------------------------------------------------------------------------- trace
def save_trace_csv(trace, path) -> None:
    """pareto.hpp:886-897"""
    path = str(path)
    rows = ["elapsed_s,hv,samples"] + [f"{format_number(p.elapsed_s)},{format_number(p.hv)},{int(p.samples)}"
                                       for p in trace]
    try:
        with open(path, "w") as fh:
            fh.write("\n".join(rows) + "\n")
    except OSError:
        raise MomcRuntimeError(f"cannot open {path} for writing")
