"""Event ingestion: the EVT1 event files of the reference
(io.hpp:106-172) and the cut of one event stream into the windows of the
batched chain.

EVT1 = a 16-byte header ("EVT1", u16 width, u16 height, u64 count, little
endian) followed by ``count`` 16-byte records (u64 t_us, u16 x, u16 y, i8 p, 3
pad bytes) -- byte-identical to evcm::Event, so a payload is read straight into
the record layout (pinned host memory and one H2D copy for device slices) and
never re-packed on the host. The header checks run on the host in the
reference's order (they need no payload); the per-record checks of read_events
(coordinate, polarity, timestamp order, io.hpp:134-144) run on the device
(``Engine.validate_slice``), reporting the FIRST violating record with the
reference's error class, so a file the reference rejects is rejected here with
the same exception type.

The reference has no window slicer (its callers pass std::vector<EventSlice>
to run_window, train.hpp); ``slice_windows`` cuts a time-sorted stream into
consecutive ``window_us`` windows with one device binary search per boundary
and hands ``Engine.chain_batch`` its ``ev_offsets`` and ``window_stride_us``.
"""
from __future__ import annotations

import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

from .engine import (EVENT_DTYPE, BadMagicError, ConfigError, DimensionMismatchError, Engine,
                     EventSlice, IoError, TruncatedFileError, _is_torch, default_engine)

EVT1_MAGIC = b"EVT1"
EVT1_HEADER_BYTES = 16  # io.hpp:117
EVT1_RECORD_BYTES = 16  # io.hpp:118


def _parse_header(head: bytes, file_bytes: int, path) -> tuple:
    """read_events' header checks, in the reference's order (io.hpp:120-132)."""
    if file_bytes < EVT1_HEADER_BYTES:
        raise TruncatedFileError("EVT1: file shorter than the 16-byte header")
    if head[:4] != EVT1_MAGIC:
        raise BadMagicError(f"EVT1: bad magic in {path}")
    width = int.from_bytes(head[4:6], "little")
    height = int.from_bytes(head[6:8], "little")
    count = int.from_bytes(head[8:16], "little")
    if width == 0 or height == 0:
        raise DimensionMismatchError("EVT1: zero sensor dimension")
    payload = file_bytes - EVT1_HEADER_BYTES
    if count > payload // EVT1_RECORD_BYTES:
        raise TruncatedFileError("EVT1: header count exceeds payload size")
    if payload != count * EVT1_RECORD_BYTES:
        raise IoError("EVT1: trailing bytes after last record")
    return width, height, count


def read_events(path, device: bool = False, engine: Optional[Engine] = None) -> EventSlice:
    """read_events (io.hpp:115-154). ``device=True`` returns the events as a torch
    cuda uint8 tensor [n, 16] (one pinned H2D copy); otherwise a numpy
    EVENT_DTYPE array. The window is the tightest one holding every event:
    [first t, last t + 1) (empty file: [0, 0))."""
    path = os.fspath(path)
    try:
        size = os.path.getsize(path)
        f = open(path, "rb")
    except OSError as e:
        raise IoError(f"cannot open {path}: {e}") from None
    with f:
        head = f.read(EVT1_HEADER_BYTES)
        width, height, count = _parse_header(head, size, path)
        nbytes = count * EVT1_RECORD_BYTES
        if device:
            import torch
            eng = engine or default_engine()
            host = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
            if nbytes and f.readinto(memoryview(host.numpy())) != nbytes:
                raise TruncatedFileError("EVT1: short read")
            raw = host.numpy().view(EVENT_DTYPE) if nbytes else np.zeros(0, EVENT_DTYPE)
            events = host.view(-1, EVT1_RECORD_BYTES).to(
                torch.device("cuda", eng.opts.device), non_blocking=True) if nbytes else \
                torch.empty((0, EVT1_RECORD_BYTES), dtype=torch.uint8,
                            device=torch.device("cuda", eng.opts.device))
        else:
            buf = bytearray(nbytes)
            if nbytes and f.readinto(buf) != nbytes:
                raise TruncatedFileError("EVT1: short read")
            # copy into a zero-padded array: the reference rebuilds each Event,
            # so the 3 pad bytes of a record never survive a read (io.hpp:137-140)
            src = np.frombuffer(buf, EVENT_DTYPE)
            events = np.zeros(count, EVENT_DTYPE)
            for name in EVENT_DTYPE.names:
                events[name] = src[name]
            raw = events
    t0 = int(raw["t_us"][0]) if count else 0
    t1 = int(raw["t_us"][-1]) + 1 if count else 0
    s = EventSlice(width, height, t0, t1, events)
    if count:
        (engine or default_engine()).validate_slice(s, check_window=False)
    return s


def _host_events(slice_: EventSlice) -> np.ndarray:
    ev = slice_.events
    if _is_torch(ev):
        ev = ev.reshape(-1).cpu().numpy().view(EVENT_DTYPE)
    return np.asarray(ev, EVENT_DTYPE)


def write_events(slice_: EventSlice, path, engine: Optional[Engine] = None) -> None:
    """write_events (io.hpp:156-172): EventSlice::validate (on the device), then
    the header and zero-padded records."""
    eng = engine or default_engine()
    eng.validate_slice(slice_, check_window=True)
    ev = _host_events(slice_)
    rec = np.zeros(len(ev), EVENT_DTYPE)  # pad bytes written as 0 (io.hpp:170)
    for name in EVENT_DTYPE.names:
        rec[name] = ev[name]
    head = (EVT1_MAGIC + int(slice_.width).to_bytes(2, "little")
            + int(slice_.height).to_bytes(2, "little") + len(ev).to_bytes(8, "little"))
    try:
        with open(os.fspath(path), "wb") as f:
            f.write(head)
            f.write(rec.tobytes())
    except OSError as e:
        raise IoError(f"cannot write {path}: {e}") from None


def format_number(v: float) -> str:
    """format_number (io.hpp:295-299): std::to_chars(double) -- the shortest
    round-trip digits, printed fixed or scientific, whichever is shorter (fixed
    on a tie; a fixed integer keeps its exact digits)."""
    import decimal
    import math
    v = float(v)
    if math.isnan(v):
        return "-nan" if math.copysign(1.0, v) < 0 else "nan"
    if math.isinf(v):
        return "-inf" if v < 0 else "inf"
    sign = "-" if math.copysign(1.0, v) < 0 else ""
    if v == 0.0:
        return sign + "0"
    t = decimal.Decimal(repr(abs(v))).as_tuple()  # repr = shortest round-trip digits
    digits = "".join(map(str, t.digits)).lstrip("0")
    exp = t.exponent + (len(t.digits) - len("".join(map(str, t.digits)).rstrip("0")))
    digits = digits.rstrip("0")
    n = len(digits)
    sci_e = exp + n - 1
    sci = digits[0] + ("." + digits[1:] if n > 1 else "") + \
        ("e-" if sci_e < 0 else "e+") + f"{abs(sci_e):02d}"
    if exp >= 0:  # an integer: printf-style fixed prints all its exact digits
        fixed = str(int(abs(v)))
    elif sci_e >= 0:
        fixed = digits[: n + exp] + "." + digits[n + exp:]
    else:
        fixed = "0." + "0" * (-sci_e - 1) + digits
    return sign + (fixed if len(fixed) <= len(sci) else sci)


# ---- PFM float maps (io.hpp:178-236), used by the predictor checkpoints -------

_WS = b" \t\n\v\f\r"  # std::isspace in the "C" locale


def _next_token(data: bytes, pos: int, what: str):
    while pos < len(data) and data[pos] in _WS:
        pos += 1
    if pos >= len(data):
        raise TruncatedFileError(f"{what}: unexpected end of header")
    start = pos
    while pos < len(data) and data[pos] not in _WS:
        pos += 1
    return data[start:pos].decode("latin-1"), pos


def _parse_int(tok: str, what: str) -> int:  # std::from_chars over the whole token
    import re
    if not re.fullmatch(r"-?[0-9]+", tok):
        raise IoError(f"{what}: bad integer '{tok}'")
    v = int(tok)
    if not -2**31 <= v < 2**31:
        raise IoError(f"{what}: bad integer '{tok}'")
    return v


def _strtod(tok: str) -> float:  # std::strtod: the longest valid prefix, 0 if none
    import re
    m = re.match(r"[+-]?(?:(?:[0-9]+\.?[0-9]*|\.[0-9]+)(?:[eE][+-]?[0-9]+)?|inf(?:inity)?|nan)",
                 tok, re.IGNORECASE)
    return float(m.group(0)) if m else 0.0


def read_pfm(path) -> np.ndarray:
    """read_pfm (io.hpp:181-217): a grayscale "Pf" map as float32 [H, W], top row
    first (the file stores the bottom row first; a negative scale means little
    endian, a magnitude != 1 scales the values)."""
    try:
        data = open(os.fspath(path), "rb").read()
    except OSError as e:
        raise IoError(f"cannot open {path}: {e}") from None
    magic, pos = _next_token(data, 0, "PFM")
    if magic != "Pf":
        raise BadMagicError(f"PFM: expected grayscale magic 'Pf' in {path}")
    tok, pos = _next_token(data, pos, "PFM")
    w = _parse_int(tok, "PFM width")
    tok, pos = _next_token(data, pos, "PFM")
    h = _parse_int(tok, "PFM height")
    tok, pos = _next_token(data, pos, "PFM")
    scale = _strtod(tok)
    if scale == 0.0:
        raise IoError("PFM: zero scale")
    if w <= 0 or h <= 0:
        raise DimensionMismatchError("PFM: non-positive dimensions")
    pos += 1  # exactly one whitespace byte separates header and raster
    need = w * h * 4
    if len(data) - pos < need:
        raise TruncatedFileError("PFM: raster shorter than w*h")
    if len(data) - pos > need:
        raise IoError("PFM: trailing bytes after raster")
    little = scale < 0.0
    img = np.frombuffer(data, "<f4" if little else ">f4", w * h, pos).astype(np.float32)
    mag = np.float32(-scale if little else scale)
    if mag != np.float32(1.0):
        img = img * mag
    return img.reshape(h, w)[::-1].copy()


def write_pfm(img, path) -> None:
    """write_pfm (io.hpp:219-228): little-endian float32, bottom row first."""
    a = np.asarray(img, np.float32)
    if a.ndim != 2 or a.size == 0:
        raise DimensionMismatchError("PFM: refusing to write empty image")
    h, w = a.shape
    try:
        with open(os.fspath(path), "wb") as f:
            f.write(f"Pf\n{w} {h}\n-1.0\n".encode())
            f.write(np.ascontiguousarray(a[::-1]).astype("<f4").tobytes())
    except OSError as e:
        raise IoError(f"cannot open {path} for writing: {e}") from None


def read_csv(path):
    """read_csv (io.hpp:323-345): no quoting, comma-separated, '\r' stripped."""
    try:
        text = open(os.fspath(path), "rb").read().decode("latin-1")
    except OSError as e:
        raise IoError(f"cannot open {path}: {e}") from None
    lines = text.split("\n")
    if lines and lines[-1] == "":
        lines.pop()  # std::getline: a final newline ends the last line
    return [ln[:-1].split(",") if ln.endswith("\r") else ln.split(",") for ln in lines]


@dataclass
class Windows:
    """Consecutive windows [t0 + w*window_us, t0 + (w+1)*window_us) of one slice:
    events of window w = events[offsets[w] : offsets[w+1]]."""
    slice: EventSlice
    t0_us: int
    window_us: int
    offsets: np.ndarray  # uint64 [n_windows + 1]

    @property
    def n_windows(self) -> int:
        return len(self.offsets) - 1

    def window(self, w: int) -> EventSlice:
        """Window w as an EventSlice (a view of the events, no copy)."""
        if not 0 <= w < self.n_windows:
            raise ConfigError(f"window {w} outside [0, {self.n_windows})")
        a, b = int(self.offsets[w]), int(self.offsets[w + 1])
        t = self.t0_us + w * self.window_us
        return EventSlice(self.slice.width, self.slice.height, t, t + self.window_us,
                          self.slice.events[a:b])

    def chain_batch(self, engine: Engine, depth, poses, k, out=None, out_device=None):
        """Engine.chain_batch over every window (one clock shift per window)."""
        return engine.chain_batch(depth, poses, k, self.t0_us, self.t0_us + self.window_us,
                                  self.slice.events, self.offsets, out=out,
                                  out_device=out_device, window_stride_us=self.window_us)


def slice_windows(slice_: EventSlice, window_us: int, n_windows: Optional[int] = None,
                  t0_us: Optional[int] = None, engine: Optional[Engine] = None) -> Windows:
    """Cuts a time-sorted slice into consecutive ``window_us`` windows from
    ``t0_us`` (default: the slice's t_start); ``n_windows`` defaults to the
    windows needed to cover [t0, t_end). Boundaries come from a device binary
    search over the events (Engine.window_offsets)."""
    if window_us <= 0:
        raise ConfigError("windows: window length must be positive")
    t0 = int(slice_.t_start_us if t0_us is None else t0_us)
    if n_windows is None:
        span = max(0, int(slice_.t_end_us) - t0)
        n_windows = max(1, -(-span // int(window_us)))
    if n_windows < 1:
        raise ConfigError("windows: need at least one window")
    eng = engine or default_engine()
    offs = eng.window_offsets(slice_.events, t0, int(window_us), int(n_windows))
    return Windows(slice_, t0, int(window_us), offs)
