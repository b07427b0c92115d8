"""BERT encoder layer and stacked forward on the B200 (reference
encoder.py:1-437), drop-in for ``packbert.encoder``.

The configuration, weight containers, deterministic init, PKBW weight files
and key=value config parsing are the reference's (same names, fields, RNG
draws, byte format and error types).  ``encoder_layer`` / ``forward`` run the
padding-free pipeline of ``OptFlags.all_on()`` on sm_100a through the C ABI
(``bt_encoder_layer`` / ``bt_encoder_forward``): device plan + pack, four
tcgen05 GEMMs with fused bias / bias+GELU epilogues, fused varlen MHA, two
fused add-bias+residual+LayerNorm passes per layer, unpack.  Weights are
uploaded once per ``EncoderWeights`` object to bf16 (transposed to the
K-major operand layout) and cached.

The other ladder rungs (``OptFlags`` subsets, reference bench.py:35-41) are
served by ``ladder.py`` from the same kernels.
"""

from __future__ import annotations

import ctypes as C
import os
import struct
import threading
import weakref
from dataclasses import dataclass, field, replace
from pathlib import Path

import numpy as np

from . import _lib
from .attention import DEFAULT_CUTOFF, DEFAULT_SPLIT_SEQ_LEN
from .errors import ConfigError, ShapeError, WeightFormatError
from .fusion import LayernormParams
from .packing import PackingPlan, SeqLengths, as_seq_lengths, ensure_plan, plan_for_lengths
from .tensor import FlopCounter, Tensor, host_array, is_device, rows_cols

WEIGHT_INIT_RANGE = 0.02


@dataclass(frozen=True)
class OptFlags:
    fuse_layernorm: bool = False
    fuse_bias_gelu: bool = False
    zero_padding: bool = False
    fused_mha: bool = False

    @classmethod
    def all_on(cls) -> "OptFlags":
        return cls(True, True, True, True)


@dataclass(frozen=True)
class ModelConfig:
    layers: int
    head_num: int
    head_size: int
    max_seq_len: int
    batch_size: int
    ffn_scale: int = 4
    cutoff: int = DEFAULT_CUTOFF
    split_seq_len: int = DEFAULT_SPLIT_SEQ_LEN
    flags: OptFlags = field(default_factory=OptFlags)
    share_layer_weights: bool = False

    def __post_init__(self):
        for name in ("layers", "head_num", "head_size", "max_seq_len", "batch_size", "ffn_scale"):
            if getattr(self, name) < 1:
                raise ConfigError(f"{name} must be >= 1, got {getattr(self, name)}")
        if self.flags.fused_mha and not self.flags.zero_padding:
            raise ConfigError("fused_mha requires zero_padding: the fused kernels consume the packing plan")

    @property
    def hidden_dim(self) -> int:
        return self.head_num * self.head_size

    def with_flags(self, flags: OptFlags) -> "ModelConfig":
        return replace(self, flags=flags)


PRESETS: dict[str, dict] = {
    "bert_base": {"layers": 12, "head_num": 12, "head_size": 64, "share_layer_weights": False},
    "albert": {"layers": 12, "head_num": 16, "head_size": 64, "share_layer_weights": True},
    "distilbert": {"layers": 6, "head_num": 12, "head_size": 64, "share_layer_weights": False},
    "deberta_cfg": {"layers": 12, "head_num": 12, "head_size": 64, "share_layer_weights": False},
}
# BERT-large geometry of the north-star configs C3/C5 (not a reference preset).
BERT_LARGE = {"layers": 24, "head_num": 16, "head_size": 64, "share_layer_weights": False}


def preset_config(name: str, batch_size: int, max_seq_len: int, flags: OptFlags = OptFlags(),
                  layers: int | None = None) -> ModelConfig:
    if name not in PRESETS:
        raise ConfigError(f"unknown preset {name!r}; choose from {sorted(PRESETS)}")
    p = PRESETS[name]
    return ModelConfig(layers=layers if layers is not None else p["layers"], head_num=p["head_num"],
                       head_size=p["head_size"], max_seq_len=max_seq_len, batch_size=batch_size, flags=flags,
                       share_layer_weights=p["share_layer_weights"])


def as_model_config(cfg) -> ModelConfig:
    """Accept the reference's ModelConfig (duck-typed) or ours."""
    if isinstance(cfg, ModelConfig):
        return cfg
    f = cfg.flags
    return ModelConfig(layers=cfg.layers, head_num=cfg.head_num, head_size=cfg.head_size,
                       max_seq_len=cfg.max_seq_len, batch_size=cfg.batch_size, ffn_scale=cfg.ffn_scale,
                       cutoff=cfg.cutoff, split_seq_len=cfg.split_seq_len,
                       flags=OptFlags(f.fuse_layernorm, f.fuse_bias_gelu, f.zero_padding, f.fused_mha),
                       share_layer_weights=cfg.share_layer_weights)


@dataclass(eq=False)
class LayerWeights:
    """Per-layer parameters, [in, out] matrices, QKV as column blocks
    (reference encoder.py:108-122)."""

    qkv_weight: np.ndarray
    qkv_bias: np.ndarray
    attn_out_weight: np.ndarray
    attn_out_bias: np.ndarray
    ffn_w1: np.ndarray
    ffn_b1: np.ndarray
    ffn_w2: np.ndarray
    ffn_b2: np.ndarray
    ln0: LayernormParams
    ln1: LayernormParams


@dataclass(eq=False)
class EncoderWeights:
    layers: list
    shared: bool

    def layer(self, index: int):
        return self.layers[0] if self.shared else self.layers[index]


def _tensor_shapes(config: ModelConfig) -> list[tuple[str, tuple[int, ...]]]:
    h = config.hidden_dim
    f = config.ffn_scale * h
    return [("qkv_weight", (h, 3 * h)), ("qkv_bias", (3 * h,)), ("attn_out_weight", (h, h)),
            ("attn_out_bias", (h,)), ("ffn_w1", (h, f)), ("ffn_b1", (f,)), ("ffn_w2", (f, h)), ("ffn_b2", (h,)),
            ("ln0_gamma", (h,)), ("ln0_beta", (h,)), ("ln1_gamma", (h,)), ("ln1_beta", (h,))]


def _layer_from_arrays(a: dict) -> LayerWeights:
    return LayerWeights(qkv_weight=a["qkv_weight"], qkv_bias=a["qkv_bias"], attn_out_weight=a["attn_out_weight"],
                        attn_out_bias=a["attn_out_bias"], ffn_w1=a["ffn_w1"], ffn_b1=a["ffn_b1"],
                        ffn_w2=a["ffn_w2"], ffn_b2=a["ffn_b2"],
                        ln0=LayernormParams(gamma=a["ln0_gamma"], beta=a["ln0_beta"]),
                        ln1=LayernormParams(gamma=a["ln1_gamma"], beta=a["ln1_beta"]))


def _layer_arrays(layer) -> dict:
    return {"qkv_weight": layer.qkv_weight, "qkv_bias": layer.qkv_bias, "attn_out_weight": layer.attn_out_weight,
            "attn_out_bias": layer.attn_out_bias, "ffn_w1": layer.ffn_w1, "ffn_b1": layer.ffn_b1,
            "ffn_w2": layer.ffn_w2, "ffn_b2": layer.ffn_b2, "ln0_gamma": np.asarray(layer.ln0.gamma),
            "ln0_beta": np.asarray(layer.ln0.beta), "ln1_gamma": np.asarray(layer.ln1.gamma),
            "ln1_beta": np.asarray(layer.ln1.beta)}


def init_weights(config, seed: int = 0) -> EncoderWeights:
    """U(-0.02, 0.02), one draw per tensor in declaration order (reference
    encoder.py:168-180) -- bit-identical to the reference's weights."""
    config = as_model_config(config)
    rng = np.random.default_rng(seed)
    stored = 1 if config.share_layer_weights else config.layers
    layers = []
    for _ in range(stored):
        arrays = {name: rng.uniform(-WEIGHT_INIT_RANGE, WEIGHT_INIT_RANGE, shape).astype(np.float32)
                  for name, shape in _tensor_shapes(config)}
        layers.append(_layer_from_arrays(arrays))
    return EncoderWeights(layers=layers, shared=config.share_layer_weights)


# ---------------------------------------------------------------- PKBW files
_WEIGHT_MAGIC = b"PKBW"
_WEIGHT_VERSION = 1
_HEADER = "<4sI5I"
_HEADER_FIELDS = ("layers", "head_num", "head_size", "ffn_scale", "share_layer_weights")


def save_weights(path, weights, config) -> None:
    """PKBW v1: little-endian header + raw <f4 tensors in declaration order
    (reference encoder.py:183-206)."""
    config = as_model_config(config)
    header = struct.pack(_HEADER, _WEIGHT_MAGIC, _WEIGHT_VERSION, config.layers, config.head_num,
                         config.head_size, config.ffn_scale, 1 if config.share_layer_weights else 0)
    with open(path, "wb") as f:
        f.write(header)
        for layer in weights.layers:
            arrays = _layer_arrays(layer)
            for name, _ in _tensor_shapes(config):
                f.write(np.ascontiguousarray(arrays[name], dtype="<f4").tobytes())


def load_weights(path, config) -> EncoderWeights:
    """Strictly validated PKBW load (reference encoder.py:226-268)."""
    config = as_model_config(config)
    raw = Path(path).read_bytes()
    hsz = struct.calcsize(_HEADER)
    if len(raw) < hsz:
        raise WeightFormatError(f"{path}: file too short for a weight header")
    magic, version, *fields = struct.unpack(_HEADER, raw[:hsz])
    if magic != _WEIGHT_MAGIC:
        raise WeightFormatError(f"{path}: bad magic {magic!r}")
    if version != _WEIGHT_VERSION:
        raise WeightFormatError(f"{path}: unsupported version {version}")
    expected = (config.layers, config.head_num, config.head_size, config.ffn_scale,
                1 if config.share_layer_weights else 0)
    for name, got, want in zip(_HEADER_FIELDS, fields, expected):
        if got != want:
            raise WeightFormatError(f"{path}: {name} is {got} in file, config expects {want}")
    shapes = _tensor_shapes(config)
    stored = 1 if config.share_layer_weights else config.layers
    per_layer = sum(int(np.prod(s)) for _, s in shapes)
    want_bytes = hsz + 4 * per_layer * stored
    if len(raw) != want_bytes:
        raise WeightFormatError(f"{path}: payload is {len(raw) - hsz} bytes, expected {want_bytes - hsz}")
    off = hsz
    layers = []
    for _ in range(stored):
        arrays = {}
        for name, shape in shapes:
            n = int(np.prod(shape))
            arrays[name] = np.frombuffer(raw, dtype="<f4", count=n, offset=off).reshape(shape).astype(np.float32)
            off += 4 * n
        layers.append(_layer_from_arrays(arrays))
    return EncoderWeights(layers=layers, shared=config.share_layer_weights)


_CONFIG_BOOL_KEYS = {"fuse_layernorm", "fuse_bias_gelu", "zero_padding", "fused_mha", "share_layer_weights"}
_CONFIG_INT_KEYS = {"layers", "head_num", "head_size", "ffn_scale", "max_seq_len", "batch_size", "cutoff",
                    "split_seq_len"}


def parse_config_text(text: str) -> ModelConfig:
    """key=value config, '#' comments (reference encoder.py:290-324)."""
    values: dict = {}
    flag_values: dict = {}
    for lineno, line in enumerate(text.splitlines(), start=1):
        line = line.split("#", 1)[0].strip()
        if not line:
            continue
        if "=" not in line:
            raise ConfigError(f"line {lineno}: expected key=value, got {line!r}")
        key, _, value = line.partition("=")
        key, value = key.strip(), value.strip()
        if key in _CONFIG_INT_KEYS:
            try:
                values[key] = int(value)
            except ValueError:
                raise ConfigError(f"line {lineno}: {key} must be an integer, got {value!r}") from None
        elif key in _CONFIG_BOOL_KEYS:
            low = value.lower()
            if low in ("1", "true", "yes", "on"):
                parsed = True
            elif low in ("0", "false", "no", "off"):
                parsed = False
            else:
                raise ConfigError(f"line {lineno}: {key} must be a boolean, got {value!r}")
            if key == "share_layer_weights":
                values[key] = parsed
            else:
                flag_values[key] = parsed
        else:
            raise ConfigError(f"line {lineno}: unknown config key {key!r}")
    missing = [k for k in ("layers", "head_num", "head_size", "max_seq_len", "batch_size") if k not in values]
    if missing:
        raise ConfigError(f"missing required config keys: {', '.join(missing)}")
    return ModelConfig(flags=OptFlags(**flag_values), **values)


def parse_config_file(path) -> ModelConfig:
    return parse_config_text(Path(path).read_text())


# ---------------------------------------------------------------- device side

class DeviceLayer:
    """One layer's parameters resident in HBM: bf16 K-major matrices, fp32
    vectors, plus the C struct the library reads."""

    def __init__(self, layer, torch):
        def mat(w):  # [in, out] -> [out, in] bf16: the fp32 matrix goes up as is, transpose + cast on the device
            if is_device(w):
                return w.t().to(torch.bfloat16).contiguous()
            return torch.from_numpy(np.ascontiguousarray(w, dtype=np.float32)).to("cuda").t().to(
                torch.bfloat16).contiguous()

        def vec(v):
            if is_device(v):
                return v.to(torch.float32).contiguous().reshape(-1)
            return torch.from_numpy(np.ascontiguousarray(np.asarray(v, np.float32).reshape(-1))).to("cuda")

        self.qkv_w, self.qkv_b = mat(layer.qkv_weight), vec(layer.qkv_bias)
        self.ao_w, self.ao_b = mat(layer.attn_out_weight), vec(layer.attn_out_bias)
        self.w1, self.b1 = mat(layer.ffn_w1), vec(layer.ffn_b1)
        self.w2, self.b2 = mat(layer.ffn_w2), vec(layer.ffn_b2)
        self.ln0_g, self.ln0_b = vec(layer.ln0.gamma), vec(layer.ln0.beta)
        self.ln1_g, self.ln1_b = vec(layer.ln1.gamma), vec(layer.ln1.beta)
        self.ln0_eps = float(getattr(layer.ln0, "eps", 1e-12))
        self.ln1_eps = float(getattr(layer.ln1, "eps", 1e-12))
        self.c = _lib.LayerWeightsC(
            self.qkv_w.data_ptr(), self.qkv_b.data_ptr(), self.ao_w.data_ptr(), self.ao_b.data_ptr(),
            self.w1.data_ptr(), self.b1.data_ptr(), self.w2.data_ptr(), self.b2.data_ptr(),
            self.ln0_g.data_ptr(), self.ln0_b.data_ptr(), self.ln1_g.data_ptr(), self.ln1_b.data_ptr(),
            self.ln0_eps, self.ln1_eps)


def _check_layer_shapes(layer, config: ModelConfig) -> None:
    arrays = _layer_arrays(layer)
    for name, shape in _tensor_shapes(config):
        got = tuple(arrays[name].shape)
        if got != shape:
            raise ShapeError(f"layer tensor {name} has shape {got}, config expects {shape}")


def layer_cfg_c(config: ModelConfig) -> _lib.LayerCfgC:
    return _lib.LayerCfgC(config.head_num, config.head_size, config.ffn_scale, config.max_seq_len, config.cutoff,
                          config.split_seq_len)


# host-I/O pipeline depth of forward() on host buffers (BertEncoderB200.default_chunks)
E2E_CHUNKS_DEFAULT = 1
# forward_host_stream: batches of more sequences than this move their padded
# buffers as one DMA each way instead of one DMA per sequence
STREAM_ROW_COPIES_MAX = 512


class BertEncoderB200:
    """Device-resident encoder: uploaded weights, cached workspace, and the
    stream-ordered forward used by ``forward()`` and ``bench.py``."""

    def __init__(self, weights, config):
        torch = _lib.require_device()
        self.torch = torch
        self.config = as_model_config(config)
        if self.config.head_size != 64:
            raise ConfigError(f"the sm_100a kernels support head_size 64, got {self.config.head_size}")
        if self.config.hidden_dim % 64:
            raise ConfigError(f"hidden size {self.config.hidden_dim} must be a multiple of 64")
        stored = [weights.layers[0]] if weights.shared else list(weights.layers)
        for lw in stored:
            _check_layer_shapes(lw, self.config)
        self._stored = [DeviceLayer(lw, torch) for lw in stored]
        n = self.config.layers
        self._layers = [self._stored[0] if weights.shared else self._stored[i] for i in range(n)]
        self._c_layers = (_lib.LayerWeightsC * n)(*[dl.c for dl in self._layers])
        self._cfg_c = layer_cfg_c(self.config)
        self._ws = None
        self._ws_event = None
        self._graphs = {}
        # one forward at a time per engine: the workspace, the cached graphs
        # and their I/O buffers are shared state (the service runs requests on
        # a thread pool)
        self._lock = threading.RLock()
        self._io_streams = None  # host-I/O pipeline: H2D, compute, D2H
        self._io_events = []
        self._stage = {}  # page-locked packed staging buffer for pageable inputs
        self._stream_stage = {}  # forward_host_stream: two page-locked packed staging slots
        self._pool = None

    def layer(self, i: int) -> DeviceLayer:
        return self._layers[i]

    def workspace(self, nbytes: int, stream=None):
        """The shared activation workspace, ordered after its previous use:
        a caller on another stream waits (on the device) for the last
        launch that used it, so two threads on different streams never
        overlap on it.  Call ``_ws_used(stream)`` after queueing the launch."""
        torch = self.torch
        s = stream if stream is not None else torch.cuda.current_stream()
        if self._ws_event is not None and not torch.cuda.is_current_stream_capturing():
            s.wait_event(self._ws_event)
        if self._ws is None or self._ws.numel() < nbytes:
            self._ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device="cuda")
        return self._ws

    def _ws_used(self, stream=None):
        torch = self.torch
        if torch.cuda.is_current_stream_capturing():
            return  # (graph replays are ordered by the stream they replay on)
        s = stream if stream is not None else torch.cuda.current_stream()
        if self._ws_event is None:
            self._ws_event = torch.cuda.Event()
        self._ws_event.record(s)

    def forward_device(self, lengths_dev, bs: int, T: int, x_padded_f32, out_padded_f32, stream=None,
                       config: ModelConfig | None = None):
        """Device forward: int32 lengths [bs], fp32 padded input [bs*mx, k] ->
        fp32 padded output (exact-zero padded rows).  No host sync."""
        with self._lock:
            cfg = config or self.config
            cfg_c = self._cfg_c if config is None else layer_cfg_c(cfg)
            ws_bytes = int(_lib.load().bt_forward_workspace_bytes(C.byref(cfg_c), bs, T))
            ws = self.workspace(ws_bytes, stream)
            _lib.call("bt_encoder_forward", self._c_layers, cfg.layers, C.byref(cfg_c), lengths_dev.data_ptr(), bs, T,
                      x_padded_f32.data_ptr(), out_padded_f32.data_ptr(), ws.data_ptr(), ws_bytes,
                      _lib.stream_ptr(stream))
            self._ws_used(stream)
            return out_padded_f32

    def forward_ptrs(self, lengths_ptr: int, bs: int, T: int, x_ptr: int, out_ptr: int, stream=None,
                     config: ModelConfig | None = None):
        """Forward on raw pointers: lengths int32[bs], padded fp32 input and
        output [bs*mx, k].  Each may be device memory or pinned host memory
        (zero-copy: only valid input rows cross PCIe; no bulk memcpy)."""
        with self._lock:
            cfg = config or self.config
            cfg_c = self._cfg_c if config is None else layer_cfg_c(cfg)
            ws_bytes = int(_lib.load().bt_forward_workspace_bytes(C.byref(cfg_c), bs, T))
            ws = self.workspace(ws_bytes, stream)
            _lib.call("bt_encoder_forward", self._c_layers, cfg.layers, C.byref(cfg_c), lengths_ptr, bs, T, x_ptr,
                      out_ptr, ws.data_ptr(), ws_bytes, _lib.stream_ptr(stream))
            self._ws_used(stream)

    GRAPH_CACHE = 8  # batch (range) shapes whose packed forward is kept as a CUDA graph

    def _graph_entry(self, seqs: SeqLengths, cfg: ModelConfig, cfg_c, slot: int = 0):
        """(graph, x_packed, y_packed) for this batch shape: device buffers
        owned by the entry and a CUDA graph of bt_encoder_forward_packed over
        them (captured after one eager warm-up run, which also autotunes).
        ``slot`` keeps independent entries of one shape (double buffering in
        ``forward_host_stream``)."""
        torch = self.torch
        key = (tuple(seqs.lengths), seqs.max_seq_len, cfg.layers, cfg.cutoff, cfg.split_seq_len, slot)
        hit = self._graphs.pop(key, None)
        if hit is not None:
            self._graphs[key] = hit  # most recently used last
            return hit
        bs, T, k = seqs.batch_size, seqs.total, cfg.hidden_dim
        lengths_dev = torch.tensor(seqs.lengths, dtype=torch.int32, device="cuda")
        xp = torch.empty((T, k), dtype=torch.float32, device="cuda")
        yp = torch.empty((T, k), dtype=torch.float32, device="cuda")
        ws_bytes = int(_lib.load().bt_forward_workspace_bytes(C.byref(cfg_c), bs, T))
        ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")

        def run():
            _lib.call("bt_encoder_forward_packed", self._c_layers, cfg.layers, C.byref(cfg_c), lengths_dev.data_ptr(),
                      bs, T, xp.data_ptr(), yp.data_ptr(), ws.data_ptr(), ws_bytes, _lib.stream_ptr())

        entry = (self._capture(run), run, xp, yp, lengths_dev, ws)
        self._graphs[key] = entry
        while len(self._graphs) > self.GRAPH_CACHE:
            self._graphs.pop(next(iter(self._graphs)))
        return entry

    def _padded_entry(self, seqs: SeqLengths, cfg: ModelConfig, cfg_c, slot: int = 0):
        """As _graph_entry, over the PADDED layout: device buffers [bs*mx, k]
        fp32 in and out and a CUDA graph of bt_encoder_forward (device plan,
        pack, layers, fp32 output rows with exact-zero padded rows), so the
        host copies are one contiguous DMA each way.  Used where per-sequence
        row copies would be thousands of DMA commands per batch."""
        torch = self.torch
        key = ("padded", tuple(seqs.lengths), seqs.max_seq_len, cfg.layers, cfg.cutoff, cfg.split_seq_len, slot)
        hit = self._graphs.pop(key, None)
        if hit is not None:
            self._graphs[key] = hit
            return hit
        bs, T, k, mx = seqs.batch_size, seqs.total, cfg.hidden_dim, seqs.max_seq_len
        lengths_dev = torch.tensor(seqs.lengths, dtype=torch.int32, device="cuda")
        xp = torch.empty((bs * mx, k), dtype=torch.float32, device="cuda")
        yp = torch.empty((bs * mx, k), dtype=torch.float32, device="cuda")
        ws_bytes = int(_lib.load().bt_forward_workspace_bytes(C.byref(cfg_c), bs, T))
        ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")

        def run():
            _lib.call("bt_encoder_forward", self._c_layers, cfg.layers, C.byref(cfg_c), lengths_dev.data_ptr(), bs, T,
                      xp.data_ptr(), yp.data_ptr(), ws.data_ptr(), ws_bytes, _lib.stream_ptr())

        entry = (self._capture(run), run, xp, yp, lengths_dev, ws)
        self._graphs[key] = entry
        while len(self._graphs) > self.GRAPH_CACHE:
            self._graphs.pop(next(iter(self._graphs)))
        return entry

    def _capture(self, run):
        """A CUDA graph of run() (after one eager warm-up, which also
        autotunes the GEMMs), or None where capture is unsupported."""
        torch = self.torch
        run()
        torch.cuda.synchronize()
        try:
            g = torch.cuda.CUDAGraph()
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                run()
            torch.cuda.current_stream().wait_stream(side)
            with torch.cuda.graph(g):
                run()
            return g
        except Exception:  # noqa: BLE001 -- graph capture unsupported here: launch eagerly
            return None

    @staticmethod
    def chunk_bounds(lengths, chunks) -> list[tuple[int, int]]:
        """Sequence ranges [b0, b1) of the host-I/O pipeline.  ``chunks`` is
        a count n (token-balanced cut into n contiguous ranges) or a list of
        token fractions (e.g. (0.3, 0.7)); sequences are never split."""
        bs = len(lengths)
        if isinstance(chunks, int):
            fr = [1.0 / max(1, chunks)] * max(1, chunks)
        else:
            fr = [float(f) for f in chunks]
        n = max(1, min(len(fr), bs))
        fr = fr[:n]
        tot = float(sum(lengths))
        cum = np.cumsum(np.asarray(lengths, dtype=np.float64))
        cuts, acc = [0], 0.0
        for f in fr[:-1]:
            acc += f / sum(fr) * tot
            c = int(np.argmin(np.abs(cum - acc))) + 1  # the sequence boundary nearest the target
            c = min(max(c, cuts[-1] + 1), bs - (n - len(cuts)))
            cuts.append(c)
        cuts.append(bs)
        return [(cuts[i], cuts[i + 1]) for i in range(len(cuts) - 1) if cuts[i + 1] > cuts[i]]

    def default_chunks(self, seqs: SeqLengths):
        """Host-I/O pipeline depth (BT_E2E_CHUNKS overrides: "1", "3" or
        fractions "0.25,0.5,0.25")."""
        env = os.environ.get("BT_E2E_CHUNKS")
        if env:
            parts = [p for p in env.split(",") if p.strip()]
            return int(parts[0]) if len(parts) == 1 else [float(p) for p in parts]
        # PCIe moves ~40 GB/s each way: below ~1 MB of rows per direction the
        # copy is short next to the launch-bound forward -- one chunk
        if seqs.batch_size < 2 or seqs.total * self.config.hidden_dim * 4 < (1 << 20):
            return 1
        return E2E_CHUNKS_DEFAULT

    def forward_host_packed(self, seqs: SeqLengths, x_pinned, out_pinned, config: ModelConfig | None = None,
                            chunks=None):
        """End-to-end forward on pinned host buffers [bs*mx, k] fp32: only the
        valid rows cross PCIe (async DMA per sequence, both directions).

        The batch is cut into contiguous sequence ranges (``chunks``,
        default ``default_chunks``) -- sequences are independent, so each
        range is its own packed forward (a CUDA graph cached per range
        shape) -- and the ranges are pipelined over three streams:
        H2D(i + 1) || forward(i) || D2H(i - 1).  The padded output rows are
        zeroed on the host while the GPU works.  Synchronises."""
        with self._lock:
            cfg = config or self.config
            cfg_c = self._cfg_c if config is None else layer_cfg_c(cfg)
            bs, mx, k = seqs.batch_size, seqs.max_seq_len, cfg.hidden_dim
            lengths_h = np.ascontiguousarray(np.asarray(seqs.lengths, dtype=np.int32))
            bounds = self.chunk_bounds(seqs.lengths, self.default_chunks(seqs) if chunks is None else chunks)
            entries = [self._graph_entry(SeqLengths(seqs.lengths[b0:b1], mx), cfg, cfg_c) for b0, b1 in bounds]
            torch = self.torch
            if self._io_streams is None:
                self._io_streams = (torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream())
            h2d, comp, d2h = self._io_streams
            while len(self._io_events) < 2 * len(bounds):
                self._io_events.append(torch.cuda.Event())
            ev_in, ev_done = self._io_events[0::2], self._io_events[1::2]
            h2d.wait_stream(torch.cuda.current_stream())
            comp.wait_stream(torch.cuda.current_stream())  # the cached graphs' buffers: previous call done
            row_b = k * 4
            lp = lengths_h.ctypes.data
            xb, ob = x_pinned.data_ptr(), out_pinned.data_ptr()
            for i, ((b0, b1), e) in enumerate(zip(bounds, entries)):
                with torch.cuda.stream(h2d):
                    _lib.call("bt_copy_rows", e[2].data_ptr(), xb + b0 * mx * row_b, lp + 4 * b0, b1 - b0, mx, row_b,
                              1, _lib.stream_ptr())
                    ev_in[i].record(h2d)
            for i, e in enumerate(entries):
                comp.wait_event(ev_in[i])
                with torch.cuda.stream(comp):
                    if e[0] is not None:
                        e[0].replay()
                    else:
                        e[1]()
                    ev_done[i].record(comp)
            # padded rows of the output are exact zeros (packing.py:158-159),
            # written on the host while the GPU computes -- before the D2H
            # enqueue, which can block the host once a large batch's per-sequence
            # copies fill the DMA queue (disjoint rows: no ordering needed)
            self._zero_padded_rows(out_pinned, seqs, k)
            for i, ((b0, b1), e) in enumerate(zip(bounds, entries)):
                d2h.wait_event(ev_done[i])
                with torch.cuda.stream(d2h):
                    _lib.call("bt_copy_rows", ob + b0 * mx * row_b, e[3].data_ptr(), lp + 4 * b0, b1 - b0, mx, row_b,
                              0, _lib.stream_ptr())
            d2h.synchronize()
            torch.cuda.current_stream().wait_stream(d2h)
            return out_pinned

    def _zero_padded_rows(self, out_pinned, seqs: SeqLengths, k: int) -> None:
        """Zero the padded rows of a host output [bs*mx, k] (the DMA writes
        only valid rows).  Large batches split the memsets over the engine's
        thread pool (C5: 1.7 GB of padding, 183 ms on one thread)."""
        import concurrent.futures as cf

        bs, mx = seqs.batch_size, seqs.max_seq_len
        o = out_pinned.numpy().reshape(bs, mx, k)

        def zero(b0, b1):
            for b in range(b0, b1):
                n = seqs.lengths[b]
                if n < mx:
                    o[b, n:] = 0.0

        pad_bytes = (bs * mx - seqs.total) * k * 4
        if pad_bytes < (64 << 20) or bs < 8:
            zero(0, bs)
            return
        if self._pool is None:
            self._pool = cf.ThreadPoolExecutor(max_workers=4, thread_name_prefix="bt200-host")
        step = -(-bs // 8)
        for f in [self._pool.submit(zero, b, min(bs, b + step)) for b in range(0, bs, step)]:
            f.result()

    def forward_host_pageable(self, seqs: SeqLengths, arr, out_pinned, config: ModelConfig | None = None):
        """forward_host_packed for a pageable host input (a reference-style
        numpy ``Tensor``, fp32 [bs*mx, k]): only each sequence's valid rows
        go over PCIe, copied straight from the pageable array into the packed
        device buffer (the driver stages them page-locked and overlaps that
        with the DMA).  Batches of more than STREAM_ROW_COPIES_MAX sequences
        (or BT_PAGEABLE_STAGE=1) instead pack the valid rows into a
        write-combined staging buffer with a thread pool, then one DMA.  Then
        the cached graph and the per-sequence D2H as forward_host_packed.
        Synchronises."""
        import concurrent.futures as cf

        with self._lock:
            cfg = config or self.config
            cfg_c = self._cfg_c if config is None else layer_cfg_c(cfg)
            bs, mx, k = seqs.batch_size, seqs.max_seq_len, cfg.hidden_dim
            graph, run, xp, yp, _, _ = self._graph_entry(seqs, cfg, cfg_c)
            torch = self.torch
            T = seqs.total
            # thousands of per-sequence pageable copies (C5: 2048) cost more
            # than staging: large batches keep the staged path
            use_stage = _PAGEABLE_STAGE or bs > STREAM_ROW_COPIES_MAX
            stage = self._stage.get((T, k)) if use_stage else None
            if stage is None and use_stage:
                stage = _WcStage(T, k)
                self._stage = {(T, k): stage}  # one shape kept
            if self._pool is None:
                self._pool = cf.ThreadPoolExecutor(max_workers=4, thread_name_prefix="bt200-host")
            if self._io_streams is None:
                self._io_streams = (torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream())
            h2d, comp, d2h = self._io_streams
            cur = torch.cuda.current_stream()
            h2d.wait_stream(cur)
            comp.wait_stream(cur)
            lengths_h = np.ascontiguousarray(np.asarray(seqs.lengths, dtype=np.int32))
            if use_stage:
                starts = np.concatenate([[0], np.cumsum(lengths_h)])
                sn = stage.array
                bounds = self.chunk_bounds(seqs.lengths, min(bs, 8))

                def copy_group(b0, b1):
                    for b in range(b0, b1):
                        sn[starts[b]:starts[b + 1]] = arr[b * mx: b * mx + lengths_h[b]]

                for f in [self._pool.submit(copy_group, b0, b1) for b0, b1 in bounds]:
                    f.result()
                one = np.asarray([T], dtype=np.int32)
                with torch.cuda.stream(h2d):  # one contiguous DMA of the packed rows (a single T-row "sequence")
                    _lib.call("bt_copy_rows", xp.data_ptr(), stage.ptr, one.ctypes.data, 1, T, k * 4, 1,
                              _lib.stream_ptr())
            else:
                # each sequence's valid rows straight from the pageable array:
                # the driver stages them through its own page-locked ring and
                # overlaps that host copy with the DMA
                with torch.cuda.stream(h2d):
                    _lib.call("bt_copy_rows", xp.data_ptr(), arr.ctypes.data, lengths_h.ctypes.data, bs, mx, k * 4,
                              1, _lib.stream_ptr())
            comp.wait_stream(h2d)
            with torch.cuda.stream(comp):
                if graph is not None:
                    graph.replay()
                else:
                    run()
            self._zero_padded_rows(out_pinned, seqs, k)  # while the GPU computes (see forward_host_packed)
            d2h.wait_stream(comp)
            with torch.cuda.stream(d2h):
                _lib.call("bt_copy_rows", out_pinned.data_ptr(), yp.data_ptr(), lengths_h.ctypes.data, bs, mx, k * 4,
                          0, _lib.stream_ptr())
            d2h.synchronize()
            cur.wait_stream(d2h)
            return out_pinned

    def forward_host_stream(self, items, config: ModelConfig | None = None):
        """Serving-style stream of batches on pinned host buffers: ``items`` is
        a list of (SeqLengths, x_pinned [bs*mx, k] fp32, out_pinned).  Each
        batch is a whole forward_host_packed (valid rows DMA'd in, the cached
        graph, valid rows DMA'd out), but consecutive batches overlap on three
        streams -- H2D(i + 1) and D2H(i - 1) run under forward(i) -- with the
        device buffers double-buffered (graph entries in two slots).  An
        input may also be pageable (``_PageableRows``, a numpy caller's
        array): its valid rows are packed into one of two page-locked
        staging slots by the host thread pool while the GPU runs the
        previous batch, then DMA'd as one copy.
        Synchronises once at the end; returns the out buffers."""
        with self._lock:
            cfg = config or self.config
            cfg_c = self._cfg_c if config is None else layer_cfg_c(cfg)
            torch = self.torch
            k = cfg.hidden_dim
            row_b = k * 4
            # per-sequence valid-row DMA for small batches; a whole padded
            # buffer per direction for large ones (C5: 2 x 2048 row copies per
            # batch fill the DMA command queue and stall the host's enqueue
            # of the next batch -- 91 ms gaps between forwards, measured)
            padded = [sq.batch_size > STREAM_ROW_COPIES_MAX for sq, _, _ in items]
            entries = [self._padded_entry(sq, cfg, cfg_c, slot=i % 2) if pd else
                       self._graph_entry(sq, cfg, cfg_c, slot=i % 2)
                       for i, ((sq, _, _), pd) in enumerate(zip(items, padded))]
            if self._io_streams is None:
                self._io_streams = (torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream())
            h2d, comp, d2h = self._io_streams
            cur = torch.cuda.current_stream()
            for st in (h2d, comp, d2h):
                st.wait_stream(cur)
            n = len(items)
            ev_in = [torch.cuda.Event() for _ in range(n)]
            ev_done = [torch.cuda.Event() for _ in range(n)]
            ev_out = [torch.cuda.Event() for _ in range(n)]
            lens = [np.ascontiguousarray(np.asarray(sq.lengths, dtype=np.int32)) for sq, _, _ in items]
            whole = [np.asarray([sq.batch_size * sq.max_seq_len], dtype=np.int32) for sq, _, _ in items]
            # pageable inputs (numpy): batch i's valid rows are packed into a
            # page-locked staging slot (i % 2) by the host thread pool while
            # the GPU runs batch i - 1, then cross PCIe as one DMA
            staged = [isinstance(x, _PageableRows) and not pd for (_, x, _), pd in zip(items, padded)]
            if any(staged):
                import concurrent.futures as cf

                if self._pool is None:
                    self._pool = cf.ThreadPoolExecutor(max_workers=4, thread_name_prefix="bt200-host")
                tmax = max(sq.total for (sq, _, _), st in zip(items, staged) if st)
                slots = self._stream_stage.get((tmax, k))
                if slots is None:
                    slots = [torch.empty((tmax, k), dtype=torch.float32, pin_memory=True) for _ in range(2)]
                    self._stream_stage = {(tmax, k): slots}
            for i, ((sq, x, out), e) in enumerate(zip(items, entries)):
                bs, mx = sq.batch_size, sq.max_seq_len
                if staged[i]:
                    if i >= 2:
                        ev_in[i - 2].synchronize()  # H2D(i - 2) has read this staging slot
                    sn = slots[i % 2].numpy()
                    arr = x.arr
                    st = np.concatenate([[0], np.cumsum(lens[i])])
                    bounds = self.chunk_bounds(sq.lengths, min(bs, _STAGE_CHUNKS))

                    def copy_group(b0, b1, sn=sn, arr=arr, st=st, ln=lens[i], mx=mx):
                        for b in range(b0, b1):
                            sn[st[b]:st[b + 1]] = arr[b * mx: b * mx + ln[b]]

                    if len(bounds) == 1:
                        copy_group(*bounds[0])
                    else:
                        for f in [self._pool.submit(copy_group, b0, b1) for b0, b1 in bounds]:
                            f.result()
                if i >= 2:
                    h2d.wait_event(ev_done[i - 2])  # forward(i - 2) has read this slot's input
                with torch.cuda.stream(h2d):
                    if staged[i]:  # the packed rows as one DMA (a single T-row "sequence")
                        one = np.asarray([sq.total], dtype=np.int32)
                        _lib.call("bt_copy_rows", e[2].data_ptr(), slots[i % 2].data_ptr(), one.ctypes.data, 1,
                                  sq.total, row_b, 1, _lib.stream_ptr())
                    elif padded[i]:  # one contiguous copy of the padded input
                        _lib.call("bt_copy_rows", e[2].data_ptr(), x.data_ptr(), whole[i].ctypes.data, 1, bs * mx,
                                  row_b, 1, _lib.stream_ptr())
                    else:
                        _lib.call("bt_copy_rows", e[2].data_ptr(), x.data_ptr(), lens[i].ctypes.data, bs, mx, row_b,
                                  1, _lib.stream_ptr())
                    ev_in[i].record(h2d)
                comp.wait_event(ev_in[i])
                if i >= 2:
                    comp.wait_event(ev_out[i - 2])  # D2H(i - 2) has read this slot's output
                with torch.cuda.stream(comp):
                    if e[0] is not None:
                        e[0].replay()
                    else:
                        e[1]()
                    ev_done[i].record(comp)
                d2h.wait_event(ev_done[i])
                with torch.cuda.stream(d2h):
                    if padded[i]:  # the device wrote the exact-zero padded rows
                        _lib.call("bt_copy_rows", out.data_ptr(), e[3].data_ptr(), whole[i].ctypes.data, 1, bs * mx,
                                  row_b, 1, _lib.stream_ptr())
                    else:
                        _lib.call("bt_copy_rows", out.data_ptr(), e[3].data_ptr(), lens[i].ctypes.data, bs, mx, row_b,
                                  0, _lib.stream_ptr())
                    ev_out[i].record(d2h)
                if staged[i]:  # (host paced by the GPU here: zero this batch's padded rows now)
                    self._zero_padded_rows(out, sq, k)
            for (sq, _, out), pd, sg in zip(items, padded, staged):  # padded output rows are exact zeros
                if not pd and not sg:  # (packing.py:158-159)
                    self._zero_padded_rows(out, sq, k)
            d2h.synchronize()
            cur.wait_stream(d2h)
            return [out for _, _, out in items]

    def layer_device(self, li: int, x_bf16, plan: PackingPlan, stream=None, config: ModelConfig | None = None):
        """In-place encoder_layer on a packed bf16 [T, k] device tensor.

        The MHA geometry comes from THIS call: max_seq_len from the plan (the
        reference dispatches on plan.max_seq_len, attention.py:309-314),
        cutoff / split_seq_len from ``config`` (default: the engine's), so a
        cached engine never runs a later call with an earlier call's shape."""
        with self._lock:
            cfg = as_model_config(config) if config is not None else self.config
            cfg_c = layer_cfg_c(replace(cfg, max_seq_len=plan.max_seq_len))
            T = plan.valid_word_cnt
            ws_bytes = int(_lib.load().bt_layer_workspace_bytes(C.byref(cfg_c), T))
            ws = self.workspace(ws_bytes, stream)
            _lib.call("bt_encoder_layer", C.byref(self._layers[li].c), C.byref(cfg_c),
                      plan.seq_starts_dev.data_ptr(), plan.batch_size, T, x_bf16.data_ptr(), ws.data_ptr(), ws_bytes,
                      _lib.stream_ptr(stream))
            self._ws_used(stream)
            return x_bf16


# weights (or layer) object -> (weakref, engine, geometry); one upload per object
_engines: dict[int, tuple] = {}
_engines_lock = threading.Lock()


def _cached_engine(obj, geom, build):
    key = id(obj)
    with _engines_lock:
        hit = _engines.get(key)
        if hit is not None and hit[0]() is obj and hit[2] == geom:
            return hit[1]
        eng = build()
        try:
            ref = weakref.ref(obj, lambda _r, k=key: _engines.pop(k, None))
        except TypeError:
            ref = lambda o=obj: o  # noqa: E731  (not weak-referenceable: keep alive)
        _engines[key] = (ref, eng, geom)
        return eng


def engine_for(weights, config) -> BertEncoderB200:
    """Device engine for an EncoderWeights object (uploaded once, cached)."""
    config = as_model_config(config)
    geom = (config.layers, config.head_num, config.head_size, config.ffn_scale, config.share_layer_weights)
    return _cached_engine(weights, geom, lambda: BertEncoderB200(weights, config))


def engine_for_layer(layer, config) -> BertEncoderB200:
    """Single-layer device engine for a LayerWeights object (cached)."""
    config = replace(as_model_config(config), layers=1, share_layer_weights=False)
    geom = ("layer", config.head_num, config.head_size, config.ffn_scale)
    return _cached_engine(layer, geom, lambda: BertEncoderB200(EncoderWeights(layers=[layer], shared=False), config))


def _is_all_on(flags) -> bool:
    return bool(flags.fuse_layernorm and flags.fuse_bias_gelu and flags.zero_padding and flags.fused_mha)


def encoder_layer(x, layer, config, plan, *, workers: int = 1, counter: FlopCounter | None = None):
    """One encoder layer (reference encoder.py:337-408).  Input and output
    share a layout (packed iff zero_padding)."""
    config = as_model_config(config)
    hidden = config.hidden_dim
    xr, xc = rows_cols(x)
    if xc != hidden:
        raise ShapeError(f"input has {xc} columns, config expects {hidden}")
    plan = ensure_plan(plan)
    expected_rows = plan.valid_word_cnt if config.flags.zero_padding else plan.padded_rows
    if xr != expected_rows:
        raise ShapeError(f"input has {xr} rows, expected {expected_rows} for this layout")
    if not _is_all_on(config.flags):
        from . import ladder

        return ladder.encoder_layer_variant(x, layer, config, plan, counter=counter)
    torch = _lib.require_device()
    eng = engine_for_layer(layer, config)
    device_mode = is_device(x)
    xb = x.to(torch.bfloat16).contiguous().clone() if device_mode else \
        torch.from_numpy(host_array(x)).to("cuda").to(torch.bfloat16)
    if counter is None:
        eng.layer_device(0, xb, plan, config=config)
    else:
        from .instrument import LaunchFlops

        with LaunchFlops() as lf:  # counts come from the launches themselves
            eng.layer_device(0, xb, plan, config=config)
        lf.add_to(counter)
    return xb.float() if device_mode else Tensor(xb.float().cpu().numpy())


def forward(weights, seqs, input_padded, config, *, workers: int = 1, counter: FlopCounter | None = None):
    """Stacked encoder: plan, pack once, L layers, unpack once (reference
    encoder.py:411-437).

    Host input (reference ``Tensor`` / ndarray, fp32 ``[bs*mx, k]``) returns a
    host fp32 ``Tensor``; a CUDA fp32 tensor returns a CUDA fp32 tensor.
    Padded output rows are exactly zero."""
    config = as_model_config(config)
    seqs = as_seq_lengths(seqs)
    if seqs.batch_size != config.batch_size or seqs.max_seq_len != config.max_seq_len:
        raise ShapeError(f"lengths describe a {seqs.batch_size}x{seqs.max_seq_len} batch, config expects "
                         f"{config.batch_size}x{config.max_seq_len}")
    rows, cols = rows_cols(input_padded)
    padded_rows = seqs.batch_size * seqs.max_seq_len
    if rows != padded_rows:
        raise ShapeError(f"input has {rows} rows, expected batch_size * max_seq_len = {padded_rows}")
    if cols != config.hidden_dim:
        raise ShapeError(f"input has {cols} columns, config expects {config.hidden_dim}")
    if not _is_all_on(config.flags):
        from . import ladder

        return ladder.forward_variant(weights, seqs, input_padded, config, counter=counter)
    torch = _lib.require_device()
    eng = engine_for(weights, config)
    if is_device(input_padded) or counter is not None:
        x = input_padded.to(torch.float32).contiguous() if is_device(input_padded) else \
            torch.from_numpy(np.ascontiguousarray(host_array(input_padded), dtype=np.float32)).to("cuda")
        lengths = torch.tensor(seqs.lengths, dtype=torch.int32).to(x.device)
        out = torch.empty((padded_rows, cols), dtype=torch.float32, device=x.device)
        if counter is None:
            eng.forward_device(lengths, seqs.batch_size, seqs.total, x, out, config=config)
        else:
            # instrumented FlopCounter: an eager forward whose launches count
            # their own work (instrument.py), not the cached graph
            from .instrument import LaunchFlops

            with LaunchFlops() as lf:
                eng.forward_device(lengths, seqs.batch_size, seqs.total, x, out, config=config)
            lf.add_to(counter)
        return out if is_device(input_padded) else Tensor(out.cpu().numpy())
    # Host I/O: DMA only each sequence's valid rows into a packed device
    # buffer, run packed -> packed, DMA the valid output rows back into their
    # padded positions, and zero the padded rows on the host while the GPU works.
    out = torch.empty((padded_rows, cols), dtype=torch.float32, pin_memory=True)
    if _is_pinned_torch(input_padded):
        eng.forward_host_packed(seqs, _pinned_f32(input_padded, torch), out, config=config)
    else:  # pageable (numpy / reference Tensor): stage only the valid rows
        arr = np.ascontiguousarray(host_array(input_padded), dtype=np.float32)
        eng.forward_host_pageable(seqs, arr, out, config=config)
    return Tensor(out.numpy())


def forward_stream(weights, batches, config):
    """A stream of independent forwards on host buffers (serving): ``batches``
    is a sequence of (seqs, input_padded) pairs, each exactly what
    ``forward`` takes; returns the list of host fp32 ``Tensor`` outputs, each
    bitwise the ``forward`` result.  Consecutive batches overlap their PCIe
    copies with the previous batch's device forward
    (``BertEncoderB200.forward_host_stream``)."""
    config = as_model_config(config)
    if not _is_all_on(config.flags):
        return [forward(weights, sq, x, config) for sq, x in batches]
    torch = _lib.require_device()
    eng = engine_for(weights, config)
    items = []
    for sq, x in batches:
        sq = as_seq_lengths(sq)
        if sq.batch_size != config.batch_size or sq.max_seq_len != config.max_seq_len:
            raise ShapeError(f"lengths describe a {sq.batch_size}x{sq.max_seq_len} batch, config expects "
                             f"{config.batch_size}x{config.max_seq_len}")
        rows, cols = rows_cols(x)
        if rows != sq.batch_size * sq.max_seq_len or cols != config.hidden_dim:
            raise ShapeError(f"input is {rows}x{cols}, expected {sq.batch_size * sq.max_seq_len}x{config.hidden_dim}")
        if is_device(x):
            raise ShapeError("forward_stream takes host inputs (use forward for CUDA tensors)")
        out = torch.empty((rows, cols), dtype=torch.float32, pin_memory=True)
        items.append((sq, _host_source(x, torch), out))
    eng.forward_host_stream(items, config=config)
    return [Tensor(out.numpy()) for _, _, out in items]


# BT_PAGEABLE_STAGE=1: forward_host_pageable stages the valid rows into a
# write-combined page-locked buffer with a 4-thread pool, then one DMA (the
# earlier path, still used for batches of more than STREAM_ROW_COPIES_MAX
# sequences: C5's 2048 per-sequence pageable copies measured slower, 3.0k vs
# 3.4k seq/s per call); default 0: per-sequence copies straight from the
# pageable array.  BT_STAGE_CHUNKS: how many host threads' worth of chunks
# forward_host_stream packs a pageable batch in.  Measured at C2 (scripts/h2d_rate_probe.py): after a multi-threaded
# host write the 7.5 MB DMA runs at 12 GB/s (0.61 ms; 47 GB/s after a
# single-threaded write), while the driver-staged pageable copy moves the same
# rows in 0.39 ms of host wall time, host copy included.
_PAGEABLE_STAGE = os.environ.get("BT_PAGEABLE_STAGE", "0") == "1"
_STAGE_CHUNKS = int(os.environ.get("BT_STAGE_CHUNKS", "8"))


class _WcStage:
    """Write-combined page-locked [T, k] fp32 staging buffer (bt_host_alloc):
    the CPU only writes it, and its stores skip the CPU caches, so the DMA
    that follows reads it at the PCIe rate.  A cache-backed pinned buffer the
    CPU has just written DMAs at ~10 GB/s on this host (measured, the dirty
    lines are snooped)."""

    def __init__(self, rows: int, cols: int):
        p = C.c_void_p()
        _lib.call("bt_host_alloc", rows * cols * 4, 1, C.byref(p))
        self.ptr = p.value
        buf = (C.c_float * (rows * cols)).from_address(self.ptr)
        self.array = np.ctypeslib.as_array(buf).reshape(rows, cols)

    def __del__(self):
        try:
            self.array = None
            _lib.call("bt_host_free", self.ptr)
        except Exception:  # noqa: BLE001 -- interpreter shutdown
            pass


def _is_pinned_torch(x) -> bool:
    return type(x).__module__.startswith("torch") and not x.is_cuda and x.dtype.is_floating_point and x.is_pinned()


class _PageableRows:
    """A pageable fp32 host array as a copy source (``data_ptr``): the H2D
    copies read it directly, staged page-locked by the driver."""

    def __init__(self, arr: np.ndarray):
        self.arr = arr

    def data_ptr(self) -> int:
        return self.arr.ctypes.data


def _host_source(x, torch):
    """forward_stream's input buffer: a page-locked fp32 torch tensor in
    place, any other host input as its pageable fp32 array (no host-side
    copy into pinned memory first; BT_PAGEABLE_STAGE=1 restores that copy)."""
    if _PAGEABLE_STAGE or _is_pinned_torch(x) and x.dtype == torch.float32 and x.is_contiguous():
        return _pinned_f32(x, torch)
    return _PageableRows(np.ascontiguousarray(host_array(x), dtype=np.float32))


def _pinned_f32(x, torch):
    """Host fp32 input as a page-locked CPU tensor (used in place when it
    already is one; otherwise one host-side copy into pinned memory)."""
    if type(x).__module__.startswith("torch") and not x.is_cuda:
        t = x if x.dtype == torch.float32 else x.float()
        t = t.contiguous()
        return t if t.is_pinned() else t.pin_memory()
    arr = host_array(x)
    pinned = torch.empty(arr.shape, dtype=torch.float32, pin_memory=True)
    pinned.numpy()[...] = arr
    return pinned
