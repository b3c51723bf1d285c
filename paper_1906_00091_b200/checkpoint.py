"""Checkpoints in the reference's ``DLRMKIT1 v1`` format (ref ``cli.py:475-518``,
``save_checkpoint`` / ``load_checkpoint``): one ASCII header line
``DLRMKIT1 v1 <sha256 of the sorted-key JSON config>`` followed by an ``.npz``
payload with ``config_json`` (uint8 bytes of that JSON), ``bottom_w_<l>``,
``bottom_b_<l>``, ``top_w_<l>``, ``top_b_<l>`` and ``table_<t>``.

Files written here load with the reference's ``load_checkpoint`` and vice
versa.  Parameters are written in their training precision (fp32, exact);
``dtype="float64"`` writes the reference's own dtype.  Optimiser state — which
the reference does not save — travels as extra arrays the reference loader
ignores: ``opt_kind`` (uint8 bytes of "adagrad") and ``adagrad_<name>`` for
every parameter array ``<name>`` (the squared-gradient accumulators).

The header / payload layer (``write_arrays`` / ``read_arrays``) is pure
numpy; ``save_checkpoint`` / ``load_checkpoint`` move the parameters to and
from the GPU model.
"""

from __future__ import annotations

import dataclasses
import hashlib
import io
import json

import numpy as np

__all__ = ["CHECKPOINT_MAGIC", "CheckpointError", "config_digest", "config_json",
           "write_arrays", "read_arrays", "save_checkpoint", "load_checkpoint",
           "load_optimizer_state", "model_arrays", "adagrad_arrays",
           "restore_adagrad"]

CHECKPOINT_MAGIC = "DLRMKIT1"


class CheckpointError(ValueError):
    """Bad magic / version / digest (the reference raises its CliError)."""


def _config_dict(config) -> dict:
    d = dataclasses.asdict(config) if dataclasses.is_dataclass(config) else dict(config)
    # plain ints / lists so the JSON (and its digest) matches the reference's
    return {"embedding_sizes": [int(m) for m in d["embedding_sizes"]],
            "sparse_dim": int(d["sparse_dim"]),
            "bottom_mlp_dims": [int(x) for x in d["bottom_mlp_dims"]],
            "top_mlp_dims": [int(x) for x in d["top_mlp_dims"]],
            "interaction": str(d["interaction"]), "seed": int(d["seed"])}


def config_json(config) -> str:
    """``json.dumps(asdict(config), sort_keys=True)`` (ref cli.py:478-480)."""
    return json.dumps(_config_dict(config), sort_keys=True)


def config_digest(config) -> str:
    """sha256 hex of the config JSON (ref ``_config_digest``, cli.py:478-480)."""
    return hashlib.sha256(config_json(config).encode("ascii")).hexdigest()


def write_arrays(path: str, config, arrays: dict) -> None:
    """Header + npz payload; ``arrays`` maps the reference's names (and any
    extra names) to numpy arrays."""
    payload = {"config_json": np.frombuffer(config_json(config).encode("ascii"), dtype=np.uint8)}
    payload.update(arrays)
    with open(path, "wb") as f:
        f.write(f"{CHECKPOINT_MAGIC} v1 {config_digest(config)}\n".encode("ascii"))
        # the zip's offsets are relative to where it starts, so writing it
        # straight behind the header gives the bytes the reference produces
        # with its BytesIO round trip
        np.savez(f, **payload)


def read_arrays(path: str):
    """(config dict, {name: array}) of a checkpoint, header and digest checked
    exactly as the reference's ``load_checkpoint``."""
    with open(path, "rb") as f:
        header = f.readline().decode("ascii").split()
        if len(header) != 3 or header[0] != CHECKPOINT_MAGIC:
            raise CheckpointError(f"not a {CHECKPOINT_MAGIC} checkpoint: {path}")
        if header[1] != "v1":
            raise CheckpointError(f"unsupported checkpoint version {header[1]}")
        payload = np.load(io.BytesIO(f.read()))
        arrays = {k: payload[k] for k in payload.files}
    cfg = json.loads(bytes(arrays.pop("config_json")).decode("ascii"))
    if config_digest(cfg) != header[2]:
        raise CheckpointError("checkpoint config digest mismatch")
    return cfg, arrays


def _host(t, dtype):
    return t.detach().to("cpu").numpy().astype(dtype, copy=False)


def model_arrays(model, dtype="float32") -> dict:
    """The reference's parameter arrays of a model (host copies)."""
    out = {}
    for name, mlp in (("bottom", model.bottom), ("top", model.top)):
        for l, layer in enumerate(mlp.layers):
            out[f"{name}_w_{l}"] = _host(layer.weight, dtype)
            out[f"{name}_b_{l}"] = _host(layer.bias, dtype)
    for t, table in enumerate(model.tables):
        out[f"table_{t}"] = _host(table.weights, dtype)
    return out


def _engine_adagrad_views(engine):
    """name -> accumulator view of a StepEngine trained with Adagrad (the
    accumulators share the parameters' flat layout)."""
    p0, w0 = engine.params.data_ptr(), engine.W_all.data_ptr()
    views = {}
    for name, layers in (("bottom", engine.model.bottom.layers),
                         ("top", engine.model.top.layers)):
        for l, layer in enumerate(layers):
            off = (layer.storage.data_ptr() - p0) // 4
            st = engine.params_acc[off:off + layer.storage.numel()].view_as(layer.storage)
            views[f"{name}_w_{l}"] = st[:, :layer.n_in]
            boff = (layer.bias.data_ptr() - p0) // 4
            views[f"{name}_b_{l}"] = engine.params_acc[boff:boff + layer.n_out]
    for t, table in enumerate(engine.model.tables):
        off = (table.weights.data_ptr() - w0) // 4
        views[f"table_{t}"] = engine.W_acc[off:off + table.weights.numel()].view_as(table.weights)
    return views


def _adagrad_views(opt, model):
    """name -> accumulator tensor for an optim.Adagrad or a StepEngine built
    with optimizer="adagrad".  An Adagrad that drives a ``train_step`` engine
    holds views of that engine's live accumulators (parallel._mirror_adagrad),
    so its state is always the one to read or write."""
    if hasattr(opt, "params_acc"):
        if getattr(opt, "optimizer", None) != "adagrad":
            raise ValueError("engine was not built with Adagrad")
        return _engine_adagrad_views(opt)
    views = {}
    for name in ("bottom", "top"):
        st = opt._mlp_state.get(name)
        if st is None:
            continue
        for l, (aw, ab) in enumerate(zip(st.mlp_weights, st.mlp_biases)):
            views[f"{name}_w_{l}"] = aw
            views[f"{name}_b_{l}"] = ab
    for t, table in enumerate(model.tables):
        acc = opt._table_state.get(table.table_id)
        if acc is not None:
            views[f"table_{t}"] = acc
    return views


def adagrad_arrays(opt, model, dtype="float32") -> dict:
    """``adagrad_<name>`` host arrays of the accumulators (see module doc)."""
    out = {"opt_kind": np.frombuffer(b"adagrad", dtype=np.uint8)}
    for k, v in _adagrad_views(opt, model).items():
        out[f"adagrad_{k}"] = _host(v, dtype)
    return out


def save_checkpoint(path: str, model, optimizer=None, dtype: str = "float32") -> None:
    """Write ``model`` (and, for Adagrad, the accumulators of ``optimizer`` —
    an ``optim.Adagrad`` or the ``StepEngine`` that trained the model) in the
    reference's format."""
    if dtype not in ("float32", "float64"):
        raise ValueError("dtype must be float32 or float64")
    arrays = model_arrays(model, dtype)
    if optimizer is not None and (getattr(optimizer, "name", None) == "adagrad"
                                  or getattr(optimizer, "optimizer", None) == "adagrad"):
        arrays.update(adagrad_arrays(optimizer, model, dtype))
    write_arrays(path, model.config, arrays)


def load_checkpoint(path: str):
    """A GPU ``DlrmModel`` from a checkpoint written here or by the reference
    (values rounded to fp32).  No parameter is drawn from the init streams:
    every array comes from the file."""
    from .embedding import EmbeddingTable
    from .model import DlrmConfig, DlrmModel, MlpLayer, MlpParams
    cfg_d, arrays = read_arrays(path)
    cfg = DlrmConfig(**cfg_d)

    def mlp(name, n, acts):
        return MlpParams([MlpLayer(arrays[f"{name}_w_{l}"], arrays[f"{name}_b_{l}"], acts[l])
                          for l in range(n)])
    nb = len(cfg.bottom_mlp_dims) - 1
    chain = cfg.top_dims_chain()
    nt = len(chain) - 1
    bottom = mlp("bottom", nb, ["relu"] * nb)
    top = mlp("top", nt, ["relu"] * (nt - 1) + ["identity"])
    tables = []
    for t, m in enumerate(cfg.embedding_sizes):
        w = arrays[f"table_{t}"]
        if w.shape != (m, cfg.sparse_dim):
            raise CheckpointError(f"table_{t} has shape {w.shape}, config says "
                                  f"{(m, cfg.sparse_dim)}")
        tables.append(EmbeddingTable(w, t))
    return DlrmModel(cfg, bottom, top, tables)


def load_optimizer_state(path: str):
    """{name: host array} of the saved Adagrad accumulators, or None."""
    _, arrays = read_arrays(path)
    if "opt_kind" not in arrays:
        return None
    kind = bytes(arrays["opt_kind"]).decode("ascii")
    if kind != "adagrad":
        raise CheckpointError(f"unknown optimiser state {kind!r}")
    return {k[len("adagrad_"):]: v for k, v in arrays.items() if k.startswith("adagrad_")}


def restore_adagrad(opt, model, state: dict) -> None:
    """Copy saved accumulators into an ``optim.Adagrad`` (creating its state;
    the next ``train_step`` engine starts from it) or an Adagrad
    ``StepEngine``."""
    import torch
    if not hasattr(opt, "params_acc"):
        from .optim import AdagradState
        for name, mlp in (("bottom", model.bottom), ("top", model.top)):
            if name not in opt._mlp_state:
                opt._mlp_state[name] = AdagradState.for_mlp(mlp)
        for table in model.tables:
            if table.table_id not in opt._table_state:
                opt._table_state[table.table_id] = torch.zeros_like(table.weights)
    views = _adagrad_views(opt, model)
    for k, v in views.items():
        if k not in state:
            raise CheckpointError(f"optimiser state lacks {k}")
        v.copy_(torch.as_tensor(np.asarray(state[k], np.float32)).to(v.device))
