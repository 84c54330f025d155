"""JSON model-graph / catalog files and the synthetic instance builders.

File schema is the reference's (ls/fileio.py:1-20) so the same files load in both packages;
floats are written with repr() so a load -> save -> load round trip is bit-identical.
Instance builders mirror ls/experiments.py:422-496 (resize_model, catalog_with_gpu_variants,
simulate_type_variants), which define BASELINE.json's cfg2/cfg3/cfg5.
"""

from __future__ import annotations

import json
from dataclasses import replace
from pathlib import Path

from .errors import ConfigError, ParseError
from .model import LayerSpec, ModelGraph, ResourceCatalog, ResourceType

FIXTURE_DIR = Path(__file__).resolve().parent.parent / "tests" / "golden" / "instances"


def _read(path) -> dict:
    path = Path(path)
    try:
        text = path.read_text()
    except OSError as exc:
        raise ParseError(path, f"cannot read file: {exc}") from exc
    try:
        obj = json.loads(text)
    except json.JSONDecodeError as exc:
        raise ParseError(path, f"line {exc.lineno} column {exc.colno}: {exc.msg}") from exc
    if not isinstance(obj, dict):
        raise ParseError(path, "top-level JSON value must be an object")
    return obj


def _field(obj: dict, key: str, path, where: str = ""):
    try:
        return obj[key]
    except KeyError:
        raise ParseError(path, f"missing field '{key}'" + (f" in {where}" if where else "")) from None


def _per_type(obj, path, where) -> dict:
    if not isinstance(obj, dict):
        raise ParseError(path, f"{where} must be an object keyed by type id")
    out = {}
    for key, value in obj.items():
        try:
            out[int(key)] = float(value)
        except (TypeError, ValueError) as exc:
            raise ParseError(path, f"{where}[{key!r}]: {exc}") from exc
    return out


def graph_from_dict(obj: dict, path="<dict>") -> ModelGraph:
    raw = _field(obj, "layers", path)
    if not isinstance(raw, list):
        raise ParseError(path, "'layers' must be a list")
    layers = []
    for pos, item in enumerate(raw):
        where = f"layers[{pos}]"
        if not isinstance(item, dict):
            raise ParseError(path, f"{where} must be an object")
        tables = {name: _per_type(_field(item, name, path, where), path, f"{where}.{name}")
                  for name in ("oct", "odt", "alpha", "beta")}
        layers.append(LayerSpec(
            index=int(_field(item, "index", path, where)),
            layer_kind=str(_field(item, "kind", path, where)),
            input_size=float(_field(item, "input_size", path, where)),
            weight_size=float(_field(item, "weight_size", path, where)),
            per_type_oct=tables["oct"], per_type_odt=tables["odt"],
            per_type_alpha=tables["alpha"], per_type_beta=tables["beta"]))
    return ModelGraph(name=str(_field(obj, "name", path)), layers=tuple(layers),
                      total_samples=int(_field(obj, "total_samples", path)),
                      epochs=int(_field(obj, "epochs", path)),
                      batch_size=int(_field(obj, "batch_size", path)),
                      profile_batch_size=int(_field(obj, "profile_batch_size", path)))


def catalog_from_dict(obj: dict, path="<dict>") -> ResourceCatalog:
    raw = _field(obj, "types", path)
    if not isinstance(raw, list):
        raise ParseError(path, "'types' must be a list")
    types = []
    for pos, item in enumerate(raw):
        where = f"types[{pos}]"
        if not isinstance(item, dict):
            raise ParseError(path, f"{where} must be an object")
        types.append(ResourceType(
            id=int(_field(item, "id", path, where)), name=str(_field(item, "name", path, where)),
            price_per_hour=float(_field(item, "price_per_hour", path, where)),
            unit=str(_field(item, "unit", path, where)),
            quota=int(_field(item, "quota", path, where)),
            is_cpu=bool(_field(item, "is_cpu", path, where))))
    kinds = obj.get("layer_kinds", [])
    if not isinstance(kinds, list):
        raise ParseError(path, "'layer_kinds' must be a list of strings")
    return ResourceCatalog(types=tuple(types), layer_kinds=tuple(str(k) for k in kinds))


def load_model_graph(path) -> ModelGraph:
    return graph_from_dict(_read(path), path)


def load_catalog(path) -> ResourceCatalog:
    return catalog_from_dict(_read(path), path)


def graph_to_dict(graph) -> dict:
    def tab(m):
        return {str(t): m[t] for t in sorted(m)}
    return {"name": graph.name, "total_samples": graph.total_samples, "epochs": graph.epochs,
            "batch_size": graph.batch_size, "profile_batch_size": graph.profile_batch_size,
            "layers": [{"index": l.index, "kind": l.layer_kind, "input_size": l.input_size,
                        "weight_size": l.weight_size, "oct": tab(l.per_type_oct),
                        "odt": tab(l.per_type_odt), "alpha": tab(l.per_type_alpha),
                        "beta": tab(l.per_type_beta)} for l in graph.layers]}


def catalog_to_dict(catalog) -> dict:
    out = {"types": [{"id": t.id, "name": t.name, "price_per_hour": t.price_per_hour,
                      "unit": t.unit, "quota": t.quota, "is_cpu": t.is_cpu}
                     for t in catalog.types]}
    if catalog.layer_kinds:
        out["layer_kinds"] = list(catalog.layer_kinds)
    return out


def save_model_graph(graph, path) -> None:
    Path(path).write_text(json.dumps(graph_to_dict(graph), indent=2) + "\n")


def save_catalog(catalog, path) -> None:
    Path(path).write_text(json.dumps(catalog_to_dict(catalog), indent=2) + "\n")


def load_fixture(name: str, fixture_dir: Path | None = None):
    """(graph, catalog, throughput_limit) of a frozen BASELINE configuration ("cfg1".."cfg5")
    or parity instance, as written by tests/golden/make_instances.py."""
    root = Path(fixture_dir) if fixture_dir else FIXTURE_DIR
    index = json.loads((root / "index.json").read_text())
    if name not in index:
        raise ConfigError(f"unknown instance '{name}' (known: {', '.join(sorted(index))})")
    entry = index[name]
    return (load_model_graph(root / entry["graph"]), load_catalog(root / entry["catalog"]),
            float(entry["throughput_limit"]))


# --- synthetic instance builders (ls/experiments.py:422-496) ---------------------------

def resize_model(graph, target_layers: int, kind: str = "full-connection"):
    """Duplicate (or drop) the last layer of ``kind`` until the graph has target_layers."""
    if target_layers < 1:
        raise ConfigError("target layer count must be >= 1")
    layers = list(graph.layers)
    kinds = [l.layer_kind for l in layers]
    if kind not in kinds:
        kind = max(set(kinds), key=kinds.count)

    def last_of_kind():
        hits = [i for i, l in enumerate(layers) if l.layer_kind == kind]
        return hits[-1] if hits else len(layers) - 1

    while len(layers) > target_layers:
        layers.pop(last_of_kind())
    while len(layers) < target_layers:
        i = last_of_kind()
        layers.insert(i, layers[i])
    layers = [replace(l, index=i) for i, l in enumerate(layers)]
    return replace(graph, name=f"{graph.name}-L{target_layers}", layers=tuple(layers))


def catalog_with_gpu_variants(catalog, num_types: int):
    """Append price variants (x(1 + 0.15 v)) of the first accelerator up to num_types."""
    if num_types < catalog.num_types:
        raise ConfigError(f"cannot shrink catalog from {catalog.num_types} to {num_types} types")
    accels = [t for t in catalog.types if not t.is_cpu]
    if not accels:
        raise ConfigError("catalog has no accelerator type to derive variants from")
    base, types = accels[0], list(catalog.types)
    v = 1
    while len(types) < num_types:
        types.append(ResourceType(id=len(types), name=f"{base.name}-v{v}",
                                  price_per_hour=base.price_per_hour * (1.0 + 0.15 * v),
                                  unit=base.unit, quota=base.quota, is_cpu=False))
        v += 1
    return ResourceCatalog(types=tuple(types), layer_kinds=catalog.layer_kinds)


def simulate_type_variants(graph, catalog):
    """Give every layer a profile for every catalog type, copied from the lowest-id known
    type of the same class (CPU vs accelerator)."""
    cpu = [t.id for t in catalog.types if t.is_cpu]
    acc = [t.id for t in catalog.types if not t.is_cpu]
    out = []
    for layer in graph.layers:
        fields = {}
        for name in ("per_type_oct", "per_type_odt", "per_type_alpha", "per_type_beta"):
            table = dict(getattr(layer, name))
            for rt in catalog.types:
                if rt.id in table:
                    continue
                donors = [i for i in (cpu if rt.is_cpu else acc) if i in table]
                if not donors:
                    raise ConfigError(f"layer {layer.index} has no profile to copy for type "
                                      f"{rt.id} ({rt.name})")
                table[rt.id] = table[donors[0]]
            fields[name] = table
        out.append(replace(layer, **fields))
    return replace(graph, layers=tuple(out))
