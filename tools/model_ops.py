"""Real-model op set: the Conv2d layers of torchvision classification
models as ConvDescriptor keys, batch 1, written to configs/model_ops.json.

    python tools/model_ops.py            (CPU; torchvision models on the meta device)

Each model runs one forward pass on a meta tensor (shape propagation only: no weights,
no compute, no download); a forward hook on every nn.Conv2d records its input shape and
parameters.  The JSON keeps, per model, the ordered layer keys (duplicates included, as a
network executes them) and the set of unique keys.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

MODELS = {  # name -> input side
    "alexnet": 224, "vgg16": 224, "resnet18": 224, "resnet50": 224, "resnext50_32x4d": 224,
    "wide_resnet50_2": 224, "densenet121": 224, "googlenet": 224, "inception_v3": 299,
    "mobilenet_v2": 224, "mobilenet_v3_large": 224, "efficientnet_b0": 224,
    "shufflenet_v2_x1_0": 224, "squeezenet1_1": 224, "mnasnet1_0": 224, "regnet_y_800mf": 224,
    "convnext_tiny": 224,
}


def conv_keys(name: str, side: int) -> list[str]:
    import torch
    from torchvision import models

    from paper_2407_10730_b200.descriptor import ConvDescriptor, key_of

    kw = {"aux_logits": False, "init_weights": False} if name in ("googlenet", "inception_v3") else {}
    net = getattr(models, name)(weights=None, **kw).to("meta").eval()
    keys: list[str] = []

    def hook(mod, inp, _out):
        x = inp[0]
        n, c, h, w = x.shape
        pad = mod.padding if isinstance(mod.padding, tuple) else (mod.padding, mod.padding)
        if isinstance(mod.padding, str):  # "same" / "valid" are not in the descriptor space
            return
        d = ConvDescriptor(batch=n, in_channels=c, in_h=h, in_w=w, out_channels=mod.out_channels,
                           k_h=mod.kernel_size[0], k_w=mod.kernel_size[1],
                           stride_h=mod.stride[0], stride_w=mod.stride[1],
                           pad_h=pad[0], pad_w=pad[1], dil_h=mod.dilation[0],
                           dil_w=mod.dilation[1], groups=mod.groups,
                           has_bias=mod.bias is not None)
        keys.append(key_of(d))

    hooks = [m.register_forward_hook(hook) for m in net.modules()
             if isinstance(m, torch.nn.Conv2d)]
    with torch.no_grad():
        net(torch.empty(1, 3, side, side, device="meta"))
    for hk in hooks:
        hk.remove()
    return keys


def main() -> None:
    out = {"source": "torchvision classification models, batch 1, meta-device forward hooks",
           "models": {}}
    unique: dict[str, None] = {}
    for name, side in MODELS.items():
        keys = conv_keys(name, side)
        out["models"][name] = {"input": [1, 3, side, side], "layers": keys,
                               "unique": sorted(set(keys))}
        for k in keys:
            unique.setdefault(k, None)
        print(f"{name:20s} {len(keys):4d} conv layers, {len(set(keys)):4d} unique", flush=True)
    out["unique"] = list(unique)
    path = ROOT / "configs" / "model_ops.json"
    path.parent.mkdir(exist_ok=True)
    path.write_text(json.dumps(out, indent=1) + "\n")
    print(f"{len(unique)} unique ops -> {path.relative_to(ROOT)}")


if __name__ == "__main__":
    main()
