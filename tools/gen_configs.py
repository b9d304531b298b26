"""Generate the extension configs (ResNet-18 CIFAR, BERT-base and their toy test twins).

The reference has only chain models (H/engine/model.hpp:18-20); these use the extension keys
"from" (input = an earlier layer's output) and "with" (second operand of "add"). BatchNorm is
folded into each conv's weight/bias by the weight owner, so convs carry a bias.

  python tools/gen_configs.py     # writes configs/{resnet18,bert_base,toy_resnet,toy_bert}.json
"""
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def resnet(name, inp, widths, blocks, classes, frac_bits=20):
    L = [{"name": "conv1", "type": "conv2d", "out": widths[0], "kernel": 3, "stride": 1, "pad": 1},
         {"name": "relu1", "type": "relu"}]
    prev, cin = "relu1", widths[0]
    for si, (w, nb) in enumerate(zip(widths, blocks)):
        for bi in range(nb):
            stride = 2 if (si > 0 and bi == 0) else 1
            p = f"l{si + 1}b{bi + 1}"
            L += [{"name": p + "c1", "type": "conv2d", "out": w, "kernel": 3, "stride": stride, "pad": 1, "from": prev},
                  {"name": p + "r1", "type": "relu"},
                  {"name": p + "c2", "type": "conv2d", "out": w, "kernel": 3, "stride": 1, "pad": 1}]
            if stride != 1 or cin != w:
                L += [{"name": p + "sc", "type": "conv2d", "out": w, "kernel": 1, "stride": stride, "pad": 0,
                       "from": prev},
                      {"name": p + "add", "type": "add", "with": p + "c2"}]
            else:
                L += [{"name": p + "add", "type": "add", "with": prev}]
            L += [{"name": p + "r2", "type": "relu"}]
            prev, cin = p + "r2", w
    L += [{"name": "gap", "type": "global_avg_pool"}, {"name": "fc", "type": "dense", "out": classes}]
    return {"name": name, "frac_bits": frac_bits, "input": inp, "layers": L}


def bert(name, inp, layers, heads, ffn, frac_bits=20):
    L = []
    prev = "input"
    for i in range(layers):
        p = f"enc{i}"
        L += [{"name": p + ".attn", "type": "attention", "heads": heads, "from": prev},
              {"name": p + ".add1", "type": "add", "with": prev},
              {"name": p + ".ln1", "type": "layernorm"},
              {"name": p + ".ffn1", "type": "dense", "out": ffn},
              {"name": p + ".gelu", "type": "gelu"},
              {"name": p + ".ffn2", "type": "dense", "out": inp[2]},
              {"name": p + ".add2", "type": "add", "with": p + ".ln1"},
              {"name": p + ".ln2", "type": "layernorm"}]
        prev = p + ".ln2"
    return {"name": name, "frac_bits": frac_bits, "input": inp, "layers": L}


def dump(cfg):
    path = os.path.join(ROOT, "configs", cfg["name"] + ".json")
    with open(path, "w") as f:
        f.write("{\n")
        f.write(f'  "name": "{cfg["name"]}", "frac_bits": {cfg["frac_bits"]}, "input": {json.dumps(cfg["input"])},\n')
        f.write('  "layers": [\n')
        f.write(",\n".join("    " + json.dumps(l) for l in cfg["layers"]))
        f.write("\n  ]\n}\n")
    print("wrote", path)


if __name__ == "__main__":
    dump(resnet("resnet18", [128, 3, 32, 32], [64, 128, 256, 512], [2, 2, 2, 2], 10))
    dump(resnet("toy_resnet", [2, 3, 8, 8], [4, 8], [1, 1], 10))
    # frac 16 (CrypTen's default, the reference MLP's): the reference's 2PC truncation (local sar,
    # H/protocols/trunc.hpp:25-42) fails with probability ~|x|/2^64 per element, and BERT-base
    # truncates ~1.7e9 values per inference — at frac 20 that is tens of 2^(64-f) errors.
    dump(bert("bert_base", [8, 128, 768], 12, 12, 3072, frac_bits=16))
    dump(bert("toy_bert", [2, 8, 16], 2, 2, 32))
