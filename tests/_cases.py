"""Shared case table: golden config name -> (variant, quantizer kwargs)."""

CONFIGS = {
    "ocp32": ("ocp32", {}),
    "mx16": ("mx16", {}),
    "mx16_oas": ("mx16_oas", {}),
    "mbs_s": ("mbs_s", {}),
    "mbs_d": ("mbs_d", {}),
    "nvfp4": ("nvfp4", {}),
    "mbs_d_cand3": ("mbs_d", {"candidates": (0, 37, 200), "augment_static": False}),
    "mbs_d_noaug": ("mbs_d", {"augment_static": False}),
    "mbs_s_m64": ("mbs_s", {"macro_size": 64}),
    "mbs_d_m256": ("mbs_d", {"macro_size": 256}),
    "mbs_d_m512": ("mbs_d", {"macro_size": 512}),
    "mbs_d_m32": ("mbs_d", {"macro_size": 32}),
    "mbs_d_lut": ("mbs_d", {"mbs_mode": "lut"}),
}

FIELDS = ("codes", "block_scales", "e4m3_scales", "mbs_mantissas", "tensor_scale")


def golden_cases(golden):
    """Yield (tensor_name, config_name) for every quantizer case in golden.npz."""
    seen = set()
    for k in golden.files:
        if k.startswith("q/"):
            _, t, c = k.split("/")[:3]
            if (t, c) not in seen:
                seen.add((t, c))
                yield t, c


def split_pair(pair):
    """'mbs_sxmbs_d' -> ('mbs_s', 'mbs_d')."""
    names = ("ocp32", "mx16_oas", "mx16", "mbs_s", "mbs_d", "nvfp4")
    for v in names:
        if pair.startswith(v + "x") and pair[len(v) + 1:] in names:
            return v, pair[len(v) + 1:]
    raise ValueError(pair)
