"""__graft_entry__.smoke(): one small load-and-serve pass on cuda:0 checked
against the oracle (the reference's own trailer/touch + the CPU transform)."""
import os
import tempfile

import numpy as np


def run_smoke() -> None:
    import torch

    import oracle
    from paper_1811_09732_b200 import catalog as C
    from paper_1811_09732_b200 import format as F
    from paper_1811_09732_b200.client import Client, TensorView
    from paper_1811_09732_b200.store import Store, StoreOptions
    from paper_1811_09732_b200.models import BoundNet
    from tests import torch_ref
    from tests.golden_data import load
    from tests.gpu_util import expected_resident

    assert torch.cuda.is_available(), "smoke needs cuda:0"
    g = {e["name"]: e for e in load("catalog.json.gz")["tiny_seed1"]}
    with tempfile.TemporaryDirectory(prefix="trims-smoke-") as d:
        # 1. identity path: catalog model, disk -> pinned -> HBM, bytes == reference trailer
        C.gen_catalog("tiny", d, seed=1, only=["alexnet"])
        with Store(StoreOptions(disk_cache_dir=d, fast_capacity_bytes=64 << 20, host_capacity_bytes=64 << 20)) as s:
            cli = Client(s)
            v = cli.open(F.ModelKey("zoo", "alexnet", "1.0.0"), force_shared=True)
            n = v.blob_bytes()
            blob = TensorView("b", [n], "i8", "native", 0, n, v.base_ptr).torch().view(torch.uint8).cpu().numpy()
            assert F.sha256(blob).hex() == g["alexnet"]["trailer"], "resident bytes differ from the reference blob"
            assert cli.touch(v) == g["alexnet"]["touch"], "touch differs from the reference"
            assert v.export.ingest_checksum == oracle.port().block_checksum(blob)
            cli.close(v)
        # 2. converting path: real-shape AlexNet / ResNet-50 fp32 -> bf16 KRSC, bit-exact
        #    vs the CPU oracle; 3. a ResNet-50 batch-1 forward (tcgen05 GEMMs) on the
        #    shared weights vs the bf16-emulating CPU oracle (tolerance: tests/test_gpu_forward.py).
        opts = StoreOptions(disk_cache_dir=d, fast_capacity_bytes=1 << 30, host_capacity_bytes=1 << 30,
                            convert_to="bf16", permute_4d=True)
        with Store(opts) as s:
            cli = Client(s)
            for name in ("alexnet", "resnet50"):
                arch = C.ARCHS[name]()
                C.write_arch(arch, d, seed=1)
                src_json, src_blob = C.arch_blob(arch, seed=1)
                v = cli.open(C.arch_key(arch), force_shared=True)
                n = v.blob_bytes()
                got = TensorView("b", [n], "i8", "native", 0, n, v.base_ptr).torch().view(torch.uint8).cpu().numpy()
                want = expected_resident(src_json, src_blob, v.manifest_json)
                assert np.array_equal(got, want), f"{name}: converted resident blob differs from the oracle"
                assert v.export.ingest_checksum == oracle.port().block_checksum(want)
                if name == "resnet50":
                    net = BoundNet(v, arch, batch=1)
                    x = torch.randn(1, 3, 224, 224, generator=torch.Generator().manual_seed(2))
                    out = torch.from_numpy(net.infer(x.numpy()))
                    ref = torch_ref.forward_bf16(arch, torch_ref.weights_from_resident(v.manifest_json, got), x)
                    rel = ((out - ref).norm() / ref.norm()).item()
                    assert rel <= 1e-2 and torch.equal(out.argmax(1), ref.argmax(1)), f"forward rel L2 {rel:.3g}"
                    net.close()
                cli.close(v)
    print("smoke ok")
