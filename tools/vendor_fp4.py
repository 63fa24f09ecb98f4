"""cuBLASLt FP4 via torch._scaled_mm on the box (vendor reference point)."""
import torch, time
dev = "cuda"
for n in (4096, 8192):
    try:
        a = torch.randint(0, 255, (n, n // 2), dtype=torch.uint8, device=dev).view(torch.float4_e2m1fn_x2)
        b = torch.randint(0, 255, (n, n // 2), dtype=torch.uint8, device=dev).view(torch.float4_e2m1fn_x2)
        # NVFP4: block-16 E4M3 scales, swizzled layout expected by cuBLASLt
        sa = torch.full((n * n // 16,), 1.0, device=dev).to(torch.float8_e4m3fn)
        sb = torch.full((n * n // 16,), 1.0, device=dev).to(torch.float8_e4m3fn)
        f = lambda: torch._scaled_mm(a, b.t(), sa, sb, out_dtype=torch.bfloat16)
        f(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(10): f()
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        print(f"cuBLASLt nvfp4 {n}^3: {ms*1e3:.1f} us {2*n**3/ms/1e9:.0f} TFLOP/s")
    except Exception as ex:
        print(f"nvfp4 {n}: unavailable: {type(ex).__name__}: {str(ex)[:200]}")
    try:
        a = torch.randint(0, 255, (n, n // 2), dtype=torch.uint8, device=dev).view(torch.float4_e2m1fn_x2)
        b = torch.randint(0, 255, (n, n // 2), dtype=torch.uint8, device=dev).view(torch.float4_e2m1fn_x2)
        sa = torch.full((n * n // 32,), 127, dtype=torch.uint8, device=dev).view(torch.float8_e8m0fnu)
        sb = torch.full((n * n // 32,), 127, dtype=torch.uint8, device=dev).view(torch.float8_e8m0fnu)
        f = lambda: torch._scaled_mm(a, b.t(), sa, sb, out_dtype=torch.bfloat16)
        f(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(10): f()
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        print(f"cuBLASLt mxfp4 {n}^3: {ms*1e3:.1f} us {2*n**3/ms/1e9:.0f} TFLOP/s")
    except Exception as ex:
        print(f"mxfp4 {n}: unavailable: {type(ex).__name__}: {str(ex)[:200]}")
