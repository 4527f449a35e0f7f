# usage: bash tools/gpu_sanitize.sh <tool>  -- one compute-sanitizer tool over small nested / OLA / direct runs
TOOL=${1:-memcheck}
mkdir -p gpurun_out
cat > /tmp/san_case.py <<'PY'
import sys, torch
sys.path.insert(0, '.')
import synth, paper_2102_13272_b200 as nw
for name, kw in (("c2k9", dict(N=2, H=29, W=31, Cin=32, Cout=32)), ("c3", dict(N=1, H=20, W=19, Cin=64, Cout=64)),
                 ("c4b", dict(N=1, H=22, W=23, Cin=8, Cout=16)), ("c5_deconv", dict(N=1, H=11, W=13)), ("c1", {})):
    l = synth.small(synth.CONFIGS[name], **kw) if kw else synth.CONFIGS[name]
    t = synth.make_inputs(l)
    for math in (nw.MATH_BF16X3, nw.MATH_FP32_SIMT):
        conv = nw.NestedConv2d(t["w"].cuda(), l.stride, l.pad, l.m_o, l.m_i, math, transposed=l.transposed,
                               output_padding=l.output_padding)
        for path in ("nested", "ola", "direct"):
            conv(t["x"].cuda(), path=path)
    torch.cuda.synchronize()
print("ok")
PY
timeout 1200 compute-sanitizer --tool $TOOL --print-limit 20 python /tmp/san_case.py > gpurun_out/sanitize_$TOOL.txt 2>&1; echo "sanitizer $TOOL rc=$?"
tail -15 gpurun_out/sanitize_$TOOL.txt
