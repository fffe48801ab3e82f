# compute-sanitizer over the kernel-family probe (round 2 kernels included)
mkdir -p gpurun_out/san
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_probe.py > gpurun_out/san/$tool.log 2>&1
  echo "$tool: $(tail -2 gpurun_out/san/$tool.log | tr '\n' ' ')"
done
SDCT_COLC=1 timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python -c "
import torch, paper_2110_01172_b200 as sd
x = torch.rand((4096, 64), dtype=torch.float64, device='cuda')
for f in (sd.dct_2d, sd.idct_2d): f(x)
torch.cuda.synchronize(); print('colc probe done')" > gpurun_out/san/colc_memcheck.log 2>&1
echo "colc memcheck: $(tail -2 gpurun_out/san/colc_memcheck.log | tr '\n' ' ')"
