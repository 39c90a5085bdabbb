out=gpurun_out/r2n; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "batched_multi_rhs or multi_rhs" 2>&1 | grep -E "Error|assert|passed|failed" | head -20
cat > /tmp/pv.py <<'PY'
import sys, torch; sys.path.insert(0, '.')
from paper_1403_6015_b200 import inputs; import paper_1403_6015_b200.hodlr as hb
cfg = inputs.CONFIGS['cfg3']; x = torch.from_numpy(inputs.points(cfg)).cuda(); y = torch.from_numpy(inputs.rhs(cfg)).cuda()
h = hb.HODLR(x, cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf, cfg.eps).factor()
xt = torch.linspace(cfg.lo, cfg.hi, 32, dtype=torch.float64, device='cuda')
for _ in range(2): m, v = h.predict(y, xt)
Y = torch.randn(cfg.n, 32, dtype=torch.float64, device='cuda')
for _ in range(2): h.solve(Y)
torch.cuda.synchronize()
PY
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/pv.csv python /tmp/pv.py > /dev/null 2>&1
python tools/launch_summary.py $out/pv.csv | head -12
