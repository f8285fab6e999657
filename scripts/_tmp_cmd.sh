timeout 600 python -m pytest tests/test_gpu_model.py tests/test_gpu_sampling.py -x -q 2>&1 | tail -2
SPECTRE_PAR_DRAFT_CTAS=48 SPECTRE_PAR_TARGET_CTAS=100 timeout 600 python -m pytest tests/test_gpu_model.py -x -q -k lossless 2>&1 | tail -2
for dc in 0 32 48 64; do tc=$((148-dc)); if [ $dc = 0 ]; then tc=0; fi; echo "== draft $dc target $tc"; SPECTRE_PAR_DRAFT_CTAS=$dc SPECTRE_PAR_TARGET_CTAS=$tc timeout 600 python scripts/r_sweep.py --gammas 4 --alphas 1.0 --out-len 256 --out gpurun_out/rs_$dc.json 2>&1 | grep -v Warn | grep variant | python3 -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['variant'], 'tok/s', round(d['tok_s']), 'L', d['mean_L'], 't_ord', d['t_ord_ms'], 't_par', d['t_par_ms'], 'ord_share', d['ordinary_share'])
"; done
