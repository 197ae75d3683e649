python -c "import sys; sys.path.insert(0,'tests'); from conftest import ensure_cfg2; ensure_cfg2('cfg2')"
FSIGPU_SETUP_TRACE=1 python -c "
import sys, time; sys.path.insert(0,'.')
from paper_1909_13201_b200 import fsigpu
from paper_1909_13201_b200.problem import load_case
P=load_case('data_cfg2/cfg2.fsix'); fsigpu.init(0)
t=time.time(); G=fsigpu.GmgPreconditioner(P.levels); print('setup', time.time()-t)
t=time.time(); lv=[P.levels[0]]+[fsigpu.build_block_sets(l) for l in P.levels[1:]]; print('device sets', time.time()-t)
"
