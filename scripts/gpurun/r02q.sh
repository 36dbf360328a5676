# lone 4608 chain anatomy (INV_TRACE build)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
KFAC_NVCC_EXTRA=-DINV_TRACE python -c "import sys; sys.path.insert(0,'paper_1811_12019_b200'); import build; build.build(force=True)" > /dev/null 2>&1
timeout -s KILL 300 python scripts/trace_one.py 4608 gpurun_out/trace_one.txt > /dev/null 2>&1; echo "trace1 rc=$?"
python scripts/trace_analyze.py gpurun_out/trace_one.txt | tail -14
python paper_1811_12019_b200/build.py --force > /dev/null
for p in 0 1; do timeout -s KILL 300 python -c "
import sys; sys.argv=['x','4608','64']; sys.path.insert(0,'scripts')
import paper_1811_12019_b200 as K
orig=K.KfacStep.__init__
def init(self,*a,**k): k['inv_precision']=$p; orig(self,*a,**k)
K.KfacStep.__init__=init
exec(open('scripts/one_inverse.py').read())"; done
