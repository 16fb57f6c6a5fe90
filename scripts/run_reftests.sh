# GPU box: the reference's own test modules through the drop-in; the scratch
# harness (_reftests/, built in the container by scripts/make_reftests.py) is
# removed afterwards.  Summary into gpurun_out/reftests.log.
cd _reftests && timeout 1500 python -m pytest tests -q -p no:cacheprovider -rfE --tb=line -W ignore \
    > ../gpurun_out/reftests.log 2>&1; echo "reftests rc=$?"
cd .. && rm -rf _reftests
tail -40 gpurun_out/reftests.log
