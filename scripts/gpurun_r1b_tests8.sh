python -c "import __graft_entry__ as g; g.build()" > gpurun_out/t8_build.log 2>&1; echo build=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/t8_smoke.log 2>&1; echo smoke=$?
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=8 > gpurun_out/t8_pytest.log 2>&1; echo pytest=$?
tail -14 gpurun_out/t8_pytest.log
