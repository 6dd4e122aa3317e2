"""Test harness around the hot path (not product code): the paper's scenario
builders, the reference's run metrics and the criterion-sweep / paired-timing
driver.  They set up inputs and post-process runs; the
package `paper_2505_17025_b200` keeps only the step path and its API."""
