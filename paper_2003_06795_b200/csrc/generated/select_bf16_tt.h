#ifndef SELECT_BF16_TT_H
#define SELECT_BF16_TT_H

#include <stdint.h>

typedef struct {
    uint32_t acc;
    uint32_t row_tile;
    uint32_t col_tile;
    uint32_t wg_rows;
    uint32_t wg_cols;
} select_bf16_tt_config;

static inline select_bf16_tt_config select_bf16_tt(int64_t m, int64_t k, int64_t n) {
    (void)m;
    (void)k;
    (void)n;
    if (m < INT64_C(17740)) {
        if (m < INT64_C(3584)) {
            if (n < INT64_C(1620)) {
                if (m < INT64_C(448)) {
                    if (n < INT64_C(79)) {
                        select_bf16_tt_config out = {2u, 1u, 1u, 8u, 8u};
                        return out;
                    } else {
                        if (k < INT64_C(111)) {
                            if (m < INT64_C(278)) {
                                select_bf16_tt_config out = {4u, 1u, 1u, 16u, 16u};
                                return out;
                            } else {
                                if (k < INT64_C(79)) {
                                    select_bf16_tt_config out = {2u, 1u, 1u, 16u, 16u};
                                    return out;
                                } else {
                                    select_bf16_tt_config out = {4u, 1u, 1u, 16u, 16u};
                                    return out;
                                }
                            }
                        } else {
                            if (k < INT64_C(2173)) {
                                if (m < INT64_C(159)) {
                                    if (k < INT64_C(1620)) {
                                        if (k < INT64_C(744)) {
                                            if (n < INT64_C(1109)) {
                                                if (m < INT64_C(70)) {
                                                    select_bf16_tt_config out = {4u, 1u, 1u, 16u, 16u};
                                                    return out;
                                                } else {
                                                    if (k < INT64_C(304)) {
                                                        select_bf16_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        select_bf16_tt_config out = {4u, 1u, 1u, 16u, 16u};
                                                        return out;
                                                    }
                                                }
                                            } else {
                                                if (m < INT64_C(70)) {
                                                    select_bf16_tt_config out = {2u, 1u, 1u, 16u, 16u};
                                                    return out;
                                                } else {
                                                    select_bf16_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        } else {
                                            if (m < INT64_C(29)) {
                                                select_bf16_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                if (k < INT64_C(992)) {
                                                    select_bf16_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    if (m < INT64_C(70)) {
                                                        select_bf16_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        select_bf16_tt_config out = {2u, 1u, 1u, 16u, 16u};
                                                        return out;
                                                    }
                                                }
                                            }
                                        }
                                    } else {
                                        if (m < INT64_C(12)) {
                                            if (m < INT64_C(3)) {
                                                select_bf16_tt_config out = {4u, 1u, 1u, 16u, 16u};
                                                return out;
                                            } else {
                                                if (m < INT64_C(6)) {
                                                    select_bf16_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_bf16_tt_config out = {1u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        } else {
                                            select_bf16_tt_config out = {4u, 1u, 1u, 16u, 16u};
                                            return out;
                                        }
                                    }
                                } else {
                                    if (n < INT64_C(1145)) {
                                        if (m < INT64_C(317)) {
                                            if (k < INT64_C(544)) {
                                                if (k < INT64_C(444)) {
                                                    select_bf16_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    if (n < INT64_C(512)) {
                                                        select_bf16_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        select_bf16_tt_config out = {4u, 1u, 1u, 16u, 16u};
                                                        return out;
                                                    }
                                                }
                                            } else {
                                                if (k < INT64_C(992)) {
                                                    if (k < INT64_C(744)) {
                                                        if (n < INT64_C(124)) {
                                                            select_bf16_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                                            return out;
                                                        } else {
                                                            select_bf16_tt_config out = {1u, 1u, 1u, 8u, 8u};
                                                            return out;
                                                        }
                                                    } else {
                                                        select_bf16_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    }
                                                } else {
                                                    if (k < INT64_C(1449)) {
                                                        if (n < INT64_C(363)) {
                                                            select_bf16_tt_config out = {2u, 1u, 1u, 16u, 16u};
                                                            return out;
                                                        } else {
                                                            select_bf16_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                                            return out;
                                                        }
                                                    } else {
                                                        select_bf16_tt_config out = {1u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    }
                                                }
                                            }
                                        } else {
                                            if (k < INT64_C(992)) {
                                                if (n < INT64_C(124)) {
                                                    if (k < INT64_C(471)) {
                                                        select_bf16_tt_config out = {1u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        select_bf16_tt_config out = {4u, 1u, 1u, 16u, 16u};
                                                        return out;
                                                    }
                                                } else {
                                                    if (k < INT64_C(203)) {
                                                        select_bf16_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        if (n < INT64_C(227)) {
                                                            select_bf16_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                                            return out;
                                                        } else {
                                                            select_bf16_tt_config out = {2u, 1u, 1u, 16u, 16u};
                                                            return out;
                                                        }
                                                    }
                                                }
                                            } else {
                                                select_bf16_tt_config out = {4u, 1u, 1u, 16u, 16u};
                                                return out;
                                            }
                                        }
                                    } else {
                                        select_bf16_tt_config out = {1u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                if (m < INT64_C(2)) {
                                    select_bf16_tt_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    if (m < INT64_C(8)) {
                                        select_bf16_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(29)) {
                                            select_bf16_tt_config out = {2u, 1u, 2u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (m < INT64_C(278)) {
                                                if (m < INT64_C(70)) {
                                                    select_bf16_tt_config out = {2u, 1u, 1u, 16u, 16u};
                                                    return out;
                                                } else {
                                                    if (m < INT64_C(139)) {
                                                        select_bf16_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        if (k < INT64_C(3259)) {
                                                            select_bf16_tt_config out = {2u, 1u, 1u, 16u, 16u};
                                                            return out;
                                                        } else {
                                                            select_bf16_tt_config out = {1u, 1u, 1u, 8u, 8u};
                                                            return out;
                                                        }
                                                    }
                                                }
                                            } else {
                                                select_bf16_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    }
                                }
                            }
                        }
                    }
                } else {
                    if (n < INT64_C(351)) {
                        if (n < INT64_C(46)) {
                            if (m < INT64_C(2218)) {
                                if (m < INT64_C(1109)) {
                                    select_bf16_tt_config out = {2u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_tt_config out = {2u, 1u, 1u, 16u, 16u};
                                    return out;
                                }
                            } else {
                                if (k < INT64_C(167)) {
                                    select_bf16_tt_config out = {1u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_tt_config out = {8u, 1u, 8u, 16u, 16u};
                                    return out;
                                }
                            }
                        } else {
                            if (m < INT64_C(1109)) {
                                if (n < INT64_C(144)) {
                                    if (n < INT64_C(111)) {
                                        if (n < INT64_C(79)) {
                                            select_bf16_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_bf16_tt_config out = {1u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        select_bf16_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (n < INT64_C(287)) {
                                        if (k < INT64_C(702)) {
                                            if (k < INT64_C(128)) {
                                                select_bf16_tt_config out = {4u, 1u, 1u, 16u, 16u};
                                                return out;
                                            } else {
                                                select_bf16_tt_config out = {2u, 1u, 1u, 16u, 16u};
                                                return out;
                                            }
                                        } else {
                                            if (k < INT64_C(992)) {
                                                select_bf16_tt_config out = {1u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                if (k < INT64_C(1536)) {
                                                    select_bf16_tt_config out = {4u, 1u, 1u, 16u, 16u};
                                                    return out;
                                                } else {
                                                    select_bf16_tt_config out = {1u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        }
                                    } else {
                                        select_bf16_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                if (n < INT64_C(136)) {
                                    if (k < INT64_C(222)) {
                                        if (m < INT64_C(2218)) {
                                            select_bf16_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (k < INT64_C(111)) {
                                                select_bf16_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_bf16_tt_config out = {4u, 1u, 1u, 16u, 16u};
                                                return out;
                                            }
                                        }
                                    } else {
                                        if (n < INT64_C(111)) {
                                            if (k < INT64_C(471)) {
                                                if (m < INT64_C(2218)) {
                                                    if (n < INT64_C(79)) {
                                                        select_bf16_tt_config out = {4u, 1u, 1u, 16u, 16u};
                                                        return out;
                                                    } else {
                                                        select_bf16_tt_config out = {2u, 1u, 1u, 16u, 16u};
                                                        return out;
                                                    }
                                                } else {
                                                    if (n < INT64_C(79)) {
                                                        select_bf16_tt_config out = {2u, 1u, 1u, 16u, 16u};
                                                        return out;
                                                    } else {
                                                        select_bf16_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    }
                                                }
                                            } else {
                                                if (m < INT64_C(2218)) {
                                                    select_bf16_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_bf16_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        } else {
                                            if (m < INT64_C(2218)) {
                                                if (k < INT64_C(768)) {
                                                    select_bf16_tt_config out = {2u, 1u, 1u, 16u, 16u};
                                                    return out;
                                                } else {
                                                    select_bf16_tt_config out = {4u, 1u, 1u, 16u, 16u};
                                                    return out;
                                                }
                                            } else {
                                                select_bf16_tt_config out = {2u, 1u, 1u, 16u, 16u};
                                                return out;
                                            }
                                        }
                                    }
                                } else {
                                    if (k < INT64_C(1630)) {
                                        if (m < INT64_C(2218)) {
                                            if (k < INT64_C(128)) {
                                                select_bf16_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                if (k < INT64_C(725)) {
                                                    select_bf16_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_bf16_tt_config out = {4u, 1u, 1u, 16u, 16u};
                                                    return out;
                                                }
                                            }
                                        } else {
                                            if (k < INT64_C(128)) {
                                                if (k < INT64_C(28)) {
                                                    select_bf16_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_bf16_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            } else {
                                                select_bf16_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    } else {
                                        select_bf16_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                }
                            }
                        }
                    } else {
                        if (m < INT64_C(2218)) {
                            if (k < INT64_C(203)) {
                                if (k < INT64_C(111)) {
                                    if (m < INT64_C(1109)) {
                                        select_bf16_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(79)) {
                                            select_bf16_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_bf16_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                } else {
                                    select_bf16_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                if (m < INT64_C(634)) {
                                    select_bf16_tt_config out = {1u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(3259)) {
                                        if (k < INT64_C(2173)) {
                                            if (k < INT64_C(725)) {
                                                if (m < INT64_C(1109)) {
                                                    if (n < INT64_C(1145)) {
                                                        select_bf16_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        select_bf16_tt_config out = {2u, 1u, 2u, 8u, 8u};
                                                        return out;
                                                    }
                                                } else {
                                                    if (k < INT64_C(363)) {
                                                        select_bf16_tt_config out = {1u, 1u, 2u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        select_bf16_tt_config out = {2u, 1u, 2u, 8u, 8u};
                                                        return out;
                                                    }
                                                }
                                            } else {
                                                if (k < INT64_C(1449)) {
                                                    select_bf16_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_bf16_tt_config out = {1u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        } else {
                                            select_bf16_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        select_bf16_tt_config out = {2u, 1u, 2u, 8u, 8u};
                                        return out;
                                    }
                                }
                            }
                        } else {
                            if (k < INT64_C(363)) {
                                if (n < INT64_C(544)) {
                                    select_bf16_tt_config out = {1u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(157)) {
                                        select_bf16_tt_config out = {2u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_bf16_tt_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                select_bf16_tt_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        }
                    }
                }
            } else {
                if (m < INT64_C(278)) {
                    if (m < INT64_C(29)) {
                        if (m < INT64_C(12)) {
                            if (k < INT64_C(10138)) {
                                select_bf16_tt_config out = {2u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                select_bf16_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        } else {
                            select_bf16_tt_config out = {4u, 1u, 1u, 16u, 16u};
                            return out;
                        }
                    } else {
                        if (k < INT64_C(725)) {
                            select_bf16_tt_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            if (m < INT64_C(70)) {
                                select_bf16_tt_config out = {2u, 1u, 1u, 16u, 16u};
                                return out;
                            } else {
                                if (m < INT64_C(139)) {
                                    select_bf16_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            }
                        }
                    }
                } else {
                    select_bf16_tt_config out = {2u, 1u, 2u, 8u, 8u};
                    return out;
                }
            }
        } else {
            if (k < INT64_C(1630)) {
                if (n < INT64_C(222)) {
                    if (n < INT64_C(91)) {
                        if (n < INT64_C(28)) {
                            if (m < INT64_C(8870)) {
                                select_bf16_tt_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                select_bf16_tt_config out = {4u, 1u, 1u, 16u, 16u};
                                return out;
                            }
                        } else {
                            if (k < INT64_C(168)) {
                                if (k < INT64_C(42)) {
                                    select_bf16_tt_config out = {2u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(96)) {
                                        select_bf16_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(146)) {
                                            select_bf16_tt_config out = {2u, 1u, 1u, 16u, 16u};
                                            return out;
                                        } else {
                                            select_bf16_tt_config out = {2u, 1u, 2u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            } else {
                                if (m < INT64_C(8870)) {
                                    if (k < INT64_C(384)) {
                                        select_bf16_tt_config out = {2u, 1u, 1u, 16u, 16u};
                                        return out;
                                    } else {
                                        select_bf16_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (k < INT64_C(222)) {
                                        select_bf16_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(384)) {
                                            select_bf16_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_bf16_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            }
                        }
                    } else {
                        if (m < INT64_C(8870)) {
                            if (k < INT64_C(91)) {
                                select_bf16_tt_config out = {1u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(363)) {
                                    select_bf16_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_tt_config out = {2u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            select_bf16_tt_config out = {2u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    }
                } else {
                    if (k < INT64_C(91)) {
                        if (m < INT64_C(8870)) {
                            select_bf16_tt_config out = {2u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            select_bf16_tt_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    } else {
                        select_bf16_tt_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    }
                }
            } else {
                if (n < INT64_C(363)) {
                    if (m < INT64_C(8870)) {
                        select_bf16_tt_config out = {2u, 1u, 2u, 8u, 8u};
                        return out;
                    } else {
                        select_bf16_tt_config out = {8u, 1u, 8u, 16u, 16u};
                        return out;
                    }
                } else {
                    select_bf16_tt_config out = {8u, 1u, 8u, 16u, 16u};
                    return out;
                }
            }
        }
    } else {
        if (k < INT64_C(815)) {
            if (m < INT64_C(35480)) {
                if (n < INT64_C(46)) {
                    select_bf16_tt_config out = {4u, 1u, 1u, 8u, 8u};
                    return out;
                } else {
                    if (k < INT64_C(97)) {
                        select_bf16_tt_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    } else {
                        if (k < INT64_C(384)) {
                            select_bf16_tt_config out = {2u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            select_bf16_tt_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    }
                }
            } else {
                if (n < INT64_C(111)) {
                    if (n < INT64_C(28)) {
                        if (k < INT64_C(68)) {
                            select_bf16_tt_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            select_bf16_tt_config out = {2u, 1u, 1u, 16u, 16u};
                            return out;
                        }
                    } else {
                        select_bf16_tt_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    }
                } else {
                    if (m < INT64_C(70960)) {
                        select_bf16_tt_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    } else {
                        select_bf16_tt_config out = {8u, 1u, 8u, 16u, 16u};
                        return out;
                    }
                }
            }
        } else {
            if (m < INT64_C(35480)) {
                select_bf16_tt_config out = {1u, 1u, 2u, 8u, 8u};
                return out;
            } else {
                select_bf16_tt_config out = {8u, 1u, 8u, 16u, 16u};
                return out;
            }
        }
    }
}

#endif /* SELECT_BF16_TT_H */
