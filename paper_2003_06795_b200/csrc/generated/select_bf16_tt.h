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
    if (k < INT64_C(1087)) {
        if (k < INT64_C(351)) {
            if (n < INT64_C(222)) {
                if (m < INT64_C(8870)) {
                    if (n < INT64_C(46)) {
                        if (k < INT64_C(118)) {
                            if (m < INT64_C(4435)) {
                                select_bf16_tt_config out = {2u, 1u, 8u, 16u, 16u};
                                return out;
                            } else {
                                select_bf16_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (m < INT64_C(2218)) {
                                if (m < INT64_C(1109)) {
                                    select_bf16_tt_config out = {8u, 1u, 2u, 16u, 16u};
                                    return out;
                                } else {
                                    if (k < INT64_C(167)) {
                                        select_bf16_tt_config out = {8u, 1u, 4u, 16u, 16u};
                                        return out;
                                    } else {
                                        select_bf16_tt_config out = {8u, 1u, 2u, 16u, 16u};
                                        return out;
                                    }
                                }
                            } else {
                                if (n < INT64_C(28)) {
                                    if (m < INT64_C(4435)) {
                                        select_bf16_tt_config out = {8u, 1u, 4u, 16u, 16u};
                                        return out;
                                    } else {
                                        select_bf16_tt_config out = {8u, 1u, 2u, 16u, 16u};
                                        return out;
                                    }
                                } else {
                                    select_bf16_tt_config out = {1u, 1u, 4u, 8u, 8u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        if (m < INT64_C(2218)) {
                            if (m < INT64_C(555)) {
                                if (m < INT64_C(224)) {
                                    select_bf16_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_tt_config out = {1u, 1u, 4u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                select_bf16_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (k < INT64_C(111)) {
                                if (k < INT64_C(28)) {
                                    if (m < INT64_C(4435)) {
                                        select_bf16_tt_config out = {8u, 1u, 2u, 16u, 16u};
                                        return out;
                                    } else {
                                        select_bf16_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_bf16_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                if (k < INT64_C(222)) {
                                    select_bf16_tt_config out = {8u, 1u, 2u, 16u, 16u};
                                    return out;
                                } else {
                                    if (m < INT64_C(4435)) {
                                        select_bf16_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (n < INT64_C(91)) {
                                            select_bf16_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_bf16_tt_config out = {8u, 1u, 2u, 16u, 16u};
                                            return out;
                                        }
                                    }
                                }
                            }
                        }
                    }
                } else {
                    if (n < INT64_C(46)) {
                        if (k < INT64_C(30)) {
                            if (m < INT64_C(17740)) {
                                select_bf16_tt_config out = {8u, 1u, 4u, 16u, 16u};
                                return out;
                            } else {
                                if (m < INT64_C(70960)) {
                                    select_bf16_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (m < INT64_C(141920)) {
                                        select_bf16_tt_config out = {8u, 2u, 8u, 16u, 16u};
                                        return out;
                                    } else {
                                        select_bf16_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                }
                            }
                        } else {
                            if (m < INT64_C(35480)) {
                                if (k < INT64_C(167)) {
                                    if (m < INT64_C(17740)) {
                                        if (k < INT64_C(118)) {
                                            if (k < INT64_C(56)) {
                                                select_bf16_tt_config out = {8u, 1u, 2u, 16u, 16u};
                                                return out;
                                            } else {
                                                select_bf16_tt_config out = {1u, 1u, 4u, 8u, 8u};
                                                return out;
                                            }
                                        } else {
                                            select_bf16_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        select_bf16_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_bf16_tt_config out = {8u, 1u, 2u, 16u, 16u};
                                    return out;
                                }
                            } else {
                                select_bf16_tt_config out = {8u, 1u, 2u, 16u, 16u};
                                return out;
                            }
                        }
                    } else {
                        if (k < INT64_C(20)) {
                            if (m < INT64_C(70960)) {
                                select_bf16_tt_config out = {8u, 1u, 4u, 16u, 16u};
                                return out;
                            } else {
                                select_bf16_tt_config out = {1u, 1u, 4u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (m < INT64_C(283839)) {
                                if (k < INT64_C(194)) {
                                    if (k < INT64_C(28)) {
                                        if (m < INT64_C(35480)) {
                                            select_bf16_tt_config out = {8u, 2u, 8u, 16u, 16u};
                                            return out;
                                        } else {
                                            select_bf16_tt_config out = {8u, 1u, 2u, 16u, 16u};
                                            return out;
                                        }
                                    } else {
                                        if (m < INT64_C(17740)) {
                                            if (k < INT64_C(46)) {
                                                select_bf16_tt_config out = {8u, 1u, 2u, 16u, 16u};
                                                return out;
                                            } else {
                                                if (k < INT64_C(97)) {
                                                    select_bf16_tt_config out = {2u, 1u, 8u, 16u, 16u};
                                                    return out;
                                                } else {
                                                    select_bf16_tt_config out = {8u, 1u, 2u, 16u, 16u};
                                                    return out;
                                                }
                                            }
                                        } else {
                                            select_bf16_tt_config out = {8u, 1u, 2u, 16u, 16u};
                                            return out;
                                        }
                                    }
                                } else {
                                    if (m < INT64_C(17740)) {
                                        if (n < INT64_C(91)) {
                                            select_bf16_tt_config out = {8u, 1u, 2u, 16u, 16u};
                                            return out;
                                        } else {
                                            select_bf16_tt_config out = {8u, 2u, 8u, 16u, 16u};
                                            return out;
                                        }
                                    } else {
                                        if (m < INT64_C(35480)) {
                                            select_bf16_tt_config out = {1u, 1u, 4u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_bf16_tt_config out = {8u, 2u, 8u, 16u, 16u};
                                            return out;
                                        }
                                    }
                                }
                            } else {
                                if (m < INT64_C(567677)) {
                                    select_bf16_tt_config out = {1u, 1u, 4u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_tt_config out = {8u, 2u, 8u, 16u, 16u};
                                    return out;
                                }
                            }
                        }
                    }
                }
            } else {
                if (m < INT64_C(2218)) {
                    if (k < INT64_C(79)) {
                        if (m < INT64_C(555)) {
                            select_bf16_tt_config out = {1u, 1u, 4u, 8u, 8u};
                            return out;
                        } else {
                            select_bf16_tt_config out = {8u, 1u, 4u, 16u, 16u};
                            return out;
                        }
                    } else {
                        if (m < INT64_C(1109)) {
                            if (n < INT64_C(744)) {
                                if (m < INT64_C(278)) {
                                    select_bf16_tt_config out = {8u, 1u, 2u, 16u, 16u};
                                    return out;
                                } else {
                                    if (m < INT64_C(555)) {
                                        select_bf16_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(182)) {
                                            select_bf16_tt_config out = {8u, 1u, 2u, 16u, 16u};
                                            return out;
                                        } else {
                                            select_bf16_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            } else {
                                if (m < INT64_C(278)) {
                                    if (m < INT64_C(70)) {
                                        select_bf16_tt_config out = {8u, 1u, 2u, 16u, 16u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(139)) {
                                            if (k < INT64_C(227)) {
                                                select_bf16_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_bf16_tt_config out = {8u, 1u, 2u, 16u, 16u};
                                                return out;
                                            }
                                        } else {
                                            if (k < INT64_C(287)) {
                                                select_bf16_tt_config out = {8u, 1u, 2u, 16u, 16u};
                                                return out;
                                            } else {
                                                select_bf16_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    }
                                } else {
                                    select_bf16_tt_config out = {8u, 1u, 2u, 16u, 16u};
                                    return out;
                                }
                            }
                        } else {
                            if (n < INT64_C(768)) {
                                select_bf16_tt_config out = {8u, 1u, 2u, 16u, 16u};
                                return out;
                            } else {
                                select_bf16_tt_config out = {8u, 1u, 4u, 16u, 16u};
                                return out;
                            }
                        }
                    }
                } else {
                    if (m < INT64_C(35480)) {
                        if (n < INT64_C(768)) {
                            if (m < INT64_C(4435)) {
                                select_bf16_tt_config out = {8u, 1u, 4u, 16u, 16u};
                                return out;
                            } else {
                                if (k < INT64_C(182)) {
                                    if (m < INT64_C(8870)) {
                                        select_bf16_tt_config out = {1u, 1u, 4u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(17740)) {
                                            if (k < INT64_C(91)) {
                                                select_bf16_tt_config out = {2u, 1u, 8u, 16u, 16u};
                                                return out;
                                            } else {
                                                select_bf16_tt_config out = {8u, 1u, 4u, 16u, 16u};
                                                return out;
                                            }
                                        } else {
                                            select_bf16_tt_config out = {8u, 1u, 4u, 16u, 16u};
                                            return out;
                                        }
                                    }
                                } else {
                                    select_bf16_tt_config out = {2u, 1u, 8u, 16u, 16u};
                                    return out;
                                }
                            }
                        } else {
                            select_bf16_tt_config out = {1u, 1u, 4u, 8u, 8u};
                            return out;
                        }
                    } else {
                        select_bf16_tt_config out = {8u, 2u, 8u, 16u, 16u};
                        return out;
                    }
                }
            }
        } else {
            if (m < INT64_C(4435)) {
                if (n < INT64_C(725)) {
                    if (k < INT64_C(992)) {
                        select_bf16_tt_config out = {2u, 1u, 1u, 8u, 8u};
                        return out;
                    } else {
                        if (m < INT64_C(278)) {
                            select_bf16_tt_config out = {2u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            if (m < INT64_C(1109)) {
                                select_bf16_tt_config out = {8u, 1u, 2u, 16u, 16u};
                                return out;
                            } else {
                                select_bf16_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        }
                    }
                } else {
                    if (m < INT64_C(555)) {
                        if (k < INT64_C(725)) {
                            if (m < INT64_C(278)) {
                                select_bf16_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (n < INT64_C(1449)) {
                                    select_bf16_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_tt_config out = {8u, 1u, 2u, 16u, 16u};
                                    return out;
                                }
                            }
                        } else {
                            if (m < INT64_C(70)) {
                                select_bf16_tt_config out = {8u, 1u, 4u, 16u, 16u};
                                return out;
                            } else {
                                if (m < INT64_C(139)) {
                                    select_bf16_tt_config out = {1u, 1u, 4u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        if (m < INT64_C(1568)) {
                            select_bf16_tt_config out = {8u, 1u, 4u, 16u, 16u};
                            return out;
                        } else {
                            select_bf16_tt_config out = {2u, 1u, 8u, 16u, 16u};
                            return out;
                        }
                    }
                }
            } else {
                if (n < INT64_C(91)) {
                    if (m < INT64_C(8870)) {
                        select_bf16_tt_config out = {2u, 1u, 1u, 8u, 8u};
                        return out;
                    } else {
                        select_bf16_tt_config out = {8u, 1u, 2u, 16u, 16u};
                        return out;
                    }
                } else {
                    if (m < INT64_C(35480)) {
                        if (m < INT64_C(8870)) {
                            select_bf16_tt_config out = {8u, 1u, 2u, 16u, 16u};
                            return out;
                        } else {
                            select_bf16_tt_config out = {1u, 1u, 4u, 8u, 8u};
                            return out;
                        }
                    } else {
                        if (m < INT64_C(141920)) {
                            select_bf16_tt_config out = {8u, 1u, 4u, 16u, 16u};
                            return out;
                        } else {
                            select_bf16_tt_config out = {8u, 2u, 8u, 16u, 16u};
                            return out;
                        }
                    }
                }
            }
        }
    } else {
        if (m < INT64_C(2509)) {
            if (n < INT64_C(1432)) {
                if (m < INT64_C(12)) {
                    if (m < INT64_C(3)) {
                        if (k < INT64_C(2897)) {
                            select_bf16_tt_config out = {8u, 1u, 4u, 16u, 16u};
                            return out;
                        } else {
                            select_bf16_tt_config out = {1u, 1u, 4u, 8u, 8u};
                            return out;
                        }
                    } else {
                        select_bf16_tt_config out = {1u, 1u, 4u, 8u, 8u};
                        return out;
                    }
                } else {
                    if (m < INT64_C(555)) {
                        if (k < INT64_C(4345)) {
                            if (m < INT64_C(40)) {
                                select_bf16_tt_config out = {8u, 1u, 2u, 16u, 16u};
                                return out;
                            } else {
                                if (m < INT64_C(139)) {
                                    select_bf16_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_tt_config out = {8u, 1u, 2u, 16u, 16u};
                                    return out;
                                }
                            }
                        } else {
                            if (m < INT64_C(70)) {
                                select_bf16_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (m < INT64_C(139)) {
                                    select_bf16_tt_config out = {8u, 1u, 4u, 16u, 16u};
                                    return out;
                                } else {
                                    select_bf16_tt_config out = {1u, 1u, 4u, 8u, 8u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        if (m < INT64_C(1109)) {
                            if (n < INT64_C(363)) {
                                select_bf16_tt_config out = {8u, 1u, 4u, 16u, 16u};
                                return out;
                            } else {
                                select_bf16_tt_config out = {1u, 1u, 4u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (n < INT64_C(363)) {
                                if (k < INT64_C(1630)) {
                                    select_bf16_tt_config out = {8u, 1u, 2u, 16u, 16u};
                                    return out;
                                } else {
                                    select_bf16_tt_config out = {1u, 1u, 4u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                select_bf16_tt_config out = {2u, 1u, 8u, 16u, 16u};
                                return out;
                            }
                        }
                    }
                }
            } else {
                if (m < INT64_C(12)) {
                    select_bf16_tt_config out = {2u, 1u, 8u, 16u, 16u};
                    return out;
                } else {
                    if (m < INT64_C(182)) {
                        if (k < INT64_C(10138)) {
                            select_bf16_tt_config out = {8u, 1u, 4u, 16u, 16u};
                            return out;
                        } else {
                            select_bf16_tt_config out = {2u, 1u, 8u, 16u, 16u};
                            return out;
                        }
                    } else {
                        select_bf16_tt_config out = {2u, 1u, 8u, 16u, 16u};
                        return out;
                    }
                }
            }
        } else {
            if (k < INT64_C(2661)) {
                if (m < INT64_C(17740)) {
                    if (n < INT64_C(182)) {
                        if (m < INT64_C(8870)) {
                            select_bf16_tt_config out = {2u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            select_bf16_tt_config out = {8u, 1u, 4u, 16u, 16u};
                            return out;
                        }
                    } else {
                        if (m < INT64_C(8870)) {
                            if (k < INT64_C(1630)) {
                                if (m < INT64_C(4435)) {
                                    select_bf16_tt_config out = {8u, 1u, 2u, 16u, 16u};
                                    return out;
                                } else {
                                    select_bf16_tt_config out = {8u, 1u, 4u, 16u, 16u};
                                    return out;
                                }
                            } else {
                                select_bf16_tt_config out = {2u, 1u, 8u, 16u, 16u};
                                return out;
                            }
                        } else {
                            if (n < INT64_C(363)) {
                                select_bf16_tt_config out = {2u, 1u, 8u, 16u, 16u};
                                return out;
                            } else {
                                select_bf16_tt_config out = {8u, 2u, 8u, 16u, 16u};
                                return out;
                            }
                        }
                    }
                } else {
                    if (k < INT64_C(1630)) {
                        if (m < INT64_C(35480)) {
                            select_bf16_tt_config out = {1u, 1u, 4u, 8u, 8u};
                            return out;
                        } else {
                            if (m < INT64_C(70960)) {
                                select_bf16_tt_config out = {8u, 1u, 4u, 16u, 16u};
                                return out;
                            } else {
                                if (m < INT64_C(141920)) {
                                    select_bf16_tt_config out = {8u, 2u, 8u, 16u, 16u};
                                    return out;
                                } else {
                                    select_bf16_tt_config out = {8u, 1u, 4u, 16u, 16u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        select_bf16_tt_config out = {8u, 2u, 8u, 16u, 16u};
                        return out;
                    }
                }
            } else {
                select_bf16_tt_config out = {8u, 2u, 8u, 16u, 16u};
                return out;
            }
        }
    }
}

#endif /* SELECT_BF16_TT_H */
